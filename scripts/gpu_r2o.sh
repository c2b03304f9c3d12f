mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py -m gpu -q -x > gpurun_out/r2o_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2o_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --pif-fused > gpurun_out/r2o_pif_fused.json 2> gpurun_out/r2o_pif_fused.err
CONFIG=c3e4 PROFILE="scatter|bin_count|interp_sub" COUNT=3 bash scripts/gpu_profile_cfg.sh r2o
