mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py tests/test_loopback_gpu.py -m gpu -q -x > gpurun_out/r2r_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2r_tests.log
for cfg in c3e4 c3; do timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2r_$cfg.json 2>/dev/null; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err
CONFIG=c3e4 PROFILE="interp_subg" COUNT=1 bash scripts/gpu_profile_cfg.sh r2r
