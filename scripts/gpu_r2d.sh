mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py -m gpu -q -x -k "sub_bin or real_type1" > gpurun_out/r2d_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2d_tests.log
timeout 600 python bench.py --config c3e4 --steps 5 --warmup 3 --no-cpu-baseline --spread-warps 5 > gpurun_out/r2d_c3e4_sw5.json 2> gpurun_out/r2d_c3e4_sw5.err
CONFIG=c3e4 EXTRA="--spread-warps 5" PROFILE="spread_sub" COUNT=1 bash scripts/gpu_profile_cfg.sh r2d
