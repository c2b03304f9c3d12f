mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py -m gpu -q -k "sub_bin or real_type1" > gpurun_out/r2c_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c_tests.log
CONFIG=c3e4 EXTRA="--spread-warps 5" PROFILE="spread_sub|interp_tile" COUNT=2 bash scripts/gpu_profile_cfg.sh r2c
