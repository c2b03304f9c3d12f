mkdir -p gpurun_out
NUFFT_SUB_GLOBAL=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py -m gpu -q -x -k "sub_bin or real_type1 or three_field" > gpurun_out/r2g_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2g_tests.log
for gl in 1 0; do
NUFFT_SUB_GLOBAL=$gl timeout 600 python bench.py --config c3e4 --steps 5 --warmup 3 --no-cpu-baseline --spread-warps 5 > gpurun_out/r2g_c3e4_g$gl.json 2> gpurun_out/r2g_c3e4_g$gl.err
done
NUFFT_SUB_GLOBAL=1 CONFIG=c3e4 EXTRA="--spread-warps 5" PROFILE="spread_subg" COUNT=1 bash scripts/gpu_profile_cfg.sh r2g
