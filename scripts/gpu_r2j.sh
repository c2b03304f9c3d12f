mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_loopback_gpu.py -m gpu -q -x -k "pif or sub_bins" > gpurun_out/r2j_loop.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2j_loop.log
NUFFT_SUB_GLOBAL=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py -m gpu -q -x -k "sub_bin or real_type1 or three_field" > gpurun_out/r2j_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2j_tests.log
for cfg in c3e4 c4n; do
NUFFT_SUB_GLOBAL=1 timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-pif --spread-warps 5 > gpurun_out/r2j_${cfg}_g1.json 2> gpurun_out/r2j_${cfg}_g1.err
done
NUFFT_SUB_GLOBAL=1 CONFIG=c3e4 EXTRA="--spread-warps 5" PROFILE="spread_subg|interp_sub" COUNT=2 bash scripts/gpu_profile_cfg.sh r2j
