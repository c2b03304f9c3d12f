mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py -m gpu -q -x -k "sub_bin or real_type1 or three_field" > gpurun_out/r2f_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2f_tests.log
for nw in 16 8; do
NUFFT_SUB_WARPS=$nw timeout 600 python bench.py --config c3e4 --steps 5 --warmup 3 --no-cpu-baseline --spread-warps 5 > gpurun_out/r2f_c3e4_nw$nw.json 2> gpurun_out/r2f_c3e4_nw$nw.err
done
CONFIG=c3e4 EXTRA="--spread-warps 5" PROFILE="spread_sub|interp_sub" COUNT=2 bash scripts/gpu_profile_cfg.sh r2f
