mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py tests/test_loopback_gpu.py -m gpu -q -x > gpurun_out/r2p_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2p_tests.log
for cfg in c3e4 c4n; do
timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/r2p_${cfg}.json 2> gpurun_out/r2p_${cfg}.err
done
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2p_pif.json 2> gpurun_out/r2p_pif.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --pif-fused > gpurun_out/r2p_pif_fused.json 2> gpurun_out/r2p_pif_fused.err
CONFIG=c3e4 PROFILE="interp_subg|spread_subg" COUNT=2 bash scripts/gpu_profile_cfg.sh r2p
