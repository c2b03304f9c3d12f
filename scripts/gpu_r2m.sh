mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py -m gpu -q -x -k "sub_bin or real_type1 or three_field or config1" > gpurun_out/r2m_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2m_tests.log
for cfg in c3e4 c4n; do
timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/r2m_${cfg}.json 2> gpurun_out/r2m_${cfg}.err
done
CONFIG=c3e4 PROFILE="spread_subg|scatter|bin_count" COUNT=3 bash scripts/gpu_profile_cfg.sh r2m
