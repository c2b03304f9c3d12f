# spread: evict-last policy on the block reductions, evict-first records / strengths
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py tests/test_pif_gpu.py -m gpu -q -x > gpurun_out/r3j_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r3j_tests.log
for cfg in c4n c3 c3e4; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/r3j_$cfg.json 2>gpurun_out/r3j_$cfg.err
done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"spread_subg" -s 1 -c 1 -o gpurun_out/r3j_dram_spread python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/r3j_ncu.log 2>&1
