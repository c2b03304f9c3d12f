# row-block interpolation (w <= 5): parity + A/B against the 8^3 register block
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -m gpu -q -x > gpurun_out/r3a_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r3a_tests.log
for cfg in c4n c3e4; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3a_$cfg.json 2>gpurun_out/r3a_$cfg.err
  NUFFT_ROW_BLOCKS=0 timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3a_${cfg}_off.json 2>/dev/null
done
