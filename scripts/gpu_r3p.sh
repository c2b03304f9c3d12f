# interp: slot stores after both points' chains
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py tests/test_pif_gpu.py -m gpu -q -x > gpurun_out/r3p_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r3p_tests.log
for cfg in c4n c3 c3e4; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3p_$cfg.json 2>gpurun_out/r3p_$cfg.err
done
