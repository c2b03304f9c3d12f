mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py -m gpu -q -x -k "sub_bin or real_type1 or three_field or config1 or every_width" > gpurun_out/r2v_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2v_tests.log
for cfg in c3e4 c3 c4n; do timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/r2v_$cfg.json 2>/dev/null; done
