mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py -m gpu -q -x -k "sub_bin or real_type1 or three_field or every_width" > gpurun_out/r2q_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2q_tests.log
for sw in 5 0; do
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --spread-warps $sw > gpurun_out/r2q_c3_sw$sw.json 2>/dev/null
timeout 300 python bench.py --config c2b --steps 10 --warmup 3 --no-cpu-baseline --spread-warps $sw > gpurun_out/r2q_c2b_sw$sw.json 2>/dev/null
done
timeout 600 python bench.py --config c3e4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2q_c3e4.json 2>/dev/null
