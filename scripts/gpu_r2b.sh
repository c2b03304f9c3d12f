mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py -m gpu -x -q -k "sub_bin or real_type1" > gpurun_out/r2b_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_tests.log
for sw in 5 0; do
timeout 600 python bench.py --config c3e4 --steps 5 --warmup 3 --no-cpu-baseline --spread-warps $sw > gpurun_out/r2b_c3e4_sw$sw.json 2> gpurun_out/r2b_c3e4_sw$sw.err
done
timeout 900 python bench.py --config c4n --steps 5 --warmup 3 --no-cpu-baseline --no-pif --spread-warps 5 > gpurun_out/r2b_c4n_sw5.json 2> gpurun_out/r2b_c4n_sw5.err
