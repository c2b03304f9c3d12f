mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_real_gpu.py tests/test_pif_gpu.py tests/test_loopback_gpu.py -m gpu -q -x > gpurun_out/r2t_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2t_tests.log
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --pif-fused > gpurun_out/r2t_pif_fused.json 2> gpurun_out/r2t_pif_fused.err
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2t_pif.json 2> gpurun_out/r2t_pif.err
timeout 1800 python bench.py --config c4e8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2t_pif_e8.json 2> gpurun_out/r2t_pif_e8.err
