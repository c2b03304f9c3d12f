mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_fullsize_gpu.py > gpurun_out/r2l_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2l_tests.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_c1.py > gpurun_out/r2l_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/r2l_memcheck.log
