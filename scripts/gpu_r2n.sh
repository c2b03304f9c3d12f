mkdir -p gpurun_out
# bounds-checked library over the GPU suite (the substitute for compute-sanitizer)
NUFFT_LIB=$PWD/paper_2605_10678_b200/libnufft_debug.so timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_fullsize_gpu.py::test_c4_fp64_landau_full_size > gpurun_out/r2n_bounds.log 2>&1
echo "pytest(bounds) rc=$?" >> gpurun_out/r2n_bounds.log
NUFFT_LIB=$PWD/paper_2605_10678_b200/libnufft_debug.so timeout 600 python bench.py --config c3e4 --steps 2 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/r2n_bounds_bench.json 2> gpurun_out/r2n_bounds_bench.err
echo "bench(bounds) rc=$?" >> gpurun_out/r2n_bounds_bench.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
