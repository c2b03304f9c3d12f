# bounds-checked build (NUFFT_DEBUG_BOUNDS: NUFFT_CHECK asserts on every shared-memory
# block index, bulk-copy alignment and sorted slot) over the GPU suite, final sources
mkdir -p gpurun_out
NUFFT_LIB=$PWD/paper_2605_10678_b200/libnufft_debug.so timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_fullsize_gpu.py::test_c4_fp64_landau_full_size > gpurun_out/r3o_bounds.log 2>&1
echo "pytest(bounds) rc=$?" >> gpurun_out/r3o_bounds.log
NUFFT_LIB=$PWD/paper_2605_10678_b200/libnufft_debug.so timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/r3o_bounds_bench.json 2> gpurun_out/r3o_bounds_bench.err
echo "bench(bounds, C4) rc=$?" >> gpurun_out/r3o_bounds_bench.err
