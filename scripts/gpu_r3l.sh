# sanity of the final in-tree build: smoke, GPU suite, one short default bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3l_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r3l_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3l_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r3l_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3l_bench.json 2> gpurun_out/r3l_bench.err
