mkdir -p gpurun_out
nproc > gpurun_out/r2a_env.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
NUFFT_PARITY_LOG=gpurun_out/r2a_parity.jsonl timeout 1800 python -m pytest tests -m gpu -x -q -s --durations=30 > gpurun_out/r2a_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_gputests.log
timeout 1200 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
echo "bench rc=$?" >> gpurun_out/r2a_bench.err
