mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2k_smoke.log
NUFFT_PARITY_LOG=gpurun_out/r2k_parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2k_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2k_tests.log
timeout 1200 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
for sw in 5 0; do timeout 300 python bench.py --config c2a --steps 10 --warmup 3 --no-cpu-baseline --spread-warps $sw > gpurun_out/r2k_c2a_sw$sw.json 2>/dev/null; done
timeout 600 python bench.py --config c4n --steps 3 --warmup 3 --no-cpu-baseline --no-pif --fft-method 1 > gpurun_out/r2k_c4n_pruned.json 2> gpurun_out/r2k_c4n_pruned.err
