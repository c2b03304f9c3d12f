#!/bin/bash
# round-2 final evidence: default bench line (C4), the ncu launch list of the same
# command, one --set full capture of the dominant kernels at C4 (traffic), GPU suite
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/final_tests.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?" >> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bin_|scan_|scatter|spread|interp|pad_|trunc|fft|weights|halo|pif_|migrate" -c 300 --csv --log-file gpurun_out/final_launches_c4n.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/final_ncu_launch.log 2>&1; echo "ncu launch rc=$?" >> gpurun_out/final_ncu_launch.log
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"spread_subg|interp_subg" -s 2 -c 2 -o gpurun_out/final_full_c4n python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/final_ncu_full.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/final_ncu_full.log
