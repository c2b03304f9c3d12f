#!/bin/bash
# one ncu --set full capture of the tensor-core spread at C2b (after a plain run)
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_tcp.log 2>&1 || { echo BUILD FAILED; exit 1; }
A="--config ${CFG:-c2b} --spread-warps 3 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 python bench.py $A > gpurun_out/tcp_plain.log 2>&1 || { echo plain failed; tail -5 gpurun_out/tcp_plain.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spread_tc -s 3 -c 1 \
    -o gpurun_out/prof_tc python bench.py $A > gpurun_out/tcp_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_tc.ncu-rep --page source --csv -k regex:spread_tc > gpurun_out/tc_src.csv 2>/dev/null
python scripts/ncu_sass_summary.py gpurun_out/tc_src.csv 30 > gpurun_out/tc_sass_summary.txt
bash scripts/ncu_details.sh gpurun_out/prof_tc.ncu-rep > gpurun_out/tc_details.txt
ncu -i gpurun_out/prof_tc.ncu-rep --page details --csv > gpurun_out/tc_details_full.csv 2>/dev/null
gzip -f gpurun_out/tc_src.csv; rm -f gpurun_out/prof_tc.ncu-rep
cat gpurun_out/tc_details.txt; head -50 gpurun_out/tc_sass_summary.txt
