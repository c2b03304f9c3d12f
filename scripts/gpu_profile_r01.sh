#!/bin/bash
# Round-1 evidence for the default bench line (C2b): plain run, launch list (ours + cuFFT),
# one ncu --set full capture of the two hot kernels, and C3 launch list.
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_prof.log 2>&1 || { echo BUILD FAILED; exit 1; }
A="--steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 python bench.py $A > gpurun_out/plain_c2b.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"nufft|fft" -c 300 --csv --log-file gpurun_out/launches_c2b_r01.csv python bench.py $A > gpurun_out/ncu_launch_c2b.log 2>&1; echo "launch_c2b=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spread_rows|interp_tile" -s 6 -c 2 -o gpurun_out/prof_c2b_r01 python bench.py $A > gpurun_out/ncu_full_c2b.log 2>&1; echo "full_c2b=$?"
timeout 300 python bench.py --config c3 $A > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"nufft|fft" -c 120 --csv --log-file gpurun_out/launches_c3_r01.csv python bench.py --config c3 $A > gpurun_out/ncu_launch_c3.log 2>&1; echo "launch_c3=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spread_tile|interp_tile|scatter|bin_count" -s 4 -c 4 -o gpurun_out/prof_c3_r01 python bench.py --config c3 $A > gpurun_out/ncu_full_c3.log 2>&1; echo "full_c3=$?"
