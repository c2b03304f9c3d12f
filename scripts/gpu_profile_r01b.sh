#!/bin/bash
# Round-1 (second pass) evidence: per config a plain bench run, then the ncu launch
# list of the same command, then one --set full capture of spread + interp.
# usage: CONFIGS="c2b c3" bash scripts/gpu_profile_r01b.sh
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_prof.log 2>&1 || { echo BUILD FAILED; exit 1; }
for cfg in ${CONFIGS:-c2b c3}; do
  A="--config $cfg --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 600 python bench.py $A > gpurun_out/plain_$cfg.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_${cfg}_${TAG:-r01b}.csv python bench.py $A > gpurun_out/ncu_launch_$cfg.log 2>&1
  echo "$cfg launch list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"${KREGEX:-spread_outer|interp_tile|spread_tile|bin_count|scatter}" -s ${SKIP:-5} -c ${COUNT:-4} \
      -o gpurun_out/prof_${cfg}_${TAG:-r01b} python bench.py $A > gpurun_out/ncu_full_$cfg.log 2>&1
  echo "$cfg full rc=$?"
  [ -n "$EXPORT" ] && bash scripts/ncu_export.sh gpurun_out/prof_${cfg}_${TAG:-r01b}.ncu-rep
done
