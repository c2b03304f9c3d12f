#!/bin/bash
# usage: CONFIG=c3e4 TILE=8 PROFILE="regex" bash scripts/gpu_profile_cfg.sh TAG  -- launch list + one full capture
TAG=${1:-dev}
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
ARGS="--config ${CONFIG:-c2b} --steps 2 --warmup 3 --no-cpu-baseline --no-pif ${TILE:+--tile $TILE} ${EXTRA}"
timeout 300 python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bin_|scan_|scatter|spread|interp|pad_|trunc|fft|weights|halo|pif_|migrate" -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu_launch=$?"
if [ -n "$PROFILE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$PROFILE" -s ${SKIP:-0} -c ${COUNT:-4} -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu_full=$?"
fi
