#!/bin/bash
# usage: bash scripts/gpu_check.sh TAG [bench args...]  -- GPU tests, smoke, bench, launch list, one ncu full capture
TAG=${1:-dev}; shift
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python bench.py "$@" > gpurun_out/bench_$TAG.log 2>&1; echo "bench=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-1500
if [ -n "$PROFILE" ]; then
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu_launch=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$PROFILE" -s 4 -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu_full=$?"
fi
