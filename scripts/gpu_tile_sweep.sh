#!/bin/bash
# usage: CONFIG=c2b TILES="8 9 10 12 13" bash scripts/gpu_tile_sweep.sh TAG
TAG=${1:-dev}
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_$TAG.log; exit 1; }
for cfg in ${CONFIGS:-c2b}; do
for t in ${TILES:-8 10 12}; do
  timeout 300 python bench.py --config $cfg --tile $t --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/sweep_${TAG}_${cfg}_$t.log 2>&1
  python - gpurun_out/sweep_${TAG}_${cfg}_$t.log $cfg $t <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['stage_ms_median']
    print(f"{sys.argv[2]} T={sys.argv[3]:>6}: {d['value']:.3e} pts/s  step {d['ms_per_step']:.3f} ms  spread {s['ms_spread']:.3f}  interp {s['ms_interp']:.3f}  setpts {s['ms_setpts']:.3f}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], 'failed', open(sys.argv[1]).read()[-300:])
PY
done; done
