#!/bin/bash
# usage: SWEEP="c3e4:8:8 c3e4:11:2" bash scripts/gpu_sweep_real.sh TAG   (config:tile:spread_warps, real path)
TAG=${1:-dev}
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
for item in $SWEEP; do
  IFS=: read cfg t nw <<< "$item"
  timeout 600 python bench.py --config $cfg --tile $t --spread-warps $nw --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline ${REAL:---real} > gpurun_out/swr_${TAG}_${cfg}_${t}_${nw}.log 2>&1
  python - gpurun_out/swr_${TAG}_${cfg}_${t}_${nw}.log "$item" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['stage_ms_median']
    print(f"{sys.argv[2]:>12}: {d['value']:.4g} {d['unit']} step {d['ms_per_step']:.3f} ms spread {s['ms_spread']:.3f} interp {s['ms_interp']:.3f} setpts {s['ms_setpts']:.3f} fft {s['ms_fft']:.3f}")
except Exception as e:
    print(sys.argv[2], 'failed', open(sys.argv[1]).read()[-400:])
PY
done
