#!/bin/bash
# weight-table A/B per config: precompute -1 (phi in the kernels) vs 1 (setpts table)
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_pc.log 2>&1 || { echo BUILD FAILED; exit 1; }
for cfg in ${CONFIGS:-c2b c2a c3 c3e4}; do
  for pc in -1 1; do
    timeout 300 python bench.py --config $cfg --precompute $pc --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pc_${cfg}_$pc.log 2>&1
    python - gpurun_out/pc_${cfg}_$pc.log "$cfg pc=$pc" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['stage_ms_median']
    print(f"{sys.argv[2]:>12}: {d['value']:.3e} step {d['ms_per_step']:.3f} ms spread {s['ms_spread']:.3f} interp {s['ms_interp']:.3f} setpts {s['ms_setpts']:.3f}")
except Exception as e:
    print(sys.argv[2], 'failed', open(sys.argv[1]).read()[-400:])
PY
  done
done
