#!/bin/bash
# usage: bash scripts/gpu_bench_configs.sh TAG -- bench every config once (device timing + stages)
TAG=${1:-dev}; shift
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_$TAG.log; exit 1; }
for cfg in ${CONFIGS:-c2b c2a c1 c3e4 c3}; do
  timeout 600 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline "$@" > gpurun_out/bench_${TAG}_$cfg.log 2>&1; echo "$cfg rc=$?"
  python - gpurun_out/bench_${TAG}_$cfg.log <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"  value={d['value']:.3e} pts/s  ms/step={d['ms_per_step']:.3f}  e2e={d['e2e']['value']:.3e}  stages={ {k:round(v,3) for k,v in d['stage_ms_median'].items()} }  roof={d['roofline']['frac']:.4f}")
except Exception as e:
    print('  parse failed', e); print(open(sys.argv[1]).read()[-2000:])
PY
done
