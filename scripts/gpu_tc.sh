#!/bin/bash
# tensor-core spread (spread_warps = 3): parity, then C2b / C2a / C3-f32 timing vs the default
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_tc.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "every_spread_kernel" > gpurun_out/tc_tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/tc_tests.log
for cfg in ${CONFIGS:-c2b c2a}; do
  for sw in 0 3; do
    timeout 300 python bench.py --config $cfg --spread-warps $sw --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tc_${cfg}_$sw.log 2>&1
    python - gpurun_out/tc_${cfg}_$sw.log "$cfg sw=$sw" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['stage_ms_median']
    print(f"{sys.argv[2]:>12}: {d['value']:.3e} step {d['ms_per_step']:.3f} ms spread {s['ms_spread']:.3f} interp {s['ms_interp']:.3f}")
except Exception as e:
    print(sys.argv[2], 'failed', open(sys.argv[1]).read()[-600:])
PY
  done
done
