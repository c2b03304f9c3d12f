#!/bin/bash
# the paper's spread / interp variants against the default kernels.
# Parity tests first, then C2b and C3 with (spread_warps, interp_method) =
#   default (0,0) | Atomic caller order (-1,1) | Atomic / Direct bin-sorted (-2,2).
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_var.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "ablation or precomputed" > gpurun_out/var_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/var_tests.log
for cfg in ${CONFIGS:-c2b c3}; do
  for v in "0 0" "-1 1" "-2 2" "8 0"; do
    set -- $v
    timeout 600 python bench.py --config $cfg --spread-warps $1 --interp-method $2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/var_${cfg}_$1_$2.log 2>&1
    python - gpurun_out/var_${cfg}_$1_$2.log "$cfg sw=$1 im=$2" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['stage_ms_median']
    print(f"{sys.argv[2]:>18}: {d['value']:.3e} pts/s step {d['ms_per_step']:.3f} ms spread {s['ms_spread']:.3f} interp {s['ms_interp']:.3f} setpts {s['ms_setpts']:.3f} fft {s['ms_fft']:.3f}")
except Exception as e:
    print(sys.argv[2], 'failed', open(sys.argv[1]).read()[-400:])
PY
  done
done
