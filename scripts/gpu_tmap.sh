#!/bin/bash
# TMA tensor-map interp staging: parity tests, then C2b / C3 / C3e4 with and without
# the map (NUFFT_NO_TMAP=1 keeps the per-row bulk copies).
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_tmap.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py tests/test_pif_gpu.py -m gpu -x -q > gpurun_out/tmap_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tmap_tests.log
for cfg in c2b c3 c3e4 c2a; do
  for mode in tmap rows; do
    if [ $mode = rows ]; then export NUFFT_NO_TMAP=1; else unset NUFFT_NO_TMAP; fi
    timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tm_${cfg}_${mode}.log 2>&1
    python - gpurun_out/tm_${cfg}_${mode}.log "$cfg $mode" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['stage_ms_median']
    print(f"{sys.argv[2]:>12}: {d['value']:.3e} step {d['ms_per_step']:.3f} ms spread {s['ms_spread']:.3f} interp {s['ms_interp']:.3f} setpts {s['ms_setpts']:.3f}")
except Exception as e:
    print(sys.argv[2], 'failed', open(sys.argv[1]).read()[-400:])
PY
  done
done
unset NUFFT_NO_TMAP
