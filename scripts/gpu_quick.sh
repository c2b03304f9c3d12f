#!/bin/bash
# parity (single GPU) + C2b / C3 stage times
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_q.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py tests/test_pif_gpu.py -m gpu -x -q > gpurun_out/q_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/q_tests.log
for cfg in ${CONFIGS:-c2b c3}; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_$cfg.log 2>&1
  python - gpurun_out/q_$cfg.log $cfg <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['stage_ms_median']
print(f"{sys.argv[2]}: {d['value']:.3e} step {d['ms_per_step']:.3f} ms", {k: round(v, 4) for k, v in s.items()})
PY
done
