#!/bin/bash
# end-of-round check: full gpu suite, smoke, default bench (+cpu baseline), reference arm,
# per-config bench lines, then the ncu launch list of the default bench command
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final_build.log 2>&1 || { echo BUILD FAILED; tail -5 gpurun_out/final_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/final_bench.log | cut -c1-600
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/final_ref.log | cut -c1-300
for cfg in c2a c3 c3e4; do
  timeout 400 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/final_$cfg.log 2>&1
  python - gpurun_out/final_$cfg.log $cfg <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['stage_ms_median']
print(f"{sys.argv[2]}: {d['value']:.3e} step {d['ms_per_step']:.3f} ms spread {s['ms_spread']:.3f} interp {s['ms_interp']:.3f} setpts {s['ms_setpts']:.3f} frac {d['roofline']['frac']:.3f}")
PY
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_c2b_r01h.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu.log 2>&1
echo "ncu rc=$?"
