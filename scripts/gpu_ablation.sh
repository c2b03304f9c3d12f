#!/bin/bash
# Spread-kernel / tile ablation: every variant on the C2b / C3 / C3e4
# workloads; one JSON line per run under gpurun_out/abl_*.log, summary on stdout.
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_abl.log 2>&1 || { echo BUILD FAILED; exit 1; }
run() {  # cfg tile warps
  timeout 600 python bench.py --config $1 --tile $2 --spread-warps $3 --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > gpurun_out/abl_$1_$2_$3.log 2>&1
  python - gpurun_out/abl_$1_$2_$3.log "$1 T=$2 kernel=$3" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['stage_ms_median']
    print(f"{sys.argv[2]:>24}: step {d['ms_per_step']:8.3f} ms  spread {s['ms_spread']:8.3f}  interp {s['ms_interp']:8.3f}  setpts {s['ms_setpts']:7.3f}")
except Exception as e:
    print(f"{sys.argv[2]:>24}: failed", open(sys.argv[1]).read()[-200:].replace(chr(10),' '))
PY
}
# C2b fp32 w=7: rows / outer need T = 9; plane kernels any T
for k in 1 2; do run c2b 9 $k; done
for t in 6 8 9 10; do for k in 4 8; do run c2b $t $k; done; done
# C3 fp64 w=7
for k in 1 2; do run c3 9 $k; done
for t in 6 8 9; do for k in 4 8; do run c3 $t $k; done; done
# C3e4 fp64 w=5: rows / outer need T = 11
for k in 1 2; do run c3e4 11 $k; done
for t in 6 8 11; do for k in 4 8; do run c3e4 $t $k; done; done
