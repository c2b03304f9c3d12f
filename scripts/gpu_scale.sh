#!/bin/bash
# usage: NGPUS="1 2" CONFIGS="c2b c3e4" bash scripts/gpu_scale.sh TAG   -- bench at several GPU counts
TAG=${1:-dev}
mkdir -p gpurun_out
python -m paper_2605_10678_b200.build > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
for cfg in ${CONFIGS:-c2b}; do for n in ${NGPUS:-1 2}; do
  if [ "$n" = "1" ]; then
    timeout 400 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/scale_${TAG}_${cfg}_$n.log 2>&1
  else
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29600+n)) bench.py --gpus $n --config $cfg --steps ${STEPS:-10} --warmup 3 > gpurun_out/scale_${TAG}_${cfg}_$n.log 2>&1
  fi
  python - gpurun_out/scale_${TAG}_${cfg}_$n.log $cfg $n <<'PY'
import json,sys
try:
    line=[l for l in open(sys.argv[1]).read().strip().splitlines() if l.startswith('{')][-1]
    d=json.loads(line); s=d['stage_ms_median']
    print(f"{sys.argv[2]} N={sys.argv[3]}: {d['value']:.3e} pts/s step {d['ms_per_step']:.3f} ms e2e {d['e2e']['value']:.3e} stages { {k:round(v,3) for k,v in s.items()} }")
except Exception as e:
    print(sys.argv[2], sys.argv[3], 'failed', open(sys.argv[1]).read()[-1500:])
PY
done; done
