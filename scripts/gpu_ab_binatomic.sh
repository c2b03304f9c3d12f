mkdir -p gpurun_out
for mode in agg plain; do
  if [ $mode = plain ]; then NUFFT_EXTRA_NVCC_FLAGS=-DNUFFT_PLAIN_BIN_ATOMIC python -m paper_2605_10678_b200.build --force > /dev/null 2>&1; else python -m paper_2605_10678_b200.build --force > /dev/null 2>&1; fi
  for cfg in c2b c3; do
    timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${mode}_$cfg.log 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab_${mode}_$cfg.log').read().strip().splitlines()[-1]); print('$mode $cfg', round(d['ms_per_step'],4), round(d['stage_ms_median']['ms_setpts'],4))"
  done
done
