# clustered-points stress case (same-address setpts atomics)
mkdir -p gpurun_out
for cfg in c3e4 c4n; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/r3m_$cfg.json 2>gpurun_out/r3m_$cfg.err
  timeout 900 python bench.py --config $cfg --points clustered --steps 5 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/r3m_${cfg}_clustered.json 2>gpurun_out/r3m_${cfg}_clustered.err
done
