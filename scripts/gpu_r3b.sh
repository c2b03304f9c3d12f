# row-block interpolation, ILP fix: parity subset + C4 / C3e4 timing + one ncu capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_real_gpu.py tests/test_pif_gpu.py -m gpu -q -x > gpurun_out/r3b_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r3b_tests.log
for cfg in c4n c3e4; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3b_$cfg.json 2>gpurun_out/r3b_$cfg.err
done
CONFIG=c3e4 PROFILE="interp_subr" COUNT=1 bash scripts/gpu_profile_cfg.sh r3b
