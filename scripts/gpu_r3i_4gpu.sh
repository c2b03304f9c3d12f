# 4 B200 after the setpts L2-policy change: slab checks + C4 bench over NCCL + the 2-GPU pytest
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tests/dist_check.py > gpurun_out/r3i_dist_check.log 2>&1
echo "dist_check rc=$?" >> gpurun_out/r3i_dist_check.log
timeout 900 python -m pytest tests/test_dist_gpu.py -m gpu -q > gpurun_out/r3i_dist_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r3i_dist_tests.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r3i_bench2.json 2> gpurun_out/r3i_bench2.err
echo "bench2 rc=$?" >> gpurun_out/r3i_bench2.err
