#!/bin/bash
# 2-rank dry run of the N>1 bench path on one GPU (gloo collectives) + sharded tests
mkdir -p gpurun_out
CORUTV_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e --no-extra > gpurun_out/r18_bench_n2.json 2> gpurun_out/r18_bench_n2.err
echo "n2 rc=$?" > gpurun_out/r18_status.txt
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_nccl.py -m gpu -q 2>&1 | tail -3 >> gpurun_out/r18_status.txt
