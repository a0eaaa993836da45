#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/r12_gputest.log
timeout 1200 python bench.py > gpurun_out/r12_bench.json 2> gpurun_out/r12_bench.err
echo "bench rc=$?" >> gpurun_out/r12_gputest.log
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r12_ref.json 2> gpurun_out/r12_ref.err
echo "ref rc=$?" >> gpurun_out/r12_gputest.log
