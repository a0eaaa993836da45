#!/bin/bash
# round-2 re-entry check: box facts, the whole -m gpu suite, the default bench line
mkdir -p gpurun_out
(nvidia-smi; free -g; nproc) > gpurun_out/r2_box.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -40 > gpurun_out/r2_gputest.log
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo bench_rc=$?
tail -3 gpurun_out/r2_gputest.log
