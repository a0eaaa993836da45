#!/bin/bash
# final-build stress pass (randomised vs the oracle) + the new strided dual-sketch test
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dual_sketch.py -m gpu -q 2>&1 | tail -2 > gpurun_out/r35_tests.txt
timeout 400 python tools/stress.py 180 > gpurun_out/r35_stress.log 2>&1
timeout 400 python tools/stress2.py 180 > gpurun_out/r35_stress2.log 2>&1
timeout 300 python tools/stress3.py 120 > gpurun_out/r35_stress3.log 2>&1
cat gpurun_out/r35_tests.txt; tail -2 gpurun_out/r35_stress.log; tail -2 gpurun_out/r35_stress2.log; tail -2 gpurun_out/r35_stress3.log
