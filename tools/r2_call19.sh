#!/bin/bash
# randomised stress of the round-2 build against the oracle
mkdir -p gpurun_out
timeout 400 python tools/stress.py 240 > gpurun_out/r19_stress.log 2>&1
timeout 400 python tools/stress2.py 240 > gpurun_out/r19_stress2.log 2>&1
timeout 300 python tools/stress3.py 150 > gpurun_out/r19_stress3.log 2>&1
tail -3 gpurun_out/r19_stress.log gpurun_out/r19_stress2.log gpurun_out/r19_stress3.log
