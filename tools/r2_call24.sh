#!/bin/bash
# dual sketch v2 after the cursor fix: timing + ncu (full set, source) of the kernel
mkdir -p gpurun_out
O=gpurun_out/r24_dual.txt
: > $O
timeout 600 python -m pytest tests/test_gpu_dual_sketch.py -m gpu -q -x 2>&1 | tail -3 >> $O
echo "--- dual on" >> $O
timeout 300 python tools/tsr_probe.py >> $O 2>&1
timeout 300 python tools/tsr_ncu_target.py >> $O 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dual_sketch -c 4 -o gpurun_out/r24_dual python tools/tsr_ncu_target.py > gpurun_out/r24_ncu.log 2>&1
cat $O
