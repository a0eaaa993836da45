#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
echo "streamk147: $(timeout 120 python tools/snorm_probe.py 3 2>&1 | tail -2 | tr '\n' ' ')" >> gpurun_out/r6_snorm_ab.txt
echo "classic: $(CORUTV_NO_STREAMK=1 timeout 120 python tools/snorm_probe.py 3 2>&1 | tail -2 | tr '\n' ' ')" >> gpurun_out/r6_snorm_ab.txt
done
