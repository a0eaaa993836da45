#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
echo "minb2: $(timeout 120 python tools/snorm_probe.py 3 2>&1 | tail -1)" >> gpurun_out/r7_ab.txt
echo "minb1: $(CORUTV_GEMM_MINB=1 timeout 120 python tools/snorm_probe.py 3 2>&1 | tail -1)" >> gpurun_out/r7_ab.txt
done
for wl in c1 c2; do
echo "$wl minb2: $(timeout 120 python tools/run_corutv.py $wl 30 2>&1 | tail -20 | sort -n | head -3 | tr '\n' ' ')" >> gpurun_out/r7_ab.txt
echo "$wl minb1: $(CORUTV_GEMM_MINB=1 timeout 120 python tools/run_corutv.py $wl 30 2>&1 | tail -20 | sort -n | head -3 | tr '\n' ' ')" >> gpurun_out/r7_ab.txt
done
CORUTV_DEBUG_PLAN=1 timeout 60 python tools/snorm_probe.py 1 2>&1 | grep "\[corutv\]" | sort | uniq -c | head -4 >> gpurun_out/r7_ab.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l.csv python tools/snorm_probe.py 1 > /dev/null 2>&1
python tools/launch_summary.py /tmp/l.csv | head -8 >> gpurun_out/r7_ab.txt
