#!/bin/bash
# the ALM's ell = 1 decompositions: time per call and the launch list of one
mkdir -p gpurun_out
O=gpurun_out/r38_ell1.txt
timeout 200 python tools/ell1_probe.py 1 30 > $O 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r38_ell1_launches.csv python tools/ell1_probe.py 1 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r38_ell1_launches.csv 2>/dev/null | head -30 >> $O
cat $O
