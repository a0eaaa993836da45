#!/bin/bash
# final round-2 profile pass: ALM update ncu (r = 50 and r = 0), C4 launch list, reference arm line
mkdir -p gpurun_out
ALM_R=50 timeout 300 python tools/alm_update_probe.py > gpurun_out/r30_alm_r50.txt 2>&1
ALM_R=0 timeout 300 python tools/alm_update_probe.py > gpurun_out/r30_alm_r0.txt 2>&1
ALM_R=50 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lowrank_kernel -c 1 -o gpurun_out/r30_alm_r50 -f python tools/alm_update_probe.py 1 > gpurun_out/r30_ncu_alm.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r30_c4_launches.csv python tools/run_rpca.py > gpurun_out/r30_ncu_c4.log 2>&1
