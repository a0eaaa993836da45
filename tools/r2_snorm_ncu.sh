#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:finalize_kernel -s 20 -c 2 -o gpurun_out/r2_snorm_fin python tools/snorm_probe.py 1 > gpurun_out/r2_snorm_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_kernel -s 40 -c 2 -o gpurun_out/r2_snorm_apply python tools/snorm_probe.py 1 >> gpurun_out/r2_snorm_ncu2.log 2>&1
