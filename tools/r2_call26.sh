#!/bin/bash
# dual sketch: which side paces it?  kernel time with the y / z products skipped (results wrong, timing only)
mkdir -p gpurun_out
O=gpurun_out/r26_dual.txt
: > $O
for d in 0 1 2 3; do
  echo "--- dbg=$d" >> $O
  CORUTV_DUAL_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:dual_sketch -c 2 python tools/tsr_ncu_target.py 2>&1 | grep -E "duration|bytes_read" >> $O
done
cat $O
