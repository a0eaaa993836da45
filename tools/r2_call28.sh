#!/bin/bash
# dual sketch (16 warps): ring depth sweep on the kernel alone + the C3-shape probe at the best depths
# variant builds (not kept in the tree): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include -DDUAL_SMAX=<S> -o paper_1906_04572_b200/libcorutv_b200_s<S>.so paper_1906_04572_b200/csrc/corutv_b200.cu
mkdir -p gpurun_out
O=gpurun_out/r28_dual.txt
: > $O
for s in 3 4 5 6 7; do
  lib=paper_1906_04572_b200/libcorutv_b200_s$s.so
  [ $s = 7 ] && lib=""
  echo "--- S=$s" >> $O
  CORUTV_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:dual_sketch -c 2 python tools/tsr_ncu_target.py 2>&1 | grep -E "duration|bytes_read" >> $O
done
for s in 3 4; do
  echo "--- probe S=$s" >> $O
  CORUTV_LIB=paper_1906_04572_b200/libcorutv_b200_s$s.so timeout 300 python tools/tsr_probe.py 2>&1 | head -1 >> $O
done
cat $O
