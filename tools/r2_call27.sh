#!/bin/bash
# dual sketch (16 warps): ring depth 7 vs 4 on the kernel alone, with and without the products
# variant builds (not kept in the tree): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include -DDUAL_SMAX=<S> -o paper_1906_04572_b200/libcorutv_b200_s<S>.so paper_1906_04572_b200/csrc/corutv_b200.cu
mkdir -p gpurun_out
O=gpurun_out/r27_dual.txt
: > $O
for lib in "" paper_1906_04572_b200/libcorutv_b200_s4.so; do
  for d in 0 3; do
    echo "--- lib=$lib dbg=$d" >> $O
    CORUTV_LIB=$lib CORUTV_DUAL_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dual_sketch -c 2 python tools/tsr_ncu_target.py 2>&1 | grep -E "duration" >> $O
  done
done
cat $O
