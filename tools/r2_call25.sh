#!/bin/bash
# dual sketch: ring depth 8 vs 5 (bytes in flight) on the kernel alone
# variant builds (not kept in the tree): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include -DDUAL_SMAX=<S> -o paper_1906_04572_b200/libcorutv_b200_s<S>.so paper_1906_04572_b200/csrc/corutv_b200.cu
mkdir -p gpurun_out
O=gpurun_out/r25_dual.txt
: > $O
for lib in "" paper_1906_04572_b200/libcorutv_b200_s5.so; do
  echo "--- lib=$lib" >> $O
  CORUTV_LIB=$lib timeout 300 python tools/tsr_probe.py >> $O 2>&1
  CORUTV_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:dual_sketch -c 4 python tools/tsr_ncu_target.py 2>&1 | grep -E "dual_sketch|duration|bytes_read" >> $O
done
cat $O
