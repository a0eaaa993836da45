#!/bin/bash
# ALM update: 3-stage TMA ring for the rank-r product (build variant) vs the 2-stage default
# variant build: as the default build command with LR_STAGES = 3 in csrc/gemm.cuh -> libcorutv_b200_lr3.so
mkdir -p gpurun_out
O=gpurun_out/r34_alm.txt
: > $O
for r in 1 20 50; do
  for lib in "" paper_1906_04572_b200/libcorutv_b200_lr3.so; do
    echo "r=$r lib=$lib: $(ALM_R=$r CORUTV_LIB=$lib timeout 120 python tools/alm_update_probe.py 2>&1 | tail -1) $(ALM_R=$r CORUTV_LIB=$lib timeout 120 python tools/alm_update_probe.py 2>&1 | tail -1)" >> $O
  done
done
cat $O
