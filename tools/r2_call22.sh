#!/bin/bash
# ALM update: constant-divisor division (div_const) + trimmed last k tile; A/B and the bitwise division test
mkdir -p gpurun_out
O=gpurun_out/r22_alm.txt
: > $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "alm_update or lowrank" 2>&1 | tail -5 >> $O
for r in 0 1 20 40 50; do
  echo "r=$r new:        $(ALM_R=$r timeout 120 python tools/alm_update_probe.py 2>&1 | tail -1)" >> $O
  echo "r=$r plain div:  $(ALM_R=$r CORUTV_ALM_PLAIN_DIV=1 timeout 120 python tools/alm_update_probe.py 2>&1 | tail -1)" >> $O
  echo "r=$r full k:     $(ALM_R=$r CORUTV_LR_FULLK=1 timeout 120 python tools/alm_update_probe.py 2>&1 | tail -1)" >> $O
  echo "r=$r both old:   $(ALM_R=$r CORUTV_LR_FULLK=1 CORUTV_ALM_PLAIN_DIV=1 timeout 120 python tools/alm_update_probe.py 2>&1 | tail -1)" >> $O
done
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k c4 2>&1 | tail -2 >> $O
cat $O
