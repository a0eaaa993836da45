#!/bin/bash
# one-pass dual sketch v2 (all warps feed both products from their own rows): parity + A/B timing
mkdir -p gpurun_out
O=gpurun_out/r23_dual.txt
: > $O
timeout 600 python -m pytest tests/test_gpu_dual_sketch.py -m gpu -q -x 2>&1 | tail -15 >> $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "alm_update" 2>&1 | tail -4 >> $O
echo "--- dual on" >> $O
timeout 300 python tools/tsr_probe.py >> $O 2>&1
echo "--- dual off" >> $O
CORUTV_DUAL_OFF=1 timeout 300 python tools/tsr_probe.py >> $O 2>&1
cat $O
