#!/bin/bash
# spectral norm: row kernels (finalize) on 256 CTAs instead of one per SM
mkdir -p gpurun_out
O=gpurun_out/r37_snorm.txt
: > $O
for c in 0 256 200; do
  echo "--- CORUTV_SNORM_CTAS=$c" >> $O
  CORUTV_SNORM_CTAS=$c timeout 200 python tools/snorm_probe.py 4 2>&1 | tail -3 >> $O
done
cat $O
