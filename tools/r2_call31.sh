#!/bin/bash
# spectral norm with the deferred CholeskyQR on the side stream: parity tests + A/B timing
mkdir -p gpurun_out
O=gpurun_out/r31_snorm.txt
: > $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py -m gpu -q -k "spectral or snorm or alm or rpca" 2>&1 | tail -5 >> $O
echo "--- deferred" >> $O
timeout 200 python tools/snorm_probe.py 4 >> $O 2>&1
echo "--- CORUTV_SNORM_DEFER=0" >> $O
CORUTV_SNORM_DEFER=0 timeout 200 python tools/snorm_probe.py 4 >> $O 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k c4 2>&1 | tail -3 >> $O
cat $O
