#!/bin/bash
mkdir -p gpurun_out
CORUTV_SNORM_DEBUG=1 timeout 120 python tools/snorm_probe.py 2 2>&1 | grep "prof" > gpurun_out/r21_prof.txt
timeout 120 python tools/snorm_probe.py 3 >> gpurun_out/r21_prof.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_dist.py tests/test_gpu_nccl.py -m gpu -q 2>&1 | tail -3 >> gpurun_out/r21_prof.txt
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k c4 2>&1 | tail -2 >> gpurun_out/r21_prof.txt
