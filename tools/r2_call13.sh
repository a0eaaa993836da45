#!/bin/bash
# one-pass dual sketch for tsr_svd (l <= 16): parity, A/B timing, ncu DRAM bytes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_harness.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -6 > gpurun_out/r13_tests.log
timeout 300 python tools/tsr_probe.py > gpurun_out/r13_tsr.txt 2>&1
CORUTV_DUAL_OFF=1 timeout 300 python tools/tsr_probe.py > gpurun_out/r13_tsr_off.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dual_sketch|gemm_kernel" -c 6 --csv --log-file gpurun_out/r13_tsr_ncu.csv python tools/tsr_probe.py > /dev/null 2>&1
