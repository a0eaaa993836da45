#!/bin/bash
# fused spectral-norm sweeps: A/B timing, parity, launch list
mkdir -p gpurun_out
for i in 1 2; do
echo "fused: $(timeout 120 python tools/snorm_probe.py 3 2>&1 | tail -1)" >> gpurun_out/r9_ab.txt
echo "unfused: $(CORUTV_SNORM_UNFUSED=1 timeout 120 python tools/snorm_probe.py 3 2>&1 | tail -1)" >> gpurun_out/r9_ab.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_nccl.py tests/test_gpu_dist.py -m gpu -q 2>&1 | tail -5 > gpurun_out/r9_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "c4" 2>&1 | tail -3 >> gpurun_out/r9_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l.csv python tools/snorm_probe.py 1 > /dev/null 2>&1
python tools/launch_summary.py /tmp/l.csv | head -8 >> gpurun_out/r9_ab.txt
