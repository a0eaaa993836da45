#!/bin/bash
# stream-K partial sweeps for the spectral norm: timing A/B, parity, plan
mkdir -p gpurun_out
echo "streamk: $(timeout 120 python tools/snorm_probe.py 3 2>&1 | tail -2 | tr '\n' ' ')" > gpurun_out/r5_snorm_ab.txt
echo "classic: $(CORUTV_NO_STREAMK=1 timeout 120 python tools/snorm_probe.py 3 2>&1 | tail -2 | tr '\n' ' ')" >> gpurun_out/r5_snorm_ab.txt
CORUTV_DEBUG_PLAN=1 timeout 60 python tools/snorm_probe.py 1 2>&1 | grep "\[corutv\]" | sort | uniq -c | head >> gpurun_out/r5_snorm_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_nccl.py tests/test_gpu_dist.py -m gpu -q 2>&1 | tail -5 > gpurun_out/r5_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "c4" 2>&1 | tail -3 >> gpurun_out/r5_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5_snorm_launches.csv python tools/snorm_probe.py 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r5_snorm_launches.csv > gpurun_out/r5_snorm_launches.txt
rm -f gpurun_out/r5_snorm_launches.csv
