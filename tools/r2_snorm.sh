#!/bin/bash
# round-2 spectral-norm check: parity tests, timing, launch list
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "spectral or alm" 2>&1 | tail -15 > gpurun_out/r2_snorm_tests.log
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "c4" 2>&1 | tail -5 >> gpurun_out/r2_snorm_tests.log
timeout 120 python tools/snorm_probe.py 3 > gpurun_out/r2_snorm_fused.log 2>&1
CORUTV_SNORM_LEGACY=1 timeout 120 python tools/snorm_probe.py 2 > gpurun_out/r2_snorm_legacy.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_snorm_launches.csv python tools/snorm_probe.py 1 > gpurun_out/r2_snorm_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r2_snorm_launches.csv > gpurun_out/r2_snorm_launches.txt 2>&1
