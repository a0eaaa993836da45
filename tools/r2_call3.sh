#!/bin/bash
# register QRCP / Cholesky + speculative CholQR schedule: parity, C1/C2 timing A/B, launch lists
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not fullsize and not reference_suite" 2>&1 | tail -25 > gpurun_out/r3_tests.log
for wl in c1 c2; do
  timeout 120 python tools/run_corutv.py $wl 30 > gpurun_out/r3_${wl}_time.log 2>&1
  CORUTV_QRCP_LEGACY=1 CORUTV_CHOL_LEGACY=1 timeout 120 python tools/run_corutv.py $wl 30 > gpurun_out/r3_${wl}_time_legacy.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_${wl}_launches.csv python tools/run_corutv.py $wl 2 > /dev/null 2>&1
done
