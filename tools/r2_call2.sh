#!/bin/bash
# C5 oracle record, the reference's own suite through install(), launch lists of C1/C2/mu0
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_reference_suite.py -m gpu -q -s 2>&1 | tail -15 > gpurun_out/r2_refsuite.log
for wl in c1 c2; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_${wl}_launches.csv python tools/run_corutv.py $wl 3 > gpurun_out/r2_${wl}_ncu.log 2>&1
  python tools/launch_summary.py gpurun_out/r2_${wl}_launches.csv > gpurun_out/r2_${wl}_launches.txt 2>&1
  timeout 120 python tools/run_corutv.py $wl 20 > gpurun_out/r2_${wl}_time.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_snorm_launches.csv python tools/snorm_probe.py 1 > gpurun_out/r2_snorm_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r2_snorm_launches.csv > gpurun_out/r2_snorm_launches.txt 2>&1
timeout 1500 python tools/c5_oracle.py > gpurun_out/r2_c5_oracle.log 2>&1
echo c5_rc=$?
