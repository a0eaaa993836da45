#!/bin/bash
# ALM update: 128 x 32 tiles at 3 CTAs/SM vs round 1's 128 x 64 at 2
mkdir -p gpurun_out
for r in 0 1 20 50; do
  echo "r=$r J2x3: $(ALM_R=$r timeout 120 python tools/alm_update_probe.py 3 2>&1 | tail -1)  J4x2: $(CORUTV_ALM_J=4 ALM_R=$r timeout 120 python tools/alm_update_probe.py 3 2>&1 | tail -1)"
done > gpurun_out/r11_alm_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_props.py tests/test_gpu_dist.py tests/test_gpu_large_ell.py -m gpu -q 2>&1 | tail -4 > gpurun_out/r11_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "c4" 2>&1 | tail -3 >> gpurun_out/r11_tests.log
timeout 300 python tools/rpca_timeline.py > gpurun_out/r11_rpca_timeline.txt 2>&1
ALM_R=50 timeout 600 ncu --set full --clock-control none -k regex:lowrank_kernel -s 3 -c 1 -o /tmp/alm python tools/alm_update_probe.py 4 > /dev/null 2>&1
ncu -i /tmp/alm.ncu-rep --page details --csv > gpurun_out/r11_alm_r50_ncu.csv 2>&1
for wl in c1 c2; do
  echo "$wl cta: $(timeout 120 python tools/run_corutv.py $wl 30 2>&1 | tail -20 | sort -n | head -3 | tr '\n' ' ')" >> gpurun_out/r11_c12_ab.txt
  echo "$wl nocta: $(CORUTV_CHOLQR_CTA_OFF=1 timeout 120 python tools/run_corutv.py $wl 30 2>&1 | tail -20 | sort -n | head -3 | tr '\n' ' ')" >> gpurun_out/r11_c12_ab.txt
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/c1.csv python tools/run_corutv.py c1 2 > /dev/null 2>&1
python tools/launch_summary.py /tmp/c1.csv > gpurun_out/r11_c1_launches.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_svd.py tests/test_gpu_harness.py tests/test_gpu_ialm.py -m gpu -q 2>&1 | tail -4 >> gpurun_out/r11_tests.log
