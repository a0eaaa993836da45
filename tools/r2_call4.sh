#!/bin/bash
# ALM update A/B, ALM parity, C4 timeline, ncu summaries (reports exported to text, binaries dropped)
mkdir -p gpurun_out
for r in 0 1 50 100; do
  echo "r=$r new: $(ALM_R=$r timeout 120 python tools/alm_update_probe.py 3 2>&1 | tail -1)  legacy: $(CORUTV_ALM_LEGACY=1 ALM_R=$r timeout 120 python tools/alm_update_probe.py 3 2>&1 | tail -1)"
done > gpurun_out/r4_alm_ab.txt 2>&1
for wl in c1 c2; do
  for v in "CORUTV_QRCP_REG_G=1 CORUTV_CHOL_REG_G=1" "CORUTV_QRCP_REG_G=4 CORUTV_CHOL_REG_G=2" "CORUTV_QRCP_LEGACY=1 CORUTV_CHOL_LEGACY=1"; do
    echo "$wl [$v] $(env $v timeout 120 python tools/run_corutv.py $wl 30 2>&1 | tail -20 | sort -n | head -5 | tr '\n' ' ')"
  done
done > gpurun_out/r4_small_ab.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_c2_launches.csv python tools/run_corutv.py c2 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_c1_launches.csv python tools/run_corutv.py c1 2 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_props.py tests/test_gpu_qrcp.py -m gpu -q 2>&1 | tail -8 > gpurun_out/r4_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "c4" 2>&1 | tail -4 >> gpurun_out/r4_tests.log
timeout 300 python tools/rpca_timeline.py > gpurun_out/r4_rpca_timeline.txt 2>&1
prof() {  # name, kernel regex, skip, command...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 600 ncu --set full --clock-control none -k regex:$kre -s $skip -c 1 -o /tmp/$name "$@" > /dev/null 2>&1
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/$name.csv 2>&1
  rm -f /tmp/$name.ncu-rep
}
ALM_R=50 prof r4_alm_ws_r50 alm_update_kernel 3 python tools/alm_update_probe.py 4
prof r4_snorm_fin1 "finalize_kernel<1>" 20 python tools/snorm_probe.py 1
prof r4_snorm_fin0 "finalize_kernel<0>" 20 python tools/snorm_probe.py 1
prof r4_snorm_apply apply_kernel 40 python tools/snorm_probe.py 1
prof r4_snorm_gemm gemm_kernel 20 python tools/snorm_probe.py 1
prof r4_qrcp_reg qrcp_reg_kernel 1 python tools/run_corutv.py c2 2
prof r4_chol_reg chol_reg_kernel 1 python tools/run_corutv.py c2 2
du -sh gpurun_out
