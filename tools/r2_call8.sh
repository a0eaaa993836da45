#!/bin/bash
# source-level ncu of the latency kernels (stall reasons per line), exported to CSV
mkdir -p gpurun_out
src() {  # name, kernel regex, skip, command...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$kre -s $skip -c 1 -o /tmp/$name "$@" > /dev/null 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$name.src.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/$name.csv 2>&1
  rm -f /tmp/$name.ncu-rep
}
src r8_chol_reg chol_reg_kernel 1 python tools/run_corutv.py c1 2
src r8_fin1 "finalize_kernel<1>" 20 python tools/snorm_probe.py 1
src r8_apply apply_kernel 40 python tools/snorm_probe.py 1
src r8_qrcp_reg qrcp_reg_kernel 1 python tools/run_corutv.py c2 2
ls -la gpurun_out/ | tail
du -sh gpurun_out
