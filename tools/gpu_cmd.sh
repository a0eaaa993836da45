set -x
python tools/prof_gemm.py 16384 > gpurun_out/prof_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches_gemm.csv python tools/prof_gemm.py 16384 > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -s 4 -c 1 -o gpurun_out/prof_gemm_kk python tools/prof_gemm.py 16384 > gpurun_out/ncu_gemm.log 2>&1
nvidia-smi --help-query-gpu | grep -i -A2 "reasons.active" | head -8 > gpurun_out/smi_help.log
