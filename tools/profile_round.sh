#!/bin/bash
# Round profiling recipe (run on the GPU box from the repo root):
#   1. the bench command alone (must exit 0)
#   2. its ncu launch list (gpu__time_duration, clocks not locked)
#   3. ncu --set full of the two C3 A-sweep GEMM launches (KK, MM)
set -e
R=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-e2e --no-rpca --no-cpu > gpurun_out/${R}_bench_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file gpurun_out/${R}_c3_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-rpca --no-cpu > gpurun_out/${R}_ncu_launches.log 2>&1
python tools/prof_c3.py > gpurun_out/${R}_prof_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 2 \
    -o gpurun_out/${R}_c3_gemm_full -f python tools/prof_c3.py > gpurun_out/${R}_ncu_full.log 2>&1
