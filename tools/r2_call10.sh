#!/bin/bash
# round-2 measurement pass: whole -m gpu suite, default bench line, C3 launch list, ncu --set full of the C3 sweeps
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/r10_gputest.log
timeout 1200 python bench.py > gpurun_out/r10_bench.json 2> gpurun_out/r10_bench.err
echo "bench rc=$?" >> gpurun_out/r10_gputest.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file /tmp/c3l.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-rpca --no-cpu --no-extra > /dev/null 2>&1
python tools/launch_summary.py /tmp/c3l.csv > gpurun_out/r10_c3_bench_launches_summary.txt
gzip -c /tmp/c3l.csv > gpurun_out/r10_c3_bench_launches.csv.gz
timeout 900 ncu --set full --clock-control none -k regex:gemm_kernel -c 2 -o /tmp/c3full -f python tools/prof_c3.py > /dev/null 2>&1
ncu -i /tmp/c3full.ncu-rep --page details --csv > gpurun_out/r10_c3_gemm_full.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/sn.csv python tools/snorm_probe.py 1 > /dev/null 2>&1
python tools/launch_summary.py /tmp/sn.csv > gpurun_out/r10_snorm_launches.txt
for wl in c1 c2; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/$wl.csv python tools/run_corutv.py $wl 2 > /dev/null 2>&1
  python tools/launch_summary.py /tmp/$wl.csv > gpurun_out/r10_${wl}_launches.txt
done
du -sh gpurun_out
