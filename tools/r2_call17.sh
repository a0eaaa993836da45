#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/r17_gputest.log
timeout 1200 python bench.py > gpurun_out/r17_bench.json 2> gpurun_out/r17_bench.err
echo "bench rc=$?" >> gpurun_out/r17_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r17_gputest.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/c1.csv python tools/run_corutv.py c1 4 > /dev/null 2>&1
python tools/launch_summary.py /tmp/c1.csv > gpurun_out/r17_c1_launches.txt
