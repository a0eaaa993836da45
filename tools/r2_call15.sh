#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graph.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r15_tests.log
for wl in c1 c2; do
  echo "$wl graph: $(timeout 120 python tools/run_corutv.py $wl 30 2>&1 | tail -20 | sort -n | head -3 | tr '\n' ' ')" >> gpurun_out/r15_ab.txt
  echo "$wl nograph: $(CORUTV_NO_GRAPH=1 timeout 120 python tools/run_corutv.py $wl 30 2>&1 | tail -20 | sort -n | head -3 | tr '\n' ' ')" >> gpurun_out/r15_ab.txt
done
timeout 600 python bench.py --no-e2e --no-rpca --no-cpu --steps 3 --warmup 3 > gpurun_out/r15_bench.json 2> gpurun_out/r15_bench.err
timeout 1200 python -m pytest tests -m gpu -q -x -k "not fullsize and not reference_suite" 2>&1 | tail -5 >> gpurun_out/r15_tests.log
