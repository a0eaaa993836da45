#!/bin/bash
mkdir -p gpurun_out
CORUTV_DEBUG_GRAPH=1 timeout 120 python tools/run_corutv.py c1 4 > gpurun_out/r16_dbg.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r16_tests.log
for wl in c1 c2; do
  echo "$wl graph: $(timeout 120 python tools/run_corutv.py $wl 30 2>&1 | tail -20 | sort -n | head -3 | tr '\n' ' ')" >> gpurun_out/r16_ab.txt
  echo "$wl nograph: $(CORUTV_NO_GRAPH=1 timeout 120 python tools/run_corutv.py $wl 30 2>&1 | tail -20 | sort -n | head -3 | tr '\n' ' ')" >> gpurun_out/r16_ab.txt
done
timeout 600 python bench.py --no-e2e --no-rpca --no-cpu --steps 3 --warmup 3 > gpurun_out/r16_bench.json 2> gpurun_out/r16_bench.err
