python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gputest14.log
python tools/debug_gpu.py 2>&1 | tail -6 > gpurun_out/debug5.log
python bench.py > gpurun_out/bench_full2.log 2>&1
python tools/c4_parity.py > gpurun_out/c4_parity.log 2>&1
