set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gputest3.log
python tools/debug_gpu.py 2>&1 | tail -8 > gpurun_out/debug3.log
python bench.py --steps 3 --warmup 2 --no-rpca --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c3b.log
python bench.py --workload c2 --steps 10 --warmup 3 --no-rpca --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c2b.log
