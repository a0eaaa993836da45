python tools/c4_iter0.py > gpurun_out/c4_iter0.log 2>&1
python tools/c4_parity.py > gpurun_out/c4_parity.log 2>&1
