#!/bin/bash
# dual sketch at ring depth 6: tests, C3-shape probe (one pass vs two sweeps), ncu launch metrics
mkdir -p gpurun_out
O=gpurun_out/r29_dual.txt
: > $O
timeout 600 python -m pytest tests/test_gpu_dual_sketch.py tests/test_gpu_svd.py -m gpu -q 2>&1 | tail -3 >> $O
echo "--- one pass" >> $O
timeout 300 python tools/tsr_probe.py >> $O 2>&1
echo "--- two sweeps" >> $O
CORUTV_DUAL_OFF=1 timeout 300 python tools/tsr_probe.py >> $O 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dual_sketch|gemm_kernel" -c 8 python tools/tsr_ncu_target.py 2>&1 | grep -E "dual_sketch|gemm_kernel|duration|bytes" >> $O
cat $O
