#!/bin/bash
# KK operand row map (conflict-free quarter-warp LDS.128) as a variant build: correctness + A/B
# variant build: the default build is the row-mapped one now; -DKK_RHO=0 gives the old fragment rows (then swap the two lib paths below)
mkdir -p gpurun_out
O=gpurun_out/r36_rho.txt
: > $O
V=paper_1906_04572_b200/libcorutv_b200_rho.so
CORUTV_LIB=$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_svd.py tests/test_gpu_large_ell.py -m gpu -q -x 2>&1 | tail -3 >> $O
for lib in "" $V; do
  echo "--- lib=$lib" >> $O
  CORUTV_LIB=$lib timeout 200 python tools/snorm_probe.py 3 2>&1 | tail -2 >> $O
  for r in 20 50; do echo "alm r=$r $(ALM_R=$r CORUTV_LIB=$lib timeout 120 python tools/alm_update_probe.py 2>&1 | tail -1)" >> $O; done
  CORUTV_LIB=$lib timeout 600 python bench.py --no-e2e --no-rpca --no-cpu --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['ms_per_step'], d['roofline']['frac'], {k:v['ms_per_step'] for k,v in d.get('workloads',{}).items()})" >> $O
done
CORUTV_LIB=$V timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:gemm_kernel --launch-skip 20 -c 2 python tools/snorm_probe.py 1 2>&1 | grep -E "gemm_kernel|duration|shared" >> $O
cat $O
