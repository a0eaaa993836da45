python -m pytest tests/test_gpu_parity.py -m gpu -q -k "lowrank_store or alm_update_matches" 2>&1 | tail -30 > gpurun_out/gputest16.log
