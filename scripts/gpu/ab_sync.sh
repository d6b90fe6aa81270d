mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sync.py tests/test_gpu_golden.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_sync.txt 2>&1; tail -2 gpurun_out/t_sync.txt
timeout 300 python scripts/sync_sweep.py rcv1 realsim w8a news20 > gpurun_out/sweep_new.jsonl 2>&1
SGDB_CSC_VEC=0 timeout 300 python scripts/sync_sweep.py rcv1 realsim w8a news20 > gpurun_out/sweep_oldcsc.jsonl 2>&1
