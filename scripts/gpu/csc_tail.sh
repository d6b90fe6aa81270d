mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_segments.py tests/test_gpu_golden.py tests/test_gpu_multirank.py tests/test_gpu_linalg.py -x -q > gpurun_out/t_tail.txt 2>&1; tail -2 gpurun_out/t_tail.txt
timeout 300 python scripts/sync_sweep.py realsim rcv1 news20 w8a > gpurun_out/sync_tail.jsonl 2>&1
