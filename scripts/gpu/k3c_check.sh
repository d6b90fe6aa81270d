mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_segments.py tests/test_gpu_golden.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_k3c.txt 2>&1; tail -3 gpurun_out/t_k3c.txt
timeout 400 python scripts/sync_sweep.py w8a realsim rcv1 news20 > gpurun_out/sync_k3c.jsonl 2>&1
