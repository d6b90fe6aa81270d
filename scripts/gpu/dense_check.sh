mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_golden.py -x -q > gpurun_out/t_dense.txt 2>&1; tail -2 gpurun_out/t_dense.txt
timeout 300 python scripts/sync_sweep.py covtype dense1000 > gpurun_out/sync_dense.jsonl 2>&1
