mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 400 python scripts/sync_sweep.py > gpurun_out/sync_sweep_now.jsonl 2> gpurun_out/sync_sweep_now.err
