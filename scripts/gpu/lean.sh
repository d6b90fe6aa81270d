mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hogwild.py tests/test_gpu_multirank.py tests/test_gpu_golden.py -x -q > gpurun_out/t_lean.txt 2>&1; tail -2 gpurun_out/t_lean.txt
timeout 300 python scripts/async_sweep.py w8a rcv1 realsim > gpurun_out/async_lean.jsonl 2>&1
