mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hogwild.py tests/test_gpu_exact.py -x -q > gpurun_out/t_hog.txt 2>&1; tail -2 gpurun_out/t_hog.txt
timeout 300 python scripts/async_sweep.py w8a news20 rcv1 realsim > gpurun_out/async_u2.jsonl 2>&1
