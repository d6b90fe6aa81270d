mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hogwild.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_hog.txt 2>&1; tail -2 gpurun_out/t_hog.txt
timeout 300 python scripts/async_sweep.py rcv1 realsim news20 > gpurun_out/async_k6c.jsonl 2>&1
SGDB_HOGWILD_CHUNK=0 timeout 300 python scripts/async_sweep.py rcv1 > gpurun_out/async_k6.jsonl 2>&1
