mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hogwild.py tests/test_gpu_golden.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_hog.txt 2>&1; tail -3 gpurun_out/t_hog.txt
timeout 300 python scripts/async_sweep.py w8a rcv1 news20 realsim > gpurun_out/async_chunk.jsonl 2>&1
SGDB_HOGWILD_CHUNK=0 timeout 300 python scripts/async_sweep.py w8a > gpurun_out/async_nochunk.jsonl 2>&1
