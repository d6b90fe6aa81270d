mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hogwild.py tests/test_gpu_multirank.py tests/test_gpu_golden.py -x -q > gpurun_out/t_short.txt 2>&1; tail -1 gpurun_out/t_short.txt
timeout 300 python scripts/async_sweep.py w8a > gpurun_out/short_on.jsonl 2>&1
SGDB_HOGWILD_SHORT=0 timeout 300 python scripts/async_sweep.py w8a > gpurun_out/short_off.jsonl 2>&1
timeout 300 python scripts/gpu/bgm.py > gpurun_out/short_loss.jsonl 2>&1
