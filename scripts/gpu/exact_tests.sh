mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_exact.py tests/test_gpu_hogwild.py -x -q > gpurun_out/t_exact.txt 2>&1; tail -3 gpurun_out/t_exact.txt
