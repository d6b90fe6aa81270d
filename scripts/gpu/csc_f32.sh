mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_segments.py tests/test_gpu_golden.py -x -q > gpurun_out/t_f32.txt 2>&1; tail -2 gpurun_out/t_f32.txt
timeout 300 python scripts/sync_sweep.py rcv1 realsim > gpurun_out/sync_f32.jsonl 2>&1
SGDB_CSC_F64=1 timeout 300 python scripts/sync_sweep.py rcv1 realsim > gpurun_out/sync_f64.jsonl 2>&1
