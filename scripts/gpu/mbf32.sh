mkdir -p gpurun_out
SGDB_MB_F32=1 timeout 600 python -m pytest tests/test_gpu_sync.py -x -q > gpurun_out/t_mbf32.txt 2>&1; tail -1 gpurun_out/t_mbf32.txt
SGDB_MB_F32=1 timeout 300 python scripts/sync_sweep.py w8a rcv1 realsim news20 > gpurun_out/graph_f32.jsonl 2>&1
