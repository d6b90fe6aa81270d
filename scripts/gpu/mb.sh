mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_golden.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_mb.txt 2>&1; tail -1 gpurun_out/t_mb.txt
SGDB_NO_EPOCH_GRAPH=1 timeout 300 python scripts/sync_sweep.py w8a rcv1 realsim news20 > gpurun_out/nograph.jsonl 2>&1
timeout 300 python scripts/sync_sweep.py w8a rcv1 realsim news20 > gpurun_out/graph.jsonl 2>&1
