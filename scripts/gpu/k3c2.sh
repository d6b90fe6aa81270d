mkdir -p gpurun_out
SGDB_SPARSE_EPOCH=1 timeout 600 python -m pytest tests/test_gpu_sync.py -x -q > gpurun_out/t_k3c2.txt 2>&1; tail -1 gpurun_out/t_k3c2.txt
SGDB_SPARSE_EPOCH=1 timeout 300 python scripts/sync_sweep.py w8a rcv1 realsim news20 > gpurun_out/k3c2.jsonl 2>&1
