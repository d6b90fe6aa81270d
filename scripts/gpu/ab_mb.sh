mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_golden.py tests/test_gpu_linalg.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_mb.txt 2>&1; tail -3 gpurun_out/t_mb.txt
: > gpurun_out/ab_mb.jsonl
for ch in 1 0; do
echo "chunks $ch" >> gpurun_out/ab_mb.jsonl
SGDB_BATCH_CHUNKS=$ch timeout 300 python scripts/sync_sweep.py realsim news20 rcv1 w8a 2>&1 | grep '"B": 4096' | cut -c1-250 >> gpurun_out/ab_mb.jsonl
done
