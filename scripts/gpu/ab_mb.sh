mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_golden.py tests/test_gpu_linalg.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_mb.txt 2>&1; tail -3 gpurun_out/t_mb.txt
SGDB_BATCH_FUSED=0 timeout 600 python -m pytest tests/test_gpu_sync.py -x -q > gpurun_out/t_mb0.txt 2>&1; tail -1 gpurun_out/t_mb0.txt
: > gpurun_out/ab_mb.jsonl
for f in 1 0; do
echo "fused $f" >> gpurun_out/ab_mb.jsonl
SGDB_BATCH_FUSED=$f timeout 300 python scripts/sync_sweep.py realsim news20 rcv1 w8a 2>&1 | grep '"B": 4096' | cut -c1-250 >> gpurun_out/ab_mb.jsonl
done
