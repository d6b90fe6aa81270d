mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_golden.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_pf.txt 2>&1; tail -1 gpurun_out/t_pf.txt
: > gpurun_out/ab_pf.jsonl
for pf in 1 0; do
  echo "{\"prefetch\": $pf}" >> gpurun_out/ab_pf.jsonl
  for k in 1 2; do
  SGDB_BATCH_PREFETCH=$pf timeout 300 python scripts/sync_sweep.py realsim news20 rcv1 2>&1 | grep '"B": 4096' | cut -c1-200 >> gpurun_out/ab_pf.jsonl
  done
done
