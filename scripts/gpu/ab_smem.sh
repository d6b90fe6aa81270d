mkdir -p gpurun_out
: > gpurun_out/ab_smem.jsonl
for sm in 1 0; do
  for nt in 1024 512; do
    echo "{\"seg_smem\": $sm, \"threads\": $nt}" >> gpurun_out/ab_smem.jsonl
    SGDB_SEG_SMEM=$sm SGDB_SEG_THREADS=$nt timeout 300 python scripts/sync_sweep.py realsim rcv1 w8a 2>&1 | grep -v '"B": 4096' | cut -c1-330 >> gpurun_out/ab_smem.jsonl
  done
done
