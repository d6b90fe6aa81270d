mkdir -p gpurun_out
out=gpurun_out/ab_seg.jsonl; : > $out
timeout 300 python -m pytest tests/test_gpu_segments.py tests/test_gpu_sync.py tests/test_gpu_golden.py -x -q > gpurun_out/t_seg.txt 2>&1; tail -5 gpurun_out/t_seg.txt
for nt in 512 768 1024; do
  echo "{\"nt\": $nt}" >> $out
  SGDB_SEG_THREADS=$nt timeout 200 python scripts/sync_sweep.py rcv1 realsim w8a news20 2>&1 | grep -v '"B": 4096' | cut -c1-330 >> $out
done
