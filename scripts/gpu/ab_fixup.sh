mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_segments.py tests/test_gpu_golden.py tests/test_gpu_multirank.py tests/test_gpu_linalg.py -x -q > gpurun_out/t_fx.txt 2>&1; tail -1 gpurun_out/t_fx.txt
SGDB_SEG_SPLIT=1 timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_segments.py -x -q > gpurun_out/t_fx1.txt 2>&1; tail -1 gpurun_out/t_fx1.txt
: > gpurun_out/ab_fx.jsonl
for fx in 1 0; do
  echo "{\"fused_fixup\": $fx}" >> gpurun_out/ab_fx.jsonl
  for k in 1 2; do
  SGDB_SEG_FUSED_FIXUP=$fx timeout 300 python scripts/sync_sweep.py news20 rcv1 2>&1 | grep -v '"B": 4096' | cut -c1-300 >> gpurun_out/ab_fx.jsonl
  done
done
