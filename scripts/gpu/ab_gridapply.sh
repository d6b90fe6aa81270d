mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_segments.py tests/test_gpu_golden.py tests/test_gpu_multirank.py tests/test_gpu_linalg.py -x -q > gpurun_out/t_ga.txt 2>&1; tail -2 gpurun_out/t_ga.txt
for m in 1 2 0; do SGDB_CSC=$m timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_segments.py -x -q > gpurun_out/t_ga$m.txt 2>&1; tail -1 gpurun_out/t_ga$m.txt; done
: > gpurun_out/ab_ga.jsonl
for ga in 1 0; do
  echo "{\"grid_apply\": $ga}" >> gpurun_out/ab_ga.jsonl
  for k in 1 2; do
  SGDB_CSC_GRID_APPLY=$ga timeout 300 python scripts/sync_sweep.py realsim rcv1 2>&1 | grep -v '"B": 4096' | cut -c1-300 >> gpurun_out/ab_ga.jsonl
  done
done
