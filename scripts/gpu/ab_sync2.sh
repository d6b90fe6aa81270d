mkdir -p gpurun_out
out=gpurun_out/ab2.jsonl; : > $out
timeout 300 python -m pytest tests/test_gpu_sync.py tests/test_gpu_golden.py -x -q > gpurun_out/t_sync.txt 2>&1; tail -2 gpurun_out/t_sync.txt
for nt in 512 768 1024; do for rl in 16 32; do
  echo "{\"nt\": $nt, \"rl\": $rl}" >> $out
  SGDB_COEF_THREADS=$nt SGDB_ROW_LANES=$rl timeout 120 python scripts/sync_sweep.py rcv1 2>&1 | grep -v '"B": 4096' | cut -c1-330 >> $out
done; done
for cl in 8 16 32; do
  echo "{\"cl\": $cl}" >> $out
  SGDB_COL_LANES=$cl timeout 120 python scripts/sync_sweep.py rcv1 realsim 2>&1 | grep -v '"B": 4096' | cut -c1-330 >> $out
done
