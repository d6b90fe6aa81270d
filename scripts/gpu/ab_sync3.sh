mkdir -p gpurun_out
out=gpurun_out/ab3.jsonl; : > $out
for nt in 768 1024; do for rl in 4 8; do
  echo "{\"k2s_nt\": $nt, \"rl\": $rl, \"cl\": $rl}" >> $out
  SGDB_SEG=0 SGDB_COEF_THREADS=$nt SGDB_ROW_LANES=$rl SGDB_COL_LANES=$rl timeout 120 python scripts/sync_sweep.py rcv1 realsim news20 2>&1 | grep -v '"B": 4096' | cut -c1-330 >> $out
done; done
