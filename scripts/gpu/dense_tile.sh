mkdir -p gpurun_out
: > gpurun_out/dense_tile.jsonl
for t in 16384 32768 49152 65536 98304; do
  echo "{\"tile\": $t}" >> gpurun_out/dense_tile.jsonl
  SGDB_DENSE_TILE=$t timeout 300 python scripts/sync_sweep.py covtype dense1000 2>&1 | grep -v '"B": 4096' >> gpurun_out/dense_tile.jsonl
done
