mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_k3c.txt 2>&1; tail -2 gpurun_out/t_k3c.txt
: > gpurun_out/k3c_ab.jsonl
for v in f64 f32; do
  echo "{\"variant\": \"$v\"}" >> gpurun_out/k3c_ab.jsonl
  if [ $v = f32 ]; then export SGDB_EPOCH_F32G=1; else unset SGDB_EPOCH_F32G; fi
  timeout 300 python scripts/sync_sweep.py w8a realsim rcv1 news20 2>&1 | grep '"B": 4096' >> gpurun_out/k3c_ab.jsonl
done
