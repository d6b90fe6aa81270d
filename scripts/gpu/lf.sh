mkdir -p gpurun_out
: > gpurun_out/lf.jsonl
SGDB_DENSE_LF416=1 timeout 300 python -m pytest tests/test_gpu_sync.py -x -q -k "dense" > gpurun_out/t_lf.txt 2>&1; tail -1 gpurun_out/t_lf.txt
for v in 0 1; do echo "{\"lf416\": $v}" >> gpurun_out/lf.jsonl; SGDB_DENSE_LF416=$v timeout 300 python scripts/sync_sweep.py covtype >> gpurun_out/lf.jsonl 2>&1; done
