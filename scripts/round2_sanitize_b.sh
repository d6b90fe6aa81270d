# compute-sanitizer over the round-2 kernels (full-batch sparse K2s/K3s with PDL and the
# arrival-wait apply, direct-update mini-batch steps, NCCL path, multi-rank hook).
mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --print-limit 20"
timeout 1500 $CS --tool memcheck python -m pytest -q -x -p no:cacheprovider tests/test_gpu_segments.py tests/test_gpu_nccl.py tests/test_gpu_multirank.py tests/test_gpu_sync.py -k "not more_row_blocks" > gpurun_out/san_memcheck_b.txt 2>&1; echo "memcheck b rc=$?" >> gpurun_out/san_memcheck_b.txt
timeout 1200 $CS --tool racecheck python -m pytest -q -x -p no:cacheprovider tests/test_gpu_segments.py -k "mixed_pareto or empty_runs or long_rows or many_short" > gpurun_out/san_racecheck_b.txt 2>&1; echo "racecheck b rc=$?" >> gpurun_out/san_racecheck_b.txt
timeout 1200 $CS --tool synccheck python -m pytest -q -x -p no:cacheprovider tests/test_gpu_segments.py tests/test_gpu_sync.py -k "mixed_pareto or one_slot or (per_epoch_parity and sparse)" > gpurun_out/san_synccheck_b.txt 2>&1; echo "synccheck b rc=$?" >> gpurun_out/san_synccheck_b.txt
for f in gpurun_out/san_*.txt; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
