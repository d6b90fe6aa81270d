# compute-sanitizer evidence (profiles/round2_sanitizer_*.txt): memcheck over the
# GPU parity suites at small sizes (every shipped kernel family is launched by
# them), racecheck + synccheck over the kernels with shared-memory staging and
# cross-warp / cross-CTA hand-offs (sparse full batch, dense full batch and
# persistent epoch, Hogwild block scope, mini-batch chunks).
mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --print-limit 20"
SMALL="tests/test_gpu_sync.py tests/test_gpu_hogwild.py tests/test_gpu_linalg.py tests/test_gpu_exact.py tests/test_gpu_golden.py tests/test_gpu_generator.py"
timeout 2400 $CS --tool memcheck --leak-check no python -m pytest -q -x -p no:cacheprovider $SMALL > gpurun_out/san_memcheck_a.txt 2>&1; echo "memcheck a rc=$?" >> gpurun_out/san_memcheck_a.txt
timeout 1200 $CS --tool memcheck python -m pytest -q -x -p no:cacheprovider tests/test_gpu_segments.py tests/test_gpu_nccl.py tests/test_gpu_multirank.py -k "not more_row_blocks" > gpurun_out/san_memcheck_b.txt 2>&1; echo "memcheck b rc=$?" >> gpurun_out/san_memcheck_b.txt
timeout 1800 $CS --tool racecheck python -m pytest -q -x -p no:cacheprovider tests/test_gpu_segments.py tests/test_gpu_sync.py -k "mixed_pareto or empty_runs or long_rows or (per_epoch_parity and 64)" > gpurun_out/san_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.txt
timeout 1200 $CS --tool synccheck python -m pytest -q -x -p no:cacheprovider tests/test_gpu_segments.py tests/test_gpu_hogwild.py -k "mixed_pareto or block" > gpurun_out/san_synccheck.txt 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_synccheck.txt
for f in gpurun_out/san_*.txt; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|rc=" $f | tail -4; done
