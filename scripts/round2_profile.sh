# ncu evidence for profiles/ (one GPU; never under torchrun). Raw reports land in
# gpurun_out/; scripts/ncu_summary.py turns them into the committed summaries.
set -x
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
# Launch list of the bench command itself (cold-cache, serialised: shares, not absolutes).
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu --no-convergence --no-extra > gpurun_out/bench_under_ncu.txt 2>&1
# Full captures of the headline kernels (rcv1 B = N) and the others named in DESIGN.md.
# (models that fit in SMEM run both passes in one launch: glued_step_kernel = K23g)
$NCU -k regex:"glued_step|k2s_margin|blocked_pass" -s 1 -c 1 -f -o gpurun_out/ncu_rcv1 python scripts/prof_targets.py sync_rcv1 3 > /dev/null 2>&1
$NCU -k regex:"glued_step|k2s_margin|blocked_pass" -s 1 -c 1 -f -o gpurun_out/ncu_realsim python scripts/prof_targets.py sync_realsim 3 > /dev/null 2>&1
$NCU -k regex:"k2s_margin|blocked_pass" -s 2 -c 2 -f -o gpurun_out/ncu_news20 python scripts/prof_targets.py sync_news20 3 > /dev/null 2>&1
for r in rcv1 realsim news20; do python scripts/ncu_summary.py gpurun_out/ncu_$r.ncu-rep > gpurun_out/ncu_${r}_summary.txt 2>&1; done
ls -la gpurun_out
