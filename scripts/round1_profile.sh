# HISTORICAL (round 1): the sparse kernels this script captures (csr_coef*, csc_*, apply_partials)
# were replaced in round 2 by K2s / K2w / K3s; scripts/round2_profile.sh is the current recipe.
# ncu evidence for profiles/ (one GPU; never under torchrun). Raw reports land in
# gpurun_out/; scripts/ncu_summary.py turns them into the committed summaries.
set -x
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-convergence --no-extra > gpurun_out/bench_under_ncu.txt 2>&1
$NCU -k regex:hogwild_kernel -s 3 -c 1 -f -o gpurun_out/ncu_hogwild python scripts/prof_targets.py hogwild_w8a 5 > /dev/null 2>&1
$NCU -k regex:dense_full_kernel -s 2 -c 1 -f -o gpurun_out/ncu_c5 python scripts/prof_targets.py sync_c5 3 > /dev/null 2>&1
$NCU -k regex:"csr_coef|csc_|apply_partials" -s 4 -c 4 -f -o gpurun_out/ncu_rcv1 python scripts/prof_targets.py sync_rcv1 3 > /dev/null 2>&1
$NCU -k regex:dense_full_kernel -s 2 -c 1 -f -o gpurun_out/ncu_covtype python scripts/prof_targets.py sync_covtype 3 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
# Summaries on the box (the raw reports are too large to bring back together).
for r in hogwild c5 rcv1 covtype; do python scripts/ncu_summary.py gpurun_out/ncu_$r.ncu-rep > gpurun_out/ncu_${r}_summary.txt 2>&1; done
for r in c5 rcv1 covtype; do rm -f gpurun_out/ncu_$r.ncu-rep; done
du -sh gpurun_out
