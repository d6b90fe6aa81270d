# ncu --set full of the kernels DESIGN.md names outside the headline (one capture each).
set -x
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:dense_epoch_kernel -s 1 -c 1 -f -o gpurun_out/ncu_k1c python scripts/prof_targets.py minibatch_covtype 2 > /dev/null 2>&1
$NCU -k regex:"mb_margin|mb_scatter" -s 40 -c 2 -f -o gpurun_out/ncu_k3c python scripts/prof_targets.py minibatch_rcv1 2 > /dev/null 2>&1
$NCU -k regex:hogwild_smem_kernel -s 2 -c 1 -f -o gpurun_out/ncu_k6 python scripts/prof_targets.py hogwild_rcv1_block 3 > /dev/null 2>&1
$NCU -k regex:"hogwild_kernel" -s 2 -c 1 -f -o gpurun_out/ncu_k6g python scripts/prof_targets.py hogwild_rcv1_block8 3 > /dev/null 2>&1
$NCU -k regex:hogwild_example_kernel -s 2 -c 1 -f -o gpurun_out/ncu_k5x python scripts/prof_targets.py hogwild_w8a_example 3 > /dev/null 2>&1
$NCU -k regex:hogwild_kernel -s 3 -c 1 -f -o gpurun_out/ncu_k5 python scripts/prof_targets.py hogwild_w8a 5 > /dev/null 2>&1
$NCU -k regex:dense_full_kernel -s 2 -c 1 -f -o gpurun_out/ncu_k1 python scripts/prof_targets.py sync_c5 3 > /dev/null 2>&1
for r in k1c k3c k6 k6g k5x k5 k1; do python scripts/ncu_summary.py gpurun_out/ncu_$r.ncu-rep > gpurun_out/ncu_${r}_summary.txt 2>&1; done
rm -f gpurun_out/*.ncu-rep
