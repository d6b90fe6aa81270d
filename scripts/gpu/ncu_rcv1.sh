mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:"csr_coef|csc_vec|apply_partials" -s 3 -c 3 -f -o gpurun_out/ncu_rcv1_k2s python scripts/prof_targets.py sync_rcv1 3 > gpurun_out/ncu_rcv1.log 2>&1
ls -la gpurun_out/
