mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
SGDB_SEG_THREADS=1024 $NCU -k regex:"csr_coef|csc_seg" -s 2 -c 2 -f -o gpurun_out/ncu_rcv1_seg4 python scripts/prof_targets.py sync_rcv1 2 > gpurun_out/ncu_seg.log 2>&1
tail -3 gpurun_out/ncu_seg.log
