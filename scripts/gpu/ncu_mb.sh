# ncu --set full of the sparse mini-batch step kernels (news20 / rcv1 shapes, B = 4096)
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:"csr_batch|apply_kernel" -s 6 -c 2 -f -o gpurun_out/ncu_mb_news20 python scripts/sync_sweep.py news20 > gpurun_out/ncu_mb.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_mb_news20.ncu-rep > gpurun_out/ncu_mb_news20.txt 2>&1
ncu -i gpurun_out/ncu_mb_news20.ncu-rep --page source --csv -k regex:csr_batch > gpurun_out/ncu_mb_news20_src.csv 2>&1
