mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:csr_coef_seg -s 1 -c 1 -f -o gpurun_out/ncu_k2t python scripts/prof_targets.py sync_rcv1 2 > gpurun_out/ncu_k2t.log 2>&1
ncu -i gpurun_out/ncu_k2t.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_k2t_sass.csv 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_k2t.ncu-rep > gpurun_out/ncu_k2t_summary.txt
rm -f gpurun_out/ncu_k2t.ncu-rep
