mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:hogwild_smem -s 2 -c 1 -f -o gpurun_out/ncu_k6 python scripts/prof_targets.py hogwild_rcv1_block 3 > gpurun_out/ncu_k6.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_k6.ncu-rep > gpurun_out/ncu_k6_summary.txt
ncu -i gpurun_out/ncu_k6.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_k6_sass.csv 2>&1
rm -f gpurun_out/ncu_k6.ncu-rep
