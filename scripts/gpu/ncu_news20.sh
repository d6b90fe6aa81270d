mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"csr_coef|csc_|apply_partials" -s 4 -c 4 -f -o gpurun_out/ncu_news20 python scripts/prof_targets.py sync_news20 3 > gpurun_out/ncu_news20.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_news20.ncu-rep > gpurun_out/ncu_news20_summary.txt
ncu -i gpurun_out/ncu_news20.ncu-rep --page source --csv --print-source sass --kernel-name regex:csc_seg > gpurun_out/ncu_news20_csc_sass.csv 2>&1
rm -f gpurun_out/ncu_news20.ncu-rep
