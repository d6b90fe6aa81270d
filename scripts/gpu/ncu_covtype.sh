mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:dense_full -s 2 -c 1 -f -o gpurun_out/ncu_cov python scripts/prof_targets.py sync_covtype 3 > gpurun_out/ncu_cov.log 2>&1
ncu -i gpurun_out/ncu_cov.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_cov_sass.csv 2>&1
ncu -i gpurun_out/ncu_cov.ncu-rep --page raw --csv > gpurun_out/ncu_cov_raw.csv 2>&1
rm -f gpurun_out/ncu_cov.ncu-rep
