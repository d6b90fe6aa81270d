mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:hogwild_chunk -s 3 -c 1 -f -o gpurun_out/ncu_k5c python scripts/prof_targets.py hogwild_w8a 5 > gpurun_out/ncu_k5c.log 2>&1
tail -2 gpurun_out/ncu_k5c.log
