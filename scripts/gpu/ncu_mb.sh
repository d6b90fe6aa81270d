# ncu --set full of the sparse mini-batch step kernels (K3c) on the rcv1 / news20 shapes, B = 4096
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
for shape in rcv1 news20; do
  $NCU -k regex:"mb_margin|mb_scatter|apply_kernel" -s 30 -c 3 -f -o gpurun_out/ncu_mb_$shape python scripts/sync_sweep.py $shape > gpurun_out/ncu_mb_$shape.log 2>&1
  python scripts/ncu_summary.py gpurun_out/ncu_mb_$shape.ncu-rep > gpurun_out/ncu_mb_$shape.txt 2>&1
  rm -f gpurun_out/ncu_mb_$shape.ncu-rep
done
