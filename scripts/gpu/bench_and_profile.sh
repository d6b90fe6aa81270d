mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 900 bash scripts/round1_profile.sh > gpurun_out/profile.log 2>&1
