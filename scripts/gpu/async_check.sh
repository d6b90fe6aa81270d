mkdir -p gpurun_out
timeout 600 python scripts/async_sweep.py > gpurun_out/async_sweep.jsonl 2> gpurun_out/async_sweep.err; tail -3 gpurun_out/async_sweep.err
timeout 400 python scripts/sync_sweep.py > gpurun_out/sync_sweep_async.jsonl 2> gpurun_out/sync_sweep_async.err
