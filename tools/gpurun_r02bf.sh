nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python tools/halo_probe.py > gpurun_out/r02bf_halo_probe.jsonl 2> gpurun_out/r02bf_halo_probe.err; echo probe=$?
cat gpurun_out/r02bf_halo_probe.jsonl; tail -20 gpurun_out/r02bf_halo_probe.err
