timeout 900 python tools/halo_probe.py cfg1 sweep128 sweep256 sweep512 sweep16384 > gpurun_out/r02bg_halo_probe.jsonl 2> gpurun_out/r02bg_halo_probe.err; echo probe=$?
cat gpurun_out/r02bg_halo_probe.jsonl; tail -5 gpurun_out/r02bg_halo_probe.err
