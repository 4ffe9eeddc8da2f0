timeout 1200 python tools/halo_probe.py pair ext512 sweep128 sweep256 sweep512 sweep1024 > gpurun_out/r02bm_halo_probe.jsonl 2> gpurun_out/r02bm_halo_probe.err; echo probe=$?
cat gpurun_out/r02bm_halo_probe.jsonl; tail -5 gpurun_out/r02bm_halo_probe.err
timeout 900 python -m pytest tests/test_gpu_halo.py -q -x > gpurun_out/r02bm_pytest_halo.log 2>&1; echo pytest=$?; tail -15 gpurun_out/r02bm_pytest_halo.log
