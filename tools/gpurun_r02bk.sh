timeout 1200 python tools/halo_probe.py pair ext512 sweep1024 sweep2048 sweep4096 sweep8192 sweep16384 > gpurun_out/r02bk_halo_probe.jsonl 2> gpurun_out/r02bk_halo_probe.err; echo probe=$?
cat gpurun_out/r02bk_halo_probe.jsonl; tail -5 gpurun_out/r02bk_halo_probe.err
timeout 900 python -m pytest tests/test_gpu_halo.py -q -x > gpurun_out/r02bk_pytest_halo.log 2>&1; echo pytest=$?; tail -5 gpurun_out/r02bk_pytest_halo.log
