timeout 600 python tools/short_probe.py RSB_RW_LAZY 0 4,16,32,48,63 1,10,100 > gpurun_out/r02dj_lazy_probe.jsonl 2>&1; cat gpurun_out/r02dj_lazy_probe.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py tests/test_gpu_acceptance.py tests/test_gpu_pystep.py tests/test_gpu_scenarios.py -x -q 2>&1 | tail -3
