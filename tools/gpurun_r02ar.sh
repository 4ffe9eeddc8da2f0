timeout 600 python tools/bw_probe.py --rods 65536 --launches 20 --precision f32 --shapes 1,3 > gpurun_out/r02ar_f32.json 2> gpurun_out/r02ar_f32.err; echo rc=$?
cat gpurun_out/r02ar_f32.json; tail -2 gpurun_out/r02ar_f32.err
timeout 600 python tools/bw_probe.py --rods 65536 --launches 20 --precision f64_fast --shapes 1,3 > gpurun_out/r02ar_f64f.json 2> gpurun_out/r02ar_f64f.err; echo rc=$?
cat gpurun_out/r02ar_f64f.json
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch_scale.py -x -q -k "f32 or fp32 or reduced or fast" > gpurun_out/r02ar_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02ar_pytest.log
