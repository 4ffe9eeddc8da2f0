set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch_scale.py -x -q -k "golden or cfg2 or cfg3 or set_params or batch" -s > gpurun_out/r02a_pytest.log 2>&1; echo pytest=$?
timeout 600 python tools/fp32_tolerance.py > gpurun_out/r02a_fp32_tol.json 2> gpurun_out/r02a_fp32_tol.err; echo tol=$?
tail -5 gpurun_out/r02a_pytest.log
