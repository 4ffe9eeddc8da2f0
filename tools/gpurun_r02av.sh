timeout 1800 python -m pytest tests/test_gpu_selfcollide.py tests/test_gpu_scenarios.py tests/test_gpu_mesh.py -x -q > gpurun_out/r02av.log 2>&1; echo pytest=$?
tail -15 gpurun_out/r02av.log
