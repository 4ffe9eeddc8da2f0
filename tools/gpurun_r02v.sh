ls baseline/_ref/rodsim | head -3
timeout 1200 python -m pytest tests/test_gpu_refcore.py -x -q > gpurun_out/r02v_refcore.log 2>&1; echo pytest=$?
tail -30 gpurun_out/r02v_refcore.log
