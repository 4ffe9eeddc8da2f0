timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or redo or speculat or stream or back" > gpurun_out/r02an.log 2>&1; echo pytest=$?
tail -15 gpurun_out/r02an.log
