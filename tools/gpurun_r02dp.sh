for r in 1 2; do
RSB_XFER=0 timeout 300 python tools/frame_probe.py 2>&1 | head -1
timeout 300 python tools/frame_probe.py 2>&1 | head -1
done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02dp_pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02dp_pytest_gpu.log
