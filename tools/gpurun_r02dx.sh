timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02dx_pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02dx_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02dx_smoke.log 2>&1; echo smoke=$?
timeout 300 python tools/haptic_ab.py 2>&1 | tail -1
