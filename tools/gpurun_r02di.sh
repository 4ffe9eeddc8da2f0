timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02di_pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02di_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02di_smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py --no-cpu > gpurun_out/r02di_bench.json 2> gpurun_out/r02di_bench.err; echo bench=$?
