nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ba_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02ba_pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02ba_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02ba_bench.json 2> gpurun_out/r02ba_bench.err; echo bench=$?
tail -c 3000 gpurun_out/r02ba_bench.json
