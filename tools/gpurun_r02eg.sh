nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02eg_pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02eg_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02eg_smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/r02eg_bench.json 2> gpurun_out/r02eg_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02eg_bench_reference.json 2> gpurun_out/r02eg_bench_reference.err; echo ref=$?
