nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02bl_pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02bl_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bl_smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/r02bl_bench.json 2> gpurun_out/r02bl_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02bl_bench_reference.json 2> gpurun_out/r02bl_bench_reference.err; echo ref=$?
tail -c 400 gpurun_out/r02bl_bench.json
