nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02dz_smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/r02dz_bench.json 2> gpurun_out/r02dz_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02dz_bench_reference.json 2> gpurun_out/r02dz_bench_reference.err; echo ref=$?
timeout 600 python -m pytest tests/test_gpu_bench.py -q 2>&1 | tail -1
