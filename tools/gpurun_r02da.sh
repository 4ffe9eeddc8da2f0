nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02da_pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02da_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02da_smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/r02da_bench.json 2> gpurun_out/r02da_bench.err; echo bench=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rod_batch_kernel -c 1 -o gpurun_out/r02da_batch python bench.py --steps 1 --warmup 1 --no-single --no-cpu > gpurun_out/r02da_ncu_batch.log 2>&1; echo ncu_batch=$?
