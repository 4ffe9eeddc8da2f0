timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02eb_pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02eb_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02eb_smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/r02eb_bench.json 2> gpurun_out/r02eb_bench.err; echo bench=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02eb_launches_hair_k1.csv python bench.py --steps 2 --warmup 1 --no-single --no-cpu > /dev/null 2>&1; echo ncu_l=$?
