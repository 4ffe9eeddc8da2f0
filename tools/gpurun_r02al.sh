nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/r02al_bench.json 2> gpurun_out/r02al_bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02al_launches_hair_k1.csv python bench.py --steps 2 --warmup 1 --no-single --no-cpu > gpurun_out/r02al_ncu_bench.log 2>&1; echo ncu=$?
tail -c 1500 gpurun_out/r02al_bench.json
