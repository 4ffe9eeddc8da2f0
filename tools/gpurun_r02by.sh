nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py > gpurun_out/r02by_bench.json 2> gpurun_out/r02by_bench.err; echo bench=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rod_halo_kernel -c 1 -o gpurun_out/r02by_halo_pair python tools/prof_case.py pair --k 10 --launches 3 > gpurun_out/r02by_ncu_pair.log 2>&1; echo ncu_pair=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rod_halo_kernel -c 1 -o gpurun_out/r02by_halo_s16384 python tools/prof_case.py sweep --n 16384 --k 10 --launches 3 > gpurun_out/r02by_ncu_s16384.log 2>&1; echo ncu_s=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02by_launches_hair_k1.csv python bench.py --steps 2 --warmup 1 --no-single --no-cpu > /dev/null 2>&1; echo ncu_l=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02by_launches_pair_k10.csv python tools/prof_case.py pair --k 10 --launches 5 > /dev/null 2>&1; echo ncu_l2=$?
