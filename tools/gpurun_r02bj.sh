nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py > gpurun_out/r02bj_bench.json 2> gpurun_out/r02bj_bench.err; echo bench=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rod_halo_kernel -c 1 -o gpurun_out/r02bj_halo_pair python tools/prof_case.py pair --k 10 --launches 3 > gpurun_out/r02bj_ncu_pair.log 2>&1; echo ncu_pair=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rod_halo_kernel -c 1 -o gpurun_out/r02bj_halo_s16384 python tools/prof_case.py sweep --n 16384 --k 10 --launches 3 > gpurun_out/r02bj_ncu_s16384.log 2>&1; echo ncu_s=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02bj_launches_pair.csv python tools/prof_case.py pair --k 10 --launches 5 > /dev/null 2>&1; echo ncu_l=$?
tail -c 600 gpurun_out/r02bj_bench.json
