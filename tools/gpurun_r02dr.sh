nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02dr_smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/r02dr_bench.json 2> gpurun_out/r02dr_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02dr_bench_reference.json 2> gpurun_out/r02dr_bench_reference.err; echo ref=$?
timeout 300 python tools/k1_launch_probe.py > gpurun_out/r02dr_k1_launch_probe.txt 2>&1; echo k1=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02dr_launches_hair_k1.csv python bench.py --steps 2 --warmup 1 --no-single --no-cpu > /dev/null 2>&1; echo ncu_l=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02dr_launches_pair_k10.csv python tools/prof_case.py pair --k 10 --launches 5 > /dev/null 2>&1; echo ncu_l2=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02dr_launches_n16_k10.csv python tools/prof_case.py sweep --n 16 --k 10 --launches 5 > /dev/null 2>&1; echo ncu_l3=$?
