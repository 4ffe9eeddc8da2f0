timeout 600 ncu --set full --import-source on --clock-control none -k regex:rod_warp --launch-skip 1 -c 1 -f -o gpurun_out/r02af_rw python tools/prof_case.py sweep --n 16 --k 1000 --launches 2 > gpurun_out/r02af_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/r02af_ncu.log
