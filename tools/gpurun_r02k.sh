RSB_BW_SHAPE=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:rod_batch --launch-skip 1 -c 1 -f -o gpurun_out/r02k_bw1 python tools/prof_case.py hair --launches 2 > gpurun_out/r02k_ncu1.log 2>&1; echo ncu1=$?
timeout 600 python tools/bw_probe.py --rods 65536 --launches 20 --shapes 1,2 > gpurun_out/r02k_k1.json 2> gpurun_out/r02k_k1.err; echo k1=$?
cat gpurun_out/r02k_k1.json
