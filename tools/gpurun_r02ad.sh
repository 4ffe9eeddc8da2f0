timeout 600 python tools/bw_probe.py --rods 65536 --launches 20 --shapes 1,3 > gpurun_out/r02ad_k1.json 2> gpurun_out/r02ad_k1.err; echo k1=$?
cat gpurun_out/r02ad_k1.json; tail -3 gpurun_out/r02ad_k1.err
