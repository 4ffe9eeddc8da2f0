timeout 600 python tools/bw_probe.py --rods 65536 --launches 20 --shapes 1 > gpurun_out/r02x_k1.json 2> gpurun_out/r02x_k1.err; echo k1=$?
cat gpurun_out/r02x_k1.json; tail -3 gpurun_out/r02x_k1.err
timeout 600 python tools/bw_breakdown.py > gpurun_out/r02x_bd.json 2> gpurun_out/r02x_bd.err; cat gpurun_out/r02x_bd.json
