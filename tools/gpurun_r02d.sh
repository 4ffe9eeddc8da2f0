set -x
timeout 300 python tools/bw_probe.py --rods 2048 --launches 5 --shapes 3,2,0 > gpurun_out/r02d_small.json 2> gpurun_out/r02d_small.err; echo s=$?
timeout 600 python tools/bw_probe.py --rods 65536 --launches 20 --shapes 3,2,1,0 > gpurun_out/r02d_k1.json 2> gpurun_out/r02d_k1.err; echo k1=$?
timeout 300 python tools/bw_probe.py --rods 65536 --launches 3 --k 10 --shapes 3,0 > gpurun_out/r02d_k10.json 2> gpurun_out/r02d_k10.err; echo k10=$?
cat gpurun_out/r02d_small.json gpurun_out/r02d_k1.json gpurun_out/r02d_k10.json; tail -5 gpurun_out/r02d_small.err
