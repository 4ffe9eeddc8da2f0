set -x
timeout 600 python -m pytest tests/test_gpu_selftest.py -x -q > gpurun_out/r02e_selftest.log 2>&1; echo st=$?
tail -3 gpurun_out/r02e_selftest.log
timeout 600 python tools/bw_probe.py --rods 65536 --launches 20 --shapes 0,1 > gpurun_out/r02e_k1.json 2> gpurun_out/r02e_k1.err; echo k1=$?
cat gpurun_out/r02e_k1.json; tail -3 gpurun_out/r02e_k1.err
