set -x
timeout 600 python -m pytest tests/test_gpu_selftest.py -x -q > gpurun_out/r02g_selftest.log 2>&1; echo st=$?
tail -2 gpurun_out/r02g_selftest.log
timeout 600 python tools/bw_probe.py --rods 65536 --launches 20 --shapes 0,1 > gpurun_out/r02g_k1.json 2> gpurun_out/r02g_k1.err; echo k1=$?
cat gpurun_out/r02g_k1.json; tail -3 gpurun_out/r02g_k1.err
RSB_BW_SHAPE=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:rod_batch --launch-skip 1 -c 1 -f -o gpurun_out/r02g_bw1 python tools/prof_case.py hair --launches 2 > gpurun_out/r02g_ncu1.log 2>&1; echo ncu1=$?
