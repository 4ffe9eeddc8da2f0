set -x
timeout 600 python -m pytest tests/test_gpu_selftest.py -x -q > gpurun_out/r02f_selftest.log 2>&1; echo st=$?
tail -3 gpurun_out/r02f_selftest.log
for sh in 0 1; do
RSB_BW_SHAPE=$sh timeout 600 ncu --set full --import-source on --clock-control none -k regex:rod_batch --launch-skip 1 -c 1 -f -o gpurun_out/r02f_bw$sh python tools/prof_case.py hair --launches 2 > gpurun_out/r02f_ncu$sh.log 2>&1; echo ncu$sh=$?
done
tail -3 gpurun_out/r02f_ncu0.log
