timeout 600 python tools/bw_breakdown.py > gpurun_out/r02l.json 2> gpurun_out/r02l.err; echo rc=$?; cat gpurun_out/r02l.json; tail -3 gpurun_out/r02l.err
