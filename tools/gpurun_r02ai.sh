timeout 600 python tools/rw_probe.py > gpurun_out/r02ai_rw.json 2> gpurun_out/r02ai_rw.err; echo rw=$?
cat gpurun_out/r02ai_rw.json; tail -5 gpurun_out/r02ai_rw.err
