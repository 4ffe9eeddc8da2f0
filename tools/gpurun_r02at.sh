timeout 300 python tools/coupled_probe.py > gpurun_out/r02at.json 2> gpurun_out/r02at.err; echo rc=$?
cat gpurun_out/r02at.json; tail -5 gpurun_out/r02at.err
