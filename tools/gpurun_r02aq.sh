timeout 600 python tools/bw_probe.py --rods 65536 --launches 20 --precision f32 --shapes 0,1,2,3 > gpurun_out/r02aq_f32.json 2> gpurun_out/r02aq_f32.err; echo rc=$?
cat gpurun_out/r02aq_f32.json; tail -2 gpurun_out/r02aq_f32.err
