for pad in 0 6000 12000; do
RSB_BW_PAD=$pad timeout 600 python tools/bw_probe.py --rods 65536 --launches 20 --shapes 1 > gpurun_out/r02y_$pad.json 2>&1; echo pad=$pad $(python -c "import json;d=json.load(open('gpurun_out/r02y_$pad.json'));print(d['shape1']['ms_per_launch'])")
done
