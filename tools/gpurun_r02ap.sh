for prec in f32; do
timeout 600 python bench.py --precision $prec --no-single --no-cpu --steps 20 > gpurun_out/r02ap_bench_$prec.json 2> gpurun_out/r02ap_bench_$prec.err; echo $prec=$?
python -c "import json;d=json.loads(open('gpurun_out/r02ap_bench_$prec.json').read().strip().splitlines()[-1]);print('$prec', d['value'], d['ms_per_step'], d['value_k10'], d['e2e']['value'], d['e2e']['value_k10'], d['roofline']['frac'], d['config']['plan'][0].get('warp_per_rod'))"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch_scale.py -x -q -k "f32 or fp32 or reduced" > gpurun_out/r02ap_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02ap_pytest.log
