# A/B: next rod's loads interleaved with the write-back (BW_ILV=1) vs after it (0)
for r in 1 2; do
for v in 0 1; do
  timeout 300 python tools/bw_probe.py --lib scratch/lib_ilv$v.so --k 1 --launches 30 --shapes 3 >> gpurun_out/r02db_ab.jsonl 2>>gpurun_out/r02db_ab.err
  timeout 300 python tools/bw_probe.py --lib scratch/lib_ilv$v.so --k 10 --launches 5 --shapes 3 >> gpurun_out/r02db_ab.jsonl 2>>gpurun_out/r02db_ab.err
done; done
cat gpurun_out/r02db_ab.jsonl
