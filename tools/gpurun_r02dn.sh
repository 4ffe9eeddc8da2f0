python tools/pcie_bw.py
for c in 16 8 32 64; do echo chunks=$c; RSB_PIPE_CHUNKS=$c timeout 300 python tools/e2e_probe.py 2>&1 | head -3; done
