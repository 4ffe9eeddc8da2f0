python - <<'PY' 2>&1
import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2509_04277_b200.engine import Engine
from test_gpu_acceptance import _coupled_pair
from paper_2509_04277_b200 import workloads as wl
def run(make, env, label):
    for k, v in env.items(): os.environ[k] = str(v)
    with Engine(make()) as eng:
        dev = eng.device_world
        eng.run_epoch(10)
        dev.enable_timing(True)
        eng.run_epoch(100)
        print(label, env, "ms/100", round(dev.last_kernel_ms(), 3), "redo", dev.last_redo_count(), flush=True)
    for k in env: os.environ.pop(k)
for m in ("v0", "v1"):
    run(lambda: _coupled_pair(m), {"RSB_DEBUG": 4}, m)
    run(lambda: _coupled_pair(m), {"RSB_HALO": 0}, m)
run(wl.pair, {"RSB_DEBUG": 4}, "pair")
PY
