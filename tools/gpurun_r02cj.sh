timeout 1200 python -m pytest tests/test_gpu_halo.py tests/test_gpu_parity.py -q -x -k "pair or bind or halo or column or set_params" > gpurun_out/r02cj_pytest.log 2>&1; echo pytest=$?; tail -5 gpurun_out/r02cj_pytest.log
python - <<'PY'
import sys
sys.path.insert(0, '.')
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.engine import Engine
def us(make, k, launches):
    with Engine(make()) as eng:
        dev = eng.device_world
        dev.run(k); dev.synchronize()
        dev.timer_start()
        for _ in range(launches): dev.run(k)
        dev.timer_stop()
        return round(dev.timer_ms() * 1e3 / (k * launches), 2), dev.last_redo_count()
print("pair", {k: us(wl.pair, k, max(2, min(200, 2000 // k))) for k in (1, 10, 100)})
PY
