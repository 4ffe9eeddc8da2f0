timeout 1200 python -m pytest tests/test_gpu_mesh.py tests/test_gpu_scenarios.py tests/test_gpu_halo.py -q -x > gpurun_out/r02cf_pytest.log 2>&1; echo pytest=$?; tail -15 gpurun_out/r02cf_pytest.log
python - <<'PY'
import os, sys
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
        return round(dev.timer_ms() * 1e3 / (k * launches), 2), bool(eng.plan()["groups"][0].get("halo")), dev.last_redo_count()
for env in ({}, {"RSB_HALO": "0"}):
    os.environ.update(env)
    print(env, "insertion", {k: us(wl.insertion, k, max(2, min(100, 1000 // k))) for k in (10, 100)}, flush=True)
    for k in env: os.environ.pop(k)
PY
