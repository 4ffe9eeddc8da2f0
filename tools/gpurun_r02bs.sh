timeout 900 python -m pytest tests/test_gpu_live.py tests/test_gpu_service.py tests/test_gpu_halo.py -q -x > gpurun_out/r02bs_pytest.log 2>&1; echo pytest=$?; tail -25 gpurun_out/r02bs_pytest.log
python - <<'PY'
import sys, time
sys.path.insert(0, '.')
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.engine import Engine
for live in (False, True):
    with Engine(wl.pair(), live=live) as eng:
        g = eng.plan()["groups"][0]
        dev = eng.device_world
        dev.run(10); dev.synchronize()
        dev.timer_start()
        for _ in range(100): dev.run(10)
        dev.timer_stop()
        print("pair live", live, "halo", g["halo"] is not None, "us/step", dev.timer_ms() * 1e3 / 1000, flush=True)
PY
