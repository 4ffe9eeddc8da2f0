timeout 900 python -m pytest tests/test_gpu_live.py tests/test_gpu_service.py tests/test_gpu_halo.py tests/test_gpu_refcore.py tests/test_gpu_acceptance.py -q -x > gpurun_out/r02bt_pytest.log 2>&1; echo pytest=$?; tail -5 gpurun_out/r02bt_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "barrier_waits" > gpurun_out/r02bt_pytest2.log 2>&1; echo pytest2=$?; tail -3 gpurun_out/r02bt_pytest2.log
python - <<'PY'
import sys, time
sys.path.insert(0, '.')
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.engine import Engine
for kw in ({}, {"live": True}, {"backend": "parallel"}):
    with Engine(wl.pair(), **kw) as eng:
        g = eng.plan()["groups"][0]
        dev = eng.device_world
        dev.run(10); dev.synchronize()
        dev.timer_start()
        for _ in range(100): dev.run(10)
        dev.timer_stop()
        print("pair", kw, "halo", g["halo"] is not None, "us/step", round(dev.timer_ms() * 1e3 / 1000, 2), flush=True)
w = wl.pair()
with Engine(w, backend="parallel") as eng:
    t0 = time.perf_counter(); fr = []
    for i in range(300):
        t1 = time.perf_counter()
        eng.post_command("insert_velocity", rod=0, value=0.05 + 1e-4 * (i % 7), axis=(0.0, 0.0, 1.0))
        eng.run_epoch(10)
        fr.append(time.perf_counter() - t1)
    import numpy as np
    print("parallel-backend haptic frame median us", np.median(fr[50:]) * 1e6)
PY
