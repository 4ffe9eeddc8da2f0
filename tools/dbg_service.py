import sys, time, traceback
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_service import *
for rep in range(6):
    for backend in ("serial", "parallel"):
        app = create_app(scene(), backend=backend, frame_interval=0.005)
        with TestClient(app) as client:
            svc = app.state.service
            with client.websocket_connect("/ws") as ws:
                ws.receive_json()
                ws.send_json(cmd(0, "grab", index=10, target=[0.0, 0.05, 0.0]))
                a = until(ws, "ack")
            t0 = time.time()
            while svc.world.grab_active.any() and time.time() < t0 + 5: time.sleep(0.01)
            print(rep, backend, "ack", a, "active", svc.world.grab_active.any(), "ctrl", svc.controller, "err", repr(svc.error), "step", svc.world.step_index, flush=True)
