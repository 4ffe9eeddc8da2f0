import sys, threading, time, numpy as np
sys.path.insert(0, '/root/repo')
from oracle.oracle import OracleStepper
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.engine import Engine
def bits(a): return np.ascontiguousarray(a).view(np.int64)
steps = 20000
g = wl.cantilever()
with Engine(g) as eng:
    eng.run_epoch(1)
    box = {}
    def run():
        try: box['m'] = eng.run_epoch(steps)
        except Exception as e: box['e'] = repr(e)
    th = threading.Thread(target=run); th.start()
    time.sleep(0.02); a = eng.post_command("grab", rod=0, index=64, target=(0.3, 0.05, 0.0))
    time.sleep(0.03); b = eng.post_command("release", rod=0, index=64)
    th.join()
    sg, sr = a.wait(5), b.wait(5)
    print('live: grab', sg, 'release', sr, box.get('e'), 'err', eng._dev.error_step())
# deterministic replica on the GPU: epochs split at the apply steps
h = wl.cantilever()
with Engine(h) as eng:
    eng.run_epoch(sg)
    eng.post_command("grab", rod=0, index=64, target=(0.3, 0.05, 0.0)); eng.run_epoch(sr - sg)
    eng.post_command("release", rod=0, index=64); eng.run_epoch(1 + steps - sr)
r = wl.cantilever(); o = OracleStepper(r)
o.run(sg); r.grab(0, 64, np.array([0.3, 0.05, 0.0])); o.run(sr - sg); r.release(0, 64); o.run(1 + steps - sr)
print('split-GPU vs oracle', np.array_equal(bits(h.positions), bits(r.positions)), 'live vs oracle', np.array_equal(bits(g.positions), bits(r.positions)))
print('nan live', np.isnan(g.positions).any(), 'nan ref', np.isnan(r.positions).any(), 'oracle err', o.error_step)
