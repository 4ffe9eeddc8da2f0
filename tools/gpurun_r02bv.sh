python - <<'PY'
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2509_04277_b200.engine import Engine
from test_gpu_acceptance import _coupled_pair
for m in ("v0", "v1"):
    for kw in ({}, {"backend": "parallel"}):
        with Engine(_coupled_pair(m), **kw) as eng:
            g = eng.plan()
            print(m, kw, g["live"], [(x["tier"], x["ctas"], x["halo"]) for x in g["groups"]], flush=True)
PY
