"""The reference arm of bench.py: the UNMODIFIED reference package,
installed into baseline/_ref (`pip install --no-index --no-build-isolation
--no-deps --target baseline/_ref <copy of /root/reference/pkg>`, DESIGN.md
§8), driven through its own public API -- `rodsim.world.World`,
`rodsim.state`, `rodsim.engine.Engine(backend="serial" | "parallel")`,
`rodsim.scenarios` -- on the host cores.  Nothing of this repository's
package, kernels or oracle is on that path.

When baseline/_ref is absent (a box that got only the source tree) the arm
falls back to the reference's compiled core built into oracle/_ref
(oracle/build_ref.sh) stepped through `make_context` / `step_serial`
(`kind` says which ran).

* `batch_arm` -- cfg5, the full 65,536-rod x 128-element batch: one World
  shard of R / procs rods per host process, each stepped by
  `Engine(backend="serial")` (the parallel backend would run
  one thread per rod, partition.py:54-67); a step is every process
  advancing its shard one step, timed as the wall time from the command to
  the last process's reply; element-steps/s = R x 128 / that time.
* `single_rod_cpu` -- one rod / the pair: `Engine(backend="serial")` and
  `Engine(backend="parallel")` with block_cap chosen for min(8, cores)
  blocks (reference bench.py:33-57 style), both reported, the faster
  named.
"""

import multiprocessing as mp
import os
import platform
import sys
import time
import types

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_SITE = os.path.join(ROOT, "baseline", "_ref")
ELEMENTS = 128

_RS = None


def ref_installed():
    d = os.path.join(REF_SITE, "rodsim")
    return os.path.isdir(d) and any(f.startswith("_core") and f.endswith(".so") for f in os.listdir(d))


def import_reference():
    """The installed reference package (baseline/_ref/rodsim), or None."""
    global _RS
    if _RS is None and ref_installed():
        if REF_SITE not in sys.path:
            sys.path.insert(0, REF_SITE)
        import rodsim
        import rodsim.constraints
        import rodsim.engine
        import rodsim.scenarios
        import rodsim.scene
        import rodsim.state
        import rodsim.world
        if not rodsim.HAVE_COMPILED_CORE:
            raise ImportError("baseline/_ref/rodsim has no compiled core")
        _RS = rodsim
    return _RS


def kind():
    if import_reference() is not None:
        return "reference"
    from oracle.oracle import reference_core_path
    return "reference-core" if reference_core_path() else "port"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or platform.machine()


# ---- worlds built with the reference's own API ------------------------------

def _ref_workloads():
    """This repository's BASELINE-config builders (workloads.py) re-bound to
    the reference's modules: the same recipe, executed with the reference's
    `World`, `state`, `SolverConfig` -- a reference World, built through the
    reference API (the golden fixtures pin the two constructions equal)."""
    rs = import_reference()
    from paper_2509_04277_b200 import workloads as wl
    g = dict(vars(wl))
    g.update(st=rs.state, World=rs.world.World, SolverConfig=rs.constraints.SolverConfig,
             BIND_BIDIRECTIONAL=rs.world.BIND_BIDIRECTIONAL, __package__="rodsim",
             __name__="rodsim._bench_workloads")
    for k, v in list(g.items()):
        if isinstance(v, types.FunctionType) and v.__module__ == wl.__name__:
            g[k] = types.FunctionType(v.__code__, g, v.__name__, v.__defaults__, v.__closure__)
    return types.SimpleNamespace(**{k: g[k] for k in ("cantilever", "extensible", "pair", "sweep")})


def ref_hair(rods, first=0):
    """cfg5 shard (SURVEY Appendix B recipe) with the reference API."""
    rs = import_reference()
    st = rs.state
    from paper_2509_04277_b200.workloads import MATERIAL
    w = rs.world.World(dt=1e-4, gravity=(0.0, -9.81, 0.0),
                       solver=rs.constraints.SolverConfig(iterations=10))
    params = st.RodParams(**MATERIAL)
    for r in range(rods):
        g = first + r
        a = np.random.default_rng(g).normal(size=3)
        w.add_rod(st.init_rod(ELEMENTS + 1, 0.4, axis=a / np.linalg.norm(a),
                              origin=(0.01 * (g % 256), 0.01 * (g // 256), 0.0)), params)
    w.finalize()
    for r in range(rods):
        w.clamp_point(r, 0)
    return w


def ref_world(name, *args):
    """A reference World for a single-rod config name."""
    rs = import_reference()
    if name == "insertion":   # the reference's own bundled scenario
        cfg = rs.scenarios.default_config("insertion")
        return rs.scene.build_world(cfg)
    return getattr(_ref_workloads(), name)(*args)


# ---- cfg5: the full batch on all host cores --------------------------------

def _shard_worker(conn, rods, first, k):
    sys.path.insert(0, ROOT)
    try:
        if k == "reference":
            rs = import_reference()
            w = ref_hair(rods, first)
            eng = rs.engine.Engine(w, backend="serial")
            run = eng.run_epoch
        else:   # the reference core from oracle/_ref on our World
            from oracle.oracle import OracleStepper, ReferenceStepper
            from paper_2509_04277_b200 import workloads
            w = workloads.hair(rods, ELEMENTS, first=first)
            run = (ReferenceStepper(w) if k == "reference-core" else OracleStepper(w)).run
        conn.send(("ready", 0.0))
        while True:
            steps = conn.recv()
            if steps is None:
                break
            t0 = time.perf_counter()
            run(steps)
            conn.send(("done", time.perf_counter() - t0))
    except BaseException as exc:   # surfaced in the parent
        conn.send(("error", repr(exc)))
    conn.close()


def batch_arm(total_rods=65536, procs=None, steps=10, warmup=2):
    """Element-steps/s of the reference on the whole batch, sharded over
    `procs` host processes; per-step wall times from the parent."""
    procs = procs or os.cpu_count() or 1
    procs = max(1, min(procs, total_rods))
    k = kind()
    if k == "reference":
        import_reference()   # the compiled core is loaded in the parent before forking
    ctx = mp.get_context("fork")
    base, rem = divmod(total_rods, procs)
    shards, first = [], 0
    for i in range(procs):
        n = base + (1 if i < rem else 0)
        shards.append((first, n))
        first += n
    conns, ps = [], []
    t_build = time.perf_counter()
    for first, n in shards:
        a, b = ctx.Pipe()
        p = ctx.Process(target=_shard_worker, args=(b, n, first, k), daemon=True)
        p.start()
        conns.append(a)
        ps.append(p)

    def gather():
        out = []
        for c in conns:
            tag, v = c.recv()
            if tag == "error":
                raise RuntimeError(f"reference shard worker failed: {v}")
            out.append(v)
        return out

    try:
        gather()
        t_build = time.perf_counter() - t_build
        for _ in range(warmup):
            for c in conns:
                c.send(1)
            gather()
        walls, busy = [], []
        for _ in range(steps):
            t0 = time.perf_counter()
            for c in conns:
                c.send(1)
            per = gather()
            walls.append(time.perf_counter() - t0)
            busy.append(max(per))
    finally:
        for c in conns:
            try:
                c.send(None)
            except Exception:
                pass
        for p in ps:
            p.join(timeout=30)
    wall = float(np.sum(walls))
    value = total_rods * ELEMENTS * steps / wall
    api = ("rodsim.engine.Engine(backend='serial').run_epoch(1) per shard" if k == "reference"
           else "rodsim._core.step_serial per shard (oracle/_ref)" if k == "reference-core"
           else "C restatement (oracle/liboracle.so)")
    return {"value": value, "unit": "element-steps/s", "cores": procs, "kind": k,
            "ms_per_step": wall / steps * 1e3,
            "ms_per_step_median": float(np.median(walls)) * 1e3,
            "slowest_shard_ms_per_step": float(np.mean(busy)) * 1e3,
            "cpu_model": cpu_model(), "os_cpu_count": os.cpu_count(),
            "api": api, "build_s": t_build,
            "sample": f"the full batch: {total_rods} rods x {ELEMENTS} elements, {procs} processes "
                      f"of ~{total_rods // procs} rods, {steps} timed steps after {warmup} warm-up",
            "same_config": True}


# ---- single rods: serial and parallel backends -------------------------------

def _time_engine(make, backend, steps, block_cap, max_blocks=None):
    rs = import_reference()
    w = make()
    with rs.engine.Engine(w, backend=backend, block_cap=block_cap, max_blocks=max_blocks) as eng:
        eng.run_epoch(min(10, steps))
        t0 = time.perf_counter()
        m = eng.run_epoch(steps)
        dt = time.perf_counter() - t0
        blocks = eng.partition.block_count
    return dt / steps * 1e6, blocks, m["barrier_wait_ns"]


def single_rod_cpu(name, args=(), steps=200, par_steps=None):
    """us/step of the reference on one rod (or the pair): serial and
    parallel backends; the faster one is the baseline."""
    k = kind()
    if k != "reference":   # fallback: the compiled core's serial loop only
        from oracle.oracle import OracleStepper, ReferenceStepper
        from paper_2509_04277_b200 import workloads as wl
        w = getattr(wl, name)(*args)
        s = ReferenceStepper(w) if k == "reference-core" else OracleStepper(w)
        s.run(2)
        t0 = time.perf_counter()
        s.run(steps)
        us = (time.perf_counter() - t0) / steps * 1e6
        return {"cpu_us_per_step": us, "cpu_kind": k, "serial_us": us, "parallel_us": None}

    def make():
        return ref_world(name, *args)
    serial, _, _ = _time_engine(make, "serial", steps, 512)
    w = make()
    cores = min(8, os.cpu_count() or 1)
    npts = max(i.num_points for i in w.rod_infos)
    cap = max(2, -(-npts // cores))
    try:
        par, blocks, bns = _time_engine(make, "parallel", par_steps or max(10, steps // 4), cap, max_blocks=cores)
    except Exception as exc:   # the threaded backend refused the partition
        par, blocks, bns = None, 0, repr(exc)
    best = min(x for x in (serial, par) if x is not None)
    return {"cpu_us_per_step": best, "cpu_kind": k,
            "cpu_backend": "serial" if best == serial else "parallel",
            "serial_us": serial, "parallel_us": par, "parallel_blocks": blocks,
            "parallel_barrier_wait_ns": bns, "api": "rodsim.engine.Engine.run_epoch"}
