"""The C ABI boundary (include/rodsim_b200.h) and the launch planner, on CPU.

* every entry point the header declares is exported by librodsim_b200.so
  and typed in _lib.SIGNATURES;
* the ctypes mirror of `rs_world_desc` has the C compiler's layout;
* the planner (rs_plan_dry: the same code path rs_create runs, minus device
  queries) maps the BASELINE configs to the intended tiers;
* without a device the engine fails loudly (there is no CPU fallback).
"""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, have_gpu
from paper_2509_04277_b200 import _lib
from paper_2509_04277_b200 import state as st
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.world import BIND_BIDIRECTIONAL, World

HEADER = os.path.join(ROOT, "include", "rodsim_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^[a-z_0-9 ]+[ \*]+(rs_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_entry_point():
    lib = _lib.load_library()
    declared = header_functions()
    assert len(declared) >= 20
    typed = {name for name, _, _ in _lib.SIGNATURES}
    for name in declared:
        assert hasattr(lib, name), name
        assert name in typed, name


def test_world_desc_layout_matches_c(tmp_path):
    fields = [f for f, _ in _lib.WorldDesc._fields_]
    src = tmp_path / "probe.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "rodsim_b200.h"\n'
        "int main(void){printf(\"%zu\\n\", sizeof(rs_world_desc));\n"
        + "".join(f'printf("%zu\\n", offsetof(rs_world_desc, {f}));\n' for f in fields)
        + "return 0;}\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    out = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert out[0] == ctypes.sizeof(_lib.WorldDesc)
    for f, off in zip(fields, out[1:]):
        assert getattr(_lib.WorldDesc, f).offset == off, f


# -- planner ---------------------------------------------------------------------

def plan(world, **kw):
    return _lib.plan_dry(world, **kw)["groups"]


def test_plan_single_rods_by_size():
    g = plan(wl.cantilever())
    assert len(g) == 1 and g[0]["tier"] == "cta" and g[0]["ctas"] == 1 and g[0]["uniform"]
    # without distance projection a rod steps in 3 phases: one CTA up to 320
    # points, a cluster above (the CTA would be bound by one SM's fp64 issue)
    assert plan(wl.extensible(256))[0]["tier"] == "cta"
    g = plan(wl.extensible())[0]
    assert g["tier"] == "cluster" and g["ctas"] >= 2
    assert plan(wl.cantilever(512))[0]["tier"] == "cta"   # inextensible: 23 phases
    g = plan(wl.sweep(4096))[0]
    assert g["tier"] == "cluster" and 2 <= g["ctas"] <= 16 and g["cluster"] == g["ctas"]
    g = plan(wl.sweep(16384))[0]
    assert g["tier"] == "cluster" and g["ctas"] <= 16
    g = plan(wl.sweep(32768))[0]
    assert g["tier"] == "grid" and g["ctas"] > 16


def test_plan_pair_keeps_bound_rods_together_with_parallel_bindings():
    g = plan(wl.pair())
    # both rods in one 9-CTA cluster of 128-point CTAs (1026 points)
    assert len(g) == 1 and g[0]["tier"] == "cluster" and g[0]["points"] == 1026
    assert g[0]["ctas"] == 9 and g[0]["cluster"] == 9
    # a matching: each binding applied in parallel by the CTA owning point a
    assert 0 < g[0]["bind_cap"] <= 128
    g = plan(wl.pair(), force_tier=0)
    assert g[0]["tier"] == "cta" and g[0]["bind_cap"] == 513


def test_plan_batched_rods_use_occupancy_variant():
    g = plan(wl.hair(2048))[0]
    # persistent stream tier: 2048 rod tasks over <= 8 CTAs per SM; a
    # 129-point rod is 64 threads x 2 slots plus the tip as thread 0's tail
    assert g["tier"] == "stream" and g["variant"] == 7 and g["ctas"] == 2048
    assert g["threads"] == 64 and g["grid"] <= 8 * 148
    strided = plan(wl.hair(2048), force_variant=5)[0]
    assert strided["tier"] == "stream" and strided["threads"] == 128
    small = plan(wl.hair(16))[0]
    assert small["tier"] == "cta"


def test_plan_forced_tiers_and_variants():
    w = wl.cantilever(200, 0.4)
    assert plan(w, force_tier=1, force_ctas=5)[0]["ctas"] == 5
    assert plan(w, force_tier=2, force_ctas=3)[0]["tier"] == "grid"
    assert plan(w, force_variant=4)[0]["variant"] == 4
    with pytest.raises(ValueError):
        plan(wl.cantilever(300, 0.6), force_variant=0)


def test_plan_segments_span_bound_non_adjacent_rods():
    w = World()
    for n in (10, 20, 10):
        w.add_rod(st.init_rod(n, 0.01 * n), st.RodParams())
    w.finalize()
    w.add_bindings(0, 2, BIND_BIDIRECTIONAL)
    g = plan(w)
    assert len(g) == 1 and g[0]["ctas"] == 1 and g[0]["points"] == 40


def test_plan_rejects_inconsistent_layouts():
    w = wl.cantilever(10, 0.1)
    w.junction_valid[-1] = True          # a junction past the rod end
    with pytest.raises(ValueError, match="junction_valid"):
        plan(w)
    # coupled rods past one 16-CTA cluster: the wide-halo grid exchange
    # steps two equal rods bound at the same local index; anything else is
    # rejected (no general kernel binds across a grid)
    big = World()
    for _ in range(2):
        big.add_rod(st.init_rod(12000, 24.0), st.RodParams())
    big.finalize()
    big.add_bindings(0, 1, BIND_BIDIRECTIONAL, stride=100)
    g = plan(big)[0]
    assert g["tier"] == "grid" and g["halo"]["exchange"] == "grid" and g["halo"]["rods"] == 2
    odd = World()
    odd.add_rod(st.init_rod(12000, 24.0), st.RodParams())
    odd.add_rod(st.init_rod(11000, 22.0), st.RodParams())
    odd.finalize()
    odd.add_bindings(0, 1, BIND_BIDIRECTIONAL, stride=100)
    with pytest.raises(NotImplementedError):
        plan(odd)


@pytest.mark.skipif(have_gpu(), reason="checks the no-device failure path")
def test_engine_fails_loudly_without_a_device():
    from paper_2509_04277_b200.engine import Engine
    with pytest.raises((ValueError, _lib.RodsimError)):
        Engine(wl.cantilever())


def test_engine_rejects_out_of_scope_scenes():
    from paper_2509_04277_b200.engine import Engine
    with pytest.raises(ValueError):
        Engine(wl.cantilever(), backend="gpu")


def test_self_collision_plan_is_one_cta():
    g = plan(wl.knot())
    assert len(g) == 1 and g[0]["tier"] == "cta" and g[0]["ctas"] == 1 and g[0]["points"] == 96
    from paper_2509_04277_b200.constraints import SolverConfig
    from paper_2509_04277_b200.selfcollide import SelfCollisionConfig
    # the paper's knot size (2 x 257 points) and up to the largest one-CTA
    # variant (1153 points) plan into one CTA; beyond that, rejected
    big = plan(wl.crossing(points=257, length=0.512))
    assert len(big) == 1 and big[0]["tier"] == "cta" and big[0]["points"] == 514 and big[0]["variant"] == 4
    w = World(dt=1e-4, solver=SolverConfig(), self_collision=SelfCollisionConfig())
    for _ in range(5):
        w.add_rod(st.init_rod(300, 0.3), st.RodParams())
    w.finalize()
    with pytest.raises(NotImplementedError, match="self-collision"):
        plan(w)


def test_desc_binds_the_mesh_tree():
    from paper_2509_04277_b200 import _lib
    w = wl.insertion(points=20, length=0.05, tube={"rings": 12, "segments": 8})
    d, keep = _lib.build_desc(w)
    assert d.has_mesh == 1 and d.n_tris == w.tree.triangles.shape[0]
    assert d.n_nodes == w.tree.node_min.shape[0] and d.mesh_depth == w.tree.max_depth
    assert d.coll_interval == 4 and d.coll_margin == 5e-4
    assert keep["tris"].dtype == np.int64 and keep["cact"] is w.contact_active
    p = _lib.plan_dry(w)
    assert p["groups"][0]["tier"] == "cta"


def test_contact_batches_stay_off_the_stream_tier():
    from paper_2509_04277_b200 import bvh, meshes
    w = wl.hair(2048)
    assert plan(w)[0]["tier"] == "stream"
    w.set_mesh(bvh.build_aabb_tree(*meshes.floor_mesh(y=-1.0, cells=2)))
    assert plan(w)[0]["tier"] == "cta"


def test_plan_barriers_per_step():
    # the latency roofline's n_sync: 3 + I x (2 colour phases + contacts +
    # pairs + bindings + grabs), as the kernel issues them (rod_step.cuh)
    assert plan(wl.cantilever())[0]["sync_per_step"] == 23      # 2I + 3
    assert plan(wl.extensible())[0]["sync_per_step"] == 3       # no colour sweeps
    assert plan(wl.pair())[0]["sync_per_step"] == 33            # 3I + 3
    assert plan(wl.insertion())[0]["sync_per_step"] == 33       # + contact phase
    assert plan(wl.knot())[0]["sync_per_step"] == 3 + 15 * 3    # + self-collision pairs
    assert plan(wl.hair(2048))[0]["sync_per_step"] == 23


def test_plan_wide_halo_kernel():
    # rod_halo.cuh: rods beyond one CTA (and one-CTA rods: spread over a cluster from 100 points)
    # step with one inter-CTA exchange per step; cluster up to 16 CTAs of <=
    # 256 threads, a co-resident grid beyond; the cfg1 cantilever, forced
    # layouts and overlapping couplings keep the general kernel
    def halo(w, **kw):
        return plan(w, **kw)[0]["halo"]
    h = halo(wl.pair())
    assert h == {"ctas": 16, "threads": 160, "ghost": 21, "rods": 2, "bindings": True, "exchange": "cluster",
                 "steps_per_exchange": 1, "short_epochs_only": False}
    assert halo(wl.extensible())["ghost"] == 2          # no colour sweeps: radius 1, 2 steps
    assert halo(wl.sweep(16384))["steps_per_exchange"] == 3
    assert halo(wl.sweep(16384))["exchange"] == "grid"
    assert halo(wl.sweep(256))["exchange"] == "cluster"
    assert halo(wl.cantilever())["ctas"] == 1                   # one CTA, no ghosts (65 points)
    assert halo(wl.sweep(48))["short_epochs_only"]             # the one-warp kernel for K >= 32
    h16 = halo(wl.sweep(16))                                   # every one-CTA rod, K < 32 only
    assert h16["ctas"] == 1 and h16["short_epochs_only"]
    assert halo(wl.sweep(1024), force_tier=1, force_ctas=4) is None
    assert halo(wl.hair(2048)) is None
    w = wl.pair()
    w.add_bindings(0, 1, 0, stride=5)
    assert halo(w) is None
