#!/usr/bin/env python
"""Benchmark: CoRdE rod step on B200 (BASELINE.json metric).

Headline line (one JSON line on rank 0):
  metric  BASELINE.json's metric; value = batched element-steps/s of cfg5
          (65536 hair rods x 128 elements, fp64 mirror mode, K physics steps
          per launch), whole job over N GPUs, rods sharded across ranks
          (strong scaling: the 65536-rod batch is fixed), device-resident
          state, CUDA events on the launching stream, max over ranks.
  e2e     the same metric through Engine.run_epoch with the World's host
          numpy arrays: H2D of the state every step, D2H of the result.
  single_rod  (N == 1) µs per time step vs element count for one rod
          (cfg1, cfg2, cfg3 pair incl. the 1 kHz haptic frame loop, cfg4
          sweep) with the reference CPU core timed beside it.
  roofline    dominant kernel, HBM bytes against MEASURED_PEAKS.json.
  cpu_baseline  the unmodified reference package (baseline/_ref, its own
          Engine API; bench_reference.py) on all host cores, on the same
          full batch (5 timed steps).

`--impl reference` times the reference CPU implementation on the same
metric/config (rank 0 only; other ranks exit): bench_reference.batch_arm.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = ("µs/time-step vs #elements (1 rod); element-steps/s batched at "
          "1/2/4/8 GPUs")
TOTAL_RODS = 65536
ELEMENTS = 128


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32", "f64_fast"])
    ap.add_argument("--rods", type=int, default=TOTAL_RODS)
    ap.add_argument("--k", type=int, default=1, help="physics steps per launch")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-single", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-variant", type=int, default=-1)
    return ap.parse_args()


# ---- algorithmic bytes -----------------------------------

def algorithmic_bytes_per_rod(points, elems, real_bytes=8):
    """pos, vel, q, w read + written once per launch; rest + u* read once."""
    return real_bytes * (2 * (6 * points + 7 * elems) + 4 * elems)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# fp64 pipe instructions the fp64 mirror kernel issues per slot-step (ncu
# smsp__sass_thread_inst_executed_op_{dadd,dmul,dfma}_pred_on of the
# warp-per-rod batched kernel, profiles/r02n_ncu_full_warp_kernel.json
# capture: 5.85e9 per launch / 8.45e6 slots; the general variant-7 kernel
# issued 685): the compute cross-check
FP64_INST_PER_SLOT_STEP = 692


def fp64_peak():
    """Measured DADD issue rate (ops/s) on this device (rs_pipe_peak)."""
    from paper_2509_04277_b200 import _lib
    try:
        return _lib.pipe_peak(1)
    except Exception:
        return None


def pcie_bidir_gbs(nbytes=256 << 20):
    """Pinned host <-> device bandwidth with both directions in flight (the
    e2e path's bound: every epoch moves the full state both ways)."""
    import torch
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    both()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        both()
    e1.record()
    torch.cuda.synchronize()
    return 2 * 4 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9


def load_traffic(key):
    """(dram bytes read + written per launch, source) from the committed
    ncu --set full capture of the same workload, or (None, None)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh).get(key)
        return float(t["bytes"]), t["source"]
    except Exception:
        return None, None


# ---- clocks sampled during the timed region --------------------------------

class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML
    polled every 2 ms from a thread (the timed region is tens of ms), or
    `nvidia-smi -lms 100` when NVML cannot be loaded."""
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, index):
        self.index = index
        self.sm, self.mx, self.reasons = [], 0.0, set()
        self._stop = threading.Event()
        self._thread = None
        self.proc = None
        self.source = None

    def _nvml_loop(self, nv, h):
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for n, b in zip(self.NAMES, self.BITS):
                    if bits & b:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self._thread.start()
            self.source = "nvml"
            time.sleep(0.01)   # first samples before the region starts
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._thread = threading.Thread(target=self._smi_loop, daemon=True)
            self._thread.start()
            self.source = "nvidia-smi"
        except Exception:
            self.proc = None
        return self

    def _smi_loop(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                self.sm.append(float(parts[0]))
                self.mx = max(self.mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[2:6]):
                if v.lower() == "active":
                    self.reasons.add(n)

    def __exit__(self, *exc):
        self._stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self._thread is not None and self.source == "nvml":
            self._thread.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.mx or None, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": self.source}


# ---- distributed plumbing ---------------------------------------------------

def dist_env():
    """(world size, rank, device).  RSB_BENCH_DEVICE pins every rank to one
    device -- with RSB_BENCH_DIST=gloo that runs the multi-rank code path on
    a one-GPU box (a test of the sharding / max-over-ranks / gather logic,
    never a scaling number)."""
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "RSB_BENCH_DEVICE" in os.environ:
        local = int(os.environ["RSB_BENCH_DEVICE"])
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), local)


class Dist:
    def __init__(self, world, rank, local):
        self.world, self.rank, self.local = world, rank, local
        self.pg = None
        self.backend = os.environ.get("RSB_BENCH_DIST", "nccl")
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local)
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group(self.backend)
            self.dist = dist
            self.torch = torch
            self.pg = True

    def barrier(self):
        if self.pg:
            self.dist.barrier()

    def max(self, x):
        if not self.pg:
            return x
        t = self.torch.tensor([float(x)], device="cuda" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.dist.destroy_process_group()


class _CudaArray:
    """__cuda_array_interface__ view of a device buffer owned by the library."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": shape,
                                         "typestr": typestr, "version": 3}


# ---- single-rod latency measurements (rank 0, N = 1) ------------------------

# Dependent-chain length of each phase of one step (SURVEY §8(d) t_chain),
# counted from the kernel's critical path (rod_step.cuh; the longest chain
# from the phase's first shared-memory load to its last store):
#   d     dependent fp64 add/mul/fma    sqrt, rcp   the square root / 1/x
#   lds   shared-memory loads on the chain (DSMEM when the slot is remote)
# scatter:   pos load -> d -> |d|^2 (mul, 2 add) -> sqrt -> 1/|d| -> t
#            (div_fast: 3) -> er -> er.t (3) -> pair (4) -> ef (1)       16 d
#            (+6 for the stretch term of an extensible element)
# gather:    F = ff_own + ff_next(e-1) -> F.q (4) -> F - (F.q)q (2) ->
#            vec(conj(q)F) (4) -> x0.5 -> +jtau -jtau(e-1) -> tau - gyro ->
#            dt x -> div_fast (3) -> w + dw                            20 d
# integrate: q (x) (0,w) (4) -> q + h dq (2) -> |q|^2 (4) -> sqrt -> 1/x
#            -> div_fast (3)                                            15 d
# colour:    v loads -> vb - va -> x n -> +, + -> + bias -> lambda
#            (mul, fma, fma) -> im lambda -> x n -> va -                11 d
# binding:   v loads -> vrel (4) -> + bias -> lambda (3) -> w lam n (2) -> +  11 d
# contact:   normal impulse with accumulator + box friction            ~24 d + 1 div
PHASE_CHAIN = {
    "scatter": {"d": 16, "sqrt": 1, "rcp": 1, "lds": 1},
    "gather": {"d": 20, "lds": 1},
    "integrate": {"d": 15, "sqrt": 1, "rcp": 1, "lds": 1},
    "colour": {"d": 11, "lds": 1},
    "binding": {"d": 11, "lds": 1},
    "contact": {"d": 24, "div": 1, "lds": 1},
}


def micro_latencies():
    """Measured dependent latencies (cycles) and the SM clock (rs_micro)."""
    from paper_2509_04277_b200 import _lib
    lat = {}
    for key, kind in (("d", "dadd"), ("sqrt", "sqrt_add"), ("rcp", "rcp"), ("div", "div"),
                      ("lds", "lds"), ("dsmem", "dsmem")):
        cyc, ns = _lib.micro(kind)
        lat[key] = cyc
        if key == "d" and ns > 0:
            lat["ghz"] = cyc / ns
    lat["sqrt"] = max(lat["sqrt"] - lat["d"], 0.0)   # the kind-4 chain is sqrt + add
    return lat


def barrier_ns(plan):
    """Measured cost of one phase barrier of a plan's tier (rs_micro)."""
    from paper_2509_04277_b200 import _lib
    if plan["tier"] in ("cluster", "grid"):
        return _lib.micro("cluster_barrier", max(2, min(16, plan["ctas"])))[1]
    return _lib.micro("bar_sync", plan["threads"])[1]


def latency_floor(plan, us, k, lat, iters=10, ext=False, t_launch_us=0.0):
    """t_floor = n_sync t_sync + t_chain + t_launch / K.
    n_sync: the barriers the kernel issues per step (from the plan: 3 + I x
    (2 colour phases when any element is distance-projected, + contacts,
    self-collision pairs, bindings, grabs)); t_sync: the tier's measured
    barrier; t_chain: the phases' dependent chains at the measured latencies
    (PHASE_CHAIN; halo loads of a multi-CTA tier are DSMEM reads)."""
    n_sync = plan["sync_per_step"]
    t_sync = barrier_ns(plan)
    halo = plan.get("halo")
    if halo and halo.get("short_epochs_only") and k >= 32:
        halo = None   # (long epochs of such rods run the speculative CTA kernel)
    if halo:
        # wide-halo kernel (rod_halo.cuh): every phase ends at a CTA barrier
        # of halo["threads"], the step at one inter-CTA exchange (cluster
        # barrier, or the grid's neighbour flags)
        from paper_2509_04277_b200 import _lib
        sweeps = plan["any_dist"] or plan["bindings"]
        n_sync = 1 + ((1 + iters * (2 + (1 if plan["bindings"] else 0))) if sweeps else 0) + \
            (1 if halo["exchange"] == "grid" else 0)
        t_sync = _lib.micro("bar_sync", halo["threads"])[1]
        if halo["ctas"] > 1:
            t_x = (_lib.micro("grid_flags", halo["ctas"])[1] if halo["exchange"] == "grid"
                   else _lib.micro("cluster_barrier", halo["ctas"])[1])
        else:
            t_x = t_sync

    def cyc(ph, extra_d=0):
        # (a multi-CTA tier's halo loads are DSMEM reads; its measured t_sync
        # already includes one DSMEM read per phase, so they count as LDS here)
        c = PHASE_CHAIN[ph]
        ld = lat["lds"]
        return ((c.get("d", 0) + extra_d) * lat["d"] + c.get("sqrt", 0) * lat["sqrt"] +
                c.get("rcp", 0) * lat["rcp"] + c.get("div", 0) * lat["div"] + c.get("lds", 0) * ld)
    chain = cyc("scatter", 6 if ext else 0) + cyc("gather") + cyc("integrate")
    per_it = 0.0
    if plan["sync_per_iteration"] >= 2 and (plan["any_dist"] or plan["bindings"]):
        per_it += 2 * cyc("colour")
    if plan["bindings"]:
        per_it += cyc("binding")
    if plan["contacts"]:
        per_it += cyc("contact")
    chain += iters * per_it
    t_chain_us = chain / lat["ghz"] / 1e3
    t_sync_us = n_sync * t_sync / 1e3
    out = {"n_sync": n_sync, "t_sync_ns": t_sync}
    if halo:
        t_sync_us += t_x / 1e3
        out.update({"n_exchange": 1, "t_exchange_ns": t_x, "exchange": halo["exchange"],
                    "model": "n_sync t_bar(CTA) + t_exchange + t_chain + t_launch/K"})
    else:
        out["model"] = "n_sync t_sync + t_chain + t_launch/K"
    floor = t_sync_us + t_chain_us + t_launch_us / k
    out.update({"sync_us": t_sync_us, "t_chain_us": t_chain_us, "chain_cycles": chain,
                "t_launch_us": t_launch_us, "k": k, "t_floor_us": floor, "frac": floor / us})
    return out


def single_rod_suite(precision):
    import bench_reference as br
    from paper_2509_04277_b200 import workloads as wl
    from paper_2509_04277_b200.engine import Engine

    def device_us(make, k, launches):
        w = make()
        with Engine(w, precision=precision) as eng:
            dev = eng.device_world
            dev.run(k)
            dev.synchronize()
            dev.timer_start()
            for _ in range(launches):
                dev.run(k)
            dev.timer_stop()
            ms = dev.timer_ms()
            plan = eng.plan()["groups"][0]
        return ms * 1e3 / (k * launches), plan

    lat = micro_latencies()
    # launch overhead: one launch per step minus the per-step cost at K = 100
    us1, _ = device_us(lambda: wl.sweep(16), 1, 200)
    us100, _ = device_us(lambda: wl.sweep(16), 100, 20)
    t_launch = max(us1 - us100, 0.0)
    out = {"latencies_cycles": lat, "t_launch_us": t_launch}

    def row(name, make, k, launches, cpu_name, cpu_args=(), cpu_steps=200, ext=False, **extra):
        us, plan = device_us(make, k, launches)
        r = {"us_per_step": us, "k": k, "tier": plan["tier"], "ctas": plan["ctas"], "halo": plan.get("halo"),
             "roofline": latency_floor(plan, us, k, lat, ext=ext, t_launch_us=t_launch)}
        r.update(br.single_rod_cpu(cpu_name, cpu_args, steps=cpu_steps))
        r["speedup_vs_cpu"] = r["cpu_us_per_step"] / us
        r.update(extra)
        out[name] = r
        return r

    row("cfg1_cantilever_64", wl.cantilever, 1000, 3, "cantilever", cpu_steps=1000)
    row("cfg2_extensible_512", wl.extensible, 10, 100, "extensible", ext=True)
    pair = row("cfg3_pair_2x512", wl.pair, 10, 100, "pair", cpu_steps=100)
    pair["steps_per_s"] = 1e6 / pair["us_per_step"]
    # haptic frame loop: commands in, K = 10 steps (1 ms simulated), state out
    w = wl.pair()
    frames = []
    with Engine(w, precision=precision) as eng:
        for i in range(1100):
            t0 = time.perf_counter()
            eng.post_command("insert_velocity", rod=0, value=0.05 + 1e-4 * (i % 7),
                             axis=(0.0, 0.0, 1.0))
            eng.run_epoch(10)
            tip = w.positions[w.rod_infos[0].point_offset + w.rod_infos[0].num_points - 1]
            frames.append(time.perf_counter() - t0)
            _ = float(tip[2])
    frames = np.array(frames[100:]) * 1e6
    pair["haptic_frame_us"] = {"median": float(np.median(frames)),
                               "p99": float(np.percentile(frames, 99)),
                               "frames": int(frames.size),
                               "rate_hz_median": float(1e6 / np.median(frames))}
    # the paper's insertion scene: mesh contacts
    row("insertion_128_tube", wl.insertion, 100, 10, "insertion", mesh_triangles=15360,
        collision_interval=4)
    sweep = {}
    for n in (16, 64, 256, 1024, 4096, 16384):
        r = {}
        for k in (1, 10, 100):
            launches = max(2, min(200, 2000 // k))
            us, plan = device_us(lambda: wl.sweep(n), k, launches)
            r[f"k{k}"] = us
        r["tier"] = plan["tier"]
        r["ctas"] = plan["ctas"]
        r["halo"] = plan.get("halo")
        r["roofline_k100"] = latency_floor(plan, r["k100"], 100, lat, t_launch_us=t_launch)
        r["roofline_k1"] = latency_floor(plan, r["k1"], 1, lat, t_launch_us=t_launch)
        c = br.single_rod_cpu("sweep", (n,), steps=max(3, 20000 // n), par_steps=max(3, 5000 // n))
        r.update(c)
        r["speedup_vs_cpu_k100"] = c["cpu_us_per_step"] / r["k100"]
        sweep[str(n)] = r
    out["cfg4_sweep_us_per_step"] = sweep
    return out


# ---- arms ---------------------------------------------------------------------

def run_reference(args):
    """The reference arm: the unmodified reference package (baseline/_ref)
    through its own API on the host cores, the same cfg5 batch and metric
    (bench_reference.batch_arm); rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import bench_reference as br
    procs = os.cpu_count() or 1
    r = br.batch_arm(args.rods, procs, steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"],
        "unit": "element-steps/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg5 hair: 65536 rods x 128 elements, roots clamped, "
                               "sharded over host processes",
                   "rods": args.rods, "elements_per_rod": ELEMENTS, "steps_per_launch": 1,
                   "iterations": 10, "dt": 1e-4},
        "cpu_baseline": dict(r),
        "e2e": {"value": r["value"], "unit": "element-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def compute_roofline(rods, launch_ms, precision):
    """fp64 pipe cross-check: issued fp64 instructions (ncu count per
    slot-step) per second against the measured DADD issue peak."""
    if precision == "f32":
        return None
    peak = fp64_peak()
    slots = rods * (ELEMENTS + 1)
    achieved = FP64_INST_PER_SLOT_STEP * slots / (launch_ms * 1e-3)
    return {"pipe": "fp64", "achieved": achieved, "peak": peak, "unit": "inst/s",
            "frac": (achieved / peak) if peak else None,
            "inst_per_slot_step": FP64_INST_PER_SLOT_STEP}


def run_ours(args):
    world, rank, local = dist_env()
    D = Dist(world, rank, local)
    from paper_2509_04277_b200 import workloads as wl
    from paper_2509_04277_b200._lib import RS_STATE
    from paper_2509_04277_b200.engine import Engine

    first, per = wl.shard(args.rods, world, rank)
    t_build = time.perf_counter()
    w = wl.hair(per, ELEMENTS, first=first)
    t_build = time.perf_counter() - t_build
    eng = Engine(w, precision=args.precision, device=local,
                 force_variant=args.force_variant)
    dev = eng.device_world
    plan = eng.plan()
    P, E = w.num_points, w.num_elements
    real = 4 if args.precision == "f32" else 8

    # ---- device-resident timed region --------------------------------
    for _ in range(args.warmup):
        dev.run(args.k)
    dev.synchronize()
    D.barrier()
    launches0 = dev.launch_count()
    with ClockSampler(local) as clk:
        dev.timer_start()
        for _ in range(args.steps):
            dev.run(args.k)
        dev.timer_stop()
        ms = dev.timer_ms()
    dev.synchronize()
    D.barrier()
    launches = dev.launch_count() - launches0
    ms_max = D.max(ms)
    elem_steps = args.rods * ELEMENTS * args.k * args.steps
    value = elem_steps / (ms_max * 1e-3)

    # roofline: algorithmic bytes of one step over the time of one step --
    # the speculative launch plus the exact launch over its redo list (empty
    # after the first step from rest; a few microseconds), so per step, not
    # per launch
    launch_ms = ms / max(args.steps, 1)
    bytes_per_launch = per * algorithmic_bytes_per_rod(ELEMENTS + 1, ELEMENTS, real)
    peak, peak_src = load_peaks()
    achieved = bytes_per_launch / (launch_ms * 1e-3) / 1e9
    traffic, traffic_src = load_traffic(f"hair_{args.precision}_k{args.k}_r{per}")

    # ---- e2e through the public API (host numpy arrays) --------------
    state_bytes = 8 * (6 * P + 7 * E)
    control_bytes = w.driver_velocity.nbytes + w.driver_rotation.nbytes + \
        w.grab_target.nbytes + w.grab_point.nbytes + w.grab_active.nbytes
    eng.run_epoch(args.k)
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        eng.run_epoch(args.k)
    e2e_s = time.perf_counter() - t0
    e2e_max = D.max(e2e_s)
    e2e_value = args.rods * ELEMENTS * args.k * args.e2e_steps / e2e_max
    pcie = pcie_bidir_gbs() if rank == 0 else None
    # (the control arrays are compared with their last upload on the host
    # every epoch and sent only when they changed: not copied here)
    e2e_gbs = state_bytes * 2 * args.e2e_steps / e2e_max / 1e9
    # the same public call with 10 steps per epoch: one state round trip over
    # PCIe per 10 steps (the host arrays are authoritative between epochs)
    eng.run_epoch(10)
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(2):
        eng.run_epoch(10)
    e2e10_max = D.max(time.perf_counter() - t0)
    e2e_value_k10 = args.rods * ELEMENTS * 10 * 2 / e2e10_max

    # the same batch at K = 10 steps per launch (state stays on chip)
    dev.run(10)
    dev.synchronize()
    dev.timer_start()
    for _ in range(3):
        dev.run(10)
    dev.timer_stop()
    ms10 = D.max(dev.timer_ms())
    value_k10 = args.rods * ELEMENTS * 30 / (ms10 * 1e-3)

    # ---- NCCL gather of the final state (results only) ---------------
    # positions (P,3) and frames (E,4) of every rank's shard, concatenated in
    # rod order on rank 0; the digest of the gathered bits
    # lets the tests compare an N-rank run with a single-process one
    import hashlib
    import torch
    gathered = 0
    digest = hashlib.sha256()
    tdt = torch.float64 if real == 8 else torch.float32
    for which, n in ((0, P * 3), (2, E * 4)):
        src = torch.as_tensor(_CudaArray(dev.device_ptr(which), (n,), "<f8" if real == 8 else "<f4"),
                              device=f"cuda:{local}")
        assert src.dtype == tdt
        if world > 1:
            if D.backend != "nccl":   # gloo test path: gather through host memory
                src = src.cpu()
            out = torch.empty(world * n, dtype=src.dtype, device=src.device)
            D.dist.all_gather_into_tensor(out, src.contiguous())
        else:
            out = src
        torch.cuda.synchronize()
        gathered += int(out.numel())
        if rank == 0:
            digest.update(out.cpu().numpy().tobytes())

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "element-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": {"f64": "f64", "f32": "f32", "f64_fast": "f64"}[args.precision],
            "data": "synthetic",
            "config": {"workload": "cfg5 hair: 65536 rods x 128 elements, roots "
                                   "clamped, sharded over ranks",
                       "rods": args.rods, "rods_per_gpu": per,
                       "elements_per_rod": ELEMENTS, "steps_per_launch": args.k,
                       "iterations": 10, "dt": 1e-4,
                       "parity_mode": args.precision,
                       "l2": "inputs larger than L2 (state %.0f MB/GPU)" % (state_bytes / 1e6),
                       "plan": plan["groups"]},
            "e2e": {"value": e2e_value, "unit": "element-steps/s", "value_k10": e2e_value_k10,
                    "h2d_bytes_per_step": state_bytes,
                    "d2h_bytes_per_step": state_bytes,
                    "control_bytes_checked_per_step": control_bytes,
                    "steps": args.e2e_steps, "api": "Engine.run_epoch",
                    "roofline": {"bound": "pcie", "achieved": e2e_gbs, "peak": pcie,
                                 "unit": "GB/s", "frac": (e2e_gbs / pcie) if pcie else None,
                                 "peak_source": "pinned H2D+D2H both in flight, measured in this run"}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src, "peak_source": peak_src,
                         "bytes_per_launch": bytes_per_launch,
                         "launch_ms": launch_ms,
                         "launches_per_step": launches / max(args.steps, 1)},
            "compute_roofline": compute_roofline(per, launch_ms, args.precision),
            "value_k10": value_k10,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "build_s": t_build,
        }
        line["nccl_gather_elems"] = gathered
        line["state_sha256"] = digest.hexdigest()
        if world == 1 and not args.no_cpu:
            import bench_reference as br
            line["cpu_baseline"] = br.batch_arm(args.rods, os.cpu_count() or 1, steps=5, warmup=1)
        if world == 1 and not args.no_single:
            line["single_rod"] = single_rod_suite(args.precision)
        print(json.dumps(line))
    eng.close()
    D.close()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
