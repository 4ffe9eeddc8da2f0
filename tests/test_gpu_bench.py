"""bench.py contract on the GPU: the JSON line's keys, and the multi-rank
path (rod shards, max over ranks, the results gather) run as two ranks on
one device over gloo -- the code a torchrun --nproc-per-node N launch takes,
minus NCCL."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "gpu_launches",
        "clocks")


def _line(out):
    return json.loads(out.strip().splitlines()[-1])


def test_bench_line_contract():
    out = subprocess.run([sys.executable, "bench.py", "--rods", "4096", "--steps", "5", "--warmup", "3",
                          "--no-single", "--no-cpu", "--e2e-steps", "2"], cwd=ROOT, check=True,
                         capture_output=True, text=True, timeout=600).stdout
    d = _line(out)
    for k in KEYS:
        assert k in d, k
    # a speculative batched step is two launches (the exact one over the redo list)
    assert d["gpu_launches"] in (5, 10) and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.5
    assert d["config"]["workload"].startswith("cfg5")


def test_bench_two_ranks_one_device():
    env = dict(os.environ, RSB_BENCH_DIST="gloo", RSB_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "2",
           "--rods", "4096", "--steps", "3", "--warmup", "3", "--no-single", "--e2e-steps", "1"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, check=True, capture_output=True, text=True,
                         timeout=600).stdout
    d = _line(out)
    assert d["n_gpus"] == 2 and d["config"]["rods_per_gpu"] == 2048
    assert d["nccl_gather_elems"] == 4096 * (129 * 3 + 128 * 4) and "cpu_baseline" not in d
    # the gathered positions + frames equal one process stepping the whole
    # batch through the same sequence of epochs, bit for bit
    one = subprocess.run([sys.executable, "bench.py", "--rods", "4096", "--steps", "3", "--warmup", "3",
                          "--no-single", "--no-cpu", "--e2e-steps", "1"], cwd=ROOT, check=True,
                         capture_output=True, text=True, timeout=600).stdout
    s = _line(one)
    assert s["nccl_gather_elems"] == d["nccl_gather_elems"]
    assert s["state_sha256"] == d["state_sha256"]
