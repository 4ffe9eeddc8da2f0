#!/usr/bin/env python
"""Per-code-region stall breakdown of one kernel from an ncu report's source
page (SASS): instructions per unit and warp-stall samples by reason, in
address windows.

  python tools/ncu_regions.py rep.ncu-rep --units 65536 --window 0x1000
"""
import argparse
import collections
import csv
import io
import subprocess

REASONS = ["stall_wait", "stall_no_inst", "stall_long_sb", "stall_short_sb", "stall_math", "stall_mio",
           "stall_lg", "stall_selected", "stall_not_selected", "stall_branch_resolving", "stall_dispatch",
           "stall_barrier", "stall_membar"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--units", type=float, default=1.0)
    ap.add_argument("--window", type=lambda x: int(x, 0), default=0x1000)
    ap.add_argument("--ops", type=int, default=0, help="top opcodes per region")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = rows[1], rows[2:]
    ix = {k: h.index(k) for k in ["Address", "Source", "Instructions Executed"] + REASONS}
    base = None
    reg = collections.defaultdict(collections.Counter)
    ops = collections.defaultdict(collections.Counter)
    tot = collections.Counter()
    for r in data:
        if len(r) <= max(ix.values()):
            continue
        adr = int(r[ix["Address"]], 16)
        base = adr if base is None else base
        w = (adr - base) // a.window
        n = int(r[ix["Instructions Executed"]] or 0)
        reg[w]["inst"] += n
        src = r[ix["Source"]].split()
        if src:
            ops[w][src[1] if src[0].startswith("@") and len(src) > 1 else src[0]] += n
        for k in REASONS:
            v = int(r[ix[k]] or 0)
            reg[w][k] += v
            tot[k] += v
    allw = sum(tot.values())
    print("total stall samples", allw, {k[6:]: round(100 * v / allw, 1) for k, v in tot.most_common(8)})
    for w in sorted(reg):
        c = reg[w]
        s = sum(c[k] for k in REASONS)
        if s < 0.01 * allw:
            continue
        top = ", ".join(f"{k[6:]} {100 * c[k] / allw:.1f}" for k in sorted(REASONS, key=lambda k: -c[k])[:4])
        print(f"{hex(w * a.window):>8} {100 * s / allw:5.1f}%  inst/unit {c['inst'] / a.units:7.0f}  {top}")
        if a.ops:
            print("          ", ", ".join(f"{o} {n / a.units:.0f}" for o, n in ops[w].most_common(a.ops)))


if __name__ == "__main__":
    main()
