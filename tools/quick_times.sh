#!/bin/bash
# Quick device timings of the BASELINE cases (tools/prof_case.py), one line each.
cd "$(dirname "$0")/.."
t() { python tools/prof_case.py "$@" | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$*', '->', round(d['us_per_step'],3), 'us/step', d['plan']['tier'], 'v%d' % d['plan']['variant'])"; }
t hair --launches 10
t pair --k 10 --launches 20
t extensible --k 10 --launches 20
t cantilever --k 1000 --launches 3
for n in 16 64 256 1024 4096 16384; do t sweep --n $n --k 100 --launches 5; done
