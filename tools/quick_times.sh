#!/bin/bash
# Quick device timings of the BASELINE cases (tools/prof_case.py), one line each.
cd "$(dirname "$0")/.."
python tools/prof_case.py hair --launches 5
python tools/prof_case.py pair --k 10 --launches 20
python tools/prof_case.py extensible --k 10 --launches 20
python tools/prof_case.py cantilever --k 1000 --launches 3
for n in 256 1024 4096 16384; do python tools/prof_case.py sweep --n $n --k 100 --launches 3; done
python tools/prof_case.py hair --launches 5 --force-variant 6
python tools/prof_case.py hair --launches 5 --force-variant 7
