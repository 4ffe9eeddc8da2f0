for args in "sweep --n 512 --k 10 --launches 20 --force-tier 0" "sweep --n 512 --k 10 --launches 20" "pair --k 10 --launches 20" "sweep --n 256 --k 10 --launches 20"; do
timeout 120 python tools/prof_case.py $args 2>&1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read().strip().splitlines()[-1]); print('$args', '->', round(d['us_per_step'],2), d['plan']['tier'], d['plan']['ctas'], d['plan']['threads'])"
done
