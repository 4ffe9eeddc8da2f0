P="python tools/prof_case.py"
for a in "sweep --n 1024 --k 100 --launches 3" ; do
 for cfg in "2 2" "4 1" "8 0" "16 0"; do set -- $cfg; $P $a --force-tier 1 --force-ctas $1 --force-variant $2 | cut -c1-60; done
done
for cfg in "2 2" "4 1" "8 0" "16 0"; do set -- $cfg; $P pair --k 10 --launches 20 --force-tier 1 --force-ctas $1 --force-variant $2 | cut -c1-60; done
for cfg in "2 1" "4 0" "8 0"; do set -- $cfg; $P extensible --k 10 --launches 20 --force-tier 1 --force-ctas $1 --force-variant $2 | cut -c1-60; done
for cfg in "2 0" "4 0"; do set -- $cfg; $P sweep --n 256 --k 100 --launches 3 --force-tier 1 --force-ctas $1 --force-variant $2 | cut -c1-60; done
for cfg in "8 2" "16 1"; do set -- $cfg; $P sweep --n 4096 --k 100 --launches 3 --force-tier 1 --force-ctas $1 --force-variant $2 | cut -c1-60; done
for cfg in "16 4" "32 2" "48 2"; do set -- $cfg; $P sweep --n 16384 --k 100 --launches 3 --force-tier 2 --force-ctas $1 --force-variant $2 | cut -c1-60; done
