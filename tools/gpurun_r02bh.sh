timeout 1200 python -m pytest tests/test_gpu_halo.py -x -q > gpurun_out/r02bh_pytest_halo.log 2>&1; echo pytest=$?
tail -30 gpurun_out/r02bh_pytest_halo.log
python -c "
from paper_2509_04277_b200 import _lib
for c in (2, 16, 48, 91, 148): print('grid_flags', c, _lib.micro('grid_flags', c))
for c in (2, 16): print('cluster', c, _lib.micro('cluster_barrier', c))
for t in (64, 128, 160, 224, 320): print('bar', t, _lib.micro('bar_sync', t))
"
