python -c "
from paper_2509_04277_b200 import _lib
for mode in (0, 1, 2):
    for c in (2, 16, 48, 91, 148): print('grid_flags mode', mode, c, _lib.micro('grid_flags', c | (mode << 16)))
"
timeout 1200 python -m pytest tests/test_gpu_halo.py -q > gpurun_out/r02bi_pytest_halo.log 2>&1; echo pytest=$?
tail -30 gpurun_out/r02bi_pytest_halo.log
