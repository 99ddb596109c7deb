"""Which rates / shapes make the encode-stream race show (mismatching runs out of 12)."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import test_gpu_engine as E  # noqa: E402
from gpu_util import bits  # noqa: E402

for (nx, ny, nz, T, P) in ((40, 16, 80, 2, 20), (64, 64, 128, 2, 32)):
    u, up, m = E._fields(nx, ny, nz, 152)
    for rates in ((64, 3, 12), (16, 16, 16), (0, 0, 0), (0, 0, 16), (16, 16, 0), (3, 3, 3), (64, 64, 64)):
        calls = [2, 2, 2]
        ou, oup = E._run_oracle(u, up, m, T, rates, calls)
        bad = 0
        for rep in range(12):
            gu, gup, _, _ = E._run_gpu(u, up, m, T, P, rates, 1, calls, slots=2)
            bad += int(not (np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup))))
        print((nx, ny, nz, T, P), rates, "bad", bad, flush=True)
