"""Encode-stream race: mismatching runs (of 20) per rate vector, host store, 2 sets, m streamed."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import test_gpu_engine as E  # noqa: E402
from gpu_util import bits  # noqa: E402

nx, ny, nz, T, P = 40, 16, 80, 2, 20
u, up, m = E._fields(nx, ny, nz, 152)
for rates in ((64, 3, 12), (64, 3, 0), (64, 0, 12), (0, 3, 12), (16, 16, 12), (64, 64, 12), (3, 3, 12), (64, 3, 64)):
    calls = [4, 7]
    ou, oup = E._run_oracle(u, up, m, T, rates, calls)
    bad_u = bad_up = 0
    for rep in range(20):
        gu, gup, _, _ = E._run_gpu(u, up, m, T, P, rates, 0, calls, slots=4)
        bad_u += int(not np.array_equal(bits(gu), bits(ou)))
        bad_up += int(not np.array_equal(bits(gup), bits(oup)))
    print(rates, "bad u", bad_u, "bad u-", bad_up, flush=True)
