"""Repeat one stepper configuration against the oracle and count mismatches."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import test_gpu_engine as E  # noqa: E402
from gpu_util import bits  # noqa: E402

nx, ny, nz, T, P, rates, store = 40, 16, 80, 2, 20, (64, 3, 12), int(os.environ.get("STORE", "0"))
calls = [4, 7]
u, up, m = E._fields(nx, ny, nz, 152)
ou, oup = E._run_oracle(u, up, m, T, rates, calls)
for sets in (2, 3, 4):
    for mres in (0, 1):
        bad = 0
        for rep in range(int(os.environ.get("REPS", "20"))):
            gu, gup, _, _ = E._run_gpu(u, up, m, T, P, rates, store, calls, slots=4, slab_sets=sets, serpentine=0,
                                      m_resident=mres)
            bad += int(not (np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup))))
        print(os.path.basename(os.environ.get("OOCZ_LIB", "liboocz.so")), "store", store, "sets", sets,
              "m_resident", mres, "mismatching runs", bad, flush=True)
