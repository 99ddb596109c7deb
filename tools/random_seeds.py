"""Extra seeds for the randomized stepper parity sweep (tests/test_gpu_engine.py
test_random_configurations_bit_exact, 96 configurations per seed)."""
import os
import sys
import time
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(R, "tests"))
sys.path.insert(0, R)
import test_gpu_engine as E  # noqa: E402
import test_gpu_fp64 as F  # noqa: E402

seeds = [int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "11,12,13,14").split(",")]
for sd in seeds:
    t = time.time()
    E.test_random_configurations_bit_exact(sd)
    if os.environ.get("PARTITIONED", "0") == "1":
        E.test_random_partitioned_configurations_bit_exact(sd)
    if os.environ.get("F64", "0") == "1":
        F.test_random_configurations64_bit_exact(sd)
    print("seed", sd, "ok", round(time.time() - t, 1), "s", flush=True)
