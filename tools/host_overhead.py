"""Host enqueue time of oocz_step (wall) against its device time, per config."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402

torch.cuda.set_device(0)
for n, P, T, store in ((512, 128, 4, 1), (512, 128, 4, 0), (64, 32, 2, 1), (64, 32, 2, 0), (128, 32, 4, 1)):
    u = synth.dense(n, n, n, seed=1)
    m = synth.layered(n, n, n)
    cfg = Z.oocz_default_config(n, n, n, tb=T, block_planes=P, rate=[16] * 3, store=store, m_resident=1)
    with Z.Stepper(cfg) as s:
        s.set(u, u, m)
        s.step(3 * T)
        st0 = s.stats()
        s.step(10 * T)
        st = s.stats()
    wall = st["step_ms"] - st0["step_ms"]
    print(f"{n}^3 P={P} T={T} store={'dev' if store else 'host'}: device {st['last_step_device_ms']:.2f} ms, "
          f"host wall {wall:.2f} ms for 10 sweeps ({st['kernel_launches'] - st0['kernel_launches']} launches)",
          flush=True)
