"""One library build (OOCZ_LIB=...): C2 value at rate 16 and raw (store in HBM,
m resident), e2e at rate 16 (host store, serpentine + m resident, 3 slots);
plus the isolated kernels on one slab.  For A/B of compile-time variants
(build with `python -m paper_2109_05410_b200.build -DNAME --out lib.so`)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402

torch.cuda.set_device(0)
fields = bench.make_fields_c2()
steps = 10
cells = bench.NX * bench.NY * bench.NZ * bench.T * steps
out = [os.path.basename(os.environ.get("OOCZ_LIB", "liboocz.so"))]
for label, store, rates, serp, slots in (("zfp_dev", 1, (16,) * 3, 0, 2), ("raw_dev", 1, (0,) * 3, 0, 2),
                                         ("zfp_host", 0, (16,) * 3, 1, 3)):
    best = 0.0
    for _ in range(2):
        dev_s, st, evs, launches, ctx = bench.run_mode_c2(Z, store, rates, fields, 0, steps, 3, 0,
                                                         m_resident=1, serpentine=serp, slots=slots)
        Z.oocz_destroy(ctx)
        best = max(best, cells / dev_s / 1e9)
    out.append(f"{label} {best:.1f} G")
iso = bench.isolated_kernels(Z, fields, 6457.1)
for k in ("stencil25_kernel", "zfp_encode_kernel", "zfp_decode_kernel", "zfp_encode64_kernel", "zfp_decode64_kernel"):
    out.append("%s %.1f us" % (k.replace("_kernel", ""), iso[k]["ms"] * 1e3))
print("  ".join(out), flush=True)
