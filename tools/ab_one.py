"""One library build (OOCZ_LIB=...): value at rate 16 and raw (store in HBM),
e2e at rate 16 (host store, 3 slots), headline schedule, C2; plus the isolated
stencil launch on one slab.  For A/B of compile-time variants."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402

torch.cuda.set_device(0)
fields = bench.make_fields(0, bench.NZ)
cells = bench.NX * bench.NY * bench.NZ * bench.T * 10
out = [os.path.basename(os.environ.get("OOCZ_LIB", "liboocz.so"))]
for label, store, rates, serp, slots in (("zfp_dev", 1, (16,) * 3, 0, 2), ("raw_dev", 1, (0,) * 3, 0, 2),
                                         ("zfp_host", 0, (16,) * 3, 1, 3)):
    best = 0.0
    for _ in range(2):
        dev_s, st, evs, launches, ctx = bench.run_mode(Z, store, rates, fields, 0, 1, None, 0, 10, 3, None, 0,
                                                      m_resident=1, serpentine=serp, slots=slots)
        Z.oocz_destroy(ctx)
        best = max(best, cells / dev_s / 1e9)
    out.append(f"{label} {best:.1f} G")
iso = bench.isolated_kernels(Z, fields, 6457.1)
for k in ("stencil25_kernel", "zfp_encode_kernel", "zfp_decode_kernel", "zfp_encode64_kernel", "zfp_decode64_kernel"):
    out.append("%s %.1f us" % (k.replace("_kernel", ""), iso[k]["ms"] * 1e3))
print("  ".join(out), flush=True)
