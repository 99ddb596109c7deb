"""Host-link rate out of a large pinned arena vs a small pinned buffer, and
with the arena's pages as transparent huge pages (mmap + madvise(HUGEPAGE) +
cudaHostRegister) vs cudaHostAlloc: the C3 headline's store is a 155 GB
arena, and on some boxes its copies run below the small-buffer probe.

  python tools/link_probe_arena.py [GB]
"""
import ctypes
import json
import mmap
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05410_b200 import oocz as Z  # noqa: E402

GB = float(sys.argv[1]) if len(sys.argv) > 1 else 64.0
nbytes = int(GB * 1e9) // (2 << 20) * (2 << 20)
chunk = 2 << 30
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
from cuda.bindings import runtime as rt  # noqa: E402
out = {"thp": open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
       "thp_defrag": open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip()}
d = torch.empty(chunk, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()


def rate(ptr, offsets, h2d=True):
    best = []
    for off in offsets:
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        if h2d:
            rt.cudaMemcpyAsync(d.data_ptr(), ptr + off, chunk, rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s.cuda_stream)
        else:
            rt.cudaMemcpyAsync(ptr + off, d.data_ptr(), chunk, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        best.append(chunk / (a.elapsed_time(b) / 1e3) / 1e9)
    return round(sum(best) / len(best), 2), round(min(best), 2), round(max(best), 2)


offs = [int(i * (nbytes - chunk) / 7) // 4096 * 4096 for i in range(8)]
small = torch.empty(chunk, dtype=torch.uint8, pin_memory=True)
out["small_2GiB_h2d"] = rate(small.data_ptr(), [0] * 4)
out["small_2GiB_d2h"] = rate(small.data_ptr(), [0] * 4, h2d=False)
t0 = time.time()
p = Z.oocz_host_alloc(nbytes)
out["hostalloc_s"] = round(time.time() - t0, 1)
out["hostalloc_h2d"] = rate(p, offs)
out["hostalloc_d2h"] = rate(p, offs, h2d=False)
Z.oocz_host_free(p)
t0 = time.time()
MAP_PRIVATE, MAP_ANON = 0x02, 0x20
q = libc.mmap(None, nbytes + (2 << 20), 3, MAP_PRIVATE | MAP_ANON, -1, 0)
q2 = (q + (2 << 20) - 1) // (2 << 20) * (2 << 20)
out["madvise_rc"] = libc.madvise(ctypes.c_void_p(q2), nbytes, 14)      # MADV_HUGEPAGE
ctypes.memset(q2, 0, 1)
r = rt.cudaHostRegister(q2, nbytes, 0)
out["register_rc"] = str(r)
out["register_s"] = round(time.time() - t0, 1)
ah = [l for l in open("/proc/meminfo") if l.startswith("AnonHugePages")]
out["AnonHugePages"] = ah[0].strip() if ah else None
out["thp_h2d"] = rate(q2, offs)
out["thp_d2h"] = rate(q2, offs, h2d=False)
print(json.dumps(out))
