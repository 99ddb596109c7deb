"""Host-link probe: pinned H2D and D2H with 1 or 2 streams per direction, alone
and concurrent (does splitting a transfer across copy engines add bandwidth?)."""
import torch

n = 512 << 20
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
ss = [torch.cuda.Stream() for _ in range(4)]


def run(nh, nd, reps=5):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(ss[0])
        for s in ss:
            s.wait_event(e0)
        ends = []
        for k in range(nh):
            with torch.cuda.stream(ss[k]):
                lo, hi = k * n // nh, (k + 1) * n // nh
                d_a[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
        for k in range(nd):
            with torch.cuda.stream(ss[2 + k]):
                lo, hi = k * n // nd, (k + 1) * n // nd
                h_out[lo:hi].copy_(d_b[lo:hi], non_blocking=True)
        for s in ss:
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            ends.append(e)
        torch.cuda.synchronize()
        ms = max(e0.elapsed_time(e) for e in ends)
        best = ms if best is None else min(best, ms)
    return best


for nh, nd in ((1, 0), (2, 0), (0, 1), (0, 2), (1, 1), (2, 2), (2, 1), (1, 2)):
    ms = run(nh, nd)
    gb = n / (ms / 1e3) / 1e9
    print(f"h2d streams {nh} d2h streams {nd}: {ms:.2f} ms, {gb:.1f} GB/s per active direction", flush=True)
