#!/bin/bash
# One-off probe of the GPU box: hardware, host memory, host-link bandwidth.
mkdir -p gpurun_out
{
nvidia-smi; nvidia-smi topo -m; lscpu; free -g; ulimit -l; numactl -H 2>/dev/null; cat /proc/meminfo | head -5
nvidia-smi --query-gpu=index,name,pcie.link.gen.max,pcie.link.width.max,memory.total,clocks.max.sm --format=csv
python - <<'PY'
import torch, time
d = torch.device('cuda:0')
for size_mb in (64, 512, 2048):
    n = size_mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    g = torch.empty(n, dtype=torch.uint8, device=d)
    g2 = torch.empty(n, dtype=torch.uint8, device=d)
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    for mode in ('h2d', 'd2h', 'both'):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            if mode in ('h2d', 'both'):
                with torch.cuda.stream(s1): g.copy_(h, non_blocking=True)
            if mode in ('d2h', 'both'):
                with torch.cuda.stream(s2): h2.copy_(g2, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{mode} {size_mb}MiB: {reps*n/dt/1e9:.1f} GB/s per direction")
t0=time.perf_counter(); big = torch.empty(32<<30, dtype=torch.uint8, pin_memory=True); print("pin 32GiB s", time.perf_counter()-t0)
PY
} > gpurun_out/probe.txt 2>&1
