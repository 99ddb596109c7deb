"""Pinned host memory from oocz_host_alloc: large buffers are THP-backed
mappings registered with cudaHostRegister, small ones cudaHostAlloc; both must
be usable as pinned copy sources / targets and freed through oocz_host_free."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2109_05410_b200 import oocz as Z

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nbytes", [64 << 20, (1 << 30) + (3 << 20)])
def test_host_alloc_round_trip(nbytes):
    p = Z.oocz_host_alloc(nbytes)
    try:
        assert p and p % 4096 == 0
        host = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)), shape=(nbytes,))
        rng = np.random.default_rng(nbytes % 97)
        # the first, a middle and the last 32 MB of the buffer, through the device
        for off in (0, nbytes // 2 // 4096 * 4096, nbytes - (32 << 20)):
            pat = rng.integers(0, 256, 32 << 20, dtype=np.uint8)
            host[off:off + pat.size] = pat
            t = torch.from_numpy(host[off:off + pat.size])      # shares the pinned memory
            d = t.to("cuda", non_blocking=True)
            torch.cuda.synchronize()
            d.add_(1)
            t.copy_(d, non_blocking=True)
            torch.cuda.synchronize()
            assert np.array_equal(host[off:off + pat.size], (pat + 1).astype(np.uint8))
    finally:
        Z.oocz_host_free(p)


def test_host_store_context_uses_pinned_store():
    """A host-store context whose store exceeds 1 GiB (the THP path) steps and
    reads back like a small one: same bits as the device store."""
    nx = ny = 1024
    nz = 256                                   # u, u-, m at rate 32: 3 x 1 GiB + stores
    rng = np.random.default_rng(3)
    u = (rng.standard_normal((nz, ny, nx)) * 0.1).astype(np.float32)
    m = np.full((nz, ny, nx), 0.05, np.float32)
    out = {}
    for store in (Z.OOCZ_STORE_HOST, Z.OOCZ_STORE_DEVICE):
        cfg = Z.oocz_default_config(nx, ny, nz, tb=2, block_planes=64, rate=[32, 32, 32], store=store)
        ctx = Z.oocz_create(cfg)
        try:
            Z.oocz_set_field(ctx, Z.OOCZ_U, u)
            Z.oocz_set_field(ctx, Z.OOCZ_UPREV, u)
            Z.oocz_set_field(ctx, Z.OOCZ_M, m)
            Z.oocz_step(ctx, 4)
            out[store] = Z.oocz_get_field(ctx, Z.OOCZ_U, np.empty_like(u))
            if store == Z.OOCZ_STORE_HOST:
                assert Z.oocz_get_stats(ctx)["host_bytes_pinned"] >= 3 * (1 << 30)
        finally:
            Z.oocz_destroy(ctx)
    assert np.array_equal(out[Z.OOCZ_STORE_HOST].view(np.uint32), out[Z.OOCZ_STORE_DEVICE].view(np.uint32))


def test_host_alloc_without_thp_falls_back_to_cudahostalloc():
    """OOCZ_NO_THP=1 (read at allocation time): the >= 1 GiB path is cudaHostAlloc
    instead, usable and freed the same way (a fresh process: the variable is read
    by the library, not cached by this one)."""
    import os
    import subprocess
    import sys
    code = (
        "import ctypes as C, numpy as np, torch\n"
        "from paper_2109_05410_b200 import oocz as Z\n"
        "n = (1 << 30) + (1 << 20)\n"
        "p = Z.oocz_host_alloc(n)\n"
        "h = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)), shape=(n,))\n"
        "h[-4096:] = 7\n"
        "d = torch.from_numpy(h[-4096:]).to('cuda')\n"
        "assert int(d.sum()) == 7 * 4096\n"
        "Z.oocz_host_free(p)\n"
        "print('ok')\n")
    env = dict(os.environ, OOCZ_NO_THP="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
