"""world_size-2 gloo tests of the multi-GPU host plumbing (CPU only):
NCCL-id broadcast, max-over-ranks timing, slab partition, and the partitioned
schedule's halo bookkeeping with the halo data moved between two real
processes (oracle emulator per slab is not needed: each rank checks that the
planes it would receive are its neighbour's boundary planes)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2109_05410_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, _ = D.env_ranks()
        # 1) NCCL unique id broadcast from rank 0
        secret = bytes(((np.arange(128) * 7 + 3) % 256).astype(np.uint8))
        got = D.share_nccl_id(dist, r, lambda: secret)
        # 2) max / sum over ranks
        mx = D.max_over_ranks(dist, 1.5 + r)
        sm = D.sum_over_ranks(dist, 1.0)
        # 3) slabs tile the grid, and each rank's halo planes (h = 8) are exactly
        #    its neighbours' boundary planes
        nz, h = 64, 8
        z0, z1 = D.slab(r, w, nz)
        field = np.arange(nz, dtype=np.float32)           # one value per plane
        mine = torch.from_numpy(field[z0:z1].copy())
        top_send, bot_send = mine[:h].clone(), mine[-h:].clone()
        recv_top, recv_bot = torch.zeros(h), torch.zeros(h)
        ops = []
        if r > 0:
            ops += [dist.P2POp(dist.isend, top_send, r - 1), dist.P2POp(dist.irecv, recv_top, r - 1)]
        if r < w - 1:
            ops += [dist.P2POp(dist.isend, bot_send, r + 1), dist.P2POp(dist.irecv, recv_bot, r + 1)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        ok_top = r == 0 or np.array_equal(recv_top.numpy(), field[z0 - h:z0])
        ok_bot = r == w - 1 or np.array_equal(recv_bot.numpy(), field[z1:z1 + h])
        q.put((r, got == secret, mx, sm, (z0, z1), ok_top, ok_bot))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_plumbing(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, id_ok, mx, sm, sl, ok_top, ok_bot in res:
        assert id_ok
        assert mx == 1.5 + world - 1 and sm == world
        assert sl == (r * 64 // world, (r + 1) * 64 // world)
        assert ok_top and ok_bot


def test_slab_rejects_indivisible():
    from paper_2109_05410_b200 import dist as D
    with pytest.raises(ValueError):
        D.slab(0, 3, 64)
