"""The multi-process NCCL transport: one process per GPU,
oocz_get_nccl_id on rank 0 broadcast over a gloo group, oocz_create(world=2)
with the id, each rank stepping its own z-slab and exchanging compressed
radius-4 halos with ncclSend / ncclRecv (one communicator per direction).
The concatenated result must equal the oracle (= world 1) bit for bit.  A
second case kills one rank before it steps: the other must return OOCZ_ENCCL
from its watchdog (OOCZ_NCCL_TIMEOUT_S) instead of hanging.

Needs >= 2 GPUs (NCCL refuses two ranks on one device); skipped otherwise --
the same protocol runs on one GPU through the in-process local group
(test_gpu_engine.py, test_gpu_fp64.py)."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth

pytestmark = pytest.mark.gpu


def _ngpus() -> int:
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


needs2 = pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (NCCL: one rank per device)")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


NX, NY, NZ = 32, 24, 128


def _fields():
    u = synth.dense(NX, NY, NZ, seed=31)
    return u, (u * np.float32(0.95)).astype(np.float32), synth.layered(NX, NY, NZ)


def _worker(rank, world, port, case, outdir):
    import torch
    import torch.distributed as dist
    from paper_2109_05410_b200 import dist as D
    from paper_2109_05410_b200 import oocz as Z
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    T, P, rates, opts, n, die = case
    nid = D.share_nccl_id(dist, rank, Z.oocz_get_nccl_id)
    cfg = Z.oocz_default_config(NX, NY, NZ, tb=T, block_planes=P, rate=list(rates), **opts)
    ctx = Z.oocz_create(cfg, rank, world, nid, rank)
    S = NZ // world
    u, up, m = _fields()
    status = "ok"
    try:
        for f, a in ((Z.OOCZ_U, u), (Z.OOCZ_UPREV, up), (Z.OOCZ_M, m)):
            Z.oocz_set_field(ctx, f, np.ascontiguousarray(a[rank * S:(rank + 1) * S]))
        if die and rank == 1:
            os._exit(0)                                  # a dead peer: never steps
        try:
            Z.oocz_step(ctx, n)
            np.save(os.path.join(outdir, f"u{rank}.npy"), Z.oocz_get_field(ctx, Z.OOCZ_U, np.empty((S, NY, NX), np.float32)))
            np.save(os.path.join(outdir, f"up{rank}.npy"),
                    Z.oocz_get_field(ctx, Z.OOCZ_UPREV, np.empty((S, NY, NX), np.float32)))
            st = Z.oocz_get_stats(ctx)
            assert st["halo_bytes"] > 0
        except Z.OoczError as e:
            status = f"error {e.status}"
    finally:
        with open(os.path.join(outdir, f"status{rank}.txt"), "w") as fh:
            fh.write(status)
        if not (die and rank == 0):
            Z.oocz_destroy(ctx)
        os._exit(0)


def _spawn(case, tmp_path, timeout=240):
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout)
        if p.is_alive():
            p.kill()
            raise AssertionError("a rank hung")


@needs2
@pytest.mark.parametrize("T,P,rates,opts,n", [
    (2, 16, (16, 16, 16), {}, 7),
    (2, 16, (8, 12, 16), dict(serpentine=1, m_resident=1, slots=3), 9),
    (1, 8, (0, 0, 0), dict(store=1), 5),
    (4, 32, (16, 16, 16), dict(serpentine=1), 12),
])
def test_nccl_two_ranks_bit_identical_to_oracle(T, P, rates, opts, n, tmp_path):
    _spawn((T, P, rates, opts, n, False), tmp_path)
    for r in range(2):
        assert (tmp_path / f"status{r}.txt").read_text() == "ok"
    gu = np.concatenate([np.load(tmp_path / f"u{r}.npy") for r in range(2)])
    gup = np.concatenate([np.load(tmp_path / f"up{r}.npy") for r in range(2)])
    u, up, m = _fields()
    ou, oup = oracle.run(u, up, m, T, rates, n)
    assert np.array_equal(gu.view(np.uint32), ou.view(np.uint32))
    assert np.array_equal(gup.view(np.uint32), oup.view(np.uint32))


@needs2
def test_nccl_dead_peer_is_an_error_not_a_hang(tmp_path, monkeypatch):
    monkeypatch.setenv("OOCZ_NCCL_TIMEOUT_S", "10")
    _spawn((2, 16, (16, 16, 16), {}, 4, True), tmp_path, timeout=180)
    assert (tmp_path / "status0.txt").read_text() == "error -8"      # OOCZ_ENCCL
