"""GPU stencil parity: the TMA-staged 25-point kernel vs the fp32 oracle.
The arithmetic order is prescribed (R5), so the bar is bit-exact
(stronger than the north star's 1e-5 per step / 1e-4 after 100 steps)."""
import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth
from gpu_util import Z, bits, to_dev

pytestmark = pytest.mark.gpu


def _state(nx, ny, nz, seed):
    u = synth.dense(nx, ny, nz, seed=seed)
    up = synth.dense(nx, ny, nz, seed=seed + 100) * np.float32(0.5)
    m = synth.layered(nx, ny, nz)
    return u.astype(np.float32), up.astype(np.float32), m


@pytest.mark.parametrize("shape", [(64, 64, 64), (136, 10, 37), (12, 20, 9), (256, 24, 70), (4, 4, 4)])
def test_single_step_bit_exact(shape):
    import torch
    nx, ny, nz = shape
    u, up, m = _state(nx, ny, nz, 7)
    want = oracle.step(u, up, m)
    du, dup, dm = to_dev(u), to_dev(up), to_dev(m)
    z = Z()
    z.oocz_stencil_step_planes(du, dup, dm, nx, ny, nz, z.default_coeffs(), 0, nz, 0, nz,
                               torch.cuda.current_stream())
    torch.cuda.synchronize()
    got = dup.cpu().numpy()
    assert np.array_equal(bits(got), bits(want))
    assert np.array_equal(du.cpu().numpy(), u)          # u is read-only


@pytest.mark.parametrize("n", [1, 2, 5, 10])
def test_many_steps_bit_exact(n):
    import torch
    nx, ny, nz = 72, 40, 48
    u, up, m = _state(nx, ny, nz, 8)
    a, b = u, up
    for _ in range(n):
        a, b = oracle.step(a, b, m), a
    du, dup, dm = to_dev(u), to_dev(up), to_dev(m)
    z = Z()
    z.oocz_stencil_steps(du, dup, dm, nx, ny, nz, z.default_coeffs(), n, torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert np.array_equal(bits(du.cpu().numpy()), bits(a))
    assert np.array_equal(bits(dup.cpu().numpy()), bits(b))


def test_hundred_steps_within_north_star_tolerance():
    import torch
    nx, ny, nz = 64, 64, 64
    u = synth.pulse(nx, ny, nz, sigma=4.0)
    m = synth.layered(nx, ny, nz)
    a, b = u, u
    for _ in range(100):
        a, b = oracle.step(a, b, m), a
    du, dup, dm = to_dev(u), to_dev(u), to_dev(m)
    z = Z()
    z.oocz_stencil_steps(du, dup, dm, nx, ny, nz, z.default_coeffs(), 100, torch.cuda.current_stream())
    torch.cuda.synchronize()
    got = du.cpu().numpy().astype(np.float64)
    err = np.abs(got - a).max() / np.abs(a).max()
    assert err <= 1e-4
    assert err == 0.0                                    # in fact bit-exact


@pytest.mark.parametrize("z0,z1,zv0,zv1", [(8, 40, 0, 48), (4, 44, 4, 44), (10, 30, 6, 34), (0, 48, 0, 48)])
def test_cone_limited_step_and_ghost(z0, z1, zv0, zv1):
    import torch
    nx, ny, nz = 40, 28, 48
    u, up, m = _state(nx, ny, nz, 9)
    # reference: planes outside [zv0, zv1) are zero ghosts
    sub = oracle.step(u[zv0:zv1], up[zv0:zv1], m[zv0:zv1])
    # poison everything the kernel must not read
    upois = u.copy()
    upois[: max(zv0, z0 - 4)] = np.nan
    upois[min(zv1, z1 + 4):] = np.nan
    du, dup, dm = to_dev(upois), to_dev(up), to_dev(m)
    z = Z()
    z.oocz_stencil_step_planes(du, dup, dm, nx, ny, nz, z.default_coeffs(), z0, z1, zv0, zv1,
                               torch.cuda.current_stream())
    torch.cuda.synchronize()
    got = dup.cpu().numpy()
    assert np.array_equal(bits(got[z0:z1]), bits(sub[z0 - zv0:z1 - zv0]))
    assert np.array_equal(bits(got[:z0]), bits(up[:z0]))
    assert np.array_equal(bits(got[z1:]), bits(up[z1:]))


def test_impulse_response_matches_closed_form():
    import torch
    n = 17
    u = np.zeros((n, n, n), np.float32)
    u[8, 8, 8] = 1
    up = np.zeros_like(u)
    m = np.full_like(u, np.float32(0.15))
    du, dup, dm = to_dev(u), to_dev(up), to_dev(m)
    z = Z()
    # nx = 17 is not a multiple of 4: rejected (float4 rows)
    with pytest.raises(z.OoczError):
        z.oocz_stencil_step_planes(du, dup, dm, n, n, n, z.default_coeffs(), 0, n, 0, n, None)
    u = np.zeros((16, 16, 16), np.float32)
    u[8, 8, 8] = 1
    up = np.zeros_like(u)
    m = np.full_like(u, np.float32(0.15))
    want = oracle.step(u, up, m)
    du, dup, dm = to_dev(u), to_dev(up), to_dev(m)
    z.oocz_stencil_step_planes(du, dup, dm, 16, 16, 16, z.default_coeffs(), 0, 16, 0, 16, None)
    torch.cuda.synchronize()
    assert np.array_equal(bits(dup.cpu().numpy()), bits(want))


@pytest.mark.parametrize("shape,cone", [((1024, 304, 40), (4, 36, 0, 40)),   # 8 x 21 = 168 tiles > 148 SMs
                                        ((512, 608, 28), (8, 20, 4, 24)),    # 4 x 41 tiles, ragged y
                                        ((2048, 64, 20), (0, 20, 0, 20))])   # 16 x 5 = 80 tiles, one column each
def test_chunked_persistent_schedule_bit_exact(shape, cone):
    """More tiles than SMs: 148 persistent CTAs take (z chunk, tile) items in
    chunk-major order (the schedule C3-sized planes use); fewer: one CTA per
    tile column.  Both equal the oracle bit for bit, cone limits included."""
    import torch
    nx, ny, nz = shape
    z0, z1, zv0, zv1 = cone
    u, up, m = _state(nx, ny, nz, 12)
    sub = oracle.step(u[zv0:zv1], up[zv0:zv1], m[zv0:zv1])
    du, dup, dm = to_dev(u), to_dev(up), to_dev(m)
    z = Z()
    z.oocz_stencil_step_planes(du, dup, dm, nx, ny, nz, z.default_coeffs(), z0, z1, zv0, zv1,
                               torch.cuda.current_stream())
    torch.cuda.synchronize()
    got = dup.cpu().numpy()
    assert np.array_equal(bits(got[z0:z1]), bits(sub[z0 - zv0:z1 - zv0]))
    assert np.array_equal(bits(got[:z0]), bits(up[:z0])) and np.array_equal(bits(got[z1:]), bits(up[z1:]))


def test_chunked_persistent_schedule_fp64():
    import torch
    nx, ny, nz = 1024, 160, 24                       # 8 x 20 = 160 tiles of 128 x 8 > 148
    u, up, m = (a.astype(np.float64) for a in _state(nx, ny, nz, 13))
    want = oracle.step_f64(u, up, m)
    du, dup, dm = to_dev(u), to_dev(up), to_dev(m)
    z = Z()
    z.oocz_stencil_step_planes_f64(du, dup, dm, nx, ny, nz, z.default_coeffs64(), 0, nz, 0, nz,
                                   torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert np.array_equal(dup.cpu().numpy().view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("seed", [11, 12])
def test_random_shapes_and_cones_bit_exact(seed):
    """Seeded random grids (ragged tiles in x and y, chunked and one-column
    schedules) and cone limits, each launched three times, against the oracle."""
    import torch
    rng = np.random.default_rng(seed)
    z = Z()
    for case in range(16):
        nx = 4 * int(rng.integers(1, 80))
        ny = int(rng.integers(1, 70))
        nz = int(rng.integers(9, 40))
        zv0 = int(rng.integers(0, 4))
        zv1 = int(rng.integers(max(zv0 + 1, nz - 4), nz + 1))
        z0 = int(rng.integers(zv0, zv1))
        z1 = int(rng.integers(z0, zv1 + 1))
        u, up, m = _state(nx, ny, nz, 200 + case)
        want = oracle.step(u[zv0:zv1], up[zv0:zv1], m[zv0:zv1])
        du, dm = to_dev(u), to_dev(m)
        for rep in range(3):
            dup = to_dev(up)
            z.oocz_stencil_step_planes(du, dup, dm, nx, ny, nz, z.default_coeffs(), z0, z1, zv0, zv1,
                                       torch.cuda.current_stream())
            torch.cuda.synchronize()
            got = dup.cpu().numpy()
            assert np.array_equal(bits(got[z0:z1]), bits(want[z0 - zv0:z1 - zv0])), (nx, ny, nz, z0, z1, zv0, zv1)
            assert np.array_equal(bits(got[:z0]), bits(up[:z0])) and np.array_equal(bits(got[z1:]), bits(up[z1:]))


@pytest.mark.parametrize("shape", [(64, 30, 24), (1024, 304, 24)])   # one tile column each / chunked (168 tiles)
def test_every_short_plane_range_bit_exact(shape):
    """The fp32 kernel marches two planes per iteration (the second predicated
    off at an odd range end) and, with more tiles than SMs, in z chunks: every
    update range [z0, z0 + n) with n = 1..9 at the slab's ends and middle,
    against the oracle bit for bit, planes outside the range untouched."""
    import torch
    nx, ny, nz = shape
    u, up, m = _state(nx, ny, nz, 21)
    want = oracle.step(u, up, m)
    du, dm = to_dev(u), to_dev(m)
    z = Z()
    for n in range(1, 10):
        for z0 in sorted({0, (nz - n) // 2, nz - n}):
            dup = to_dev(up)
            z.oocz_stencil_step_planes(du, dup, dm, nx, ny, nz, z.default_coeffs(), z0, z0 + n, 0, nz,
                                       torch.cuda.current_stream())
            torch.cuda.synchronize()
            got = dup.cpu().numpy()
            assert np.array_equal(bits(got[z0:z0 + n]), bits(want[z0:z0 + n])), (n, z0)
            assert np.array_equal(bits(got[:z0]), bits(up[:z0])) and np.array_equal(bits(got[z0 + n:]), bits(up[z0 + n:]))
