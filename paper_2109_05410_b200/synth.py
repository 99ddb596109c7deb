"""Seeded synthetic inputs shaped like the paper's workload.

This module holds no arithmetic of the method (no stencil, no codec): it only
draws the initial fields.  It is the one module shared by the oracle-side
tests and the CUDA-side tests/bench, so both see bit-identical inputs.
Values are computed in fp64 and rounded (RNE) to fp32 by numpy.

Generators:
  PULSE(sigma)  u = exp(-r^2 / (2 sigma^2)), r from the grid centre; u- = u
                (zero initial velocity).  Its tails reach fp32
                denormals and zero, exercising extreme ZFP exponents.
  DENSE(seed)   u = sum_{q=1..4} a_q sin(2 pi i/lx_q + px_q) sin(2 pi j/ly_q + py_q)
                                 sin(2 pi k/lz_q + pz_q),
                lambda ~ U[8, 64] cells, phase ~ U[0, 2 pi), a ~ U[0.25, 1];
                separable, so every 4^3 block is non-trivial.
  LAYERED       m = (v(k) (1 + 0.05 sin(2 pi i/97) sin(2 pi j/89)) 0.4/4500)^2,
                v = 1500/2500/3500/4500 m/s in z-quarters: a layered velocity
                model as in the paper's geophysics setting;
                max m = 0.1764 < 105/512 (the CFL bound of DESIGN.md R2).
Random numbers come from splitmix64 (a counter-based generator).
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1


def splitmix64(state: int):
    """Yield an endless stream of 64-bit outputs (Steele et al.'s splitmix64)."""
    while True:
        state = (state + 0x9E3779B97F4A7C15) & _M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        yield z ^ (z >> 31)


def uniforms(seed: int, n: int) -> np.ndarray:
    g = splitmix64(seed)
    return np.array([(next(g) >> 11) * (1.0 / (1 << 53)) for _ in range(n)], np.float64)


def pulse(nx: int, ny: int, nz: int, sigma: float, z0: int = 0, z1: int | None = None) -> np.ndarray:
    """Planes [z0, z1) of PULSE(sigma) as fp32 (nz_sel, ny, nx)."""
    z1 = nz if z1 is None else z1
    x = (np.arange(nx, dtype=np.float64) - nx / 2) ** 2
    y = (np.arange(ny, dtype=np.float64) - ny / 2) ** 2
    z = (np.arange(z0, z1, dtype=np.float64) - nz / 2) ** 2
    r2 = z[:, None, None] + y[None, :, None] + x[None, None, :]
    return np.exp(-r2 / (2.0 * sigma * sigma)).astype(np.float32)


def dense_params(seed: int):
    u = uniforms(seed, 40)
    p = []
    for q in range(4):
        v = u[10 * q:10 * q + 10]
        lam = 8.0 + 56.0 * v[0:3]
        ph = 2.0 * np.pi * v[3:6]
        a = 0.25 + 0.75 * v[6]
        p.append((lam, ph, a))
    return p


def dense(nx: int, ny: int, nz: int, seed: int, z0: int = 0, z1: int | None = None,
          y0: int = 0, y1: int | None = None, x0: int = 0, x1: int | None = None) -> np.ndarray:
    """Box [z0, z1) x [y0, y1) x [x0, x1) of DENSE(seed) as fp32: the same
    elementwise fp64 operations on sub-ranges of the index vectors, so a box
    holds exactly the values of the whole field there."""
    z1 = nz if z1 is None else z1
    y1 = ny if y1 is None else y1
    x1 = nx if x1 is None else x1
    out = np.zeros((z1 - z0, y1 - y0, x1 - x0), np.float64)
    i = np.arange(x0, x1, dtype=np.float64)
    j = np.arange(y0, y1, dtype=np.float64)
    k = np.arange(z0, z1, dtype=np.float64)
    for lam, ph, a in dense_params(seed):
        sx = np.sin(2 * np.pi * i / lam[0] + ph[0])
        sy = np.sin(2 * np.pi * j / lam[1] + ph[1])
        sz = np.sin(2 * np.pi * k / lam[2] + ph[2])
        out += a * sz[:, None, None] * (sy[:, None] * sx[None, :])[None, :, :]
    return out.astype(np.float32)


def layered(nx: int, ny: int, nz: int, z0: int = 0, z1: int | None = None,
            y0: int = 0, y1: int | None = None, x0: int = 0, x1: int | None = None) -> np.ndarray:
    z1 = nz if z1 is None else z1
    y1 = ny if y1 is None else y1
    x1 = nx if x1 is None else x1
    i = np.arange(x0, x1, dtype=np.float64)
    j = np.arange(y0, y1, dtype=np.float64)
    k = np.arange(z0, z1)
    vel = np.array([1500.0, 2500.0, 3500.0, 4500.0])[np.minimum((4 * k) // max(nz, 1), 3)]
    lat = 1.0 + 0.05 * np.sin(2 * np.pi * j / 97.0)[:, None] * np.sin(2 * np.pi * i / 89.0)[None, :]
    m = (vel[:, None, None] * lat[None, :, :] * 0.4 / 4500.0) ** 2
    return m.astype(np.float32)


# ---- the same generators evaluated on the GPU, plane chunk by plane chunk, for
# grids that never exist whole in host memory (C3: 3 x 103 GB).  The sin tables
# are numpy's (fp64); the products and sums are the same fp64 operations in the
# same order, so the values are bit-identical to dense() / layered() (checked
# by tests/test_synth_gpu.py and on every run of the C3-scale parity test).

def dense_torch(nx: int, ny: int, nz: int, seed: int, z0: int, z1: int, device="cuda", fp64: bool = False):
    """Planes [z0, z1) of DENSE(seed) as an fp32 (or, fp64 = True, the unrounded
    fp64) torch tensor on `device`."""
    import torch
    i = np.arange(nx, dtype=np.float64)
    j = np.arange(ny, dtype=np.float64)
    k = np.arange(z0, z1, dtype=np.float64)
    out = torch.zeros((z1 - z0, ny, nx), dtype=torch.float64, device=device)
    for lam, ph, a in dense_params(seed):
        sx = torch.from_numpy(np.sin(2 * np.pi * i / lam[0] + ph[0])).to(device)
        sy = torch.from_numpy(np.sin(2 * np.pi * j / lam[1] + ph[1])).to(device)
        asz = torch.from_numpy(a * np.sin(2 * np.pi * k / lam[2] + ph[2])).to(device)   # a * sz, as numpy
        out += asz[:, None, None] * (sy[:, None] * sx[None, :])[None, :, :]
    return out if fp64 else out.to(torch.float32)


def layered_torch(nx: int, ny: int, nz: int, z0: int, z1: int, device="cuda", fp64: bool = False, _lat={}):
    """Planes [z0, z1) of LAYERED as an fp32 (or fp64) torch tensor on `device`."""
    import torch
    key = (nx, ny, str(device))
    if key not in _lat:
        i = np.arange(nx, dtype=np.float64)
        j = np.arange(ny, dtype=np.float64)
        lat = 1.0 + 0.05 * np.sin(2 * np.pi * j / 97.0)[:, None] * np.sin(2 * np.pi * i / 89.0)[None, :]
        _lat.clear()
        _lat[key] = torch.from_numpy(lat).to(device)
    k = np.arange(z0, z1)
    vel = torch.from_numpy(np.array([1500.0, 2500.0, 3500.0, 4500.0])[np.minimum((4 * k) // max(nz, 1), 3)]).to(device)
    t = vel[:, None, None] * _lat[key][None, :, :] * 0.4 / 4500.0
    return t * t if fp64 else (t * t).to(torch.float32)


def random_blocks(nblocks: int, seed: int) -> np.ndarray:
    """Adversarial 4^3 blocks for codec tests: (nblocks, 64) fp32 mixing
    random magnitudes over the whole exponent range, denormals, zeros,
    signed zeros, constants, single spikes and smooth ramps."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = np.zeros((nblocks, 64), np.float32)
    for b in range(nblocks):
        kind = b % 8
        if kind == 0:      # random normal numbers, random common scale
            e = rng.integers(-120, 120)
            out[b] = (rng.standard_normal(64) * 2.0 ** e).astype(np.float32)
        elif kind == 1:    # exponents spread across the block
            out[b] = (rng.standard_normal(64) * 2.0 ** rng.integers(-140, 100, 64)).astype(np.float32)
        elif kind == 2:    # denormals only
            out[b] = (rng.integers(-(1 << 23), 1 << 23, 64).astype(np.float64) * 2.0 ** -149).astype(np.float32)
        elif kind == 3:    # constant, possibly denormal
            out[b] = np.float32(rng.standard_normal() * 2.0 ** rng.integers(-149, 120))
        elif kind == 4:    # single spike on zeros (and signed zeros)
            out[b] = np.where(rng.random(64) < 0.5, np.float32(-0.0), np.float32(0.0))
            out[b, rng.integers(64)] = np.float32(rng.standard_normal() * 2.0 ** rng.integers(-60, 60))
        elif kind == 5:    # smooth ramp
            i, j, k = np.meshgrid(np.arange(4), np.arange(4), np.arange(4), indexing="xy")
            g = rng.standard_normal(4)
            out[b] = (g[0] + g[1] * i + g[2] * j + g[3] * k).astype(np.float32).reshape(64)
        elif kind == 6:    # max-magnitude values
            out[b] = (np.sign(rng.standard_normal(64)) * np.float32(3.4e38) * rng.random(64)).astype(np.float32)
        else:              # raw random bit patterns, made finite
            bits = rng.integers(0, 1 << 32, 64, dtype=np.uint64).astype(np.uint32)
            v = bits.view(np.float32).copy()
            v[~np.isfinite(v)] = np.float32(1.0)
            out[b] = v
    return out


def blocks_to_field(blocks: np.ndarray, nbx: int, nby: int, nbz: int) -> np.ndarray:
    """Place (nbx*nby*nbz, 64) blocks (block order bz, by, bx; local i+4j+16k)
    into a (4nbz, 4nby, 4nbx) field."""
    b = blocks.reshape(nbz, nby, nbx, 4, 4, 4)          # bz, by, bx, k, j, i
    return np.ascontiguousarray(b.transpose(0, 3, 1, 4, 2, 5).reshape(4 * nbz, 4 * nby, 4 * nbx))
