"""The torch (chunked, GPU-capable) generators equal the numpy ones bit for
bit, and numpy sub-boxes equal the whole field there (the C3-scale parity test
and the benchmark generate their inputs this way).  Runs on the CPU device
here; the GPU parity tests re-check on cuda."""
import numpy as np
import pytest

from paper_2109_05410_b200 import synth


@pytest.mark.parametrize("shape,z0,z1", [((40, 24, 32), 0, 32), ((64, 36, 48), 12, 20), ((128, 8, 16), 4, 8)])
def test_torch_generators_equal_numpy(shape, z0, z1):
    nx, ny, nz = shape
    a = synth.dense_torch(nx, ny, nz, 2, z0, z1, device="cpu").numpy()
    assert np.array_equal(a.view(np.uint32), synth.dense(nx, ny, nz, seed=2, z0=z0, z1=z1).view(np.uint32))
    b = synth.layered_torch(nx, ny, nz, z0, z1, device="cpu").numpy()
    assert np.array_equal(b.view(np.uint32), synth.layered(nx, ny, nz, z0=z0, z1=z1).view(np.uint32))


def test_boxes_equal_whole_field():
    nx, ny, nz = 52, 40, 36
    u = synth.dense(nx, ny, nz, seed=2)
    m = synth.layered(nx, ny, nz)
    for (z0, z1, y0, y1, x0, x1) in [(0, 36, 0, 40, 0, 52), (4, 12, 8, 40, 20, 52), (30, 36, 0, 3, 51, 52)]:
        assert np.array_equal(synth.dense(nx, ny, nz, 2, z0, z1, y0, y1, x0, x1), u[z0:z1, y0:y1, x0:x1])
        assert np.array_equal(synth.layered(nx, ny, nz, z0, z1, y0, y1, x0, x1), m[z0:z1, y0:y1, x0:x1])
