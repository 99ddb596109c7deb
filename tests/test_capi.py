"""CPU-side checks of the C ABI (no GPU compute): the library loads, exports
every function include/oocz.h declares, and its host-only calls (config
validation, sizes, CFL bound) follow the contract."""
import ctypes as C
import os
from fractions import Fraction

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def z():
    import __graft_entry__ as g
    g.build_library()
    from paper_2109_05410_b200 import oocz
    return oocz


def test_every_header_symbol_is_exported(z):
    names = z.header_functions()
    assert len(names) >= 20
    lib = C.CDLL(z.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version(z):
    assert z.oocz_abi_version() == z.ABI_VERSION == 6


def test_zfp_bytes_closed_form(z):
    assert z.oocz_zfp_bytes(64, 64, 64, 16) == 524_288
    assert z.oocz_zfp_bytes(512, 512, 512, 8) == 128 << 20
    assert z.oocz_zfp_bytes(4096, 4096, 1536, 16) == 51_539_607_552


def test_cfl_limit_default_coefficients(z):
    assert abs(z.oocz_cfl_limit(z.default_coeffs()) - float(Fraction(105, 512))) < 1e-6
    assert abs(z.oocz_cfl_limit_f64(z.default_coeffs64()) - float(Fraction(105, 512))) < 1e-9


@pytest.mark.parametrize("kw,world,code,msg", [
    (dict(nx=62), 1, -2, "multiples of 4"),
    (dict(block_planes=36, tb=5, nz=144), 1, -1, "P (36) < 2h (40)"),
    (dict(block_planes=48, nz=144), 1, 0, ""),                       # SPEC.md:297 analogue
    (dict(block_planes=144, tb=12, nz=1152), 1, 0, ""),             # paper: D = 8 -> P = 144, h = 48
    (dict(block_planes=40, nz=128), 1, -1, "does not divide"),
    (dict(block_planes=32, nz=128), 3, -1, "world (3) does not divide nz"),
    (dict(rate=[16, 70, 16]), 1, -1, "rate[1] (70)"),
    (dict(block_planes=30), 1, -2, "P (30)"),
    (dict(slots=1), 1, -1, "slots"),
    (dict(store=7), 1, -1, "store"),
    (dict(precision=16), 1, -1, "precision (16)"),
    (dict(precision=64, block_planes=32), 1, 0, ""),
    (dict(slab_sets=3, block_planes=32), 1, 0, ""),
    (dict(slab_sets=5, block_planes=32), 1, -1, "slab_sets (5)"),
    (dict(slab_sets=1, block_planes=32), 1, 0, ""),
    (dict(slab_sets=-1, block_planes=32), 1, -1, "slab_sets (-1)"),
    (dict(graphs=1, block_planes=32), 1, 0, ""),
    (dict(graphs=2, block_planes=32), 1, -1, "graphs (2)"),
    (dict(cone=1, block_planes=32), 1, 0, ""),
    (dict(cone=2, block_planes=32), 1, -1, "cone (2)"),
    (dict(resident_blocks=2, block_planes=32), 1, 0, ""),
    (dict(resident_blocks=4, block_planes=32), 1, 0, ""),            # K = D
    (dict(resident_blocks=5, block_planes=32), 1, -1, "resident_blocks (5) outside [-1 (auto), D = 4]"),
    (dict(resident_blocks=-1, block_planes=32), 1, 0, ""),           # auto
    (dict(resident_blocks=-2, block_planes=32), 1, -1, "resident_blocks (-2)"),
    (dict(resident_blocks=-1, block_planes=32, store=1), 1, -1, "needs store = OOCZ_STORE_HOST"),
    (dict(resident_blocks=1, block_planes=32, store=1), 1, -1, "needs store = OOCZ_STORE_HOST"),
    (dict(resident_blocks=1, block_planes=32), 2, 0, ""),             # per rank: D = 2
    (dict(resident_blocks=3, block_planes=32), 2, -1, "resident_blocks (3) outside [-1 (auto), D = 2]"),
])
def test_validate(z, kw, world, code, msg):
    base = dict(nx=64, ny=64, nz=128, tb=4, block_planes=32)
    base.update(kw)
    cfg = z.oocz_default_config(base.pop("nx"), base.pop("ny"), base.pop("nz"), **base)
    rc, m = z.oocz_validate(cfg, world)
    assert rc == code, m
    assert msg in m


def test_host_store_bytes_leave_out_the_resident_rows(z):
    """resident_blocks = K: the host store holds only the rows of blocks K .. D-1
    (each field's part rounded up to 4 KiB)."""
    rows = 64 // 4 * 64 // 4 * 8 * 16                     # one 4-plane row of a 64 x 64 plane at rate 16
    for k in range(5):
        cfg = z.oocz_default_config(64, 64, 128, tb=4, block_planes=32, resident_blocks=k)
        part = (128 - 32 * k) // 4 * rows
        assert z.oocz_host_store_bytes(cfg, 1) == 3 * ((part + 4095) // 4096 * 4096)


def test_default_config(z):
    cfg = z.oocz_default_config(16, 16, 64)
    assert (cfg.nx, cfg.ny, cfg.nz, cfg.tb, cfg.block_planes) == (16, 16, 64, 4, 64)
    assert list(cfg.rate) == [16, 16, 16] and cfg.store == 0 and cfg.slots == 2
    import oracle
    assert list(cfg.c) == list(oracle.default_coeffs())
    assert cfg.precision == 32 and list(cfg.c64) == list(oracle.C64)


def test_missing_library_fails_loudly(tmp_path):
    """No fallback: without the CUDA library the binding refuses to import."""
    import subprocess
    import sys
    env = dict(os.environ, OOCZ_LIB=str(tmp_path / "absent.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_2109_05410_b200.oocz"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "not built" in r.stderr


def test_product_never_touches_the_oracle():
    """The package (the product path) imports nothing from oracle/ (test
    infrastructure only) and links nothing from it."""
    import glob
    import re
    pkg = os.path.join(ROOT, "paper_2109_05410_b200")
    files = glob.glob(os.path.join(pkg, "*.py")) + glob.glob(os.path.join(pkg, "csrc", "*"))
    assert files
    for f in files:
        if f.endswith(".so") or f.endswith(".o"):
            continue
        src = open(f, errors="replace").read()
        assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), f
        assert "liboracle" not in src and "oracle.h" not in src, f
