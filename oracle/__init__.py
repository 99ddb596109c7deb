"""CPU oracle for arXiv 2109.05410's hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2109_05410_b200`` never imports it and shares no code with it.

The C sources (``zfp_ref.c``, ``stencil_ref.c``, ``ooc_emul.c``) are compiled
with plain gcc into ``liboracle.so`` (``-ffp-contract=off`` so that the
prescribed fp32 evaluation order of SURVEY 8(c) c.1 is kept).  This module is
argument marshalling only: numpy arrays in, numpy arrays out.

Citations: see ``oracle.h``.  Parity vs real zfp/cuZFP bitstreams is
UNPINNED (no zfp here); every other function is pinned by
``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = ["zfp_ref.c", "zfp_ref64.c", "stencil_ref.c", "ooc_emul.c", "ooc_emul64.c"]
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no CUDA)."""
    srcs = [os.path.join(_HERE, s) for s in _SRCS]
    deps = srcs + [os.path.join(_HERE, "oracle.h")]
    if not force and os.path.exists(_LIB_PATH):
        t = os.path.getmtime(_LIB_PATH)
        if all(os.path.getmtime(d) <= t for d in deps):
            return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-std=gnu11", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
           "-fno-fast-math", "-fopenmp", "-Wall", "-Wno-unused-function",
           *srcs, "-o", tmp, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB_PATH)
            f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
            f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
            i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
            u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
            u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
            i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
            ci = C.c_int
            sig = {
                "orc_exponent_max": (C.c_int32, [f32p]),
                "orc_fwd_cast": (None, [f32p, ci, i32p]),
                "orc_inv_cast": (None, [i32p, ci, f32p]),
                "orc_fwd_lift": (None, [i32p]),
                "orc_inv_lift": (None, [i32p]),
                "orc_fwd_xform": (None, [i32p]),
                "orc_inv_xform": (None, [i32p]),
                "orc_int2uint": (C.c_uint32, [C.c_int32]),
                "orc_uint2int": (C.c_int32, [C.c_uint32]),
                "orc_perm3": (C.POINTER(C.c_uint8), []),
                "orc_encode_block": (ci, [f32p, ci, u64p]),
                "orc_decode_block": (ci, [u64p, ci, f32p]),
                "orc_encode_ints": (ci, [u32p, ci, u64p, ci]),
                "orc_decode_ints": (ci, [u64p, ci, ci, u32p]),
                "orc_zfp_bytes": (C.c_size_t, [ci, ci, ci, ci]),
                "orc_zfp_encode": (ci, [f32p, ci, ci, ci, ci, u64p]),
                "orc_zfp_decode": (ci, [u64p, ci, ci, ci, ci, f32p]),
                "orc_roundtrip": (ci, [f32p, ci, ci, ci, ci]),
                "orc_default_coeffs": (None, [f32p]),
                "orc_step": (None, [f32p, f32p, f32p, f32p, ci, ci, ci, f32p]),
                "orc_step_f64": (None, [f64p, f64p, f64p, f64p, ci, ci, ci, f64p]),
                "orc_step_planes": (None, [f32p, f32p, f32p, f32p, ci, ci, ci, f32p, ci, ci]),
                "orc_advance": (ci, [f32p, f32p, f32p, ci, ci, ci, f32p, ci, i32p, C.c_long]),
                "orc_ooc_emulate": (ci, [f32p, f32p, f32p, ci, ci, ci, f32p, ci, ci, ci, i32p,
                                         C.c_long, ci, u64p]),
                "orc64_ooc_emulate": (ci, [f64p, f64p, f64p, ci, ci, ci, f64p, ci, ci, ci, i32p,
                                           C.c_long, ci, u64p]),
                "orc_step_planes_f64": (None, [f64p, f64p, f64p, f64p, ci, ci, ci, f64p, ci, ci]),
                "orc64_exponent_max": (C.c_int32, [f64p]),
                "orc64_fwd_cast": (None, [f64p, ci, i64p]),
                "orc64_inv_cast": (None, [i64p, ci, f64p]),
                "orc64_fwd_lift": (None, [i64p]),
                "orc64_inv_lift": (None, [i64p]),
                "orc64_fwd_xform": (None, [i64p]),
                "orc64_inv_xform": (None, [i64p]),
                "orc64_int2uint": (C.c_uint64, [C.c_int64]),
                "orc64_uint2int": (C.c_int64, [C.c_uint64]),
                "orc64_encode_ints": (ci, [u64p, ci, u64p, ci]),
                "orc64_decode_ints": (ci, [u64p, ci, ci, u64p]),
                "orc64_encode_block": (ci, [f64p, ci, u64p]),
                "orc64_decode_block": (ci, [u64p, ci, f64p]),
                "orc64_zfp_encode": (ci, [f64p, ci, ci, ci, ci, u64p]),
                "orc64_zfp_decode": (ci, [u64p, ci, ci, ci, ci, f64p]),
                "orc64_roundtrip": (ci, [f64p, ci, ci, ci, ci]),
                "orc64_advance": (ci, [f64p, f64p, f64p, ci, ci, ci, f64p, ci, i32p, C.c_long]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _shape3(a):
    nz, ny, nx = a.shape
    return nx, ny, nz


# ---------------------------------------------------------------- codec
def default_coeffs() -> np.ndarray:
    c = np.zeros(5, np.float32)
    lib().orc_default_coeffs(c)
    return c


def perm3() -> np.ndarray:
    p = lib().orc_perm3()
    return np.array([p[i] for i in range(64)], dtype=np.int64)


def exponent_max(block64) -> int:
    return int(lib().orc_exponent_max(_f32(block64).reshape(64)))


def fwd_cast(block64, emax):
    q = np.zeros(64, np.int32)
    lib().orc_fwd_cast(_f32(block64).reshape(64), int(emax), q)
    return q


def inv_cast(q, emax):
    x = np.zeros(64, np.float32)
    lib().orc_inv_cast(np.ascontiguousarray(q, np.int32), int(emax), x)
    return x


def fwd_lift(v):
    v = np.array(v, dtype=np.int32).copy()
    lib().orc_fwd_lift(v)
    return v


def inv_lift(v):
    v = np.array(v, dtype=np.int32).copy()
    lib().orc_inv_lift(v)
    return v


def fwd_xform(q):
    q = np.array(q, dtype=np.int32).reshape(64).copy()
    lib().orc_fwd_xform(q)
    return q


def inv_xform(q):
    q = np.array(q, dtype=np.int32).reshape(64).copy()
    lib().orc_inv_xform(q)
    return q


def int2uint(x: int) -> int:
    return int(lib().orc_int2uint(int(np.int32(x))))


def uint2int(u: int) -> int:
    return int(lib().orc_uint2int(int(u) & 0xFFFFFFFF))


def encode_block(block64, rate: int):
    out = np.zeros(rate, np.uint64)
    used = lib().orc_encode_block(_f32(block64).reshape(64), int(rate), out)
    return out, int(used)


def decode_block(words, rate: int):
    x = np.zeros(64, np.float32)
    used = lib().orc_decode_block(np.ascontiguousarray(words, np.uint64), int(rate), x)
    return x, int(used)


def encode_ints(u64coeffs, budget_bits: int):
    u = np.ascontiguousarray(u64coeffs, np.uint32)
    words = np.zeros((budget_bits + 63) // 64 + 1, np.uint64)
    used = lib().orc_encode_ints(u, int(budget_bits), words, 0)
    return words, int(used)


def decode_ints(words, budget_bits: int):
    u = np.zeros(64, np.uint32)
    used = lib().orc_decode_ints(np.ascontiguousarray(words, np.uint64), 0, int(budget_bits), u)
    return u, int(used)


def zfp_bytes(nx, ny, nz, rate) -> int:
    return int(lib().orc_zfp_bytes(nx, ny, nz, rate))


def zfp_encode(field, rate: int) -> np.ndarray:
    """field: (nz, ny, nx) fp32 -> uint64 words, block order bz, by, bx."""
    f = _f32(field)
    nx, ny, nz = _shape3(f)
    out = np.zeros(zfp_bytes(nx, ny, nz, rate) // 8, np.uint64)
    rc = lib().orc_zfp_encode(f, nx, ny, nz, int(rate), out)
    if rc:
        raise ValueError("orc_zfp_encode: bad arguments")
    return out


def zfp_decode(words, shape, rate: int) -> np.ndarray:
    nz, ny, nx = shape
    f = np.zeros((nz, ny, nx), np.float32)
    rc = lib().orc_zfp_decode(np.ascontiguousarray(words, np.uint64), nx, ny, nz, int(rate), f)
    if rc:
        raise ValueError("orc_zfp_decode: bad arguments")
    return f


def roundtrip(field, rate: int) -> np.ndarray:
    f = _f32(field).copy()
    nx, ny, nz = _shape3(f)
    if lib().orc_roundtrip(f, nx, ny, nz, int(rate)):
        raise ValueError("orc_roundtrip: bad arguments")
    return f


# ---------------------------------------------------------------- stencil
def step(u, uprev, m, c=None) -> np.ndarray:
    """One leapfrog step over the whole grid; returns u+ (new array)."""
    u, uprev, m = _f32(u), _f32(uprev), _f32(m)
    c = default_coeffs() if c is None else _f32(c)
    out = np.zeros_like(u)
    nx, ny, nz = _shape3(u)
    lib().orc_step(u, uprev, m, out, nx, ny, nz, c)
    return out


def step_f64(u, uprev, m, c=None) -> np.ndarray:
    u = np.ascontiguousarray(u, np.float64)
    uprev = np.ascontiguousarray(uprev, np.float64)
    m = np.ascontiguousarray(m, np.float64)
    if c is None:
        c = np.array([-205 / 72, 8 / 5, -1 / 5, 8 / 315, -1 / 560], np.float64)
    c = np.ascontiguousarray(c, np.float64)
    out = np.zeros_like(u)
    nx, ny, nz = _shape3(u)
    lib().orc_step_f64(u, uprev, m, out, nx, ny, nz, c)
    return out


def advance(u, uprev, m, T: int, rates, nsteps: int, c=None):
    """SURVEY 8(c) c.0 schedule (after set_field's round trip, done by the caller).

    Returns new (u, uprev) arrays."""
    u, uprev, m = _f32(u).copy(), _f32(uprev).copy(), _f32(m)
    c = default_coeffs() if c is None else _f32(c)
    nx, ny, nz = _shape3(u)
    r = np.array(list(rates), np.int32)
    rc = lib().orc_advance(u, uprev, m, nx, ny, nz, c, int(T), r, int(nsteps))
    if rc:
        raise ValueError("orc_advance: bad arguments")
    return u, uprev


def run(u0, uprev0, m0, T: int, rates, nsteps: int, c=None):
    """Whole method as the user sees it: set_field (RT of all three fields),
    then step(nsteps) in one call.  Returns (u, uprev)."""
    u = roundtrip(u0, rates[0])
    up = roundtrip(uprev0, rates[1])
    m = roundtrip(m0, rates[2])
    return advance(u, up, m, T, rates, nsteps, c)


def ooc_emulate64(u0, uprev0, m0, T: int, P: int, G: int, rates, nsteps: int,
                  poison: bool = False, c=None):
    """fp64 twin of ooc_emulate (ooc_emul64.c): the literal region-by-region
    out-of-core emulator in the paper's precision; returns (u, uprev, stats)."""
    u, up, m = _f64(u0).copy(), _f64(uprev0).copy(), _f64(m0)
    c = C64 if c is None else _f64(c)
    nx, ny, nz = _shape3(u)
    stats = np.zeros(3, np.uint64)
    r = np.array(list(rates), np.int32)
    rc = lib().orc64_ooc_emulate(u, up, m, nx, ny, nz, c, int(T), int(P), int(G), r,
                                 int(nsteps), int(bool(poison)), stats)
    if rc:
        raise ValueError("orc64_ooc_emulate: bad arguments")
    return u, up, {"h2d": int(stats[0]), "d2h": int(stats[1]), "halo": int(stats[2])}


def ooc_emulate(u0, uprev0, m0, T: int, P: int, G: int, rates, nsteps: int,
                poison: bool = False, c=None):
    """Literal region-by-region out-of-core emulator; returns (u, uprev, stats)."""
    u, up, m = _f32(u0).copy(), _f32(uprev0).copy(), _f32(m0)
    c = default_coeffs() if c is None else _f32(c)
    nx, ny, nz = _shape3(u)
    stats = np.zeros(3, np.uint64)
    r = np.array(list(rates), np.int32)
    rc = lib().orc_ooc_emulate(u, up, m, nx, ny, nz, c, int(T), int(P), int(G), r,
                               int(nsteps), int(bool(poison)), stats)
    if rc:
        raise ValueError("orc_ooc_emulate: bad arguments")
    return u, up, {"h2d": int(stats[0]), "d2h": int(stats[1]), "halo": int(stats[2])}


# ---------------------------------------------------------------- fp64 (zfp_ref64.c)
C64 = np.array([-205 / 72, 8 / 5, -1 / 5, 8 / 315, -1 / 560], np.float64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def exponent_max64(block64) -> int:
    return int(lib().orc64_exponent_max(_f64(block64).reshape(64)))


def fwd_cast64(block64, emax):
    q = np.zeros(64, np.int64)
    lib().orc64_fwd_cast(_f64(block64).reshape(64), int(emax), q)
    return q


def inv_cast64(q, emax):
    x = np.zeros(64, np.float64)
    lib().orc64_inv_cast(np.ascontiguousarray(q, np.int64), int(emax), x)
    return x


def fwd_lift64(v):
    v = np.array(v, dtype=np.int64).copy()
    lib().orc64_fwd_lift(v)
    return v


def inv_lift64(v):
    v = np.array(v, dtype=np.int64).copy()
    lib().orc64_inv_lift(v)
    return v


def fwd_xform64(q):
    q = np.array(q, dtype=np.int64).reshape(64).copy()
    lib().orc64_fwd_xform(q)
    return q


def inv_xform64(q):
    q = np.array(q, dtype=np.int64).reshape(64).copy()
    lib().orc64_inv_xform(q)
    return q


def int2uint64(x: int) -> int:
    return int(lib().orc64_int2uint(int(np.int64(x))))


def uint2int64(u: int) -> int:
    return int(lib().orc64_uint2int(int(u) & 0xFFFFFFFFFFFFFFFF))


def encode_block64(block64, rate: int):
    out = np.zeros(rate, np.uint64)
    used = lib().orc64_encode_block(_f64(block64).reshape(64), int(rate), out)
    return out, int(used)


def decode_block64(words, rate: int):
    x = np.zeros(64, np.float64)
    used = lib().orc64_decode_block(np.ascontiguousarray(words, np.uint64), int(rate), x)
    return x, int(used)


def encode_ints64(u, budget_bits: int):
    u = np.ascontiguousarray(u, np.uint64)
    words = np.zeros((budget_bits + 63) // 64 + 1, np.uint64)
    used = lib().orc64_encode_ints(u, int(budget_bits), words, 0)
    return words, int(used)


def decode_ints64(words, budget_bits: int):
    u = np.zeros(64, np.uint64)
    used = lib().orc64_decode_ints(np.ascontiguousarray(words, np.uint64), 0, int(budget_bits), u)
    return u, int(used)


def zfp_encode64(field, rate: int) -> np.ndarray:
    f = _f64(field)
    nx, ny, nz = _shape3(f)
    out = np.zeros(zfp_bytes(nx, ny, nz, rate) // 8, np.uint64)
    if lib().orc64_zfp_encode(f, nx, ny, nz, int(rate), out):
        raise ValueError("orc64_zfp_encode: bad arguments")
    return out


def zfp_decode64(words, shape, rate: int) -> np.ndarray:
    nz, ny, nx = shape
    f = np.zeros((nz, ny, nx), np.float64)
    if lib().orc64_zfp_decode(np.ascontiguousarray(words, np.uint64), nx, ny, nz, int(rate), f):
        raise ValueError("orc64_zfp_decode: bad arguments")
    return f


def roundtrip64(field, rate: int) -> np.ndarray:
    f = _f64(field).copy()
    nx, ny, nz = _shape3(f)
    if lib().orc64_roundtrip(f, nx, ny, nz, int(rate)):
        raise ValueError("orc64_roundtrip: bad arguments")
    return f


def advance64(u, uprev, m, T: int, rates, nsteps: int, c=None):
    u, uprev, m = _f64(u).copy(), _f64(uprev).copy(), _f64(m)
    c = C64 if c is None else _f64(c)
    nx, ny, nz = _shape3(u)
    r = np.array(list(rates), np.int32)
    if lib().orc64_advance(u, uprev, m, nx, ny, nz, c, int(T), r, int(nsteps)):
        raise ValueError("orc64_advance: bad arguments")
    return u, uprev


def run64(u0, uprev0, m0, T: int, rates, nsteps: int, c=None):
    """fp64 twin of run(): set_field round trips, then step(nsteps)."""
    return advance64(roundtrip64(u0, rates[0]), roundtrip64(uprev0, rates[1]), roundtrip64(m0, rates[2]),
                     T, rates, nsteps, c)
