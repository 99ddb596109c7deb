"""Thin ctypes binding of liboocz.so (include/oocz.h); same names as the C ABI.

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  There is no CPU fallback -- if liboocz.so is missing or cannot
be loaded, importing this module raises.  Device pointers may be given as
ints or as torch CUDA tensors (``.data_ptr()`` is taken); streams as ints,
torch streams, or None (legacy default stream).
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OOCZ_LIB", os.path.join(_HERE, "liboocz.so"))   # override: A/B builds only
HEADER = os.path.join(os.path.dirname(_HERE), "include", "oocz.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
_lib = C.CDLL(LIB_PATH)

# ------------------------------------------------------------------ constants
OOCZ_OK, OOCZ_EINVAL, OOCZ_EALIGN, OOCZ_ECFL, OOCZ_ECAPACITY = 0, -1, -2, -3, -4
OOCZ_ENONFINITE, OOCZ_ESTATE, OOCZ_ECUDA, OOCZ_ENCCL = -5, -6, -7, -8
OOCZ_U, OOCZ_UPREV, OOCZ_M = 0, 1, 2
OOCZ_STORE_HOST, OOCZ_STORE_DEVICE = 0, 1
STAGES = {0: "h2d", 1: "decode", 2: "stencil", 3: "encode", 4: "d2h", 5: "halo", 6: "copy"}


class oocz_config(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("c", C.c_float * 5), ("tb", C.c_int32), ("block_planes", C.c_int32),
                ("rate", C.c_int32 * 3), ("store", C.c_int32), ("slots", C.c_int32),
                ("profile", C.c_int32), ("device_bytes", C.c_uint64), ("m_resident", C.c_int32),
                ("precision", C.c_int32), ("c64", C.c_double * 5), ("serpentine", C.c_int32),
                ("slab_sets", C.c_int32), ("graphs", C.c_int32), ("cone", C.c_int32),
                ("resident_blocks", C.c_int32), ("m_hbm", C.c_int32)]


class oocz_stats(C.Structure):
    _fields_ = [("steps", C.c_uint64), ("sweeps", C.c_uint64), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("halo_bytes", C.c_uint64), ("kernel_launches", C.c_uint64),
                ("device_bytes_used", C.c_uint64), ("host_bytes_pinned", C.c_uint64),
                ("step_ms", C.c_double), ("h2d_ms", C.c_double), ("decode_ms", C.c_double),
                ("stencil_ms", C.c_double), ("encode_ms", C.c_double), ("d2h_ms", C.c_double),
                ("copy_ms", C.c_double), ("halo_ms", C.c_double),
                ("last_step_device_ms", C.c_double), ("step_device_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class oocz_event(C.Structure):
    _fields_ = [("sweep", C.c_int32), ("block", C.c_int32), ("stage", C.c_int32), ("lane", C.c_int32),
                ("start_ms", C.c_double), ("end_ms", C.c_double), ("bytes", C.c_uint64)]


_ctx_p = C.c_void_p
_vp = C.c_void_p
_i32 = C.c_int32
_SIGS = {
    "oocz_abi_version": (_i32, []),
    "oocz_status_string": (C.c_char_p, [C.c_int]),
    "oocz_default_config": (None, [C.POINTER(oocz_config), _i32, _i32, _i32]),
    "oocz_cfl_limit": (C.c_double, [C.POINTER(C.c_float)]),
    "oocz_cfl_limit_f64": (C.c_double, [C.POINTER(C.c_double)]),
    "oocz_get_config": (C.c_int, [_ctx_p, C.POINTER(oocz_config)]),
    "oocz_validate": (C.c_int, [C.POINTER(oocz_config), _i32, C.c_char_p, C.c_size_t]),
    "oocz_get_nccl_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "oocz_create": (C.c_int, [C.POINTER(oocz_config), _i32, _i32, C.POINTER(C.c_uint8), _i32, C.POINTER(_ctx_p)]),
    "oocz_create_ex": (C.c_int, [C.POINTER(oocz_config), _i32, _i32, C.POINTER(C.c_uint8), _i32, _vp, C.c_size_t,
                                 C.POINTER(_ctx_p)]),
    "oocz_host_store_bytes": (C.c_size_t, [C.POINTER(oocz_config), _i32]),
    "oocz_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "oocz_host_free": (None, [_vp]),
    "oocz_set_field": (C.c_int, [_ctx_p, _i32, _vp, C.c_size_t]),
    "oocz_set_field_device": (C.c_int, [_ctx_p, _i32, _vp, C.c_size_t]),
    "oocz_step": (C.c_int, [_ctx_p, C.c_int64]),
    "oocz_get_field": (C.c_int, [_ctx_p, _i32, _vp, C.c_size_t]),
    "oocz_get_field_device": (C.c_int, [_ctx_p, _i32, _vp, C.c_size_t]),
    "oocz_set_field_planes": (C.c_int, [_ctx_p, _i32, _i32, _i32, _vp, _i32]),
    "oocz_get_field_planes": (C.c_int, [_ctx_p, _i32, _i32, _i32, _vp, _i32]),
    "oocz_get_stats": (C.c_int, [_ctx_p, C.POINTER(oocz_stats)]),
    "oocz_store_bytes": (C.c_size_t, [_ctx_p, _i32]),
    "oocz_save_store": (C.c_int, [_ctx_p, _i32, _vp, C.c_size_t]),
    "oocz_load_store": (C.c_int, [_ctx_p, _i32, _vp, C.c_size_t]),
    "oocz_create_local_group": (C.c_int, [C.POINTER(oocz_config), _i32, _i32, C.POINTER(_ctx_p)]),
    "oocz_step_local_group": (C.c_int, [C.POINTER(_ctx_p), _i32, C.c_int64]),
    "oocz_get_events": (C.c_int, [_ctx_p, C.POINTER(oocz_event), C.c_size_t, C.POINTER(C.c_size_t)]),
    "oocz_last_error": (C.c_char_p, [_ctx_p]),
    "oocz_destroy": (None, [_ctx_p]),
    "oocz_zfp_bytes": (C.c_size_t, [_i32, _i32, _i32, _i32]),
    "oocz_zfp_encode": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "oocz_zfp_decode": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "oocz_stencil_steps": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, C.POINTER(C.c_float), _i32, _vp]),
    "oocz_stencil_step_planes": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, C.POINTER(C.c_float),
                                           _i32, _i32, _i32, _i32, _vp]),
    "oocz_zfp_encode_f64": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "oocz_zfp_decode_f64": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "oocz_stencil_steps_f64": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, C.POINTER(C.c_double), _i32, _vp]),
    "oocz_stencil_step_planes_f64": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, C.POINTER(C.c_double),
                                               _i32, _i32, _i32, _i32, _vp]),
    "oocz_kernel_launch_count": (C.c_uint64, []),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

ABI_VERSION = 6          # the oocz_config layout this binding marshals (include/oocz.h)
if _lib.oocz_abi_version() != ABI_VERSION:
    raise ImportError(f"{LIB_PATH} has ABI {_lib.oocz_abi_version()}, the binding expects {ABI_VERSION}: rebuild")


def header_functions() -> list[str]:
    """Every function include/oocz.h declares (for the export test)."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(oocz_[a-z0-9_]+)\s*\(", txt)))


class OoczError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        s = _lib.oocz_status_string(status).decode()
        super().__init__(f"{s} ({status}){': ' + msg if msg else ''}")


def _ptr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "cuda_stream"):
        return x.cuda_stream
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(f"cannot take a pointer of {type(x)}")


def _stream(s) -> int | None:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _check(rc: int, ctx=None):
    if rc != OOCZ_OK:
        msg = (_lib.oocz_last_error(ctx) or b"").decode()
        raise OoczError(rc, msg)


def _c5(c) -> C.Array:
    arr = (C.c_float * 5)(*[float(v) for v in np.asarray(c, np.float32)])
    return arr


def _c5d(c) -> C.Array:
    return (C.c_double * 5)(*[float(v) for v in np.asarray(c, np.float64)])


# ------------------------------------------------------------------ library
def oocz_abi_version() -> int:
    return _lib.oocz_abi_version()


_CFG_FIELDS = {k for k, _ in oocz_config._fields_}


def oocz_default_config(nx: int, ny: int, nz: int, **kw) -> oocz_config:
    cfg = oocz_config()
    _lib.oocz_default_config(C.byref(cfg), nx, ny, nz)
    for k, v in kw.items():
        if k == "rate":
            v = list(v) if hasattr(v, "__len__") else [v] * 3
            cfg.rate = (C.c_int32 * 3)(*v)
        elif k == "c":
            cfg.c = _c5(v)
        elif k == "c64":
            cfg.c64 = _c5d(v)
        elif k in _CFG_FIELDS:
            setattr(cfg, k, v)
        else:
            raise TypeError(f"oocz_config has no field {k!r}")
    return cfg


def oocz_cfl_limit(c) -> float:
    return float(_lib.oocz_cfl_limit(_c5(c)))


def oocz_cfl_limit_f64(c) -> float:
    return float(_lib.oocz_cfl_limit_f64(_c5d(c)))


def oocz_get_config(ctx: int) -> oocz_config:
    cfg = oocz_config()
    _check(_lib.oocz_get_config(ctx, C.byref(cfg)), ctx)
    return cfg


def field_dtype(ctx: int):
    """numpy dtype of the context's fields (precision 32 -> float32, 64 -> float64)."""
    return np.float64 if oocz_get_config(ctx).precision == 64 else np.float32


def oocz_validate(cfg: oocz_config, world: int = 1) -> tuple[int, str]:
    buf = C.create_string_buffer(256)
    rc = _lib.oocz_validate(C.byref(cfg), world, buf, 256)
    return rc, buf.value.decode()


def oocz_get_nccl_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_lib.oocz_get_nccl_id(buf))
    return bytes(buf)


def oocz_create(cfg: oocz_config, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                device: int = 0) -> int:
    out = _ctx_p()
    idp = None
    if nccl_id is not None:
        idp = (C.c_uint8 * 128)(*nccl_id)
    _check(_lib.oocz_create(C.byref(cfg), rank, world, idp, device, C.byref(out)))
    return out.value


def oocz_create_ex(cfg: oocz_config, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                   device: int = 0, host_arena: int | None = None, arena_bytes: int = 0) -> int:
    out = _ctx_p()
    idp = None
    if nccl_id is not None:
        idp = (C.c_uint8 * 128)(*nccl_id)
    _check(_lib.oocz_create_ex(C.byref(cfg), rank, world, idp, device, host_arena, arena_bytes, C.byref(out)))
    return out.value


def oocz_host_store_bytes(cfg: oocz_config, world: int = 1) -> int:
    return int(_lib.oocz_host_store_bytes(C.byref(cfg), world))


def oocz_host_alloc(nbytes: int) -> int:
    out = _vp()
    _check(_lib.oocz_host_alloc(nbytes, C.byref(out)))
    return out.value


def oocz_host_free(p: int | None) -> None:
    _lib.oocz_host_free(p)


def oocz_create_local_group(cfg: oocz_config, world: int, device: int = 0) -> list[int]:
    outs = (_ctx_p * world)()
    _check(_lib.oocz_create_local_group(C.byref(cfg), world, device, outs))
    return [o for o in outs]


def oocz_step_local_group(ctxs: list[int], nsteps: int) -> None:
    arr = (_ctx_p * len(ctxs))(*ctxs)
    rc = _lib.oocz_step_local_group(arr, len(ctxs), nsteps)
    _check(rc, ctxs[0])


def oocz_set_field(ctx: int, field: int, src: np.ndarray) -> None:
    a = np.ascontiguousarray(src, field_dtype(ctx))
    _check(_lib.oocz_set_field(ctx, field, a.ctypes.data, a.size), ctx)


def oocz_set_field_device(ctx: int, field: int, d_src, count: int) -> None:
    _check(_lib.oocz_set_field_device(ctx, field, _ptr(d_src), count), ctx)


def oocz_set_field_planes(ctx: int, field: int, z0: int, src, nplanes: int | None = None) -> None:
    """Planes [z0, z0 + nplanes) from a host array (nplanes, ny, nx) or a device
    tensor / pointer (nplanes required for a raw pointer)."""
    if isinstance(src, np.ndarray):
        a = np.ascontiguousarray(src, field_dtype(ctx))
        _check(_lib.oocz_set_field_planes(ctx, field, z0, a.shape[0], a.ctypes.data, 0), ctx)
    else:
        n = src.shape[0] if nplanes is None else nplanes
        _check(_lib.oocz_set_field_planes(ctx, field, z0, n, _ptr(src), 1), ctx)


def oocz_get_field_planes(ctx: int, field: int, z0: int, dst, nplanes: int | None = None):
    """Planes [z0, z0 + nplanes) into a host array (nplanes, ny, nx) or a device
    tensor / pointer."""
    if isinstance(dst, np.ndarray):
        assert dst.dtype == field_dtype(ctx) and dst.flags.c_contiguous
        _check(_lib.oocz_get_field_planes(ctx, field, z0, dst.shape[0], dst.ctypes.data, 0), ctx)
    else:
        n = dst.shape[0] if nplanes is None else nplanes
        _check(_lib.oocz_get_field_planes(ctx, field, z0, n, _ptr(dst), 1), ctx)
    return dst


def oocz_step(ctx: int, nsteps: int) -> None:
    _check(_lib.oocz_step(ctx, nsteps), ctx)


def oocz_get_field(ctx: int, field: int, dst: np.ndarray) -> np.ndarray:
    assert dst.dtype == field_dtype(ctx) and dst.flags.c_contiguous
    _check(_lib.oocz_get_field(ctx, field, dst.ctypes.data, dst.size), ctx)
    return dst


def oocz_get_field_device(ctx: int, field: int, d_dst, count: int) -> None:
    _check(_lib.oocz_get_field_device(ctx, field, _ptr(d_dst), count), ctx)


def oocz_store_bytes(ctx: int, field: int) -> int:
    return int(_lib.oocz_store_bytes(ctx, field))


def oocz_save_store(ctx: int, field: int) -> np.ndarray:
    buf = np.empty(oocz_store_bytes(ctx, field), np.uint8)
    _check(_lib.oocz_save_store(ctx, field, buf.ctypes.data, buf.size), ctx)
    return buf


def oocz_load_store(ctx: int, field: int, data: np.ndarray) -> None:
    a = np.ascontiguousarray(data, np.uint8)
    _check(_lib.oocz_load_store(ctx, field, a.ctypes.data, a.size), ctx)


def oocz_get_stats(ctx: int) -> dict:
    st = oocz_stats()
    _check(_lib.oocz_get_stats(ctx, C.byref(st)), ctx)
    return st.as_dict()


def oocz_get_events(ctx: int) -> list[dict]:
    n = C.c_size_t()
    _check(_lib.oocz_get_events(ctx, None, 0, C.byref(n)), ctx)
    evs = (oocz_event * max(n.value, 1))()
    _check(_lib.oocz_get_events(ctx, evs, n.value, C.byref(n)), ctx)
    return [{k: getattr(e, k) for k, _ in oocz_event._fields_} for e in evs[: n.value]]


def oocz_last_error(ctx: int) -> str:
    return _lib.oocz_last_error(ctx).decode()


def oocz_destroy(ctx: int) -> None:
    _lib.oocz_destroy(ctx)


# ------------------------------------------------------------------ codec / kernels
def oocz_zfp_bytes(nx: int, ny: int, nz: int, rate: int) -> int:
    return int(_lib.oocz_zfp_bytes(nx, ny, nz, rate))


def oocz_zfp_encode(d_in, nx, ny, nz, rate, d_out, stream=None) -> None:
    _check(_lib.oocz_zfp_encode(_ptr(d_in), nx, ny, nz, rate, _ptr(d_out), _stream(stream)))


def oocz_zfp_decode(d_in, nx, ny, nz, rate, d_out, stream=None) -> None:
    _check(_lib.oocz_zfp_decode(_ptr(d_in), nx, ny, nz, rate, _ptr(d_out), _stream(stream)))


def oocz_stencil_steps(d_u, d_uprev, d_m, nx, ny, nz, c, nsteps, stream=None) -> None:
    _check(_lib.oocz_stencil_steps(_ptr(d_u), _ptr(d_uprev), _ptr(d_m), nx, ny, nz, _c5(c), nsteps,
                                   _stream(stream)))


def oocz_stencil_step_planes(d_u, d_uprev, d_m, nx, ny, nz, c, z0, z1, zv0, zv1, stream=None) -> None:
    _check(_lib.oocz_stencil_step_planes(_ptr(d_u), _ptr(d_uprev), _ptr(d_m), nx, ny, nz, _c5(c),
                                         z0, z1, zv0, zv1, _stream(stream)))


def oocz_zfp_encode_f64(d_in, nx, ny, nz, rate, d_out, stream=None) -> None:
    _check(_lib.oocz_zfp_encode_f64(_ptr(d_in), nx, ny, nz, rate, _ptr(d_out), _stream(stream)))


def oocz_zfp_decode_f64(d_in, nx, ny, nz, rate, d_out, stream=None) -> None:
    _check(_lib.oocz_zfp_decode_f64(_ptr(d_in), nx, ny, nz, rate, _ptr(d_out), _stream(stream)))


def oocz_stencil_steps_f64(d_u, d_uprev, d_m, nx, ny, nz, c, nsteps, stream=None) -> None:
    _check(_lib.oocz_stencil_steps_f64(_ptr(d_u), _ptr(d_uprev), _ptr(d_m), nx, ny, nz, _c5d(c), nsteps,
                                       _stream(stream)))


def oocz_stencil_step_planes_f64(d_u, d_uprev, d_m, nx, ny, nz, c, z0, z1, zv0, zv1, stream=None) -> None:
    _check(_lib.oocz_stencil_step_planes_f64(_ptr(d_u), _ptr(d_uprev), _ptr(d_m), nx, ny, nz, _c5d(c),
                                             z0, z1, zv0, zv1, _stream(stream)))


def oocz_kernel_launch_count() -> int:
    return int(_lib.oocz_kernel_launch_count())


def default_coeffs() -> np.ndarray:
    cfg = oocz_default_config(4, 4, 4)
    return np.array(list(cfg.c), np.float32)


def default_coeffs64() -> np.ndarray:
    cfg = oocz_default_config(4, 4, 4)
    return np.array(list(cfg.c64), np.float64)


# ------------------------------------------------------------------ convenience
class Stepper:
    """RAII wrapper: ``with Stepper(cfg) as s: s.set(u, up, m); s.step(n); s.get(OOCZ_U)``."""

    def __init__(self, cfg: oocz_config, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 device: int = 0):
        self.cfg = cfg
        self.world = world
        self.ctx = oocz_create(cfg, rank, world, nccl_id, device)
        self.shape = (cfg.nz // world, cfg.ny, cfg.nx)
        self.dtype = np.float64 if cfg.precision == 64 else np.float32

    def set(self, u, uprev, m):
        for f, a in ((OOCZ_U, u), (OOCZ_UPREV, uprev), (OOCZ_M, m)):
            oocz_set_field(self.ctx, f, a)

    def step(self, n: int):
        oocz_step(self.ctx, n)

    def get(self, field: int) -> np.ndarray:
        return oocz_get_field(self.ctx, field, np.empty(self.shape, self.dtype))

    def stats(self) -> dict:
        return oocz_get_stats(self.ctx)

    def close(self):
        if self.ctx:
            oocz_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
