"""Helpers for the -m gpu tests: move numpy arrays through the C ABI's codec /
kernel entry points (device pointers from torch tensors) and back."""
import numpy as np


def Z():
    from paper_2109_05410_b200 import oocz
    return oocz


def to_dev(a: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_encode(field: np.ndarray, rate: int) -> np.ndarray:
    import torch
    nz, ny, nx = field.shape
    z = Z()
    d_in = to_dev(field.astype(np.float32))
    out = torch.empty(max(z.oocz_zfp_bytes(nx, ny, nz, rate) // 8, 1), dtype=torch.int64, device="cuda")
    z.oocz_zfp_encode(d_in, nx, ny, nz, rate, out, torch.cuda.current_stream())
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint64)[: z.oocz_zfp_bytes(nx, ny, nz, rate) // 8]


def gpu_decode(words: np.ndarray, shape, rate: int) -> np.ndarray:
    import torch
    nz, ny, nx = shape
    z = Z()
    d_in = to_dev(np.ascontiguousarray(words, np.uint64).view(np.int64))
    out = torch.empty((nz, ny, nx), dtype=torch.float32, device="cuda")
    z.oocz_zfp_decode(d_in, nx, ny, nz, rate, out, torch.cuda.current_stream())
    torch.cuda.synchronize()
    return out.cpu().numpy()


def bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, np.float32).view(np.uint32)
