"""paper_2511_03909_b200 -- B200-native WECT / ECF hot path of arXiv 2511.03909.

Thin Python binding over libwect.so (C ABI in include/wect.h).  The functions
take torch tensors (CUDA or CPU) or numpy arrays and only marshal arguments;
every step of the method runs in the library's sm_100a kernels.  Host (CPU)
arrays are staged through the device by the library itself (the end-to-end
path); CUDA tensors are used in place on torch's current stream.

    wect_images(img, dirs, T)        WECT of a batch of uint8 images / volumes
    wect_complex(coords, cells, dirs, T, vweights=...)
    ecf_complex(fvals, cells, T, k0=..., vweights=...)
    wect_maxheight(coords, dirs)     M = max |<x, s>|, binary64

Multi-GPU sharding lives in paper_2511_03909_b200.dist.
"""
from __future__ import annotations

import ctypes
from typing import Iterable, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import FP32_ONLY, FREUDENTHAL, TIME_MAIN, VALIDATE, WectError  # noqa: F401

__all__ = ["wect_images", "ecf_images", "wect_complex", "ecf_complex", "wect_complex_backward", "ecf_complex_backward", "wect_maxheight", "sync_status", "repair_count",
           "stats", "WectError", "VALIDATE", "FP32_ONLY", "TIME_MAIN", "load"]

load = _lib.load


def _torch():
    import torch

    return torch


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    raise TypeError(f"unsupported array type {type(x)}")


def _as(x, np_dtype, torch_dtype_name):
    """Contiguous array of the required dtype, same kind (torch/numpy) and device."""
    if x is None:
        return None
    if _is_torch(x):
        torch = _torch()
        td = getattr(torch, torch_dtype_name)
        if x.dtype != td:
            raise TypeError(f"expected {td}, got {x.dtype}")
        return x.contiguous()
    x = np.ascontiguousarray(x)
    if x.dtype != np_dtype:
        raise TypeError(f"expected {np.dtype(np_dtype)}, got {x.dtype}")
    return x


def _device_of(*xs):
    for x in xs:
        if x is not None and _is_torch(x) and x.is_cuda:
            return x.device
    return None


def _stream(dev, stream):
    if stream is not None:
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    if dev is None:
        return None
    return _torch().cuda.current_stream(dev).cuda_stream


def _grid(T, d_begin, d_count, maxheight, lo, hi, flags):
    return _lib.wect_grid(int(T), int(d_begin), int(d_count), float(maxheight), float(lo), float(hi), int(flags))


def _alloc_out(shape, torch_dtype_name, dev, out):
    """A fresh output tensor, or the caller's out= after checking that the library may
    write exactly prod(shape) elements of torch_dtype_name into it (the C ABI only sees a
    pointer: a short, mistyped or strided out would be written out of bounds)."""
    torch = _torch()
    td = getattr(torch, torch_dtype_name)
    if out is not None:
        if not _is_torch(out):
            raise TypeError("out must be a torch tensor")
        n = 1
        for d in shape:
            n *= int(d)
        if out.numel() != n:
            raise ValueError(f"out has {out.numel()} elements, expected {n} (shape {tuple(shape)})")
        if out.dtype != td:
            raise ValueError(f"out dtype {out.dtype} does not match the output dtype {td}")
        if dev is not None and out.device != dev:
            raise ValueError(f"out is on {out.device}, inputs on {dev}")
        if not out.is_contiguous():
            raise ValueError("out must be contiguous")
        return out
    return torch.empty(shape, dtype=td, device=dev if dev is not None else "cpu")


def wect_images(img, dirs, T: int, *, d_begin: int = 0, d_count: int = 0, maxheight: float = 0.0, lo: float = 0.0,
                hi: float = 0.0, out_dtype: str = "int32", out=None, flags: int = 0, freudenthal: bool = False,
                stream=None):
    """WECT of a batch of uint8 images [B, H, W] or volumes [B, Z, Y, X], as
    cubical complexes, or (freudenthal=True, 2-D) as Freudenthal triangulations.

    Returns [B, d_count or D - d_begin, T] (int32 or int64)."""
    if freudenthal:
        flags |= _lib.FREUDENTHAL
    L = _lib.load()
    img = _as(img, np.uint8, "uint8")
    dirs = _as(dirs, np.float32, "float32")
    if img.ndim not in (3, 4):
        raise ValueError("img must be [B, H, W] or [B, Z, Y, X]")
    B = int(img.shape[0])
    dims = (ctypes.c_int64 * (img.ndim - 1))(*[int(d) for d in img.shape[1:]])
    D = int(dirs.shape[0])
    rows = d_count if d_count else D - d_begin
    dev = _device_of(img, dirs)
    out = _alloc_out((B, rows, int(T)), out_dtype, dev, out)
    odt = {"int32": _lib.I32, "int64": _lib.I64}[out_dtype]
    g = _grid(T, d_begin, d_count, maxheight, lo, hi, flags)
    _lib.check(L.wect_images(_ptr(img), B, img.ndim - 1, dims, _ptr(dirs), D, ctypes.byref(g), _ptr(out), odt,
                             _stream(dev, stream)))
    return out


def ecf_images(img, T: int, *, maxheight: float = 0.0, lo: float = 0.0, hi: float = 0.0, out_dtype: str = "int32",
               out=None, flags: int = 0, stream=None):
    """ECF of a batch of uint8 images [B, H, W] or volumes [B, Z, Y, X]: intensity as the
    vertex filter, unweighted lower-star Euler characteristic (Remark "which-ecf",
    P:273-282).  Grid: [lo, hi] if lo < hi, else [-maxheight, maxheight] if maxheight > 0,
    else each image's own [-M, M].  Returns [B, T] (int32 or int64)."""
    L = _lib.load()
    img = _as(img, np.uint8, "uint8")
    if img.ndim not in (3, 4):
        raise ValueError("img must be [B, H, W] or [B, Z, Y, X]")
    B = int(img.shape[0])
    dims = (ctypes.c_int64 * (img.ndim - 1))(*[int(d) for d in img.shape[1:]])
    dev = _device_of(img)
    out = _alloc_out((B, int(T)), out_dtype, dev, out)
    odt = {"int32": _lib.I32, "int64": _lib.I64}[out_dtype]
    g = _grid(T, 0, 0, maxheight, lo, hi, flags)
    _lib.check(L.ecf_images(_ptr(img), B, img.ndim - 1, dims, ctypes.byref(g), _ptr(out), odt, _stream(dev, stream)))
    return out


def _cells_array(cells: Sequence[Tuple], is_float: bool):
    """cells: [(verts [count, arity] int32, weights [count] or None, dim), ...]"""
    arr = (_lib.wect_cells * max(1, len(cells)))()
    keep = []
    for i, (verts, weights, dim) in enumerate(cells):
        verts = _as(verts, np.int32, "int32")
        weights = _as(weights, np.float32, "float32") if (is_float and weights is not None) else (
            _as(weights, np.int32, "int32") if weights is not None else None)
        keep += [verts, weights]
        count = int(verts.shape[0])
        arity = int(verts.shape[1]) if verts.ndim == 2 else 1
        arr[i] = _lib.wect_cells(_ptr(verts), _ptr(weights), count, arity, int(dim))
    return arr, keep


def _run_complex(fn, k0, n, coords, vweights, cells, src, D, T, is_float, d_begin, d_count, maxheight, lo, hi, out,
                 flags, stream, dev_hint):
    L = _lib.load()
    arr, keep = _cells_array(cells, is_float)
    if vweights is not None:
        vweights = _as(vweights, np.float32, "float32") if is_float else _as(vweights, np.int32, "int32")
    desc = _lib.wect_complex_desc(_ptr(coords), int(k0), int(n), _ptr(vweights), arr, len(cells),
                                  _lib.F32 if is_float else _lib.I32)
    rows = d_count if d_count else D - d_begin
    dev = dev_hint
    out = _alloc_out((rows, int(T)), "float64" if is_float else "int64", dev, out)
    g = _grid(T, d_begin, d_count, maxheight, lo, hi, flags)
    _lib.check(fn(ctypes.byref(desc), _ptr(src), int(D), ctypes.byref(g), _ptr(out),
                  _lib.F64 if is_float else _lib.I64, _stream(dev, stream)))
    del keep
    return out


def wect_complex(coords, cells: Sequence[Tuple], dirs, T: int, *, vweights=None, is_float: Optional[bool] = None,
                 d_begin: int = 0, d_count: int = 0, maxheight: float = 0.0, out=None, flags: int = 0, stream=None):
    """WECT of an explicit weighted complex (Alg. 1 with FVals = V D^T).

    coords [k0, n] fp32; cells [(verts int32 [k, arity], weights or None, dim)];
    dirs [D, n] fp32.  Integer weights -> int64 [rows, T]; float weights -> float64."""
    coords = _as(coords, np.float32, "float32")
    dirs = _as(dirs, np.float32, "float32")
    if is_float is None:
        ws = [w for _, w, _ in cells if w is not None] + ([vweights] if vweights is not None else [])
        is_float = bool(ws) and str(ws[0].dtype).endswith("float32")
    k0, n = int(coords.shape[0]), int(coords.shape[1])
    return _run_complex(_lib.load().wect_complex, k0, n, coords, vweights, cells, dirs, int(dirs.shape[0]), T,
                        is_float, d_begin, d_count, maxheight, 0.0, 0.0, out, flags, stream,
                        _device_of(coords, dirs, vweights, *[c[0] for c in cells]))


def ecf_complex(fvals, cells: Sequence[Tuple], T: int, *, vweights=None, is_float: Optional[bool] = None,
                d_begin: int = 0, d_count: int = 0, maxheight: float = 0.0, lo: float = 0.0, hi: float = 0.0,
                out=None, flags: int = 0, stream=None):
    """WECFs for given vertex filters (Alg. 1).  fvals [k0, m] fp32.
    lo < hi selects an explicit height grid (reading A9)."""
    fvals = _as(fvals, np.float32, "float32")
    if fvals.ndim == 1:
        fvals = fvals.reshape(-1, 1)
    if is_float is None:
        ws = [w for _, w, _ in cells if w is not None] + ([vweights] if vweights is not None else [])
        is_float = bool(ws) and str(ws[0].dtype).endswith("float32")
    k0, m = int(fvals.shape[0]), int(fvals.shape[1])
    return _run_complex(_lib.load().ecf_complex, k0, 1, None, vweights, cells, fvals, m, T, is_float, d_begin,
                        d_count, maxheight, lo, hi, out, flags, stream,
                        _device_of(fvals, vweights, *[c[0] for c in cells]))


def _run_backward(fn, k0, n, coords, cells, src, D, T, G, d_begin, d_count, maxheight, lo, hi, flags, stream, dev_hint):
    L = _lib.load()
    arr, keep = _cells_array([(v, None, d) for v, _, d in cells], False)
    desc = _lib.wect_complex_desc(_ptr(coords), int(k0), int(n), None, arr, len(cells), _lib.I32)
    G = _as(G, np.float64, "float64")
    dev = dev_hint
    gv = _alloc_out((int(k0),), "float64", dev, None)
    gc = [_alloc_out((int(v.shape[0]),), "float64", dev, None) for v, _, _ in cells]
    ptrs = (ctypes.c_void_p * max(1, len(cells)))(*[_ptr(x) for x in gc])
    g = _grid(T, d_begin, d_count, maxheight, lo, hi, flags)
    _lib.check(fn(ctypes.byref(desc), _ptr(src), int(D), ctypes.byref(g), _ptr(G), _ptr(gv), ptrs, _stream(dev, stream)))
    del keep
    return gv, gc


def wect_complex_backward(coords, cells: Sequence[Tuple], dirs, T: int, G, *, d_begin: int = 0, d_count: int = 0,
                          maxheight: float = 0.0, flags: int = 0, stream=None):
    """dL/dweights through wect_complex for G = dL/dout [rows, T] (fp64).  Returns
    (grad_vweights [k0], [grad_cells_i [count_i]]) in float64 (include/wect.h)."""
    coords = _as(coords, np.float32, "float32")
    dirs = _as(dirs, np.float32, "float32")
    k0, n = int(coords.shape[0]), int(coords.shape[1])
    return _run_backward(_lib.load().wect_complex_backward, k0, n, coords, cells, dirs, int(dirs.shape[0]), T, G,
                         d_begin, d_count, maxheight, 0.0, 0.0, flags, stream, _device_of(coords, dirs, G))


def ecf_complex_backward(fvals, cells: Sequence[Tuple], T: int, G, *, d_begin: int = 0, d_count: int = 0,
                         maxheight: float = 0.0, lo: float = 0.0, hi: float = 0.0, flags: int = 0, stream=None):
    """dL/dweights through ecf_complex for G = dL/dout [rows, T] (fp64)."""
    fvals = _as(fvals, np.float32, "float32")
    if fvals.ndim == 1:
        fvals = fvals.reshape(-1, 1)
    k0, m = int(fvals.shape[0]), int(fvals.shape[1])
    return _run_backward(_lib.load().ecf_complex_backward, k0, 1, None, cells, fvals, m, T, G, d_begin, d_count,
                         maxheight, lo, hi, flags, stream, _device_of(fvals, G))


def wect_maxheight(coords, dirs, stream=None) -> float:
    L = _lib.load()
    coords = _as(coords, np.float32, "float32")
    dirs = _as(dirs, np.float32, "float32")
    M = ctypes.c_double(0.0)
    dev = _device_of(coords, dirs)
    _lib.check(L.wect_maxheight(_ptr(coords), int(coords.shape[0]), int(coords.shape[1]), _ptr(dirs),
                                int(dirs.shape[0]), ctypes.byref(M), _stream(dev, stream)))
    return M.value


def sync_status(stream=None) -> None:
    """Synchronise and raise WectError(WECT_ERANGE) if a kernel saw a bad vertex index."""
    L = _lib.load()
    _lib.check(L.wect_sync_status(_stream(_device_of(), stream) if stream is not None else None))


def repair_count(reset: bool = False) -> int:
    """binary64 near-edge repairs since the last reset (reading A1)."""
    L = _lib.load()
    c = ctypes.c_uint64(0)
    _lib.check(L.wect_repair_count(ctypes.byref(c), 1 if reset else 0))
    return int(c.value)


def stats(reset: bool = False):
    """(kernel launches, timed dominant-kernel launches, their summed device ms) since the
    last reset; the timed pair is recorded only for calls made with flags=TIME_MAIN."""
    L = _lib.load()
    a, b, ms = ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_double(0.0)
    _lib.check(L.wect_stats(ctypes.byref(a), ctypes.byref(b), ctypes.byref(ms), 1 if reset else 0))
    return int(a.value), int(b.value), float(ms.value)
