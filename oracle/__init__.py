"""CPU oracle for the WECT / WECF hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It shares no code with
paper_2511_03909_b200/ (the CUDA path) and never imports it.

Arms:
  O0  oracle.exact      -- exact rational arithmetic (fractions), tiny inputs.
  O1  wecfs_naive       -- naive sublevel-set enumeration in binary64.
  O2  wecfs_alg1        -- Algorithm 1 step by step in binary64.
The binary64 arms live in wect_oracle.c (built by oracle/build.py).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

from . import build as _build

_LIB = None


class _Cells(ctypes.Structure):
    _fields_ = [("verts", ctypes.c_void_p), ("weights", ctypes.c_void_p), ("count", ctypes.c_int64),
                ("arity", ctypes.c_int32), ("dim", ctypes.c_int32)]


def lib():
    global _LIB
    if _LIB is None:
        path = _build.build()
        L = ctypes.CDLL(path)
        d, i64, i32, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        L.orc_heights.argtypes = [vp, i64, i32, vp, i32, vp]
        L.orc_maxheight.argtypes = [vp, i64, i32]
        L.orc_maxheight.restype = d
        L.orc_alpha.argtypes = [d, d, d, i32]
        L.orc_alpha.restype = i32
        L.orc_beta.argtypes = [i32, d, d, i32]
        L.orc_beta.restype = d
        for f in (L.orc_wecfs_alg1, L.orc_wecfs_naive):
            f.argtypes = [vp, i64, i32, vp, vp, i32, ctypes.c_int, i32, d, d, vp]
            f.restype = ctypes.c_int
        L.orc_grid_coords.argtypes = [i32, vp, vp]
        L.orc_grid_cells.argtypes = [i32, vp, vp, vp, vp, vp]
        L.orc_wect_images.argtypes = [vp, i64, i32, vp, vp, i32, i32, d, ctypes.c_int, vp]
        L.orc_wect_images.restype = ctypes.c_int
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        _LIB = L
    return _LIB


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


# ----------------------------------------------------------------- primitives
def heights(coords: np.ndarray, dirs: np.ndarray) -> np.ndarray:
    """FVals = V * D^T in binary64 (Example "wect")."""
    coords = np.ascontiguousarray(coords, np.float32)
    dirs = np.ascontiguousarray(dirs, np.float32)
    k0, n = coords.shape
    D = dirs.shape[0]
    out = np.empty((k0, D), np.float64)
    lib().orc_heights(_p(coords), k0, n, _p(dirs), D, _p(out))
    return out


def maxheight(fvals: np.ndarray) -> float:
    fvals = np.ascontiguousarray(fvals, np.float64)
    k0 = fvals.shape[0]
    m = fvals.shape[1] if fvals.ndim == 2 else 1
    return float(lib().orc_maxheight(_p(fvals), k0, m))


def alpha(t: float, lo: float, hi: float, T: int) -> int:
    return int(lib().orc_alpha(float(t), float(lo), float(hi), int(T)))


def beta(q: int, lo: float, hi: float, T: int) -> float:
    return float(lib().orc_beta(int(q), float(lo), float(hi), int(T)))


def _cells_struct(cx):
    arr = (_Cells * max(1, len(cx.cells)))()
    keep = []
    for i, c in enumerate(cx.cells):
        v = np.ascontiguousarray(c.verts, np.int32)
        if c.weights is None:
            w = None
        elif cx.is_float:
            w = np.ascontiguousarray(c.weights, np.float64)
        else:
            w = np.ascontiguousarray(c.weights, np.int64)
        keep += [v, w]
        arr[i].verts = _p(v)
        arr[i].weights = _p(w)
        arr[i].count = v.shape[0]
        arr[i].arity = v.shape[1] if v.ndim == 2 else 1
        arr[i].dim = c.dim
    return arr, keep


def wecfs(fvals: np.ndarray, cx, T: int, lo: float, hi: float, naive: bool = False) -> np.ndarray:
    """Alg. 1 (O2) or the naive enumeration (O1) for FVals [k0, m] (binary64)."""
    fvals = np.ascontiguousarray(fvals, np.float64)
    k0 = fvals.shape[0]
    m = fvals.shape[1]
    arr, keep = _cells_struct(cx)
    if cx.vweights is None:
        vw = None
    else:
        vw = np.ascontiguousarray(cx.vweights, np.float64 if cx.is_float else np.int64)
    out = np.zeros((m, T), np.float64 if cx.is_float else np.int64)
    f = lib().orc_wecfs_naive if naive else lib().orc_wecfs_alg1
    rc = f(_p(fvals), k0, m, _p(vw), arr, len(cx.cells), 1 if cx.is_float else 0, T, float(lo), float(hi), _p(out))
    if rc != 0:
        raise IndexError("vertex index out of range")
    return out


# ---------------------------------------------------------- the three calls
def wect_complex(cx, dirs: np.ndarray, T: int, maxheight_override: float = 0.0,
                 naive: bool = False, rows: Optional[slice] = None) -> np.ndarray:
    """WECT of an explicit complex: M over ALL directions (reading A2)."""
    fv = heights(cx.coords, dirs)
    M = maxheight_override if maxheight_override > 0 else maxheight(fv)
    if rows is not None:
        fv = np.ascontiguousarray(fv[:, rows])
    return wecfs(fv, cx, T, -M, M, naive)


def ecf_complex(cx, fvals32: np.ndarray, T: int, lo: float = 0.0, hi: float = 0.0,
                maxheight_override: float = 0.0, naive: bool = False) -> np.ndarray:
    """WECFs for caller filters FVals (fp32, exact in binary64)."""
    fv = np.ascontiguousarray(fvals32, np.float32).astype(np.float64)
    if fv.ndim == 1:
        fv = fv[:, None]
    if not lo < hi:
        M = maxheight_override if maxheight_override > 0 else maxheight(fv)
        lo, hi = -M, M
    return wecfs(fv, cx, T, lo, hi, naive)


def grid_coords(dims) -> np.ndarray:
    dims = np.ascontiguousarray(dims, np.int64)
    nv = int(np.prod(dims))
    out = np.empty((nv, len(dims)), np.float32)
    lib().orc_grid_coords(len(dims), _p(dims), _p(out))
    return out


def grid_complex(img: np.ndarray):
    """Explicit cubical complex (V-construction) of ONE image / volume (P:213-215,
    P:337-338; readings A3, A5, A7), as a synth.Complex with int weights."""
    import synth  # generator container type only

    dims = np.ascontiguousarray(img.shape, np.int64)
    nd = len(dims)
    im = np.ascontiguousarray(img, np.uint8).reshape(-1)
    counts = np.zeros(4, np.int64)
    lib().orc_grid_cells(nd, _p(dims), _p(im), _p(counts), None, None)
    verts_arr = (ctypes.c_void_p * 4)()
    w_arr = (ctypes.c_void_p * 4)()
    keep = {}
    for i in range(1, nd + 1):
        keep[i] = (np.zeros((int(counts[i]), 1 << i), np.int32), np.zeros(int(counts[i]), np.int64))
        verts_arr[i] = _p(keep[i][0]) if counts[i] > 0 else None
        w_arr[i] = _p(keep[i][1]) if counts[i] > 0 else None
    lib().orc_grid_cells(nd, _p(dims), _p(im), _p(counts), verts_arr, w_arr)
    cells = [synth.Cells(keep[i][0], keep[i][1].astype(np.int32), i) for i in range(1, nd + 1)]
    return synth.Complex(grid_coords(dims), im.astype(np.int32), cells, im.shape[0], is_float=False)


def wect_images(img: np.ndarray, dirs: np.ndarray, T: int, maxheight_override: float = 0.0,
                naive: bool = False) -> np.ndarray:
    """O2 (or O1) WECT of a batch [B, dims...] of uint8 images: int64 [B, D, T]."""
    img = np.ascontiguousarray(img, np.uint8)
    B = img.shape[0]
    dims = np.ascontiguousarray(img.shape[1:], np.int64)
    dirs = np.ascontiguousarray(dirs, np.float32)
    D = dirs.shape[0]
    out = np.zeros((B, D, T), np.int64)
    rc = lib().orc_wect_images(_p(img), B, len(dims), _p(dims), _p(dirs), D, T, float(maxheight_override),
                               1 if naive else 0, _p(out))
    if rc != 0:
        raise RuntimeError(rc)
    return out


def ecf_images(img: np.ndarray, T: int, lo: float = 0.0, hi: float = 0.0, maxheight_override: float = 0.0,
               naive: bool = False) -> np.ndarray:
    """O2 (or O1) ECF of a batch [B, dims...] of uint8 images (Remark "which-ecf",
    P:273-282): per image, the explicit cubical complex with UNIT weights, the
    intensities as the one vertex filter (fp32, exact), Alg. 1 with m = 1 on the grid
    [lo, hi] if lo < hi, else [-maxheight, maxheight] if given, else the image's own
    [-M, M].  int64 [B, T]."""
    import synth  # generator container type only

    img = np.ascontiguousarray(img, np.uint8)
    out = np.zeros((img.shape[0], T), np.int64)
    for b in range(img.shape[0]):
        cx = grid_complex(img[b])
        unit = synth.Complex(cx.coords, None, [synth.Cells(c.verts, None, c.dim) for c in cx.cells], cx.k0,
                             is_float=False)
        f = img[b].reshape(-1).astype(np.float32)
        out[b] = ecf_complex(unit, f, T, lo, hi, maxheight_override, naive)[0]
    return out


# ------------------------------------------------------- weights gradient (NEXT-3)
def alpha_vec(t: np.ndarray, lo: float, hi: float, T: int) -> np.ndarray:
    """alpha (eq. left-adjoint) elementwise in binary64, in the written order:
    u = ((T-1) * (t - lo)) / (hi - lo), clamp(ceil(u), 0, T-1); hi <= lo -> 0 (reading A6)."""
    t = np.asarray(t, np.float64)
    if not hi > lo:
        return np.zeros(t.shape, np.int64)
    u = (float(T - 1) * (t - lo)) / (hi - lo)
    return np.clip(np.ceil(u), 0, T - 1).astype(np.int64)


def wecfs_grad(fvals: np.ndarray, cx, T: int, lo: float, hi: float, G: np.ndarray, vertices=None):
    """dL/dw for L with G = dL/dWECFs [m, T], straight from the closed form:
    WECFs[p, q] = sum_s w(s) (-1)^dim s [bin(s, p) <= q], bin(s, p) = max over the vertices
    of s of alpha(f_p(v)) (Alg. 1 lines 3, 7-8), so
        dL/dw(s) = sum_{p, q} G[p, q] (-1)^dim s [bin(s, p) <= q].
    The indicator is materialised ([cells, m, T]) -- small inputs only (`vertices`: an index
    subset for the vertex part, e.g. samples of a full-size complex).
    Returns (grad_vweights [k0] or [len(vertices)], [grad_cells_i]) in float64."""
    fv = np.asarray(fvals, np.float64)
    G = np.asarray(G, np.float64)
    vb = alpha_vec(fv, lo, hi, T)  # [k0, m]
    q = np.arange(T)

    def grad_of(bins, sign):  # bins [count, m]
        ind = (bins[:, :, None] <= q[None, None, :]).astype(np.float64)
        return sign * np.einsum("spq,pq->s", ind, G)

    gv = grad_of(vb if vertices is None else vb[np.asarray(vertices)], 1.0)
    gc = []
    for c in cx.cells:
        v = np.asarray(c.verts, np.int64).reshape(len(c.verts), -1)
        gc.append(grad_of(vb[v].max(axis=1), -1.0 if c.dim % 2 else 1.0))
    return gv, gc


def wect_complex_grad(cx, dirs: np.ndarray, T: int, G: np.ndarray, maxheight_override: float = 0.0):
    """Weights gradient through wect_complex (M over ALL directions, reading A2)."""
    fv = heights(cx.coords, dirs)
    M = maxheight_override if maxheight_override > 0 else maxheight(fv)
    return wecfs_grad(fv, cx, T, -M, M, G)


def ecf_complex_grad(cx, fvals32: np.ndarray, T: int, G: np.ndarray, lo: float = 0.0, hi: float = 0.0):
    fv = np.ascontiguousarray(fvals32, np.float32).astype(np.float64)
    if fv.ndim == 1:
        fv = fv[:, None]
    if not lo < hi:
        M = maxheight(fv)
        lo, hi = -M, M
    return wecfs_grad(fv, cx, T, lo, hi, G)


# ------------------------------------------------ Freudenthal images (NEXT-2)
def freudenthal_complex(img: np.ndarray):
    """Explicit weighted Freudenthal complex of ONE 2-D image: pixels
    are vertices at the grid coordinates of reading A3; edges are the horizontal, vertical
    and (r,c)-(r+1,c+1) diagonal pairs; each unit square splits along that diagonal into
    {(r,c),(r,c+1),(r+1,c+1)} and {(r,c),(r+1,c),(r+1,c+1)}; vertex weight = intensity,
    every other simplex's weight = max of its vertices' weights."""
    import synth  # generator container type only

    im = np.ascontiguousarray(img, np.uint8)
    H, W = im.shape
    idx = np.arange(H * W, dtype=np.int64).reshape(H, W)
    flat = im.reshape(-1).astype(np.int64)
    e = [np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1),      # horizontal
         np.stack([idx[:-1, :].ravel(), idx[1:, :].ravel()], 1),      # vertical
         np.stack([idx[:-1, :-1].ravel(), idx[1:, 1:].ravel()], 1)]   # diagonal (r,c)-(r+1,c+1)
    edges = np.concatenate(e, 0)
    t_up = np.stack([idx[:-1, :-1].ravel(), idx[:-1, 1:].ravel(), idx[1:, 1:].ravel()], 1)
    t_lo = np.stack([idx[:-1, :-1].ravel(), idx[1:, :-1].ravel(), idx[1:, 1:].ravel()], 1)
    tris = np.concatenate([t_up, t_lo], 0)
    ew = flat[edges].max(axis=1) if len(edges) else np.zeros(0, np.int64)
    tw = flat[tris].max(axis=1) if len(tris) else np.zeros(0, np.int64)
    cells = [synth.Cells(edges.astype(np.int32).reshape(-1, 2), ew.astype(np.int32), 1),
             synth.Cells(tris.astype(np.int32).reshape(-1, 3), tw.astype(np.int32), 2)]
    return synth.Complex(grid_coords((H, W)), flat.astype(np.int32), cells, H * W, is_float=False)


def wect_images_freudenthal(img: np.ndarray, dirs: np.ndarray, T: int, maxheight_override: float = 0.0,
                            naive: bool = False) -> np.ndarray:
    """O2 (or O1) WECT of a batch [B, H, W] of u8 images as Freudenthal complexes, M over
    ALL directions of the (image-independent) grid (reading A2): int64 [B, D, T]."""
    img = np.ascontiguousarray(img, np.uint8)
    out = np.zeros((img.shape[0], dirs.shape[0], T), np.int64)
    for b in range(img.shape[0]):
        cx = freudenthal_complex(img[b])
        out[b] = wect_complex(cx, dirs, T, maxheight_override, naive)
    return out
