"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds input GENERATORS only -- none of the method's arithmetic
(no heights, no binning, no histogram, no cumsum, no image embedding; the
image coordinate convention of DESIGN.md reading A3 is implemented separately
by oracle/ and by the library).  Both sides consume exactly the arrays made
here.  Recipes:

* images: uint8 U{0..255} (the paper's random fill of its padded set),
  or an "fmnist-like" centred textured blob on a zero background;
* directions on S^1: theta_p = 2*pi*p/D from (1, 0) (reading A4), computed in
  binary64 and rounded once to fp32;  on S^{n-1}, n >= 3: seeded standard
  normal rows normalised in binary64, rounded once to fp32;
* cfg4 mesh: a 2500 x 4000 torus grid triangulated with one diagonal per
  square (V = 1e7, E = 3e7, F = 2e7, chi = 0), fp32 coordinates with
  N(0, 1e-3) jitter, int32 weights U{0..255} on every cell;
* cfg5: 1e6 points U[-1,1]^5; 2e6 random sorted 5-subsets with all faces
  de-duplicated; fp32 weights U[0,1) on every cell;
* small random closed simplicial complexes for the parity suites.

Seed base S0 = 251103909; config c uses S0 + c (numpy PCG64).
"""
from __future__ import annotations

import dataclasses
import itertools
from typing import List, Optional

import numpy as np

S0 = 251103909


@dataclasses.dataclass
class Cells:
    verts: np.ndarray  # int32 [count, arity]
    weights: Optional[np.ndarray]  # int32 or float32 [count]; None = unit weights
    dim: int


@dataclasses.dataclass
class Complex:
    coords: Optional[np.ndarray]  # float32 [k0, n] (None for pure-filter ECF inputs)
    vweights: Optional[np.ndarray]  # int32 / float32 [k0] or None (unit)
    cells: List[Cells]
    k0: int
    is_float: bool = False  # weight dtype: False -> int32, True -> float32

    @property
    def n(self) -> int:
        return 0 if self.coords is None else int(self.coords.shape[1])

    def num_cells(self) -> int:
        return self.k0 + sum(int(c.verts.shape[0]) for c in self.cells)


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


# ---------------------------------------------------------------- directions
def directions_s1(D: int) -> np.ndarray:
    th = 2.0 * np.pi * np.arange(D, dtype=np.float64) / D
    return np.stack([np.cos(th), np.sin(th)], axis=1).astype(np.float32)


def directions_sphere(D: int, n: int, seed: int) -> np.ndarray:
    if n == 2:
        return directions_s1(D)
    g = rng(seed).standard_normal((D, n))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    return g.astype(np.float32)


# ------------------------------------------------------------------- images
def images_u8(B: int, dims, seed: int, kind: str = "uniform") -> np.ndarray:
    dims = tuple(int(d) for d in dims)
    r = rng(seed)
    if kind == "uniform":
        return r.integers(0, 256, size=(B,) + dims, dtype=np.uint8)
    if kind == "fmnist":
        # centred textured blob on a zero background (about half the pixels zero)
        grids = np.meshgrid(*[np.linspace(-1, 1, d) for d in dims], indexing="ij")
        rad = np.sqrt(sum(g * g for g in grids))
        out = np.zeros((B,) + dims, dtype=np.uint8)
        for b0 in range(0, B, 4096):
            b1 = min(B, b0 + 4096)
            scale = r.uniform(0.55, 0.85, size=(b1 - b0,) + (1,) * len(dims))
            tex = r.integers(40, 256, size=(b1 - b0,) + dims)
            mask = rad[None] < scale
            out[b0:b1] = np.where(mask, tex, 0).astype(np.uint8)
        return out
    if kind == "blobs":
        # smooth Gaussian blobs on a zero background (cfg3 variant)
        out = np.zeros((B,) + dims, dtype=np.float32)
        grids = np.meshgrid(*[np.arange(d, dtype=np.float32) for d in dims], indexing="ij")
        for b in range(B):
            for _ in range(6):
                c = [r.uniform(0, d) for d in dims]
                s = r.uniform(0.05, 0.15) * max(dims)
                d2 = sum((g - ci) ** 2 for g, ci in zip(grids, c))
                out[b] += 255.0 * np.exp(-d2 / (2 * s * s)).astype(np.float32)
        return np.clip(out, 0, 255).astype(np.uint8)
    raise ValueError(kind)


# ------------------------------------------------------------ explicit meshes
def torus_mesh(nu: int, nv: int, seed: int, R: float = 1.0, r: float = 0.4,
               jitter: float = 1e-3, shuffle: bool = False) -> Complex:
    """Torus grid nu x nv; edges right/down/diagonal, two triangles per square."""
    g = rng(seed)
    i = np.arange(nu, dtype=np.int64)[:, None]
    j = np.arange(nv, dtype=np.int64)[None, :]
    u = 2 * np.pi * np.arange(nu) / nu
    v = 2 * np.pi * np.arange(nv) / nv
    uu, vv = np.meshgrid(u, v, indexing="ij")
    xyz = np.stack([(R + r * np.cos(vv)) * np.cos(uu), (R + r * np.cos(vv)) * np.sin(uu), r * np.sin(vv)], axis=-1)
    xyz = xyz.reshape(-1, 3) + g.normal(0.0, jitter, size=(nu * nv, 3))
    coords = xyz.astype(np.float32)
    vid = (i * nv + j)
    ip = ((i + 1) % nu) * nv + j
    jp = i * nv + (j + 1) % nv
    dp = ((i + 1) % nu) * nv + (j + 1) % nv
    a, b, c, d = (np.broadcast_to(x, (nu, nv)).reshape(-1) for x in (vid, ip, jp, dp))
    edges = np.concatenate([np.stack([a, b], 1), np.stack([a, c], 1), np.stack([a, d], 1)]).astype(np.int32)
    tris = np.concatenate([np.stack([a, b, d], 1), np.stack([a, c, d], 1)]).astype(np.int32)
    k0 = nu * nv
    if shuffle:
        perm = g.permutation(k0).astype(np.int32)
        coords = coords[np.argsort(perm)]
        edges = perm[edges]
        tris = perm[tris]
        edges = edges[g.permutation(edges.shape[0])]
        tris = tris[g.permutation(tris.shape[0])]
    vw = g.integers(0, 256, size=k0, dtype=np.int32)
    ew = g.integers(0, 256, size=edges.shape[0], dtype=np.int32)
    tw = g.integers(0, 256, size=tris.shape[0], dtype=np.int32)
    return Complex(coords, vw, [Cells(edges, ew, 1), Cells(tris, tw, 2)], k0, is_float=False)


def _unique_rows(a: np.ndarray) -> np.ndarray:
    a = np.sort(a, axis=1)
    v = np.ascontiguousarray(a).view(np.dtype((np.void, a.dtype.itemsize * a.shape[1])))
    _, idx = np.unique(v, return_index=True)
    return a[np.sort(idx)]


def random_simplicial(nverts: int, nsimp: int, n: int, k: int, seed: int,
                      float_weights: bool = True) -> Complex:
    """nsimp random sorted (k+1)-subsets of nverts points in U[-1,1]^n, with all faces."""
    g = rng(seed)
    coords = g.uniform(-1.0, 1.0, size=(nverts, n)).astype(np.float32)
    top = np.empty((nsimp, k + 1), dtype=np.int64)
    filled = 0
    while filled < nsimp:
        cand = g.integers(0, nverts, size=(nsimp - filled, k + 1))
        cand.sort(axis=1)
        ok = np.all(cand[:, 1:] != cand[:, :-1], axis=1)
        cand = cand[ok]
        top[filled:filled + cand.shape[0]] = cand
        filled += cand.shape[0]
    cells = []
    for dim in range(1, k + 1):
        faces = [top[:, list(c)] for c in itertools.combinations(range(k + 1), dim + 1)]
        f = _unique_rows(np.concatenate(faces)).astype(np.int32)
        w = g.random(f.shape[0], dtype=np.float32) if float_weights else g.integers(0, 256, f.shape[0], dtype=np.int32)
        cells.append(Cells(f, w, dim))
    vw = g.random(nverts, dtype=np.float32) if float_weights else g.integers(0, 256, nverts, dtype=np.int32)
    return Complex(coords, vw, cells, nverts, is_float=float_weights)


def random_small_complex(seed: int, n: int = 3, nverts: int = 40, ntop: int = 30, kmax: int = 3,
                         float_weights: bool = False, wlo: int = -50, whi: int = 50) -> Complex:
    """A small closed simplicial complex (dim <= kmax) for parity suites: random top
    simplices of random dimension plus all their faces; vertices that no simplex
    uses stay as isolated vertices."""
    g = rng(seed)
    coords = g.uniform(-1.0, 1.0, size=(nverts, n)).astype(np.float32)
    by_dim = {d: set() for d in range(1, kmax + 1)}
    for _ in range(ntop):
        d = int(g.integers(1, kmax + 1))
        s = tuple(sorted(g.choice(nverts, size=d + 1, replace=False).tolist()))
        for dd in range(1, d + 1):
            for c in itertools.combinations(s, dd + 1):
                by_dim[dd].add(c)
    cells = []
    for d in range(1, kmax + 1):
        if not by_dim[d]:
            cells.append(Cells(np.zeros((0, d + 1), np.int32), np.zeros(0, np.float32 if float_weights else np.int32), d))
            continue
        v = np.array(sorted(by_dim[d]), dtype=np.int32)
        w = g.uniform(-1, 1, v.shape[0]).astype(np.float32) if float_weights else g.integers(wlo, whi, v.shape[0], dtype=np.int32)
        cells.append(Cells(v, w, d))
    vw = g.uniform(-1, 1, nverts).astype(np.float32) if float_weights else g.integers(wlo, whi, nverts, dtype=np.int32)
    return Complex(coords, vw, cells, nverts, is_float=float_weights)


# ------------------------------------------------------------------ configs
CONFIGS = {
    0: dict(name="cfg1_mnist1", kind="images", B=1, dims=(28, 28), D=32, T=64),
    1: dict(name="cfg2_mnist60k", kind="images", B=60000, dims=(28, 28), D=64, T=128),
    2: dict(name="cfg3_vol256", kind="images", B=1, dims=(256, 256, 256), D=512, T=256),
    3: dict(name="cfg4_torus10M", kind="complex", D=1024, T=512),
    4: dict(name="cfg5_r5_2M", kind="complex", D=256, T=256),
}


def make_config(c: int, image_kind: str = "uniform", scale: float = 1.0):
    """Return (inputs dict) for BASELINE.json configs[c]; scale < 1 shrinks batch/mesh."""
    spec = dict(CONFIGS[c])
    seed = S0 + c
    if spec["kind"] == "images":
        B = max(1, int(spec["B"] * scale))
        dims = spec["dims"]
        img = images_u8(B, dims, seed, image_kind)
        n = len(dims)
        dirs = directions_s1(spec["D"]) if n == 2 else directions_sphere(spec["D"], n, S0 + 30)
        return dict(spec, B=B, img=img, dirs=dirs)
    if c == 3:
        nu, nv = (2500, 4000) if scale >= 1.0 else (max(4, int(2500 * scale ** 0.5)), max(4, int(4000 * scale ** 0.5)))
        cx = torus_mesh(nu, nv, seed)
        return dict(spec, complex=cx, dirs=directions_sphere(spec["D"], 3, S0 + 40))
    if c == 4:
        nv = max(64, int(1_000_000 * scale))
        ns = max(16, int(2_000_000 * scale))
        cx = random_simplicial(nv, ns, 5, 4, seed, float_weights=True)
        return dict(spec, complex=cx, dirs=directions_sphere(spec["D"], 5, S0 + 50))
    raise ValueError(c)
