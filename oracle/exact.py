"""O0: exact-rational WECT/WECF oracle -- TEST INFRASTRUCTURE ONLY, tiny inputs.

Every fp32 input is converted exactly to a Fraction; nothing is rounded.
Follows the definitions literally:
  h_s(v) = l(v) . s
  M = max_{p, v} |f_p(v)|
  beta(q) = q * 2M / (T-1) - M
  F(t) = {sigma : max_{v in sigma} f(v) <= t}        (lower star)
  chi(F(t), w) = sum_{sigma in F(t)} (-1)^dim w
  WECT[p, q] = chi(F_p(beta(q)), w)
Degenerate M = 0: every cell is in F(beta(q)) for all q (reading A6).
"""
from __future__ import annotations

from fractions import Fraction
from typing import List, Optional, Sequence, Tuple

Cell = Tuple[Tuple[int, ...], object, int]  # (vertex ids, weight, dim)


def frac(x) -> Fraction:
    return Fraction(float(x))


def exact_heights(coords, dirs) -> List[List[Fraction]]:
    """[k0][D] exact heights."""
    return [[sum((frac(x) * frac(s) for x, s in zip(v, d)), Fraction(0)) for d in dirs] for v in coords]


def wecfs_exact(fvals: Sequence[Sequence[Fraction]], cells: List[Cell], T: int,
                lo: Optional[Fraction] = None, hi: Optional[Fraction] = None) -> List[List[Fraction]]:
    """fvals [k0][m] exact; cells include the vertices themselves as ((a,), w, 0)."""
    m = len(fvals[0]) if fvals else 0
    if lo is None or hi is None:
        M = max((abs(f) for row in fvals for f in row), default=Fraction(0))
        lo, hi = -M, M
    out = []
    for p in range(m):
        row = []
        for q in range(T):
            t = lo + Fraction(q) * (hi - lo) / (T - 1)
            s = Fraction(0)
            for verts, w, dim in cells:
                fmax = max(fvals[v][p] for v in verts)
                if hi == lo or fmax <= t:
                    s += (-1) ** dim * Fraction(w)
            row.append(s)
        out.append(row)
    return out


def alpha_exact(t: Fraction, lo: Fraction, hi: Fraction, T: int) -> int:
    """ceil((T-1)(t - lo)/(hi - lo)) clamped (eq. left-adjoint), exactly."""
    if hi == lo:
        return 0
    u = Fraction(T - 1) * (t - lo) / (hi - lo)
    c = -((-u.numerator) // u.denominator)
    return max(0, min(T - 1, c))


def complex_cells(cx) -> List[Cell]:
    """synth.Complex -> flat cell list (vertices first, then each dimension)."""
    cells: List[Cell] = []
    for a in range(cx.k0):
        w = 1 if cx.vweights is None else cx.vweights[a]
        cells.append(((a,), float(w) if cx.is_float else int(w), 0))
    for c in cx.cells:
        for b in range(c.verts.shape[0]):
            w = 1 if c.weights is None else c.weights[b]
            cells.append((tuple(int(x) for x in c.verts[b]), float(w) if cx.is_float else int(w), c.dim))
    return cells


def wect_exact(cx, dirs, T: int) -> List[List[Fraction]]:
    return wecfs_exact(exact_heights(cx.coords, dirs), complex_cells(cx), T)
