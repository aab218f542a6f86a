"""Pins of the CPU oracle (O0/O1/O2) against what the paper and mathematics fix.

None of these compare the oracle with itself: each checks a value printed in the
paper, a hand evaluation of a formula, a closed form (Euler characteristics,
step functions), an invariant (top bin = chi, Galois law, linearity,
refinement) or brute force in exact rational arithmetic (O0).
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from oracle import exact


def _cx(k0, cells, vw=None, coords=None, is_float=False):
    cl = []
    for dim, verts, w in cells:
        v = np.asarray(verts, np.int32).reshape(-1, len(verts[0]) if len(verts) else dim + 1)
        cl.append(synth.Cells(v, None if w is None else np.asarray(w, np.float32 if is_float else np.int32), dim))
    return synth.Complex(None if coords is None else np.asarray(coords, np.float32),
                         None if vw is None else np.asarray(vw, np.float32 if is_float else np.int32),
                         cl, k0, is_float)


def _chi(cx):
    tot = 0 if not cx.is_float else 0.0
    tot += cx.k0 if cx.vweights is None else cx.vweights.astype(np.float64 if cx.is_float else np.int64).sum()
    for c in cx.cells:
        s = c.verts.shape[0] if c.weights is None else c.weights.astype(np.float64 if cx.is_float else np.int64).sum()
        tot += (-1) ** c.dim * s
    return tot


# ----------------------------------------------------------------- alpha/beta
def test_alpha_beta_hand_values(golden):
    hv = golden["hand_values"]
    for e in hv["alpha"]:
        assert oracle.alpha(e["t"], -e["M"], e["M"], e["T"]) == e["expected"], e["cite"]
        assert exact.alpha_exact(Fraction(e["t"]), Fraction(-e["M"]), Fraction(e["M"]), e["T"]) == e["expected"]
    for e in hv["beta"]:
        assert oracle.beta(e["q"], -e["M"], e["M"], e["T"]) == e["expected"], e["cite"]


def test_alpha_degenerate_and_clamp():
    # reading A6: M = 0 -> index 0; values outside [-M, M] clamp
    assert oracle.alpha(0.0, 0.0, 0.0, 9) == 0
    assert oracle.alpha(5.0, -1.0, 1.0, 9) == 8
    assert oracle.alpha(-5.0, -1.0, 1.0, 9) == 0


def test_galois_law_binary64():
    """alpha(t) <= q  <=>  t <= beta(q)  (eq. galois) on 2e5 random pairs.
    In binary64 the law can only fail for t within rounding of beta(q); those are counted."""
    g = np.random.default_rng(1)
    bad = 0
    for T in (2, 5, 64, 257):
        M = float(g.uniform(0.1, 10))
        ts = g.uniform(-M, M, 50000)
        qs = g.integers(0, T, 50000)
        for t, q in zip(ts, qs):
            lhs = oracle.alpha(t, -M, M, T) <= q
            b = oracle.beta(int(q), -M, M, T)
            rhs = t <= b
            if lhs != rhs:
                assert abs(t - b) <= 4e-16 * M * T, (t, q, T, M)
                bad += 1
    assert bad <= 2


def test_galois_law_exact():
    g = np.random.default_rng(2)
    for _ in range(3000):
        T = int(g.integers(2, 40))
        M = Fraction(int(g.integers(1, 1000)), int(g.integers(1, 100)))
        q = int(g.integers(0, T))
        beta = Fraction(q) * 2 * M / (T - 1) - M
        # exact beta and its neighbours are the interesting points
        for t in (beta, beta - Fraction(1, 10**9), beta + Fraction(1, 10**9),
                  Fraction(g.uniform(-1, 1)) * M):
            if -M <= t <= M:
                assert (exact.alpha_exact(t, -M, M, T) <= q) == (t <= beta)


# --------------------------------------------------------- appendix A pins
def test_appendix_scatter_add(golden):
    """Appendix A scatter_add(U, V)(S) = [[1,8,5],[2,4,11]], through Alg. 1's
    scatter of VertexWeights: one vertex of weight 5 whose bins under filters 0, 1 are
    U = 1, 2 (f = 0 and 1 with M = 1, T = 3 -> alpha = 1, 2).  Alg. 1 returns cumsum(D);
    the first difference recovers D, and S + D must equal the printed result."""
    a = golden["appendix_a"]["scatter_add"]
    cx = _cx(1, [], vw=[5])
    out = oracle.wecfs(np.array([[0.0, 1.0]]), cx, 3, -1.0, 1.0)
    D = np.diff(np.concatenate([np.zeros((2, 1), np.int64), out], axis=1), axis=1)
    assert D.tolist() == a["D"]
    assert (np.array(a["S"]) + D).tolist() == a["expected"]


def test_appendix_cumsum(golden):
    """cumsum rows of T: a row r = [x, y] of DiffWECFs arises from a vertex of
    weight x at f = -1 (bin 0) and a vertex of weight y at f = +1 (bin 1), T = 2."""
    a = golden["appendix_a"]["cumsum_T"]
    for row, exp in zip(a["input"], a["expected"]):
        cx = _cx(2, [], vw=row)
        out = oracle.wecfs(np.array([[-1.0], [1.0]]), cx, 2, -1.0, 1.0)
        assert out[0].tolist() == exp


def test_appendix_rmax(golden):
    """rmax is how a cell gets its bin: an edge over two vertices whose bins are
    the row [a, b] of T lands in bin max(a, b).  Zero vertex weights, edge weight 1 (sign -1)."""
    a = golden["appendix_a"]["rmax_T_axis1"]
    T = 7
    for row, exp in zip(a["input"], a["expected"]):
        f = np.array([[oracle.beta(row[0], -1.0, 1.0, T)], [oracle.beta(row[1], -1.0, 1.0, T)]])
        f[:, 0] = np.where(np.abs(f[:, 0]) < 1e-12, 0.0, f[:, 0])
        f = np.vstack([f, [[1.0]]])  # a third isolated vertex pins M = 1
        cx = _cx(3, [(1, [[0, 1]], [1])], vw=[0, 0, 0])
        out = oracle.wecfs(f, cx, T, -1.0, 1.0)
        D = np.diff(np.concatenate([[0], out[0]]))
        assert D[exp] == -1 and np.count_nonzero(D) == 1


# ----------------------------------------------------------- hand complexes
def test_segment_hand_trace(golden):
    s = golden["hand_values"]["segment"]
    cx = _cx(2, [(1, s["edges"], None)])
    fv = np.array(s["fvals"])
    for naive in (False, True):
        out = oracle.ecf_complex(cx, fv.astype(np.float32), s["T"], naive=naive)
        assert out.tolist() == s["expected"], s["cite"]
    ex = exact.wecfs_exact([[Fraction(0)], [Fraction(1)]], exact.complex_cells(cx), s["T"])
    assert [[int(x) for x in r] for r in ex] == s["expected"]


def _octahedron():
    coords = [[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]]
    tris = [tuple(sorted((a, b, c))) for a in (0, 1) for b in (2, 3) for c in (4, 5)]
    edges = sorted({tuple(sorted(e)) for t in tris for e in itertools.combinations(t, 2)})
    return coords, edges, tris


@pytest.mark.parametrize("naive", [False, True])
def test_euler_characteristics(naive):
    """Top bin = chi of the whole complex (P:769-776 at q = T-1): octahedron boundary 2,
    triangle boundary 0, path 1, filled triangle 1 (Euler's formula)."""
    g = np.random.default_rng(3)
    dirs = synth.directions_sphere(16, 3, 7)
    coords, edges, tris = _octahedron()
    octa = _cx(6, [(1, edges, None), (2, tris, None)], coords=coords)
    tri_b = _cx(3, [(1, [[0, 1], [1, 2], [0, 2]], None)], coords=g.normal(size=(3, 3)))
    path = _cx(4, [(1, [[0, 1], [1, 2], [2, 3]], None)], coords=g.normal(size=(4, 3)))
    filled = _cx(3, [(1, [[0, 1], [1, 2], [0, 2]], None), (2, [[0, 1, 2]], None)], coords=g.normal(size=(3, 3)))
    for cx, chi in ((octa, 2), (tri_b, 0), (path, 1), (filled, 1)):
        out = oracle.wect_complex(cx, dirs, 9, naive=naive)
        assert (out[:, -1] == chi).all()


def test_single_simplex_step():
    """A k-simplex with all faces and unit weights has chi = 1 and its WECF is the step
    [q >= alpha(min_v f(v))]: the sublevel set is a face (chi 1) or empty."""
    g = np.random.default_rng(4)
    for k in range(1, 6):
        n = 5
        cells = [(d, [list(c) for c in itertools.combinations(range(k + 1), d + 1)], None) for d in range(1, k + 1)]
        cx = _cx(k + 1, cells, coords=g.normal(size=(k + 1, n)))
        dirs = synth.directions_sphere(8, n, k)
        T = 33
        out = oracle.wect_complex(cx, dirs, T)
        fv = oracle.heights(cx.coords, dirs)
        M = np.abs(fv).max()
        for p in range(8):
            a = oracle.alpha(fv[:, p].min(), -M, M, T)
            assert out[p].tolist() == [1 if q >= a else 0 for q in range(T)]


# ------------------------------------------------------------- image grids
def test_grid_coords_hand(golden):
    e = golden["hand_values"]["grid_coords_2x3"]
    assert oracle.grid_coords(e["dims"]).tolist() == e["expected"]


def test_grid_coords_hand_3d(golden):
    """A volume's axis mapping (slice -> axis 2, row -> axis 1, column -> axis 0) against
    hand values: an axis swap or a wrong S fails."""
    e = golden["hand_values"]["grid_coords_2x3x4"]
    got = oracle.grid_coords(e["dims"])[e["vertices"]]
    assert np.array_equal(got, np.array(e["expected"], np.float64).astype(np.float32))


def test_cubical_counts(golden):
    for case in golden["hand_values"]["cubical_counts"]["cases"]:
        img = np.zeros(case["dims"], np.uint8)
        cx = oracle.grid_complex(img)
        got = [cx.k0] + [c.verts.shape[0] for c in cx.cells]
        assert got == case["counts"]


def test_grid_unit_weights_step():
    """Unit-weight full grid: WECT[d, q] = [q >= alpha(min_v h_d(v))], chi = 1
    (each non-minimal vertex's lower star sums to (1-1)^k = 0)."""
    for dims in ((3, 4), (5, 5), (2, 3, 3)):
        n = len(dims)
        dirs = synth.directions_sphere(8, n, 11) if n == 3 else synth.directions_s1(8)
        cx = oracle.grid_complex(np.ones(dims, np.uint8))
        T = 9
        out = oracle.wect_complex(cx, dirs, T)
        fv = oracle.heights(cx.coords, dirs)
        M = np.abs(fv).max()
        for p in range(8):
            a = oracle.alpha(fv[:, p].min(), -M, M, T)
            assert out[p].tolist() == [1 if q >= a else 0 for q in range(T)]
        # the batched image entry point (max rule weights) agrees
        im = oracle.wect_images(np.ones((1,) + dims, np.uint8), dirs, T)[0]
        assert (im == out).all()


def test_constant_and_delta_images():
    dirs = synth.directions_s1(12)
    T = 17
    unit = oracle.wect_images(np.ones((1, 6, 7), np.uint8), dirs, T)[0]
    for c in (0, 3, 255):
        out = oracle.wect_images(np.full((1, 6, 7), c, np.uint8), dirs, T)[0]
        assert (out == c * unit).all()
    # delta image: one interior pixel of weight w: its vertex, 4 edges, 4 squares carry w
    w = 200
    img = np.zeros((1, 5, 5), np.uint8)
    img[0, 2, 2] = w
    out = oracle.wect_images(img, dirs, T)[0]
    assert (out[:, -1] == w * (1 - 4 + 4)).all()
    # hand row: the sublevel set contains the pixel's star cells once all their corners are below t
    coords = oracle.grid_coords((5, 5))
    fv = oracle.heights(coords, dirs)
    M = np.abs(fv).max()
    center = 2 * 5 + 2
    nbrs = {"l": 2 * 5 + 1, "r": 2 * 5 + 3, "u": 1 * 5 + 2, "d": 3 * 5 + 2,
            "ul": 1 * 5 + 1, "ur": 1 * 5 + 3, "dl": 3 * 5 + 1, "dr": 3 * 5 + 3}
    squares = [("ul", "u", "l"), ("ur", "u", "r"), ("dl", "d", "l"), ("dr", "d", "r")]
    for p in range(12):
        for q in range(T):
            t = oracle.beta(q, -M, M, T)
            s = 0
            if fv[center, p] <= t:
                s += w
            for e in ("l", "r", "u", "d"):
                if max(fv[center, p], fv[nbrs[e], p]) <= t:
                    s -= w
            for sq in squares:
                if max(fv[center, p], *[fv[nbrs[k], p] for k in sq]) <= t:
                    s += w
            assert out[p, q] == s


def test_image_batch_max_rule_vs_explicit():
    """wect_images (max-rule cell weights) equals Alg. 1 on the explicitly built complex,
    and the naive arm equals Alg. 1 on random u8 images."""
    g = np.random.default_rng(5)
    imgs = g.integers(0, 256, (3, 4, 5), dtype=np.uint8)
    dirs = synth.directions_s1(10)
    o2 = oracle.wect_images(imgs, dirs, 11)
    o1 = oracle.wect_images(imgs, dirs, 11, naive=True)
    # O1 (beta comparisons) and O2 (alpha) are both binary64 renditions; they may only
    # differ in directions that put a vertex within rounding of a bin edge (reading A1).
    fv = oracle.heights(oracle.grid_coords((4, 5)), dirs)
    edge_rows = _near_edge(fv, np.abs(fv).max(), 11).any(axis=0)
    assert edge_rows.sum() <= 2
    assert (o1[:, ~edge_rows] == o2[:, ~edge_rows]).all()
    for b in range(3):
        cx = oracle.grid_complex(imgs[b])
        # max rule spelled out for every cell
        for c in cx.cells:
            assert (c.weights == imgs[b].reshape(-1)[c.verts].max(axis=1)).all()
        assert (oracle.wect_complex(cx, dirs, 11) == o2[b]).all()


# ---------------------------------------------------- arms against each other
def _near_edge(fv, M, T, tol=1e-9):
    """Pairs whose binary64 u lies within tol of an interior integer (the endpoints 0 and T-1
    are exact in both arms: alpha(+-M) and beta(0), beta(T-1) are forced)."""
    u = (T - 1) * (fv + M) / (2 * M)
    r = np.round(u)
    return (np.abs(u - r) < tol) & (r > 0) & (r < T - 1)


@pytest.mark.parametrize("seed", range(12))
def test_o2_equals_o0_exact(seed):
    """Alg. 1 in binary64 (O2) equals exact rational enumeration (O0) on random small
    complexes with integer weights: bit-exact."""
    g = np.random.default_rng(100 + seed)
    n = int(g.integers(1, 5))
    cx = synth.random_small_complex(seed, n=n, nverts=int(g.integers(3, 14)), ntop=int(g.integers(1, 10)), kmax=3)
    D = int(g.integers(1, 5))
    # generic directions (no exact zero-ish components, so no binary64 near-ties; reading A1)
    dirs = g.standard_normal((D, n)).astype(np.float32)
    T = int(g.choice([2, 3, 7, 16]))
    o2 = oracle.wect_complex(cx, dirs, T)
    o0 = exact.wect_exact(cx, dirs, T)
    assert o2.tolist() == [[int(x) for x in r] for r in o0]


@pytest.mark.parametrize("seed", range(20))
def test_o2_equals_o1_random(seed):
    """S:365-style suite: dim <= 3, k <= 500, D <= 8, T in {2, 7, 64}; O1 == O2 except for
    heights within rounding of a bin edge (counted, expected none)."""
    g = np.random.default_rng(200 + seed)
    is_float = bool(seed % 2)
    cx = synth.random_small_complex(seed, n=3, nverts=60, ntop=40, kmax=3, float_weights=is_float)
    dirs = synth.directions_sphere(8, 3, seed)
    T = [2, 7, 64][seed % 3]
    fv = oracle.heights(cx.coords, dirs)
    M = np.abs(fv).max()
    assert not _near_edge(fv, M, T).any()
    o2 = oracle.wect_complex(cx, dirs, T)
    o1 = oracle.wect_complex(cx, dirs, T, naive=True)
    if is_float:
        np.testing.assert_allclose(o2, o1, rtol=0, atol=1e-9)
    else:
        assert (o1 == o2).all()
    assert np.allclose(o2[:, -1], _chi(cx))


def test_float_weights_vs_exact():
    cx = synth.random_small_complex(7, n=2, nverts=9, ntop=6, kmax=2, float_weights=True)
    dirs = synth.directions_s1(5)
    o2 = oracle.wect_complex(cx, dirs, 7)
    o0 = exact.wect_exact(cx, dirs, 7)
    np.testing.assert_allclose(o2, np.array([[float(x) for x in r] for r in o0]), rtol=0, atol=1e-12)


# ------------------------------------------------------------- invariants
def test_linearity_in_weights():
    g = np.random.default_rng(6)
    cx1 = synth.random_small_complex(9, n=3, nverts=50, ntop=30)
    cx2 = synth.random_small_complex(9, n=3, nverts=50, ntop=30, wlo=-7, whi=90)  # same cells, other weights
    assert all((a.verts == b.verts).all() for a, b in zip(cx1.cells, cx2.cells))
    s = synth.Complex(cx1.coords, cx1.vweights + cx2.vweights,
                      [synth.Cells(a.verts, a.weights + b.weights, a.dim) for a, b in zip(cx1.cells, cx2.cells)],
                      cx1.k0)
    dirs = synth.directions_sphere(6, 3, 3)
    assert (oracle.wect_complex(s, dirs, 32) == oracle.wect_complex(cx1, dirs, 32) + oracle.wect_complex(cx2, dirs, 32)).all()


def test_refinement_exact():
    """Grid nesting: beta_T(q) = beta_{2T-1}(2q), so coarse[p,q] = fine[p,2q] (O0, exact)."""
    cx = synth.random_small_complex(10, n=2, nverts=10, ntop=8, kmax=2)
    dirs = synth.directions_s1(4)
    T = 6
    coarse = exact.wect_exact(cx, dirs, T)
    fine = exact.wect_exact(cx, dirs, 2 * T - 1)
    for p in range(4):
        assert [coarse[p][q] for q in range(T)] == [fine[p][2 * q] for q in range(T)]


def test_bottom_bin_only_at_minus_M():
    """WECT[p, 0] collects only cells all of whose vertices sit exactly at -M (alpha(t) = 0
    iff t = -M for t in [-M, M])."""
    coords = np.array([[1, 0], [-1, 0], [0, 0.5], [0.25, -0.25]], np.float32)
    cx = _cx(4, [(1, [[0, 2], [1, 2], [1, 3]], [10, 20, 30])], vw=[1, 2, 3, 4], coords=coords)
    dirs = np.array([[1, 0], [0, 1], [-1, 0]], np.float32)
    out = oracle.wect_complex(cx, dirs, 5)
    assert out[:, 0].tolist() == [2, 0, 1]


def test_maxheight_over_all_directions():
    """M is taken over ALL filters: computing rows separately with the full-set M
    reproduces the rows of the full result, while each row's own M would not."""
    cx = synth.random_small_complex(11, n=3, nverts=30, ntop=20)
    dirs = synth.directions_sphere(6, 3, 5)
    dirs[2] *= 3.0  # a longer direction sets M
    full = oracle.wect_complex(cx, dirs, 16)
    fv = oracle.heights(cx.coords, dirs)
    M = np.abs(fv).max()
    for p in range(6):
        assert (oracle.wect_complex(cx, dirs, 16, rows=slice(p, p + 1))[0] == full[p]).all()
        assert (oracle.wecfs(fv[:, p:p + 1], cx, 16, -M, M)[0] == full[p]).all()
    own = oracle.wecfs(np.ascontiguousarray(fv[:, 0:1]), cx, 16, -np.abs(fv[:, 0]).max(), np.abs(fv[:, 0]).max())
    assert not (own[0] == full[0]).all()


def test_out_of_range_index_rejected():
    cx = _cx(2, [(1, [[0, 5]], None)], coords=np.zeros((2, 2)))
    with pytest.raises(IndexError):
        oracle.wect_complex(cx, synth.directions_s1(2), 4)


def test_reading_a1_binary64_tie():
    """Reading A1 documented on a real tie: direction 5 of S^1(10) is (-1, 1.2e-16); a vertex
    at x = 0, y > 0 has exact height +tiny > beta(5) = 0 (exact arithmetic puts it in bin 6),
    but binary64 absorbs M + h = M, so alpha evaluated as written gives bin 5.  O2 (and the
    CUDA path, which reproduces O2) follow the binary64 evaluation; O0 differs only there."""
    img = np.full((1, 4, 5), 7, np.uint8)
    dirs = synth.directions_s1(10)
    cx = oracle.grid_complex(img[0])
    o2 = oracle.wect_complex(cx, dirs, 11)
    o0 = np.array([[int(x) for x in r] for r in exact.wect_exact(cx, dirs, 11)])
    fv = oracle.heights(cx.coords, dirs)
    edge_rows = _near_edge(fv, np.abs(fv).max(), 11).any(axis=0)
    assert edge_rows[5]
    assert (o0[~edge_rows] == o2[~edge_rows]).all()


def test_torus_chi_zero():
    cx = synth.torus_mesh(6, 9, 1)
    cx1 = synth.Complex(cx.coords, None, [synth.Cells(c.verts, None, c.dim) for c in cx.cells], cx.k0)
    out = oracle.wect_complex(cx1, synth.directions_sphere(5, 3, 1), 12)
    assert (out[:, -1] == 0).all()
