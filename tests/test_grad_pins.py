"""Pins of the weights-gradient oracle (oracle.wecfs_grad) against what
the mathematics fixes, independently of its own code: a hand-evaluated segment
(tests/golden/grad_segment.json), Euler's identity for a linear map (L(w) = <G, WECT(w)> =
sum_s w(s) dL/dw(s), with the forward from the independently pinned O2 arm), and exact
unit finite differences of the forward (integer weights and integer-valued G: exact in
binary64)."""
import numpy as np
import pytest

import oracle
import synth


def test_grad_segment_hand_values(golden):
    g = golden["grad_segment"]
    cx = synth.Complex(None, None, [synth.Cells(np.array(g["edges"], np.int32), None, 1)], 2, is_float=False)
    gv, gc = oracle.ecf_complex_grad(cx, np.array(g["fvals"], np.float32), g["T"], np.array(g["G"]))
    assert gv.tolist() == g["grad_vertices"]
    assert gc[0].tolist() == g["grad_edges"]


def _loss(cx, dirs, T, G):
    return float((oracle.wect_complex(cx, dirs, T).astype(np.float64) * G).sum())


@pytest.mark.parametrize("seed", range(6))
def test_grad_euler_identity_and_finite_differences(seed):
    rng = np.random.default_rng(4000 + seed)
    cx = synth.random_small_complex(seed) if hasattr(synth, "random_small_complex") else synth.torus_mesh(5, 6, seed)
    D, T = int(rng.integers(1, 7)), int(rng.choice([2, 5, 17, 64]))
    dirs = synth.directions_sphere(D, cx.coords.shape[1], 4100 + seed) if cx.coords.shape[1] > 2 else synth.directions_s1(D)
    G = rng.integers(-3, 4, size=(D, T)).astype(np.float64)
    gv, gc = oracle.wect_complex_grad(cx, dirs, T, G)
    # Euler: L(w) = sum_s w(s) g(s)  (exact: small integers)
    L = _loss(cx, dirs, T, G)
    vw = cx.vweights if cx.vweights is not None else np.ones(cx.k0, np.int32)
    lin = float((vw.astype(np.float64) * gv).sum())
    for c, g in zip(cx.cells, gc):
        w = c.weights if c.weights is not None else np.ones(len(c.verts), np.int32)
        lin += float((w.astype(np.float64) * g).sum())
    assert lin == L
    # unit finite differences on a few cells of each dimension and a few vertices
    for ci, c in enumerate(cx.cells):
        for s in rng.choice(len(c.verts), size=min(3, len(c.verts)), replace=False):
            w = (c.weights if c.weights is not None else np.ones(len(c.verts), np.int32)).copy()
            w[s] += 1
            cells = [synth.Cells(x.verts, w if i == ci else x.weights, x.dim) for i, x in enumerate(cx.cells)]
            cx2 = synth.Complex(cx.coords, cx.vweights, cells, cx.k0, is_float=False)
            assert _loss(cx2, dirs, T, G) - L == gc[ci][s]
    for v in rng.choice(cx.k0, size=min(3, cx.k0), replace=False):
        w = vw.copy()
        w[v] += 1
        cx2 = synth.Complex(cx.coords, w, cx.cells, cx.k0, is_float=False)
        assert _loss(cx2, dirs, T, G) - L == gv[v]


def test_alpha_vec_matches_scalar_alpha():
    rng = np.random.default_rng(5)
    t = rng.uniform(-3, 3, 2000)
    t[:50] = np.round(t[:50] * 4) / 4  # values on bin edges
    for T in (2, 9, 64):
        got = oracle.alpha_vec(t, -3.0, 3.0, T)
        assert got.tolist() == [oracle.alpha(x, -3.0, 3.0, T) for x in t]
