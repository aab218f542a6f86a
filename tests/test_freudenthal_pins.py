"""Pins of the Freudenthal-image oracle (oracle.freudenthal_complex)
against what SPEC's derived examples and topology fix: cell counts RC,
R(C-1) + C(R-1) + (R-1)(C-1), 2(R-1)(C-1); the 2x2 image has 4 / 5 / 2 cells; the full
grid is contractible (unit-weighted chi = 1 in every direction's top bin); the max-weight
rule; and the WECT of a unit-weight grid is the step [q >= alpha(min h)] (a linear height's
sublevel set of the Freudenthal grid is contractible: the two diagonal-free corners of a
square cannot both lie strictly below the two others since h(0,1) + h(1,0) = h(0,0) + h(1,1))."""
import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("R,C", [(1, 1), (2, 2), (3, 5), (6, 4), (1, 7)])
def test_counts_and_chi(R, C):
    cx = oracle.freudenthal_complex(np.ones((R, C), np.uint8))
    ne, nt = len(cx.cells[0].verts), len(cx.cells[1].verts)
    assert (cx.k0, ne, nt) == (R * C, R * (C - 1) + C * (R - 1) + (R - 1) * (C - 1), 2 * (R - 1) * (C - 1))
    assert cx.k0 - ne + nt == 1


def test_two_by_two_hand_example():
    img = np.array([[10, 20], [30, 40]], np.uint8)
    cx = oracle.freudenthal_complex(img)
    e = {tuple(v): int(w) for v, w in zip(cx.cells[0].verts.tolist(), cx.cells[0].weights)}
    t = {tuple(v): int(w) for v, w in zip(cx.cells[1].verts.tolist(), cx.cells[1].weights)}
    assert e == {(0, 1): 20, (2, 3): 40, (0, 2): 30, (1, 3): 40, (0, 3): 40}
    assert t == {(0, 1, 3): 40, (0, 2, 3): 40}
    # total weighted chi = 10+20+30+40 - (20+40+30+40+40) + (40+40) = 10
    dirs = synth.directions_s1(8)
    out = oracle.wect_images_freudenthal(img[None], dirs, 16)
    assert (out[0, :, -1] == 10).all()


def test_unit_grid_step_function():
    dirs = synth.directions_s1(12)
    H, W, T = 5, 7, 40
    out = oracle.wect_images_freudenthal(np.ones((1, H, W), np.uint8), dirs, T)[0]
    fv = oracle.heights(oracle.grid_coords((H, W)), dirs)
    M = np.abs(fv).max()
    for p in range(len(dirs)):
        a = oracle.alpha(fv[:, p].min(), -M, M, T)
        assert out[p].tolist() == [1 if q >= a else 0 for q in range(T)]


def test_o0_exact_agrees_and_linearity():
    from oracle import exact

    g = np.random.default_rng(9)
    img = g.integers(0, 256, (2, 3, 4), dtype=np.uint8)
    dirs = g.standard_normal((5, 2)).astype(np.float32)  # generic: no binary64 near-ties (A1)
    o2 = oracle.wect_images_freudenthal(img, dirs, 9)
    for b in range(2):
        o0 = exact.wect_exact(oracle.freudenthal_complex(img[b]), dirs, 9)
        assert o2[b].tolist() == [[int(x) for x in r] for r in o0]
    c = oracle.wect_images_freudenthal(np.full((1, 3, 4), 3, np.uint8), dirs, 9)
    u = oracle.wect_images_freudenthal(np.ones((1, 3, 4), np.uint8), dirs, 9)
    assert (c == 3 * u).all()
