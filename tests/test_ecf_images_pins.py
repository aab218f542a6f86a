"""Pins of the image-ECF oracle (oracle.ecf_images) against what the
paper and topology fix, independently of the oracle's own code:

* Remark "which-ecf": the ECF of an image is the Euler characteristic of the
  lower-star filtration with the intensities as the vertex filter.  On the grid [0, 255]
  with T = 256 (reading A9) beta(q) = q, so out[q] = chi(sublevel complex {cells with all
  corners <= q}).  For the cubical V-construction of a binary pixel set X (pixels are
  vertices, a cell is present when all its corners are in X), chi = (#4-connected
  components of X) - (#holes), a hole being an 8-connected component of the complement
  that does not touch the image border (digital-topology duality of 4/8 connectivity).
  Counted here with scipy.ndimage.label -- a different algorithm and a different library.
* the top bin is chi(full grid) = 1; a constant image is a single step; an all-zero image
  with its own grid (M = 0) puts every cell in bin 0 (reading A6).
"""
import numpy as np
import pytest
from scipy import ndimage

import oracle

FOUR = np.array([[0, 1, 0], [1, 1, 1], [0, 1, 0]])
EIGHT = np.ones((3, 3), int)


def chi_by_labels(X: np.ndarray) -> int:
    if not X.any():
        return 0
    _, n4 = ndimage.label(X, structure=FOUR)
    lab, n8 = ndimage.label(~X, structure=EIGHT)
    border = set(np.unique(np.concatenate([lab[0], lab[-1], lab[:, 0], lab[:, -1]]))) - {0}
    holes = n8 - len(border)
    return int(n4 - holes)


def test_chi_by_labels_hand_cases():
    ring = np.zeros((5, 5), bool)
    ring[1:4, 1:4] = True
    ring[2, 2] = False
    assert chi_by_labels(ring) == 0  # an annulus
    diamond = np.zeros((3, 3), bool)
    diamond[0, 1] = diamond[1, 0] = diamond[1, 2] = diamond[2, 1] = True
    assert chi_by_labels(diamond) == 4  # diagonal neighbours are not joined in the V-construction
    assert chi_by_labels(np.ones((4, 6), bool)) == 1


@pytest.mark.parametrize("seed", range(8))
def test_ecf_images_equals_sublevel_euler_characteristic(seed):
    rng = np.random.default_rng(1000 + seed)
    H, W = [(6, 7), (9, 5), (1, 8), (8, 1), (12, 12), (3, 3), (10, 4), (7, 11)][seed]
    # few distinct levels so the sublevel sets have components and holes
    img = rng.choice(np.array([0, 3, 17, 64, 128, 200, 255], np.uint8), size=(2, H, W))
    got = oracle.ecf_images(img, 256, 0.0, 255.0)
    for b in range(2):
        want = [chi_by_labels(img[b] <= q) for q in range(256)]
        assert got[b].tolist() == want


def test_ecf_images_o1_agrees_on_random_u8():
    rng = np.random.default_rng(7)
    img = rng.integers(0, 256, size=(3, 6, 5), dtype=np.uint8)
    for lo, hi, mh in ((0.0, 0.0, 0.0), (0.0, 255.0, 0.0), (0.0, 0.0, 300.0)):
        a = oracle.ecf_images(img, 33, lo, hi, mh)
        b = oracle.ecf_images(img, 33, lo, hi, mh, naive=True)
        assert np.array_equal(a, b)


def test_ecf_images_top_bin_constant_and_zero():
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, size=(4, 7, 9), dtype=np.uint8)
    assert (oracle.ecf_images(img, 64)[:, -1] == 1).all()
    const = np.full((1, 5, 6), 77, np.uint8)
    # own grid [-77, 77]: every cell has value M -> top bin only
    assert oracle.ecf_images(const, 16)[0].tolist() == [0] * 15 + [1]
    # [0, 255], T = 256: step at q = 77
    assert oracle.ecf_images(const, 256, 0.0, 255.0)[0].tolist() == [0] * 77 + [1] * 179
    zero = np.zeros((1, 4, 4), np.uint8)
    assert oracle.ecf_images(zero, 8)[0].tolist() == [1] * 8  # M = 0: bin 0 (reading A6)


def test_ecf_volume_sublevel_chi_of_solid_blocks():
    # 3-D: the sublevel set of a volume holding one solid box of value 0 in a 255 background
    # is a solid box (chi = 1) for 0 <= q < 255, and the full grid (chi = 1) at q = 255
    vol = np.full((1, 5, 6, 4), 255, np.uint8)
    vol[0, 1:4, 2:5, 1:3] = 0
    got = oracle.ecf_images(vol, 256, 0.0, 255.0)[0]
    assert got.tolist() == [1] * 256
    # two separated boxes -> chi = 2 below 255
    vol[0, 1:4, 0, 0] = 0
    vol[0, 1:4, 1, :] = 255
    got = oracle.ecf_images(vol, 256, 0.0, 255.0)[0]
    assert got[:255].tolist() == [2] * 255 and got[255] == 1
