"""GPU parity of wect_images(..., freudenthal=True) against the
oracle (O2 on the explicit weighted Freudenthal complex of each image), bit-exact."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_03909_b200 as w  # noqa: E402
from paper_2511_03909_b200 import _lib  # noqa: E402

DEV = torch.device("cuda:0")


def gpu(img, dirs, T, **kw):
    out = w.wect_images(torch.from_numpy(np.ascontiguousarray(img)).to(DEV), torch.from_numpy(dirs).to(DEV), T,
                        freudenthal=True, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("H,W,B,D,T", [(28, 28, 40, 64, 128), (5, 7, 9, 9, 13), (1, 9, 3, 4, 6), (9, 1, 2, 5, 5),
                                       (1, 1, 2, 3, 2), (40, 50, 2, 40, 64), (33, 2, 3, 70, 300)])
def test_freudenthal_vs_O2(H, W, B, D, T):
    img = synth.images_u8(B, (H, W), 900 + H * 3 + W)
    dirs = synth.directions_s1(D)
    assert (gpu(img, dirs, T) == oracle.wect_images_freudenthal(img, dirs, T)).all()


def test_freudenthal_generic_directions_maxheight_int64_slices():
    g = np.random.default_rng(31)
    img = synth.images_u8(6, (17, 23), 931, "fmnist")
    dirs = g.standard_normal((50, 2)).astype(np.float32)
    ref = oracle.wect_images_freudenthal(img, dirs, 77)
    assert (gpu(img, dirs, 77, out_dtype="int64") == ref).all()
    assert (gpu(img, dirs, 77, d_begin=10, d_count=25) == ref[:, 10:35]).all()  # M over ALL rows (A2)
    ref2 = oracle.wect_images_freudenthal(img, dirs, 77, maxheight_override=5.0)
    assert (gpu(img, dirs, 77, maxheight=5.0) == ref2).all()
    host = w.wect_images(img, dirs, 77, freudenthal=True).numpy()  # host buffers
    assert (host == ref).all()


def test_freudenthal_properties_and_errors():
    dirs = synth.directions_s1(24)
    ones = np.ones((2, 11, 13), np.uint8)
    out = gpu(ones, dirs, 50)
    fv = oracle.heights(oracle.grid_coords((11, 13)), dirs)
    M = np.abs(fv).max()
    for p in range(24):  # contractible sublevel sets: the unit-grid step (test_freudenthal_pins)
        a = oracle.alpha(fv[:, p].min(), -M, M, 50)
        assert out[0, p].tolist() == [1 if q >= a else 0 for q in range(50)]
    assert (gpu(ones * 9, dirs, 50) == 9 * out).all()
    with pytest.raises(_lib.WectError):  # volumes have no Freudenthal option
        w.wect_images(torch.zeros((1, 3, 3, 3), dtype=torch.uint8, device=DEV),
                      torch.from_numpy(synth.directions_sphere(4, 3, 1)).to(DEV), 8, freudenthal=True)


def test_freudenthal_mnist_batch_sampled():
    c = synth.make_config(1, scale=0.2)  # 12,000 images of the cfg2 shape
    img, dirs, T = c["img"], c["dirs"], c["T"]
    out = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, freudenthal=True)
    torch.cuda.synchronize()
    idx = np.sort(np.random.default_rng(13).choice(img.shape[0], 24, replace=False))
    ref = oracle.wect_images_freudenthal(img[idx], dirs, T)
    assert (out[torch.from_numpy(idx).to(DEV)].cpu().numpy() == ref).all()


def test_freudenthal_sweep_near_antidiagonal_directions():
    """Directions with s_x + s_y ~ 0 (the chamber wall of the diagonal): the sweep's chamber
    regrouping needs its exact correction list there (rounded diagonal comparisons); the
    histogram path (WECT_FREUD_HIST-free shapes > 1023 pixels) needs none."""
    base = np.array([[-0.70710677, 0.70710677], [0.70710677, -0.70710677]], np.float32)
    eps = [0.0, 1e-7, -1e-7, 3e-6, -3e-6, 1e-4]
    dirs = np.concatenate([base + np.array([0.0, e], np.float32) for e in eps] + [synth.directions_s1(16)])
    dirs = dirs.astype(np.float32)
    for H, W, T in [(28, 28, 128), (13, 17, 255), (31, 33, 64)]:
        img = synth.images_u8(20, (H, W), 950 + H)
        assert (gpu(img, dirs, T) == oracle.wect_images_freudenthal(img, dirs, T)).all(), (H, W, T)


def test_freudenthal_sweep_correction_list_is_exercised():
    """A direction found by search (CPU, oracle binary64 bins) for which two diagonal pairs of
    a 20x24 grid at T = 1000 have their rounded height order opposite to the chamber of
    s_x + s_y, with a bin edge in between: the sweep must apply its correction list."""
    dirs = np.array([[0.8697633743286133, -0.8697633147239685], [0.6, 0.8], [-0.8, 0.6]], np.float32)
    fv = oracle.heights(oracle.grid_coords((20, 24)), dirs[:1])[:, 0]
    M = np.abs(oracle.heights(oracle.grid_coords((20, 24)), dirs)).max()
    vb = oracle.alpha_vec(fv, -M, M, 1000).reshape(20, 24)
    assert (vb[1:, 1:] < vb[:-1, :-1]).any()  # the designated (upper-right) vertex has the lower bin
    img = synth.images_u8(30, (20, 24), 977)
    img[:, :, :] = np.maximum(img, 1)  # every simplex weight non-zero
    assert (gpu(img, dirs, 1000) == oracle.wect_images_freudenthal(img, dirs, 1000)).all()
