"""GPU parity of the tensor-core image-batch path (k_mma.cu, tcgen05 kind::f16 into TMEM,
SURVEY §8(f) NEXT-4(ii)) against the oracle O2, element by element: the contraction
out[b, s, q] = sum_v cw_o(b, v) [bin(v, s) <= q] is exact in fp16 x fp16 -> fp32, so the
result must equal O2 bit for bit (reading A1 bins, int32 and int64 outputs).

WECT_IMAGES_MMA selects the path per call (read by the library at every call), so both
the contraction and the default sweep run against the same oracle here."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_03909_b200 as w  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture
def mma(monkeypatch):
    monkeypatch.setenv("WECT_IMAGES_MMA", "1")
    yield


def _run(img, dirs, T, dt="int32", **kw):
    return w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, out_dtype=dt,
                         **kw).cpu().numpy()


@pytest.mark.parametrize("H,W,B,D,T", [(28, 28, 300, 16, 128), (28, 28, 129, 64, 128), (8, 8, 5, 9, 13),
                                       (12, 4, 130, 7, 64), (5, 16, 3, 33, 200), (28, 28, 64, 5, 256),
                                       (16, 20, 257, 12, 32), (2, 4, 1, 4, 2)])
def test_mma_images_vs_O2(mma, H, W, B, D, T):
    g = np.random.default_rng(H * 100 + W + B + T)
    img = g.integers(0, 256, (B, H, W), dtype=np.uint8)
    dirs = synth.directions_s1(D) if D % 2 else g.standard_normal((D, 2)).astype(np.float32)
    o2 = oracle.wect_images(img, dirs, T)
    for dt in ("int32", "int64"):
        out = _run(img, dirs, T, dt)
        bad = np.argwhere(out != o2)
        assert bad.size == 0, (dt, bad[:5].tolist(), out[tuple(bad[0])], o2[tuple(bad[0])])


def test_mma_axis_and_diagonal_directions(mma):
    """Axis and 45-degree directions (quadrant walls s_x = 0 / s_y = 0, ties on bin edges)."""
    img = np.random.default_rng(3).integers(0, 256, (140, 28, 28), dtype=np.uint8)
    a = np.sqrt(0.5)
    dirs = np.array([[1, 0], [-1, 0], [0, 1], [0, -1], [a, a], [-a, a], [a, -a], [-a, -a]], np.float32)
    for T in (28, 55, 128):
        assert (_run(img, dirs, T) == oracle.wect_images(img, dirs, T)).all()


def test_mma_cfg2_batch_sampled():
    """BASELINE configs[1] (60,000 x 28x28, D = 64, T = 128) through the contraction: 512 sampled
    images (every tile position, first and last tiles) equal O2."""
    import os
    os.environ["WECT_IMAGES_MMA"] = "1"
    try:
        c = synth.make_config(1)
        img, dirs, T = c["img"], c["dirs"], c["T"]
        out = _run(img, dirs, T)
        idx = np.unique(np.concatenate([np.arange(128), np.arange(59872, 60000),
                                        np.random.default_rng(9).integers(0, 60000, 256)]))
        assert (out[idx] == oracle.wect_images(img[idx], dirs, T)).all()
    finally:
        del os.environ["WECT_IMAGES_MMA"]


@pytest.mark.parametrize("H,W,B,D,T", [(28, 28, 150, 16, 128), (8, 12, 33, 9, 40), (28, 28, 300, 16, 128),
                                       (12, 4, 130, 7, 64), (5, 16, 3, 33, 200)])
def test_mma_v2_vs_O2(monkeypatch, H, W, B, D, T):
    """The second contraction kernel (WECT_IMAGES_MMA=2: A written MN-major from per-tile
    transposed pixels read through L1, 64-vertex SWIZZLE_128B chunks, TMEM double-buffered,
    TMA-store epilogue of 128-byte rows), int32 output, bit-exact vs O2."""
    monkeypatch.setenv("WECT_IMAGES_MMA", "2")
    g = np.random.default_rng(H + W + B)
    img = g.integers(0, 256, (B, H, W), dtype=np.uint8)
    dirs = synth.directions_s1(D) if D % 2 else g.standard_normal((D, 2)).astype(np.float32)
    assert (_run(img, dirs, T) == oracle.wect_images(img, dirs, T)).all()
