"""GPU parity of ecf_images against the oracle (O2 per image on the
explicit unit-weight cubical complex), element by element, bit-exact (integer result,
bins from binary64 alpha on both sides, reading A1)."""
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


def gpu(img, T, **kw):
    out = w.ecf_images(torch.from_numpy(np.ascontiguousarray(img)).to(DEV), T, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy()


GRIDS = [dict(), dict(lo=0.0, hi=255.0), dict(maxheight=300.0), dict(lo=-10.5, hi=99.25)]


def _orc(img, T, g):
    return oracle.ecf_images(img, T, g.get("lo", 0.0), g.get("hi", 0.0), g.get("maxheight", 0.0))


@pytest.mark.parametrize("dims,B,T", [((28, 28), 70, 256), ((5, 7), 33, 13), ((1, 9), 5, 6), ((9, 1), 4, 5),
                                      ((1, 1), 3, 2), ((64, 64), 9, 100), ((70, 80), 3, 256), ((3, 300), 2, 64),
                                      ((5, 8), 40, 256), ((4, 12), 37, 31), ((7, 12), 6, 256), ((1, 16), 9, 20),
                                      ((16, 4), 9, 20)])
@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_ecf_images_2d_vs_O2(dims, B, T, gi):
    img = synth.images_u8(B, dims, 500 + dims[0] * 7 + dims[1] + gi)
    g = GRIDS[gi]
    assert (gpu(img, T, **g) == _orc(img, T, g)).all()


@pytest.mark.parametrize("dims,B,T", [((5, 6, 7), 6, 64), ((2, 3, 4), 9, 7), ((17, 18, 19), 2, 256), ((1, 1, 40), 3, 9)])
@pytest.mark.parametrize("gi", [0, 1])
def test_ecf_images_3d_vs_O2(dims, B, T, gi):
    img = synth.images_u8(B, dims, 700 + sum(dims) + gi)
    g = GRIDS[gi]
    assert (gpu(img, T, **g) == _orc(img, T, g)).all()


def test_ecf_images_fmnist_like_zero_background():
    img = synth.images_u8(120, (28, 28), 801, "fmnist")
    for g in (dict(), dict(lo=0.0, hi=255.0)):
        assert (gpu(img, 256, **g) == _orc(img, 256, g)).all()


def test_ecf_images_int64_host_buffers_and_unaligned():
    img = synth.images_u8(40, (28, 28), 802)
    ref = oracle.ecf_images(img, 256, 0.0, 255.0)
    host = w.ecf_images(img, 256, lo=0.0, hi=255.0, out_dtype="int64").numpy()
    assert (host == ref).all()
    # an input that starts 1 byte past a 16-byte boundary takes the byte-load path
    raw = torch.zeros(40 * 784 + 1, dtype=torch.uint8, device=DEV)
    raw[1:] = torch.from_numpy(img.reshape(-1)).to(DEV)
    un = raw[1:].view(40, 28, 28)
    assert (w.ecf_images(un, 256, lo=0.0, hi=255.0).cpu().numpy() == ref).all()


def test_ecf_images_degenerate_and_errors():
    zero = torch.zeros((5, 6, 6), dtype=torch.uint8, device=DEV)
    assert (w.ecf_images(zero, 8).cpu().numpy() == 1).all()  # M = 0: every cell in bin 0 (A6)
    empty = torch.zeros((0, 28, 28), dtype=torch.uint8, device=DEV)
    assert w.ecf_images(empty, 8).shape == (0, 8)
    with pytest.raises(_lib.WectError):
        w.ecf_images(zero, 1)
    top = w.ecf_images(torch.from_numpy(synth.images_u8(50, (13, 17), 803)).to(DEV), 40).cpu().numpy()
    assert (top[:, -1] == 1).all()  # chi of the full grid


def test_ecf_images_full_batch_sampled_vs_O2():
    """The bench workload (60,000 FMNIST-shaped 28x28 images, T = 256, grid [0, 255]) in the
    bench launch configuration; 64 sampled images through the oracle, top bin on all."""
    img = synth.images_u8(60000, (28, 28), synth.S0 + 60)
    out = w.ecf_images(torch.from_numpy(img).to(DEV), 256, lo=0.0, hi=255.0)
    torch.cuda.synchronize()
    idx = np.sort(np.random.default_rng(12).choice(60000, 64, replace=False))
    idx = np.concatenate([[0, 59999], idx])
    assert (out[torch.from_numpy(idx).to(DEV)].cpu().numpy() == oracle.ecf_images(img[idx], 256, 0.0, 255.0)).all()
    assert (out[:, -1] == 1).all()


def test_ecf_images_large_path_sampled():
    """1000 x 1000 ('padded ImageNet') through the large-image path."""
    img = synth.images_u8(2, (1000, 1000), synth.S0 + 61)
    out = gpu(img, 256, lo=0.0, hi=255.0)
    ref = oracle.ecf_images(img, 256, 0.0, 255.0)
    assert (out == ref).all()


def test_ecf_images_errors_and_row_args():
    zero = torch.zeros((2, 4, 4), dtype=torch.uint8, device=DEV)
    from paper_2511_03909_b200 import _lib as L
    import ctypes

    g = L.wect_grid(8, 1, 0, 0.0, 0.0, 0.0, 0)  # d_begin != 0: one filter per image
    out = torch.empty((2, 8), dtype=torch.int32, device=DEV)
    dims = (ctypes.c_int64 * 2)(4, 4)
    st = L.load().ecf_images(zero.data_ptr(), 2, 2, dims, ctypes.byref(g), out.data_ptr(), L.I32, None)
    assert st == L.EINVAL
    g = L.wect_grid(70000, 0, 0, 0.0, 0.0, 0.0, 0)  # T > 65536
    st = L.load().ecf_images(zero.data_ptr(), 2, 2, dims, ctypes.byref(g), out.data_ptr(), L.I32, None)
    assert st == L.ENOTSUP
    g = L.wect_grid(8, 0, 0, 0.0, 0.0, 0.0, 0)
    st = L.load().ecf_images(zero.data_ptr(), 2, 4, dims, ctypes.byref(g), out.data_ptr(), L.I32, None)  # ndim 4
    assert st == L.EINVAL


@pytest.mark.parametrize("dims,B", [((100, 4), 3), ((65, 132), 2), ((16, 400), 2), ((17, 300), 3)])
def test_ecf_images_large_row_block_path(dims, B):
    """Large 2-D images with W % 4 == 0 take the row-block kernel (16 rows + halo per CTA):
    row counts not a multiple of 16, W = 4, both grids; a 1-byte-misaligned input takes the
    generic large-image kernel."""
    img = synth.images_u8(B, dims, 1200 + dims[0] + dims[1])
    for g in (dict(), dict(lo=0.0, hi=255.0)):
        assert (gpu(img, 256, **g) == _orc(img, 256, g)).all()
    raw = torch.zeros(img.size + 1, dtype=torch.uint8, device=DEV)
    raw[1:] = torch.from_numpy(img.reshape(-1)).to(DEV)
    out = w.ecf_images(raw[1:].view(img.shape), 64).cpu().numpy()
    assert (out == _orc(img, 64, dict())).all()
