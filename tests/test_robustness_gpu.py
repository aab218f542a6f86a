"""GPU regressions for the round-1 advisor findings and the round-2 sweep's
store paths: every result is compared element by element with the oracle (O2)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module")
def w():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2511_03909_b200 as w

    return w


def test_histogram_path_more_than_65535_images(w):
    """32x32 images exceed the sweep's shared memory and take k_grid_hist, whose grid carries
    the image index in gridDim.z: a batch of 70,000 must be chunked (api.cu)."""
    g = np.random.default_rng(65536)
    B = 70_000
    img = g.integers(0, 256, (B, 32, 32), dtype=np.uint8)
    dirs = synth.directions_s1(3)
    out = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), 5).cpu().numpy()
    pick = np.array([0, 1, 65534, 65535, 65536, 69_999] + list(g.integers(0, B, 10)))
    assert (out[pick] == oracle.wect_images(img[pick], dirs, 5)).all()


def test_image_ecf_wide_rows_fall_back_to_the_generic_kernel(w):
    """X = 8192: the rows kernel's staged rows would need > 227 KB of shared memory, so the
    generic kernel must take it (k_ecf_images.cu)."""
    g = np.random.default_rng(8192)
    img = g.integers(0, 256, (2, 3, 8192), dtype=np.uint8)
    out = w.ecf_images(torch.from_numpy(img).to(DEV), 256, lo=0.0, hi=255.0).cpu().numpy()
    assert (out == oracle.ecf_images(img, 256, 0.0, 255.0)).all()


@pytest.mark.parametrize("dt,T", [("int32", 128), ("int64", 64), ("int32", 13)])
def test_sweep_output_not_16_byte_aligned(w, dt, T):
    """An out= view at an odd element offset (or T * size not a multiple of 16) cannot take
    the TMA tensor store: the sweep must fall back to its bounded element stores (ADVICE r1:
    16-byte stores to a misaligned out faulted)."""
    g = np.random.default_rng(T)
    img = g.integers(0, 256, (70, 28, 28), dtype=np.uint8)
    dirs = synth.directions_s1(9)
    n = 70 * 9 * T
    buf = torch.zeros(n + 1, dtype=getattr(torch, dt), device=DEV)
    view = buf[1:].view(70, 9, T)
    w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, out_dtype=dt, out=view)
    assert buf[0].item() == 0
    assert (view.cpu().numpy() == oracle.wect_images(img, dirs, T)).all()


def test_sweep_tail_group_and_partial_chunk(w):
    """B not a multiple of the 64-image group and T not a multiple of the 8-bin chunk: the
    TMA box is clipped at both tensor edges."""
    g = np.random.default_rng(99)
    img = g.integers(0, 256, (131, 20, 24), dtype=np.uint8)
    dirs = synth.directions_s1(17)
    for dt, T in (("int32", 12), ("int64", 20), ("int32", 8)):
        out = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, out_dtype=dt)
        assert (out.cpu().numpy() == oracle.wect_images(img, dirs, T)).all()


def test_one_filter_stream_without_vertex_bins_matches(w, monkeypatch):
    """WECT_STREAM_NO_VBIN=1 sends the one-filter ECF through k_stream's per-cell binning
    (the round-1 path): the same result as the k_vbin1 path and O2."""
    cx = synth.torus_mesh(40, 50, 9)
    f = np.random.default_rng(9).uniform(-1, 1, (cx.k0, 1)).astype(np.float32)
    cells = [(torch.from_numpy(c.verts).to(DEV), torch.from_numpy(c.weights).to(DEV), c.dim) for c in cx.cells]
    vw = torch.from_numpy(cx.vweights).to(DEV)
    a = w.ecf_complex(torch.from_numpy(f).to(DEV), cells, 128, vweights=vw).cpu().numpy()
    monkeypatch.setenv("WECT_STREAM_NO_VBIN", "1")
    b = w.ecf_complex(torch.from_numpy(f).to(DEV), cells, 128, vweights=vw).cpu().numpy()
    ref = oracle.ecf_complex(cx, f, 128)
    assert (a == ref).all() and (b == ref).all()


def test_stream_large_weights_take_the_direct_path(w):
    """Integer weights above the in-kernel bound (|w| > 4095) make a warp add its unit straight
    into the int64 table: exact, no max|w| pre-pass."""
    cx = synth.torus_mesh(40, 50, 10)
    g = np.random.default_rng(10)
    for c in cx.cells:
        c.weights[:] = g.integers(-2**30, 2**30, c.weights.shape[0]).astype(np.int32)
    f = g.uniform(-1, 1, (cx.k0, 1)).astype(np.float32)
    cells = [(torch.from_numpy(c.verts).to(DEV), torch.from_numpy(c.weights).to(DEV), c.dim) for c in cx.cells]
    got = w.ecf_complex(torch.from_numpy(f).to(DEV), cells, 64, vweights=torch.from_numpy(cx.vweights).to(DEV))
    assert (got.cpu().numpy() == oracle.ecf_complex(cx, f, 64)).all()
