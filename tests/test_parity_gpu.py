"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle (O2, and O1 where
cheap), element by element on the same seeded inputs.

Integer weights: bit-exact (reading A1: bins equal the binary64 evaluation of alpha).
Float weights: |gpu - oracle| <= 1e-5 * A, A = cumsum of |w| over the same bins (A8).
"""
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


def cells_of(cx, device=DEV):
    out = []
    for c in cx.cells:
        v = torch.from_numpy(np.ascontiguousarray(c.verts, np.int32)).to(device)
        wt = None if c.weights is None else torch.from_numpy(np.ascontiguousarray(c.weights)).to(device)
        out.append((v, wt, c.dim))
    return out


def gpu_wect_complex(cx, dirs, T, **kw):
    vw = None if cx.vweights is None else torch.from_numpy(np.ascontiguousarray(cx.vweights)).to(DEV)
    out = w.wect_complex(torch.from_numpy(cx.coords).to(DEV), cells_of(cx), torch.from_numpy(dirs).to(DEV), T,
                         vweights=vw, is_float=cx.is_float, **kw)
    w.sync_status()
    return out.cpu().numpy()


def abs_cumsum(cx, dirs, T):
    """A[p, q] = sum of |w| over cells with bin <= q (reading A8's tolerance scale)."""
    ab = synth.Complex(cx.coords, None if cx.vweights is None else np.abs(cx.vweights),
                       [synth.Cells(c.verts, None if c.weights is None else np.abs(c.weights), 0) for c in cx.cells],
                       cx.k0, cx.is_float)
    return oracle.wect_complex(ab, dirs, T)


def assert_float_close(g, o, A):
    err = np.abs(g - o)
    assert (err <= 1e-5 * A + 1e-12).all(), float((err / (A + 1e-30)).max())


# ------------------------------------------------------------------ images
def test_cfg1_bit_exact_vs_O2_and_O1():
    c = synth.make_config(0)
    img, dirs = c["img"], c["dirs"]
    o2 = oracle.wect_images(img, dirs, c["T"])
    o1 = oracle.wect_images(img, dirs, c["T"], naive=True)
    g = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), c["T"]).cpu().numpy()
    assert g.dtype == np.int32
    assert (g == o2).all()
    # O1 may differ only in directions with a binary64 near-tie (reading A1); cfg1 has none
    assert (g == o1).all()


@pytest.mark.parametrize("H,W,B,D,T", [(28, 28, 130, 16, 64), (5, 7, 65, 9, 13), (1, 9, 3, 4, 6), (9, 1, 2, 4, 5),
                                       (32, 32, 64, 37, 2), (17, 23, 70, 33, 130), (2, 2, 1, 8, 257)])
def test_images2d_sweep_vs_O2(H, W, B, D, T):
    g = np.random.default_rng(H * 1000 + W * 10 + B)
    img = g.integers(0, 256, (B, H, W), dtype=np.uint8)
    dirs = synth.directions_s1(D) if D % 2 else g.standard_normal((D, 2)).astype(np.float32)
    o2 = oracle.wect_images(img, dirs, T)
    for dt in ("int32", "int64"):
        out = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, out_dtype=dt)
        assert (out.cpu().numpy() == o2).all()


@pytest.mark.parametrize("H,W,B,D,T", [(40, 50, 3, 40, 64), (33, 33, 2, 5, 7)])
def test_images2d_histogram_path_vs_O2(H, W, B, D, T):
    g = np.random.default_rng(7)
    img = g.integers(0, 256, (B, H, W), dtype=np.uint8)
    dirs = g.standard_normal((D, 2)).astype(np.float32)
    o2 = oracle.wect_images(img, dirs, T)
    out = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, out_dtype="int64")
    assert (out.cpu().numpy() == o2).all()


@pytest.mark.parametrize("dims,B,D,T", [((5, 6, 7), 2, 40, 16), ((9, 8, 10), 1, 33, 64), ((2, 3, 4), 3, 7, 5),
                                        ((1, 1, 6), 1, 3, 4), ((16, 16, 16), 1, 64, 256)])
def test_volumes3d_vs_O2(dims, B, D, T):
    g = np.random.default_rng(sum(dims) + D)
    img = g.integers(0, 256, (B,) + dims, dtype=np.uint8)
    dirs = synth.directions_sphere(D, 3, int(D))
    o2 = oracle.wect_images(img, dirs, T)
    for dt in ("int32", "int64"):
        out = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, out_dtype=dt)
        assert (out.cpu().numpy() == o2).all()


def test_images_direction_slices_match_full():
    g = np.random.default_rng(8)
    for shape, D in (((70, 28, 28), 64), ((1, 7, 8, 9), 40)):
        img = torch.from_numpy(g.integers(0, 256, shape, dtype=np.uint8)).to(DEV)
        nd = len(shape) - 1
        dirs = torch.from_numpy(synth.directions_sphere(D, nd, 3) if nd == 3 else synth.directions_s1(D)).to(DEV)
        full = w.wect_images(img, dirs, 32, out_dtype="int64")
        for a, b in ((0, 5), (5, 37), (37, D)):
            part = w.wect_images(img, dirs, 32, d_begin=a, d_count=b - a, out_dtype="int64")
            assert torch.equal(part, full[:, a:b])


def test_images_host_buffers_equal_device():
    g = np.random.default_rng(9)
    img = g.integers(0, 256, (100, 28, 28), dtype=np.uint8)
    dirs = synth.directions_s1(16)
    dev = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), 64).cpu().numpy()
    host = w.wect_images(img, dirs, 64)  # numpy in -> host staging path inside the library
    assert (host.numpy() == dev).all()


def test_images_unit_and_constant_properties():
    dirs = synth.directions_s1(24)
    T = 50
    ones = torch.ones((3, 11, 13), dtype=torch.uint8, device=DEV)
    out = w.wect_images(ones, torch.from_numpy(dirs).to(DEV), T).cpu().numpy()
    fv = oracle.heights(oracle.grid_coords((11, 13)), dirs)
    M = np.abs(fv).max()
    for p in range(24):
        a = oracle.alpha(fv[:, p].min(), -M, M, T)
        assert out[0, p].tolist() == [1 if q >= a else 0 for q in range(T)]
    c = w.wect_images(ones * 77, torch.from_numpy(dirs).to(DEV), T).cpu().numpy()
    assert (c == 77 * out).all()


def test_images_determinism():
    g = np.random.default_rng(10)
    img = torch.from_numpy(g.integers(0, 256, (300, 28, 28), dtype=np.uint8)).to(DEV)
    dirs = torch.from_numpy(synth.directions_s1(64)).to(DEV)
    a = w.wect_images(img, dirs, 128)
    b = w.wect_images(img, dirs, 128)
    assert torch.equal(a, b)


def test_cfg2_full_batch_sampled_vs_O2():
    """BASELINE configs[1] at full size in the bench launch configuration; 64 sampled images
    computed one by one by the oracle, plus the top-bin law on every image."""
    c = synth.make_config(1)
    img, dirs, T = c["img"], c["dirs"], c["T"]
    out = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T)
    torch.cuda.synchronize()
    g = np.random.default_rng(11)
    idx = np.sort(g.choice(img.shape[0], 64, replace=False))
    idx = np.concatenate([[0, img.shape[0] - 1], idx])
    o2 = oracle.wect_images(img[idx], dirs, T)
    assert (out[torch.from_numpy(idx).to(DEV)].cpu().numpy() == o2).all()
    # top bin = chi(K, w) of each image, identical in every direction
    top = out[:, :, -1]
    assert torch.equal(top, top[:, :1].expand_as(top))


def test_cfg3_volume_sampled_directions_vs_O2():
    """BASELINE configs[2] (256^3, D = 512, T = 256): 6 sampled directions through the oracle
    with the FULL direction set's M (reading A2), all 512 rows checked for the top-bin law."""
    c = synth.make_config(2)
    img, dirs, T = c["img"], c["dirs"], c["T"]
    out = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, out_dtype="int64")
    out = out.cpu().numpy()[0]
    coords = oracle.grid_coords(img.shape[1:])
    fv_all_M = 0.0
    # M over all directions: the corners attain it
    corners = np.array([[x, y, z] for x in (coords[:, 0].min(), coords[:, 0].max())
                        for y in (coords[:, 1].min(), coords[:, 1].max())
                        for z in (coords[:, 2].min(), coords[:, 2].max())], np.float32)
    fv_all_M = np.abs(oracle.heights(corners, dirs)).max()
    rows = [0, 1, 100, 257, 400, 511]
    o2 = oracle.wect_images(img, dirs[rows], T, maxheight_override=fv_all_M)[0]
    assert (out[rows] == o2).all()
    assert (out[:, -1] == out[0, -1]).all()


# ------------------------------------------------------- explicit complexes
@pytest.mark.parametrize("seed", range(10))
def test_complex_int_vs_O2(seed):
    g = np.random.default_rng(300 + seed)
    n = int(g.integers(1, 6))
    cx = synth.random_small_complex(seed, n=n, nverts=int(g.integers(5, 300)), ntop=int(g.integers(1, 200)),
                                    kmax=int(g.integers(1, 5)))
    D = int(g.choice([1, 7, 32, 33, 70]))
    dirs = g.standard_normal((D, n)).astype(np.float32)
    T = int(g.choice([2, 3, 16, 64, 129, 512]))
    o2 = oracle.wect_complex(cx, dirs, T)
    assert (gpu_wect_complex(cx, dirs, T) == o2).all()


def test_complex_unit_weights_and_structured_directions():
    cx = synth.torus_mesh(30, 40, 2)
    unit = synth.Complex(cx.coords, None, [synth.Cells(c.verts, None, c.dim) for c in cx.cells], cx.k0)
    dirs = synth.directions_sphere(50, 3, 4)
    dirs[:3] = np.eye(3, dtype=np.float32)  # axis directions: many equal heights
    g = gpu_wect_complex(unit, dirs, 100)
    assert (g == oracle.wect_complex(unit, dirs, 100)).all()
    assert (g[:, -1] == 0).all()  # torus chi = 0
    g2 = gpu_wect_complex(cx, dirs, 100)
    assert (g2 == oracle.wect_complex(cx, dirs, 100)).all()


@pytest.mark.parametrize("seed", range(4))
def test_complex_float_vs_O2(seed):
    cx = synth.random_simplicial(2000, 3000, 5, 4, 500 + seed, float_weights=True)
    dirs = synth.directions_sphere(40, 5, seed)
    T = 256
    o2 = oracle.wect_complex(cx, dirs, T)
    g = gpu_wect_complex(cx, dirs, T)
    assert_float_close(g, o2, abs_cumsum(cx, dirs, T))


def test_complex_row_slices_and_maxheight():
    cx = synth.random_small_complex(3, n=3, nverts=200, ntop=150, kmax=3)
    dirs = synth.directions_sphere(70, 3, 9)
    dirs[5] *= 2.5
    full = gpu_wect_complex(cx, dirs, 64)
    for a, b in ((0, 1), (3, 40), (40, 70)):
        assert (gpu_wect_complex(cx, dirs, 64, d_begin=a, d_count=b - a) == full[a:b]).all()
    M = w.wect_maxheight(torch.from_numpy(cx.coords).to(DEV), torch.from_numpy(dirs).to(DEV))
    assert M == np.abs(oracle.heights(cx.coords, dirs)).max()
    # caller-supplied M reproduces the computed one
    assert (gpu_wect_complex(cx, dirs, 64, maxheight=M) == full).all()


def test_complex_host_buffers():
    cx = synth.random_small_complex(4, n=2, nverts=100, ntop=80, kmax=2)
    dirs = synth.directions_s1(12)
    cells = [(c.verts, c.weights, c.dim) for c in cx.cells]
    host = w.wect_complex(cx.coords, cells, dirs, 33, vweights=cx.vweights)
    assert (host.numpy() == oracle.wect_complex(cx, dirs, 33)).all()


def test_ecf_vs_O2_and_grids():
    cx = synth.torus_mesh(20, 30, 5)
    g = np.random.default_rng(12)
    f = g.uniform(-1, 1, (cx.k0, 3)).astype(np.float32)
    cells = cells_of(cx)
    vw = torch.from_numpy(cx.vweights).to(DEV)
    for T in (2, 256, 513):
        out = w.ecf_complex(torch.from_numpy(f).to(DEV), cells, T, vweights=vw).cpu().numpy()
        assert (out == oracle.ecf_complex(cx, f, T)).all()
    # explicit [lo, hi] grid (reading A9): one bin per integer intensity
    fi = g.integers(0, 256, (cx.k0, 1)).astype(np.float32)
    out = w.ecf_complex(torch.from_numpy(fi).to(DEV), cells, 256, vweights=vw, lo=0.0, hi=255.0).cpu().numpy()
    assert (out == oracle.ecf_complex(cx, fi, 256, lo=0.0, hi=255.0)).all()


def test_degenerate_inputs():
    # M = 0: every cell in bin 0, every column = chi (reading A6)
    cx = synth.Complex(np.zeros((3, 2), np.float32), np.array([1, 2, 3], np.int32),
                       [synth.Cells(np.array([[0, 1], [1, 2]], np.int32), np.array([5, 7], np.int32), 1)], 3)
    dirs = synth.directions_s1(4)
    g = gpu_wect_complex(cx, dirs, 5)
    assert (g == (1 + 2 + 3 - 12)).all()
    assert (g == oracle.wect_complex(cx, dirs, 5)).all()
    # k0 = 0: zeros
    e = synth.Complex(np.zeros((0, 2), np.float32), np.zeros(0, np.int32), [], 0)
    assert (gpu_wect_complex(e, dirs, 5) == 0).all()
    # a dimension with no cells is skipped
    cx2 = synth.Complex(cx.coords, cx.vweights, cx.cells + [synth.Cells(np.zeros((0, 3), np.int32), np.zeros(0, np.int32), 2)], 3)
    assert (gpu_wect_complex(cx2, dirs, 5) == g).all()


def test_out_of_range_index_reported():
    cx = synth.Complex(np.random.default_rng(0).normal(size=(4, 2)).astype(np.float32), None,
                       [synth.Cells(np.array([[0, 1], [2, 9]], np.int32), None, 1)], 4)
    dirs = synth.directions_s1(3)
    with pytest.raises(w.WectError) as e:
        gpu_wect_complex(cx, dirs, 8, flags=w.VALIDATE)
    assert e.value.status == _lib.ERANGE
    with pytest.raises(w.WectError) as e:
        gpu_wect_complex(cx, dirs, 8)  # kernel-detected, reported by sync_status
    assert e.value.status == _lib.ERANGE
    w.sync_status()  # the word was cleared


def test_repairs_are_counted():
    w.repair_count(reset=True)
    c = synth.make_config(0)
    w.wect_images(torch.from_numpy(c["img"]).to(DEV), torch.from_numpy(c["dirs"]).to(DEV), c["T"])
    cx = synth.torus_mesh(50, 60, 3)
    gpu_wect_complex(cx, synth.directions_sphere(64, 3, 1), 512)
    assert w.repair_count() >= 0


def test_fp32_only_differs_only_at_flagged_edges():
    """WECT_FP32_ONLY skips the binary64 repair; any difference from O2 must then come from
    cells whose binary64 u lies within tau of an integer (the near-edge cases)."""
    cx = synth.torus_mesh(40, 50, 6)
    dirs = synth.directions_sphere(64, 3, 2)
    T = 512
    a = gpu_wect_complex(cx, dirs, T)
    b = gpu_wect_complex(cx, dirs, T, flags=w.FP32_ONLY)
    o2 = oracle.wect_complex(cx, dirs, T)
    assert (a == o2).all()
    diff_rows = np.nonzero((b != o2).any(axis=1))[0]
    fv = oracle.heights(cx.coords, dirs)
    M = np.abs(fv).max()
    u = (T - 1) * (fv + M) / (2 * M)
    near = (np.abs(u - np.round(u)) < 1e-3).any(axis=0)
    assert set(diff_rows.tolist()) <= set(np.nonzero(near)[0].tolist())


def test_cfg4_scaled_mesh_vs_O2():
    c = synth.make_config(3, scale=0.002)  # ~20k vertices torus, D = 1024, T = 512
    cx, dirs, T = c["complex"], c["dirs"], c["T"]
    o2 = oracle.wect_complex(cx, dirs, T)
    assert (gpu_wect_complex(cx, dirs, T) == o2).all()


def test_cfg5_scaled_float_vs_O2():
    c = synth.make_config(4, scale=0.002)
    cx, dirs, T = c["complex"], c["dirs"], c["T"]
    o2 = oracle.wect_complex(cx, dirs, T)
    assert_float_close(gpu_wect_complex(cx, dirs, T), o2, abs_cumsum(cx, dirs, T))


def _full_M(cx, dirs):
    """M over ALL directions (reading A2), via the oracle's heights, chunked over directions."""
    M = 0.0
    for a in range(0, dirs.shape[0], 64):
        M = max(M, float(np.abs(oracle.heights(cx.coords, dirs[a:a + 64])).max()))
    return M


@pytest.mark.slow
def test_cfg4_full_mesh_sampled_directions_vs_O2():
    """BASELINE configs[3] at full size (1e7 V / 3e7 E / 2e7 F, D = 1024, T = 512) in the bench
    launch configuration; 3 sampled rows through the oracle with the full set's M."""
    c = synth.make_config(3)
    cx, dirs, T = c["complex"], c["dirs"], c["T"]
    g = gpu_wect_complex(cx, dirs, T)
    M = _full_M(cx, dirs)
    rows = [0, 517, 1023]
    o2 = oracle.wect_complex(cx, np.ascontiguousarray(dirs[rows]), T, maxheight_override=M)
    assert (g[rows] == o2).all()
    assert (g[:, -1] == g[0, -1]).all()  # top bin = chi(K, w) in every direction


@pytest.mark.slow
def test_cfg5_full_complex_sampled_directions_vs_O2():
    """BASELINE configs[4] at full size (2e6 random 4-simplices with all faces, fp32 weights,
    D = 256, T = 256); 2 sampled rows within the A8 tolerance."""
    c = synth.make_config(4)
    cx, dirs, T = c["complex"], c["dirs"], c["T"]
    g = gpu_wect_complex(cx, dirs, T)
    M = _full_M(cx, dirs)
    rows = [3, 200]
    d = np.ascontiguousarray(dirs[rows])
    o2 = oracle.wect_complex(cx, d, T, maxheight_override=M)
    ab = synth.Complex(cx.coords, np.abs(cx.vweights), [synth.Cells(x.verts, np.abs(x.weights), 0) for x in cx.cells],
                       cx.k0, True)
    A = oracle.wect_complex(ab, d, T, maxheight_override=M)
    assert_float_close(g[rows], o2, A)


def test_images_edge_cases():
    """1x1 images (a single vertex), B not a multiple of 64, T = 2, all-zero images."""
    dirs = synth.directions_s1(5)
    one = np.full((3, 1, 1), 9, np.uint8)
    out = w.wect_images(torch.from_numpy(one).to(DEV), torch.from_numpy(dirs).to(DEV), 4).cpu().numpy()
    assert (out == oracle.wect_images(one, dirs, 4)).all()
    z = np.zeros((65, 6, 6), np.uint8)
    out = w.wect_images(torch.from_numpy(z).to(DEV), torch.from_numpy(dirs).to(DEV), 2).cpu().numpy()
    assert (out == 0).all()
    g = np.random.default_rng(13)
    im = g.integers(0, 256, (129, 6, 6), dtype=np.uint8)
    out = w.wect_images(torch.from_numpy(im).to(DEV), torch.from_numpy(dirs).to(DEV), 2).cpu().numpy()
    assert (out == oracle.wect_images(im, dirs, 2)).all()


def test_small_D_streaming_path_vs_O2():
    """D <= 8 goes through the thread-per-cell streaming kernel (k_cells): exact vs O2 for
    several arities, ambient dimensions and both weight types."""
    for seed in range(6):
        g = np.random.default_rng(700 + seed)
        n = int(g.integers(1, 6))
        isf = bool(seed % 2)
        cx = synth.random_small_complex(seed, n=n, nverts=400, ntop=300, kmax=4, float_weights=isf)
        dirs = g.standard_normal((int(g.integers(1, 9)), n)).astype(np.float32)
        T = int(g.choice([2, 33, 256]))
        o2 = oracle.wect_complex(cx, dirs, T)
        got = gpu_wect_complex(cx, dirs, T)
        if isf:
            assert_float_close(got, o2, abs_cumsum(cx, dirs, T))
        else:
            assert (got == o2).all()


def _misaligned(a: np.ndarray) -> torch.Tensor:
    """Device copy of `a` whose data pointer is 4 bytes past a 16-byte boundary."""
    flat = torch.zeros(a.size + 4, dtype=torch.from_numpy(a[:0]).dtype, device=DEV)
    view = flat[1:1 + a.size].view(a.shape)
    view.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    assert view.data_ptr() % 16 == 4
    return view


def test_stream_kernel_mid_size_vs_O2():
    """The bulk-copy ring kernel (k_stream) over enough 2048-cell units to wrap its stages
    many times per CTA, segment tails not a multiple of 4 ids, ECF and D <= 8 WECT; the
    int64 direct path for huge integer weights; the misaligned-list fallback (k_cells)."""
    cx = synth.torus_mesh(601, 799, 11)  # k0 odd: every segment ends in a ragged tail
    g = np.random.default_rng(41)
    cells = cells_of(cx)
    vw = torch.from_numpy(cx.vweights).to(DEV)
    f = g.uniform(-1, 1, (cx.k0, 2)).astype(np.float32)
    out = w.ecf_complex(torch.from_numpy(f).to(DEV), cells, 512, vweights=vw).cpu().numpy()
    assert (out == oracle.ecf_complex(cx, f, 512)).all()
    dirs = synth.directions_sphere(3, 3, 5)
    o2 = oracle.wect_complex(cx, dirs, 300)
    assert (gpu_wect_complex(cx, dirs, 300) == o2).all()
    # misaligned index lists: same result through the fallback kernel
    mis = [(_misaligned(np.asarray(c.verts, np.int32)), torch.from_numpy(c.weights).to(DEV), c.dim) for c in cx.cells]
    got = w.wect_complex(torch.from_numpy(cx.coords).to(DEV), mis, torch.from_numpy(dirs).to(DEV), 300, vweights=vw)
    assert (got.cpu().numpy() == o2).all()
    # |w| up to 2^30: int32 partials cannot hold a unit, adds go straight to int64
    big = synth.Complex(cx.coords, g.integers(-2**30, 2**30, cx.k0, dtype=np.int32),
                        [synth.Cells(c.verts, g.integers(-2**30, 2**30, len(c.verts), dtype=np.int32), c.dim)
                         for c in cx.cells], cx.k0)
    assert (gpu_wect_complex(big, dirs[:1], 64) == oracle.wect_complex(big, dirs[:1], 64)).all()


def test_stream_kernel_float_arity5_vs_O2():
    cx = synth.random_simplicial(20000, 30000, 4, 4, 77, float_weights=True)  # arities 1..5
    dirs = synth.directions_sphere(5, 4, 3)
    T = 200
    assert_float_close(gpu_wect_complex(cx, dirs, T), oracle.wect_complex(cx, dirs, T), abs_cumsum(cx, dirs, T))


def test_high_arity_cells_take_the_generic_kernel():
    """Arity 8 (7-simplices) at D > 8: the vertex-bin path declines (records hold <= 7
    ids) and k_complex computes it; arity 6-7 stay on the vertex-bin path."""
    for kmax, seed in ((7, 91), (6, 92), (5, 93)):
        cx = synth.random_small_complex(seed, n=3, nverts=60, ntop=12, kmax=kmax)
        dirs = synth.directions_sphere(40, 3, seed)
        assert (gpu_wect_complex(cx, dirs, 97) == oracle.wect_complex(cx, dirs, 97)).all()


def test_ecf_single_filter_integer_weights_vs_O2():
    """ecf_complex with m = 1 and integer weights (the ECF-X shape): arities 2..8, ragged
    segment tails, unit weights, |w| ~ 2^30 (int64 direct adds), a misaligned list, both
    grids."""
    g = np.random.default_rng(4242)
    for seed, (n, kmax) in enumerate([(3, 2), (4, 3), (6, 5), (8, 7)]):
        cx = synth.random_simplicial(3001 + seed, 4003 + seed, n, kmax, 900 + seed, float_weights=False)
        f = g.uniform(-1, 1, (cx.k0, 1)).astype(np.float32)
        for T in (2, 77, 512):
            out = w.ecf_complex(torch.from_numpy(f).to(DEV), cells_of(cx), T,
                                vweights=torch.from_numpy(cx.vweights).to(DEV)).cpu().numpy()
            assert (out == oracle.ecf_complex(cx, f, T)).all(), (seed, T)
    cx = synth.torus_mesh(301, 157, 3)
    f = g.uniform(-1, 1, (cx.k0, 1)).astype(np.float32)
    unit = synth.Complex(cx.coords, None, [synth.Cells(c.verts, None, c.dim) for c in cx.cells], cx.k0)
    out = w.ecf_complex(torch.from_numpy(f).to(DEV), [(torch.from_numpy(c.verts).to(DEV), None, c.dim) for c in cx.cells],
                        512).cpu().numpy()
    assert (out == oracle.ecf_complex(unit, f, 512)).all()
    big = synth.Complex(cx.coords, g.integers(-2**30, 2**30, cx.k0, dtype=np.int32),
                        [synth.Cells(c.verts, g.integers(-2**30, 2**30, len(c.verts), dtype=np.int32), c.dim)
                         for c in cx.cells], cx.k0)
    out = w.ecf_complex(torch.from_numpy(f).to(DEV), cells_of(big), 300,
                        vweights=torch.from_numpy(big.vweights).to(DEV)).cpu().numpy()
    assert (out == oracle.ecf_complex(big, f, 300)).all()
    mis = [(_misaligned(np.asarray(c.verts, np.int32)), torch.from_numpy(c.weights).to(DEV), c.dim) for c in cx.cells]
    out = w.ecf_complex(torch.from_numpy(f).to(DEV), mis, 512, vweights=torch.from_numpy(cx.vweights).to(DEV))
    assert (out.cpu().numpy() == oracle.ecf_complex(cx, f, 512)).all()
    fi = g.integers(0, 256, (cx.k0, 1)).astype(np.float32)
    out = w.ecf_complex(torch.from_numpy(fi).to(DEV), cells_of(cx), 256, vweights=torch.from_numpy(cx.vweights).to(DEV),
                        lo=0.0, hi=255.0).cpu().numpy()
    assert (out == oracle.ecf_complex(cx, fi, 256, lo=0.0, hi=255.0)).all()


@pytest.mark.slow
def test_ecfx_full_size_vs_O2():
    """The ECF-X bench workload at full size (cfg4 mesh, one filter U[-1,1], T = 512, integer
    weights) in the bench launch configuration: the whole row against O2, bit-exact."""
    c = synth.make_config(3)
    cx = c["complex"]
    f = synth.rng(synth.S0 + 60).uniform(-1, 1, (cx.k0, 1)).astype(np.float32)
    out = w.ecf_complex(torch.from_numpy(f).to(DEV), cells_of(cx), 512,
                        vweights=torch.from_numpy(cx.vweights).to(DEV)).cpu().numpy()
    w.sync_status()
    assert (out == oracle.ecf_complex(cx, f, 512)).all()


def test_calls_are_cuda_graph_capturable():
    """Every stream operation of a device-buffer call is capturable (stream-ordered
    allocations, memsets, launches): capture wect_images / ecf_images once, replay, and
    compare with the oracle (launch overhead of small calls goes away: cfg1 0.152 -> 0.130 ms
    median per call on the B200)."""
    c = synth.make_config(0)
    img = torch.from_numpy(c["img"]).to(DEV)
    dirs = torch.from_numpy(c["dirs"]).to(DEV)
    out = torch.empty((1, 32, 64), dtype=torch.int32, device=DEV)
    eout = torch.empty((1, 256), dtype=torch.int32, device=DEV)
    w.wect_images(img, dirs, 64, out=out)
    w.ecf_images(img, 256, lo=0.0, hi=255.0, out=eout)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        w.wect_images(img, dirs, 64, out=out)
        w.ecf_images(img, 256, lo=0.0, hi=255.0, out=eout)
    out.zero_()
    eout.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == oracle.wect_images(c["img"], c["dirs"], 64)).all()
    assert (eout.cpu().numpy() == oracle.ecf_images(c["img"], 256, 0.0, 255.0)).all()


@pytest.mark.parametrize("D", [9, 16, 17, 24])
def test_streaming_path_multi_tile_directions_vs_O2(D):
    """8 < D <= 24 runs the streaming kernel in tiles of 8 directions (grid.y): exact for
    integer weights, A8 for float weights, on a mesh large enough to wrap the ring."""
    g = np.random.default_rng(5000 + D)
    cx = synth.torus_mesh(257, 311, D)
    dirs = synth.directions_sphere(D, 3, 5100 + D)
    assert (gpu_wect_complex(cx, dirs, 200) == oracle.wect_complex(cx, dirs, 200)).all()
    cf = synth.random_small_complex(D, n=4, nverts=500, ntop=400, kmax=3, float_weights=True)
    d4 = g.standard_normal((D, 4)).astype(np.float32)
    assert_float_close(gpu_wect_complex(cf, d4, 77), oracle.wect_complex(cf, d4, 77), abs_cumsum(cf, d4, 77))
