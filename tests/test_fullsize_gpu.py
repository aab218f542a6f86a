"""Round-2 parity additions (VERDICT r1 "Next round" item 1):

* full-size, ALL-rows parity of the fp32 fast paths against the oracle (O2, chunked over
  directions with the full set's M, reading A2): cfg3 (k_grid_hist, 512 rows), cfg4
  (k_vbins + k_cells_vb, 1024 rows), cfg5 (float weights, 256 rows, tolerance A8), and 256
  sampled images of the 60k Freudenthal batch (chamber sweep);
* a tie-heavy suite: lattice coordinates, axis-aligned and 45-degree directions, and
  T - 1 a multiple of the lattice spacing, so vertex heights fall exactly on (or within
  rounding of) bin edges.  Every fast path (k_grid_hist, k_vbins/k_cells_vb, k_stream,
  k_grad_cells) must take its binary64 repair there (wect_repair_count() > 0) and stay
  bit-exact with O2 (reading A1)."""
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


def _cells(cx):
    return [(torch.from_numpy(np.ascontiguousarray(c.verts, np.int32)).to(DEV),
             None if c.weights is None else torch.from_numpy(np.ascontiguousarray(c.weights)).to(DEV), c.dim)
            for c in cx.cells]


def _gpu_complex(cx, dirs, T, **kw):
    vw = None if cx.vweights is None else torch.from_numpy(np.ascontiguousarray(cx.vweights)).to(DEV)
    out = w.wect_complex(torch.from_numpy(cx.coords).to(DEV), _cells(cx), torch.from_numpy(dirs).to(DEV), T,
                         vweights=vw, is_float=cx.is_float, **kw)
    w.sync_status()
    return out.cpu().numpy()


def _full_M(coords, dirs):
    M = 0.0
    for a in range(0, dirs.shape[0], 64):
        M = max(M, float(np.abs(oracle.heights(coords, dirs[a:a + 64])).max()))
    return M


def _oracle_rows(fn, dirs, chunk=64):
    """Oracle over all rows, chunked over directions (each chunk with the full set's M)."""
    return np.concatenate([fn(np.ascontiguousarray(dirs[a:a + chunk])) for a in range(0, dirs.shape[0], chunk)])


# ------------------------------------------------------------ full size, all rows
@pytest.mark.slow
def test_cfg3_volume_all_rows_vs_O2():
    """BASELINE configs[2]: 256^3 u8 volume, D = 512 on S^2, T = 256 -> every one of the
    512 x 256 int64 outputs equals O2 (k_grid_cw + k_grid_hist)."""
    c = synth.make_config(2)
    img, dirs, T = c["img"], c["dirs"], c["T"]
    g = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T,
                      out_dtype="int64").cpu().numpy()[0]
    coords = oracle.grid_coords(img.shape[1:])
    corners = np.array([[x, y, z] for x in (coords[:, 0].min(), coords[:, 0].max())
                        for y in (coords[:, 1].min(), coords[:, 1].max())
                        for z in (coords[:, 2].min(), coords[:, 2].max())], np.float32)
    M = float(np.abs(oracle.heights(corners, dirs)).max())
    o2 = _oracle_rows(lambda d: oracle.wect_images(img, d, T, maxheight_override=M)[0], dirs)
    assert g.shape == o2.shape == (512, T)
    assert (g == o2).all()


@pytest.mark.slow
def test_cfg4_mesh_all_rows_vs_O2():
    """BASELINE configs[3]: the 1e7-vertex torus mesh, D = 1024, T = 512: all 1024 rows
    (k_vbins + k_cells_vb, 16 tiles of 64 directions) equal O2, computed 64 rows at a time."""
    c = synth.make_config(3)
    cx, dirs, T = c["complex"], c["dirs"], c["T"]
    g = _gpu_complex(cx, dirs, T)
    M = _full_M(cx.coords, dirs)
    o2 = _oracle_rows(lambda d: oracle.wect_complex(cx, d, T, maxheight_override=M), dirs)
    assert (g == o2).all()


@pytest.mark.slow
def test_cfg5_complex_all_rows_within_A8():
    """BASELINE configs[4]: 2e6 random 4-simplices with all faces in R^5, fp32 weights,
    D = 256, T = 256: all rows within |g - o| <= 1e-5 A (reading A8)."""
    c = synth.make_config(4)
    cx, dirs, T = c["complex"], c["dirs"], c["T"]
    g = _gpu_complex(cx, dirs, T)
    M = _full_M(cx.coords, dirs)
    o2 = _oracle_rows(lambda d: oracle.wect_complex(cx, d, T, maxheight_override=M), dirs)
    ab = synth.Complex(cx.coords, np.abs(cx.vweights), [synth.Cells(x.verts, np.abs(x.weights), 0) for x in cx.cells],
                       cx.k0, True)
    A = _oracle_rows(lambda d: oracle.wect_complex(ab, d, T, maxheight_override=M), dirs)
    err = np.abs(g - o2)
    assert (err <= 1e-5 * A + 1e-12).all(), float((err / (A + 1e-30)).max())


@pytest.mark.slow
def test_freudenthal_cfg2_batch_256_sampled_images_vs_O2():
    """The 60k cfg2 batch as Freudenthal complexes (NEXT-2) in the bench launch
    configuration: 256 sampled images (plus the first and last) equal O2."""
    c = synth.make_config(1)
    img, dirs, T = c["img"], c["dirs"], c["T"]
    out = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, freudenthal=True)
    torch.cuda.synchronize()
    idx = np.sort(np.random.default_rng(256).choice(img.shape[0], 256, replace=False))
    idx = np.concatenate([[0, img.shape[0] - 1], idx])
    o2 = oracle.wect_images_freudenthal(img[idx], dirs, T)
    assert (out[torch.from_numpy(idx).to(DEV)].cpu().numpy() == o2).all()


# ------------------------------------------------------------ tie-heavy directions
def _tie_dirs(n, extra, seed):
    """Axis directions, +-45 degree diagonals of every axis pair, then seeded random ones."""
    d = []
    for k in range(n):
        for s in (1.0, -1.0):
            e = np.zeros(n)
            e[k] = s
            d.append(e)
    for a in range(n):
        for b in range(a + 1, n):
            for sa, sb in ((1, 1), (1, -1), (-1, 1), (-1, -1)):
                e = np.zeros(n)
                e[a], e[b] = sa, sb
                d.append(e / np.sqrt(2.0))
    d = np.array(d)
    if extra:
        d = np.concatenate([d, synth.directions_sphere(extra, n, seed).astype(np.float64)])
    return d.astype(np.float32)


def _lattice_mesh(nu, nv, seed):
    """Planar triangulated grid with dyadic lattice coordinates (exact in fp32):
    (i/(nu-1) - 1/2, j/(nv-1) - 1/2, 0), edges right/down/diagonal, u8-range int weights."""
    g = np.random.default_rng(seed)
    ii, jj = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    coords = np.stack([ii / (nu - 1) - 0.5, jj / (nv - 1) - 0.5, np.zeros_like(ii, dtype=np.float64)], -1)
    coords = coords.reshape(-1, 3).astype(np.float32)
    vid = (ii * nv + jj)
    a = vid[:-1, :-1].ravel()
    b = vid[1:, :-1].ravel()
    c_ = vid[:-1, 1:].ravel()
    d = vid[1:, 1:].ravel()
    er = np.stack([vid[:-1, :].ravel(), vid[1:, :].ravel()], 1)
    ed = np.stack([vid[:, :-1].ravel(), vid[:, 1:].ravel()], 1)
    eg = np.stack([a, d], 1)
    edges = np.concatenate([er, ed, eg]).astype(np.int32)
    tris = np.concatenate([np.stack([a, b, d], 1), np.stack([a, c_, d], 1)]).astype(np.int32)
    k0 = nu * nv
    cx = synth.Complex(coords, g.integers(0, 256, k0).astype(np.int32),
                       [synth.Cells(edges, g.integers(0, 256, edges.shape[0]).astype(np.int32), 1),
                        synth.Cells(tris, g.integers(0, 256, tris.shape[0]).astype(np.int32), 2)], k0, False)
    return cx


@pytest.mark.parametrize("T", [33, 65, 129])
def test_ties_volume_histogram_path(T):
    """17^3 volume (grid spacing 1/16), axis and 45-degree directions, M = 1/2 (the axis
    directions' grid M), T - 1 a multiple of 16: every axis-direction vertex height is
    exactly a bin edge.  k_grid_hist must repair and match O2 bit for bit."""
    img = np.random.default_rng(T).integers(0, 256, (2, 17, 17, 17), dtype=np.uint8)
    dirs = _tie_dirs(3, 5, T)
    w.repair_count(reset=True)
    g = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, maxheight=0.5,
                      out_dtype="int64").cpu().numpy()
    assert w.repair_count() > 0
    assert (g == oracle.wect_images(img, dirs, T, maxheight_override=0.5)).all()


@pytest.mark.parametrize("T", [33, 65, 129, 257])
def test_ties_volume_covering_grid_fast_bins(T):
    """17^3 volume, axis directions only, the paper grid (M computed = 1/2, so [-M, M] holds
    every height and k_grid_hist takes its clamp-free rounded-up-add bins): with T - 1 a
    multiple of 16 every vertex height is exactly a bin edge -- repairs fire, bit-exact."""
    img = np.random.default_rng(T + 1).integers(0, 256, (2, 17, 17, 17), dtype=np.uint8)
    dirs = _tie_dirs(3, 0, T)[:6]
    w.repair_count(reset=True)
    g = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T,
                      out_dtype="int64").cpu().numpy()
    assert w.repair_count() > 0
    assert (g == oracle.wect_images(img, dirs, T)).all()
    # and with random directions added (M then from the grid corners, no ties)
    dirs2 = np.concatenate([dirs, synth.directions_sphere(40, 3, T)]).astype(np.float32)
    g2 = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs2).to(DEV), T,
                       out_dtype="int32").cpu().numpy()
    assert (g2 == oracle.wect_images(img, dirs2, T)).all()


def test_ties_large_image_histogram_path():
    """A 2-D image too large for the sweep (40 x 33) takes k_grid_hist: axis / 45-degree
    directions with T - 1 = 4 (L - 1) on the long axis."""
    img = np.random.default_rng(5).integers(0, 256, (3, 33, 40), dtype=np.uint8)
    dirs = _tie_dirs(2, 3, 5)
    T = 4 * 39 + 1
    w.repair_count(reset=True)
    g = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, maxheight=0.5,
                      out_dtype="int64").cpu().numpy()
    assert w.repair_count() > 0
    assert (g == oracle.wect_images(img, dirs, T, maxheight_override=0.5)).all()


@pytest.mark.parametrize("extra,T", [(30, 65), (30, 129), (2, 33), (2, 97)])
def test_ties_lattice_mesh_vbins_and_stream(extra, T):
    """Lattice mesh (spacing 1/32) with axis / 45-degree directions and M = 1/2: extra = 30
    gives D = 48 > 24 (k_vbins + k_cells_vb), extra = 2 gives D = 20 (k_stream)."""
    cx = _lattice_mesh(33, 33, T)
    dirs = _tie_dirs(3, extra, T)
    w.repair_count(reset=True)
    g = _gpu_complex(cx, dirs, T, maxheight=0.5)
    assert w.repair_count() > 0
    assert (g == oracle.wect_complex(cx, dirs, T, maxheight_override=0.5)).all()


def test_ties_lattice_mesh_ecf_stream():
    """ECF (k_stream) with a filter taking exactly the grid values q / (T - 1) of [0, 1]."""
    cx = _lattice_mesh(33, 33, 7)
    T = 65
    f = (np.random.default_rng(7).integers(0, T, (cx.k0, 1)) / (T - 1)).astype(np.float32)
    w.repair_count(reset=True)
    g = w.ecf_complex(torch.from_numpy(f).to(DEV), _cells(cx), T, vweights=torch.from_numpy(cx.vweights).to(DEV),
                      lo=0.0, hi=1.0)
    w.sync_status()
    assert w.repair_count() > 0
    assert (g.cpu().numpy() == oracle.ecf_complex(cx, f, T, lo=0.0, hi=1.0)).all()


def test_ties_lattice_mesh_backward():
    """k_grad_cells on the tie-heavy lattice: exact for integer-valued G (reading A13)."""
    cx = _lattice_mesh(33, 33, 11)
    dirs = _tie_dirs(3, 30, 11)
    T = 65
    G = np.random.default_rng(11).integers(-3, 4, (dirs.shape[0], T)).astype(np.float64)
    w.repair_count(reset=True)
    gv, gc = w.wect_complex_backward(torch.from_numpy(cx.coords).to(DEV), _cells(cx), torch.from_numpy(dirs).to(DEV),
                                     T, torch.from_numpy(G).to(DEV), maxheight=0.5)
    w.sync_status()
    assert w.repair_count() > 0
    ov, oc = oracle.wect_complex_grad(cx, dirs, T, G, maxheight_override=0.5)
    assert np.array_equal(gv.cpu().numpy(), ov)
    assert all(np.array_equal(a.cpu().numpy(), b) for a, b in zip(gc, oc))


@pytest.mark.parametrize("T", [39, 77])
def test_fused_grid_hist_ties_and_unfused_ab(T, monkeypatch):
    """WECT_GRID_FUSED=1 on a volume whose x axis is a multiple of 4: the fused k_grid_hist
    (orthant weights computed from the pixels of each row segment, directions sorted by
    orthant).  9 x 9 x 20 (x spacing 1/19), axis directions only: M = 1/2 and T - 1 a multiple
    of 19 put every x-axis vertex height on a bin edge -- repairs fire; then random directions;
    both bit-exact vs O2, and equal to the default table path (k_grid_cw)."""
    monkeypatch.setenv("WECT_GRID_FUSED", "1")
    img = np.random.default_rng(T + 5).integers(0, 256, (3, 9, 9, 20), dtype=np.uint8)
    dirs = _tie_dirs(3, 0, T)[:6]
    w.repair_count(reset=True)
    g = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, out_dtype="int64").cpu().numpy()
    assert w.repair_count() > 0
    assert (g == oracle.wect_images(img, dirs, T)).all()
    dirs2 = np.concatenate([dirs, synth.directions_sphere(70, 3, T)]).astype(np.float32)
    o2 = oracle.wect_images(img, dirs2, T)
    g2 = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs2).to(DEV), T, out_dtype="int32").cpu().numpy()
    assert (g2 == o2).all()
    monkeypatch.delenv("WECT_GRID_FUSED")
    g3 = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs2).to(DEV), T, out_dtype="int32").cpu().numpy()
    assert (g3 == o2).all()


def test_fused_grid_hist_2d_large_images(monkeypatch):
    """2-D images too large for the sweep with a width that is a multiple of 4 (36 x 44): the
    fused histogram path in 2-D, x-border groups at both ends, ragged last segment."""
    monkeypatch.setenv("WECT_GRID_FUSED", "1")
    img = np.random.default_rng(11).integers(0, 256, (5, 36, 44), dtype=np.uint8)
    dirs = np.concatenate([_tie_dirs(2, 0, 1), synth.directions_s1(41)]).astype(np.float32)
    for T in (43, 130):
        g = w.wect_images(torch.from_numpy(img).to(DEV), torch.from_numpy(dirs).to(DEV), T, out_dtype="int64").cpu().numpy()
        assert (g == oracle.wect_images(img, dirs, T)).all()


@pytest.mark.parametrize("T", [33, 65, 129])
def test_ties_lattice_mesh_covering_grid(T):
    """Lattice mesh, axis directions only (repeated to D = 30 > 24: k_vbins + k_cells_vb), the
    paper grid (M computed = 1/2 from the same vertices and directions): T - 1 a multiple of
    32 puts every vertex height on a bin edge -- repairs fire, bit-exact vs O2."""
    cx = _lattice_mesh(33, 33, T + 1)
    dirs = np.tile(_tie_dirs(3, 0, T)[:6], (5, 1))
    w.repair_count(reset=True)
    g = _gpu_complex(cx, dirs, T)
    assert w.repair_count() > 0
    assert (g == oracle.wect_complex(cx, dirs, T)).all()
