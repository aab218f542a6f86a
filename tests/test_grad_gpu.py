"""GPU parity of wect_complex_backward / ecf_complex_backward against
the oracle's closed-form gradient (oracle.wecfs_grad).  Integer-valued G: every partial sum
is an exact binary64 integer, so the comparison is bit-exact.  Random fp64 G: reading A13,
|gpu - oracle| <= 1e-12 * sum|G| of the rows (binary64 reassociation only)."""
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
    return [(torch.from_numpy(np.ascontiguousarray(c.verts, np.int32)).to(DEV), None, c.dim) for c in cx.cells]


def _check(gv, gc, ov, oc, G, exact):
    tol = 0.0 if exact else 1e-12 * float(np.abs(G).sum())
    assert np.abs(gv.cpu().numpy() - ov).max(initial=0.0) <= tol
    for a, b in zip(gc, oc):
        assert np.abs(a.cpu().numpy() - b).max(initial=0.0) <= tol


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("exact", [True, False])
def test_wect_backward_vs_oracle(seed, exact):
    rng = np.random.default_rng(6000 + seed)
    n = [2, 3, 3, 4, 5, 3][seed]
    cx = synth.random_small_complex(seed, n=n, nverts=60 + 20 * seed, ntop=50, kmax=min(3, n))
    D, T = [(1, 7), (9, 64), (70, 33), (64, 512), (33, 2), (130, 128)][seed]
    dirs = synth.directions_s1(D) if n == 2 else synth.directions_sphere(D, n, 6100 + seed)
    G = rng.integers(-5, 6, size=(D, T)).astype(np.float64) if exact else rng.standard_normal((D, T))
    gv, gc = w.wect_complex_backward(torch.from_numpy(cx.coords).to(DEV), _cells(cx), torch.from_numpy(dirs).to(DEV),
                                     T, torch.from_numpy(G).to(DEV))
    w.sync_status()
    ov, oc = oracle.wect_complex_grad(cx, dirs, T, G)
    _check(gv, gc, ov, oc, G, exact)


def test_wect_backward_row_slice_and_host_buffers():
    cx = synth.torus_mesh(9, 11, 3)
    dirs = synth.directions_sphere(100, 3, 6200)
    T = 40
    G = np.random.default_rng(1).integers(-4, 5, size=(100, T)).astype(np.float64)
    ov, oc = oracle.wect_complex_grad(cx, dirs, T, G)
    # host (numpy) buffers: the library stages them
    gv, gc = w.wect_complex_backward(cx.coords, [(c.verts, None, c.dim) for c in cx.cells], dirs, T, G)
    _check(gv, gc, ov, oc, G, True)
    # rows 30..79 only: the gradient of L restricted to those rows, with M over ALL rows (A2)
    ov2, oc2 = oracle.wecfs_grad(oracle.heights(cx.coords, dirs)[:, 30:80], cx, T,
                                 -oracle.maxheight(oracle.heights(cx.coords, dirs)),
                                 oracle.maxheight(oracle.heights(cx.coords, dirs)), G[30:80])
    gv2, gc2 = w.wect_complex_backward(cx.coords, [(c.verts, None, c.dim) for c in cx.cells], dirs, T,
                                       np.ascontiguousarray(G[30:80]), d_begin=30, d_count=50)
    _check(gv2, gc2, ov2, oc2, G, True)


@pytest.mark.parametrize("m,T", [(1, 512), (5, 17), (77, 256)])
def test_ecf_backward_vs_oracle(m, T):
    cx = synth.torus_mesh(12, 10, m)
    f = np.random.default_rng(m).uniform(-1, 1, (cx.k0, m)).astype(np.float32)
    G = np.random.default_rng(m + 1).integers(-3, 4, size=(m, T)).astype(np.float64)
    gv, gc = w.ecf_complex_backward(torch.from_numpy(f).to(DEV), _cells(cx), T, torch.from_numpy(G).to(DEV))
    ov, oc = oracle.ecf_complex_grad(cx, f, T, G)
    _check(gv, gc, ov, oc, G, True)
    gv, gc = w.ecf_complex_backward(torch.from_numpy(f).to(DEV), _cells(cx), T, torch.from_numpy(G).to(DEV),
                                    lo=-2.0, hi=0.5)
    ov, oc = oracle.ecf_complex_grad(cx, f, T, G, -2.0, 0.5)
    _check(gv, gc, ov, oc, G, True)


def test_backward_large_T_global_rc_path():
    cx = synth.torus_mesh(8, 9, 4)
    dirs = synth.directions_sphere(40, 3, 6300)
    T = 1000  # RC tile > 160 KB: gathered from global memory
    G = np.random.default_rng(2).integers(-3, 4, size=(40, T)).astype(np.float64)
    gv, gc = w.wect_complex_backward(cx.coords, [(c.verts, None, c.dim) for c in cx.cells], dirs, T, G)
    ov, oc = oracle.wect_complex_grad(cx, dirs, T, G)
    _check(gv, gc, ov, oc, G, True)


def test_backward_mesh_euler_identity_at_scale():
    """cfg4-shaped mesh (scaled): L(w) from the GPU forward equals sum w * grad from the GPU
    backward, exactly (integer weights, integer G)."""
    c = synth.make_config(3, scale=0.02)
    cx, dirs = c["complex"], c["dirs"][:96]
    T = 512
    G = np.random.default_rng(3).integers(-2, 3, size=(96, T)).astype(np.float64)
    cells = [(torch.from_numpy(x.verts).to(DEV), torch.from_numpy(x.weights).to(DEV), x.dim) for x in cx.cells]
    fwd = w.wect_complex(torch.from_numpy(cx.coords).to(DEV), cells, torch.from_numpy(dirs).to(DEV), T,
                         vweights=torch.from_numpy(cx.vweights).to(DEV)).cpu().numpy()
    L = float((fwd.astype(np.float64) * G).sum())
    gv, gc = w.wect_complex_backward(torch.from_numpy(cx.coords).to(DEV), cells, torch.from_numpy(dirs).to(DEV), T,
                                     torch.from_numpy(G).to(DEV))
    lin = float((cx.vweights.astype(np.float64) * gv.cpu().numpy()).sum())
    for x, g in zip(cx.cells, gc):
        lin += float((x.weights.astype(np.float64) * g.cpu().numpy()).sum())
    assert lin == L


def test_sharded_entry_points_single_rank_use_the_library():
    """dist.wect_complex_backward_sharded / ecf_images_sharded without a process group:
    the default compute is the CUDA library (no oracle, no fallback)."""
    from paper_2511_03909_b200.dist import ecf_images_sharded, wect_complex_backward_sharded

    cx = synth.torus_mesh(7, 9, 2)
    dirs = torch.from_numpy(synth.directions_sphere(20, 3, 6400)).to(DEV)
    G = torch.from_numpy(np.random.default_rng(4).integers(-3, 4, size=(20, 50)).astype(np.float64)).to(DEV)
    coords = torch.from_numpy(cx.coords).to(DEV)
    gv, gc = wect_complex_backward_sharded(coords, _cells(cx), dirs, 50, G)
    ov, oc = oracle.wect_complex_grad(cx, dirs.cpu().numpy(), 50, G.cpu().numpy())
    _check(gv, gc, ov, oc, G.cpu().numpy(), True)
    img = torch.from_numpy(synth.images_u8(9, (28, 28), 6500)).to(DEV)
    e = ecf_images_sharded(img, 256, lo=0.0, hi=255.0)
    assert (e.cpu().numpy() == oracle.ecf_images(img.cpu().numpy(), 256, 0.0, 255.0)).all()


def test_backward_edge_cases_and_errors():
    from paper_2511_03909_b200 import _lib

    cx = synth.torus_mesh(5, 6, 1)
    dirs = synth.directions_sphere(7, 3, 6600)
    cells = [(c.verts, None, c.dim) for c in cx.cells]
    G = np.ones((7, 9))
    # T < 2, bad row range, NULL G
    with pytest.raises(_lib.WectError):
        w.wect_complex_backward(cx.coords, cells, dirs, 1, np.ones((7, 1)))
    with pytest.raises(_lib.WectError):
        w.wect_complex_backward(cx.coords, cells, dirs, 9, G, d_begin=5, d_count=5)
    # arity 9 cells: not supported by the backward (documented)
    wide = [(np.zeros((3, 9), np.int32), None, 8)]
    with pytest.raises(_lib.WectError):
        w.wect_complex_backward(cx.coords, wide, dirs, 9, G)
    # out-of-range vertex index: reported by sync_status, the cell gets no gradient
    bad = [(np.array([[0, 1], [2, cx.k0 + 5]], np.int32), None, 1)]
    w.wect_complex_backward(cx.coords, bad, dirs, 9, G)
    with pytest.raises(_lib.WectError):
        w.sync_status()
    # G = 0 -> zero gradient; single direction; T = 2
    gv, gc = w.wect_complex_backward(cx.coords, cells, dirs[:1], 2, np.zeros((1, 2)))
    assert float(np.abs(gv.numpy()).max()) == 0.0 and all(float(np.abs(g.numpy()).max()) == 0.0 for g in gc)
    # top-bin-only G: every gradient is its sign times the number of rows (all cells land in bins <= T-1)
    Gt = np.zeros((7, 9))
    Gt[:, -1] = 1.0
    gv, gc = w.wect_complex_backward(cx.coords, cells, dirs, 9, Gt)
    assert (gv.numpy() == 7.0).all()
    for (v, _, d), g in zip(cells, gc):
        assert (g.numpy() == (7.0 if d % 2 == 0 else -7.0)).all()


@pytest.mark.slow
@pytest.mark.parametrize("c", [3, 4])
def test_backward_full_size_sampled_vs_oracle(c):
    """bwd3 / bwd4 at BASELINE's full sizes (cfg4 mesh, D = 1024, T = 512; cfg5 complex,
    D = 256, T = 256) in the bench launch configuration; the oracle's closed form on 64
    sampled cells of every dimension and 64 sampled vertices, M over ALL directions (A2)."""
    d = synth.make_config(c)
    cx, dirs, T = d["complex"], d["dirs"], d["T"]
    D = dirs.shape[0]
    G = synth.rng(synth.S0 + 70 + c).integers(-3, 4, size=(D, T)).astype(np.float64)
    gv, gc = w.wect_complex_backward(torch.from_numpy(cx.coords).to(DEV), _cells(cx), torch.from_numpy(dirs).to(DEV), T,
                                     torch.from_numpy(G).to(DEV))
    w.sync_status()
    g = np.random.default_rng(100 + c)
    M = 0.0  # M over ALL vertices and directions (A2), chunked over directions
    for a in range(0, D, 64):
        M = max(M, float(np.abs(oracle.heights(cx.coords, dirs[a:a + 64])).max()))
    vs = np.sort(g.choice(cx.k0, 64, replace=False))
    picks = [np.sort(g.choice(len(x.verts), 64, replace=False)) for x in cx.cells]
    # heights of the vertices the samples touch only, ids remapped into that subset
    need = np.unique(np.concatenate([vs] + [x.verts[i].reshape(-1) for x, i in zip(cx.cells, picks)]))
    remap = {int(v): k for k, v in enumerate(need)}
    fv = oracle.heights(np.ascontiguousarray(cx.coords[need]), dirs)
    sub = synth.Complex(None, None, [synth.Cells(np.vectorize(remap.get)(x.verts[i]).astype(np.int32), None, x.dim)
                                     for x, i in zip(cx.cells, picks)], len(need))
    ov, oc = oracle.wecfs_grad(fv, sub, T, -M, M, G, vertices=[remap[int(v)] for v in vs])
    assert (gv[torch.from_numpy(vs).to(DEV)].cpu().numpy() == ov).all()
    for gi, i, o in zip(gc, picks, oc):
        assert (gi[torch.from_numpy(i).to(DEV)].cpu().numpy() == o).all()
