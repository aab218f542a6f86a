"""Small invocations of each hot kernel for compute-sanitizer (memcheck / racecheck /
synccheck), checked against the oracle:  python tools/sanitize_cases.py CASE"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2511_03909_b200 as w  # noqa: E402
import synth  # noqa: E402

DEV = torch.device("cuda:0")
T_ = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731


def cells(cx):
    return [(T_(c.verts), None if c.weights is None else T_(c.weights), c.dim) for c in cx.cells]


def main(case):
    g = np.random.default_rng(1)
    if case == "sweep":  # k_sort2d + k_sweep2d (TMA stores, bulk-copy ring) + Freudenthal fix-ups
        img = g.integers(0, 256, (70, 28, 28), dtype=np.uint8)
        dirs = synth.directions_s1(17)
        got = w.wect_images(T_(img), T_(dirs), 64).cpu().numpy()
        assert (got == oracle.wect_images(img, dirs, 64)).all()
        got = w.wect_images(T_(img), T_(dirs), 64, freudenthal=True).cpu().numpy()
        assert (got == oracle.wect_images_freudenthal(img, dirs, 64)).all()
    elif case == "ecfimg":  # k_ecf_img2d_w4 (28x28) and k_ecf_img2d_rows + k_ecf_img_final (wide)
        img = g.integers(0, 256, (40, 28, 28), dtype=np.uint8)
        assert (w.ecf_images(T_(img), 256, lo=0.0, hi=255.0).cpu().numpy() == oracle.ecf_images(img, 256, 0.0, 255.0)).all()
        img = g.integers(0, 256, (2, 40, 200), dtype=np.uint8)
        assert (w.ecf_images(T_(img), 256, lo=0.0, hi=255.0).cpu().numpy() == oracle.ecf_images(img, 256, 0.0, 255.0)).all()
    elif case == "stream":  # k_stream (D <= 24 and the ECF)
        cx = synth.torus_mesh(30, 40, 2)
        dirs = synth.directions_sphere(6, 3, 2)
        got = w.wect_complex(T_(cx.coords), cells(cx), T_(dirs), 64, vweights=T_(cx.vweights)).cpu().numpy()
        w.sync_status()
        assert (got == oracle.wect_complex(cx, dirs, 64)).all()
        f = g.uniform(-1, 1, (cx.k0, 1)).astype(np.float32)
        got = w.ecf_complex(T_(f), cells(cx), 64, vweights=T_(cx.vweights)).cpu().numpy()
        assert (got == oracle.ecf_complex(cx, f, 64)).all()
    elif case == "cells_vb":  # k_vbins + k_cells_vb (D > 24)
        cx = synth.torus_mesh(30, 40, 3)
        dirs = synth.directions_sphere(40, 3, 3)
        got = w.wect_complex(T_(cx.coords), cells(cx), T_(dirs), 64, vweights=T_(cx.vweights)).cpu().numpy()
        w.sync_status()
        assert (got == oracle.wect_complex(cx, dirs, 64)).all()
    elif case == "grid_hist":  # k_grid_params + k_grid_cw + k_grid_hist + k_finalize (volumes)
        vol = g.integers(0, 256, (2, 9, 10, 11), dtype=np.uint8)
        dirs = synth.directions_sphere(40, 3, 4)
        got = w.wect_images(T_(vol), T_(dirs), 32, out_dtype="int64").cpu().numpy()
        assert (got == oracle.wect_images(vol, dirs, 32)).all()
    elif case == "grad":  # k_rcumsum + k_vbins + k_grad_cells
        cx = synth.torus_mesh(30, 40, 5)
        dirs = synth.directions_sphere(40, 3, 5)
        G = g.integers(-3, 4, (40, 64)).astype(np.float64)
        gv, gc = w.wect_complex_backward(T_(cx.coords), cells(cx), T_(dirs), 64, T_(G))
        w.sync_status()
        ov, oc = oracle.wect_complex_grad(cx, dirs, 64, G)
        assert np.array_equal(gv.cpu().numpy(), ov) and all(np.array_equal(a.cpu().numpy(), b) for a, b in zip(gc, oc))
    elif case == "mma":  # k_mma_dirs / k_mma_passes / k_mma_bimg + k_mma2d (tcgen05, TMEM, bulk copies)
        os.environ["WECT_IMAGES_MMA"] = "1"
        img = g.integers(0, 256, (200, 28, 28), dtype=np.uint8)
        dirs = synth.directions_s1(19)
        got = w.wect_images(T_(img), T_(dirs), 128).cpu().numpy()
        assert (got == oracle.wect_images(img, dirs, 128)).all()
    elif case == "grid_fused":  # k_dir_perm + the fused k_grid_hist (orthant weights from the pixels)
        os.environ["WECT_GRID_FUSED"] = "1"
        vol = g.integers(0, 256, (2, 9, 10, 12), dtype=np.uint8)
        dirs = synth.directions_sphere(40, 3, 6)
        got = w.wect_images(T_(vol), T_(dirs), 32, out_dtype="int64").cpu().numpy()
        assert (got == oracle.wect_images(vol, dirs, 32)).all()
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print(f"case {case}: ok")


if __name__ == "__main__":
    main(sys.argv[1])
