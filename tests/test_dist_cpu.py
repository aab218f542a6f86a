"""Multi-rank (world_size 2, gloo, CPU) tests of the sharding/gather logic in
paper_2511_03909_b200.dist.  The compute step is injected with the CPU oracle (test
infrastructure) so the partition + gather path runs without a GPU; on GPUs the
same code calls the CUDA library and gathers over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2511_03909_b200.dist import (ecf_images_sharded, gather_rows, global_maxheight, shard_range,
                                        wect_complex_backward_sharded, wect_complex_sharded, wect_images_sharded)


def test_shard_range_partitions():
    for n in (0, 1, 5, 64, 65, 1023):
        for w in (1, 2, 3, 8):
            cover = []
            for r in range(w):
                lo, hi = shard_range(n, w, r)
                assert 0 <= lo <= hi <= n
                cover += list(range(lo, hi))
            assert cover == list(range(n))
            sizes = [shard_range(n, w, r)[1] - shard_range(n, w, r)[0] for r in range(w)]
            assert max(sizes) - min(sizes) <= 1


def _oracle_images(img, dirs, T, d_begin, d_count, **kw):
    full = oracle.wect_images(img.numpy(), dirs.numpy(), T)  # M over ALL directions (reading A2)
    cnt = d_count if d_count else dirs.shape[0] - d_begin
    return torch.from_numpy(full[:, d_begin:d_begin + cnt].copy())


def _oracle_complex(coords, cells, dirs, T, d_begin, d_count, **kw):
    cx = synth.Complex(coords, kw["vweights"], [synth.Cells(v, w, d) for v, w, d in cells], coords.shape[0])
    full = oracle.wect_complex(cx, dirs, T, maxheight_override=kw.get("maxheight", 0.0))
    return torch.from_numpy(full[d_begin:d_begin + d_count].copy())


def _oracle_maxheight(coords, dirs):
    return oracle.maxheight(oracle.heights(coords, np.asarray(dirs)))


def _oracle_ecf_images(img, T, **kw):
    return torch.from_numpy(oracle.ecf_images(img.numpy(), T, kw.get("lo", 0.0), kw.get("hi", 0.0)))


def _oracle_backward(coords, cells, dirs, T, G_rows, d_begin, d_count, **kw):
    """the oracle's closed-form gradient of the rows [d_begin, d_begin + d_count), M over ALL rows"""
    cx = synth.Complex(coords, None, [synth.Cells(v, None, d) for v, _, d in cells], coords.shape[0])
    fv = oracle.heights(coords, dirs)
    M = oracle.maxheight(fv)
    gv, gc = oracle.wecfs_grad(fv[:, d_begin:d_begin + d_count], cx, T, -M, M, np.asarray(G_rows))
    return torch.from_numpy(gv), [torch.from_numpy(g) for g in gc]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = np.random.default_rng(0)
        img = torch.from_numpy(g.integers(0, 256, (7, 6, 5), dtype=np.uint8))  # 7 images: uneven split
        dirs = torch.from_numpy(synth.directions_s1(9))  # 9 directions: uneven split
        ref = _oracle_images(img, dirs, 16, 0, 0)
        a = wect_images_sharded(img, dirs, 16, mode="batch", compute=_oracle_images)
        b = wect_images_sharded(img, dirs, 16, mode="directions", compute=_oracle_images)
        loc = wect_images_sharded(img, dirs, 16, mode="batch", gather=False, compute=_oracle_images)
        lo, hi = shard_range(7, world, rank)
        cx = synth.random_small_complex(3, n=3, nverts=40, ntop=30)
        cells = [(c.verts, c.weights, c.dim) for c in cx.cells]
        d3 = synth.directions_sphere(5, 3, 1)
        d3[4] *= 3.0  # the row that sets M lives on the last rank
        cref = oracle.wect_complex(cx, d3, 12)
        c = wect_complex_sharded(cx.coords, cells, d3, 12, compute=_oracle_complex,
                                 maxheight_compute=_oracle_maxheight, vweights=cx.vweights)
        # M from per-shard maxima (all_reduce MAX) equals M over all directions, exactly
        mh = global_maxheight(cx.coords, d3, compute=_oracle_maxheight) == _oracle_maxheight(cx.coords, d3)
        # image ECF (NEXT-1): batch shards, no exchange
        eimg = torch.from_numpy(g.integers(0, 256, (5, 6, 8), dtype=np.uint8))
        eref = oracle.ecf_images(eimg.numpy(), 32, 0.0, 255.0)
        e = ecf_images_sharded(eimg, 32, compute=_oracle_ecf_images, lo=0.0, hi=255.0)
        # weights gradient (NEXT-3): direction shards, partial gradients all-reduced (SUM)
        G = torch.from_numpy(g.integers(-3, 4, size=(5, 12)).astype(np.float64))
        gv_ref, gc_ref = oracle.wect_complex_grad(cx, d3, 12, G.numpy())
        gv, gc = wect_complex_backward_sharded(cx.coords, cells, d3, 12, G, compute=_oracle_backward)
        gok = np.array_equal(gv.numpy(), gv_ref) and all(np.array_equal(a_.numpy(), b_) for a_, b_ in zip(gc, gc_ref))
        q.put((rank, bool(torch.equal(a, ref)), bool(torch.equal(b, ref)), bool(torch.equal(loc, ref[lo:hi])),
               bool(np.array_equal(c.numpy(), cref)), bool(np.array_equal(e.numpy(), eref)), bool(gok), bool(mh)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_unsharded():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, *oks in res:
        assert all(oks), (rank, oks)


def test_gather_rows_single_process():
    t = torch.arange(12).reshape(3, 4)
    assert torch.equal(gather_rows(t, 3, 0), t)
