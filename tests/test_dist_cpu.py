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
from paper_2511_03909_b200.dist import gather_rows, shard_range, wect_complex_sharded, wect_images_sharded


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
    full = oracle.wect_complex(cx, dirs, T)
    return torch.from_numpy(full[d_begin:d_begin + d_count].copy())


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
        c = wect_complex_sharded(cx.coords, cells, d3, 12, compute=_oracle_complex, vweights=cx.vweights)
        q.put((rank, bool(torch.equal(a, ref)), bool(torch.equal(b, ref)), bool(torch.equal(loc, ref[lo:hi])),
               bool(np.array_equal(c.numpy(), cref))))
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
