"""The sharding layer (paper_2511_03909_b200.dist) with the CUDA library doing the compute:
a 1-rank NCCL group (the production backend) and 2 ranks sharing the box's GPU over gloo
(the collectives then run on host-staged copies), each compared element by element with
the oracle (O2)."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as tdist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cases(dev):
    """(name, sharded result on this rank (gathered), oracle reference)"""
    from paper_2511_03909_b200 import dist as wd

    g = np.random.default_rng(3)
    img = g.integers(0, 256, (67, 28, 28), dtype=np.uint8)
    dirs = synth.directions_s1(13)
    ref_img = oracle.wect_images(img, dirs, 32)
    img_d, dirs_d = torch.from_numpy(img).to(dev), torch.from_numpy(dirs).to(dev)
    out = []
    out.append(("images/batch", wd.wect_images_sharded(img_d, dirs_d, 32, mode="batch").cpu().numpy(), ref_img))
    out.append(("images/directions", wd.wect_images_sharded(img_d, dirs_d, 32, mode="directions").cpu().numpy(),
                ref_img))
    vol = g.integers(0, 256, (1, 9, 10, 11), dtype=np.uint8)
    d3 = synth.directions_sphere(21, 3, 4)
    out.append(("volume/directions",
                wd.wect_images_sharded(torch.from_numpy(vol).to(dev), torch.from_numpy(d3).to(dev), 40,
                                       mode="directions", out_dtype="int64").cpu().numpy(),
                oracle.wect_images(vol, d3, 40)))
    cx = synth.torus_mesh(30, 40, 5)
    dm = synth.directions_sphere(37, 3, 5)
    dm[36] *= 2.5  # the row that sets M sits in the last shard
    cells = [(torch.from_numpy(c.verts).to(dev), torch.from_numpy(c.weights).to(dev), c.dim) for c in cx.cells]
    coords_d, dm_d = torch.from_numpy(cx.coords).to(dev), torch.from_numpy(dm).to(dev)
    out.append(("complex/directions",
                wd.wect_complex_sharded(coords_d, cells, dm_d, 64, vweights=torch.from_numpy(cx.vweights).to(dev))
                .cpu().numpy(), oracle.wect_complex(cx, dm, 64)))
    M = wd.global_maxheight(coords_d, dm_d)
    out.append(("global_maxheight", np.array([M]), np.array([oracle.maxheight(oracle.heights(cx.coords, dm))])))
    eimg = g.integers(0, 256, (45, 28, 28), dtype=np.uint8)
    out.append(("ecf_images/batch",
                wd.ecf_images_sharded(torch.from_numpy(eimg).to(dev), 256, lo=0.0, hi=255.0).cpu().numpy(),
                oracle.ecf_images(eimg, 256, 0.0, 255.0)))
    G = g.integers(-3, 4, size=(37, 64)).astype(np.float64)
    gv, gc = wd.wect_complex_backward_sharded(coords_d, cells, dm_d, 64, torch.from_numpy(G).to(dev))
    ov, oc = oracle.wect_complex_grad(cx, dm, 64, G)
    out.append(("backward/directions", np.concatenate([gv.cpu().numpy()] + [x.cpu().numpy() for x in gc]),
                np.concatenate([ov] + list(oc))))
    return out


def test_one_rank_nccl_group():
    port = _free_port()
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                             device_id=torch.device("cuda:0"))
    try:
        for name, got, ref in _cases(torch.device("cuda:0")):
            assert np.array_equal(got, ref), name
    finally:
        tdist.destroy_process_group()


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        res = [(name, bool(np.array_equal(got, ref))) for name, got, ref in _cases(torch.device("cuda:0"))]
        q.put((rank, res, None))
    except Exception as e:  # report, do not hang the parent
        q.put((rank, [], repr(e)))
    finally:
        tdist.destroy_process_group()


def test_two_ranks_gloo_sharing_one_gpu():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, oks, err in res:
        assert err is None, (rank, err)
        assert all(ok for _, ok in oks), (rank, oks)
