"""Multi-GPU sharding of the WECT hot path (one process per GPU, torch.distributed).

The method has no cross-rank data dependence: every output row
(p, q) depends only on its filter and on the global maxheight M.  So the path shards
two ways, with NCCL used only to GATHER outputs (never inside the data path):

  * batch sharding (image batches, BASELINE configs[1]): rank r takes a contiguous
    block of images; the grid M is the same for every image of a fixed-size batch.
  * direction sharding (one large complex, configs[2..4]): rank r computes the rows
    [d_lo, d_hi) of the full direction set.  The library always takes M over ALL
    directions it is given (reading A2), so every rank passes the full `dirs` and
    its row range -- the sharded result equals the unsharded one bit for bit.

`compute` hooks exist so the host-side partition/gather logic can be exercised by
CPU tests (gloo, world_size 2) with the oracle injected; the default compute is the
CUDA library, and there is no CPU fallback in the product path.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced split of [0, n): the first n % world ranks get one extra."""
    base, extra = divmod(int(n), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _world(group) -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def gather_rows(local: torch.Tensor, n_total: int, dim: int, group=None) -> torch.Tensor:
    """all_gather of uneven contiguous shards along `dim` (pad to the largest shard, trim)."""
    world, rank = _world(group)
    if world == 1:
        return local
    sizes = [shard_range(n_total, world, r)[1] - shard_range(n_total, world, r)[0] for r in range(world)]
    mx = max(sizes)
    local = local.movedim(dim, 0).contiguous()
    if local.shape[0] < mx:
        pad = torch.zeros((mx - local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        local = torch.cat([local, pad], 0)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local, group=group)
        parts = [out[r * mx: r * mx + sizes[r]] for r in range(world)]
    else:
        bufs = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(bufs, local, group=group)
        parts = [bufs[r][: sizes[r]] for r in range(world)]
    return torch.cat(parts, 0).movedim(0, dim)


def _lib_images(img, dirs, T, d_begin, d_count, **kw):
    from . import wect_images

    return wect_images(img, dirs, T, d_begin=d_begin, d_count=d_count, **kw)


def wect_images_sharded(img: torch.Tensor, dirs: torch.Tensor, T: int, *, mode: str = "batch", gather: bool = True,
                        group=None, compute: Optional[Callable] = None, **kw) -> torch.Tensor:
    """WECT of an image batch across ranks.

    mode="batch": `img` is the FULL batch on every rank (or a view of it); rank r computes
    images shard_range(B, world, r).  mode="directions": rank r computes the rows
    shard_range(D, world, r) for all images.  With gather=True the full [B, D, T] result
    is assembled on every rank via all_gather (NCCL over NVLink on GPUs); with
    gather=False the local shard is returned."""
    compute = compute or _lib_images
    world, rank = _world(group)
    B, D = int(img.shape[0]), int(dirs.shape[0])
    if mode == "batch":
        lo, hi = shard_range(B, world, rank)
        local = compute(img[lo:hi].contiguous(), dirs, T, 0, 0, **kw)
        return gather_rows(local, B, 0, group) if gather else local
    if mode == "directions":
        lo, hi = shard_range(D, world, rank)
        local = compute(img, dirs, T, lo, hi - lo, **kw) if hi > lo else torch.zeros(
            (B, 0, T), dtype=torch.int32 if kw.get("out_dtype", "int32") == "int32" else torch.int64, device=img.device)
        return gather_rows(local, D, 1, group) if gather else local
    raise ValueError(mode)


def _lib_maxheight(coords, dirs):
    from . import wect_maxheight

    return wect_maxheight(coords, dirs)


def global_maxheight(coords, dirs, *, group=None, compute: Optional[Callable] = None) -> float:
    """M = max over ALL directions and vertices of |<x_v, s_p>| (reading A2) from
    per-shard maxima: rank r evaluates only its direction rows shard_range(D, world, r)
    (wect_maxheight on that contiguous slice) and all_reduce(MAX) combines them.  Exact: each
    shard's M is the exact binary64 maximum and max is associative.  Direction-sharded
    calls pass it as `maxheight`, so no rank scans the full direction set."""
    compute = compute or _lib_maxheight
    world, rank = _world(group)
    D = int(dirs.shape[0])
    lo, hi = shard_range(D, world, rank)
    m = float(compute(coords, dirs[lo:hi])) if hi > lo else 0.0
    if world > 1:
        on_dev = dist.get_backend(group) == "nccl"
        t = torch.tensor([m], dtype=torch.float64,
                         device=torch.device("cuda", torch.cuda.current_device()) if on_dev else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        m = float(t.item())
    return m


def _lib_complex(coords, cells, dirs, T, d_begin, d_count, **kw):
    from . import wect_complex

    return wect_complex(coords, cells, dirs, T, d_begin=d_begin, d_count=d_count, **kw)


def wect_complex_sharded(coords, cells: Sequence[Tuple], dirs, T: int, *, gather: bool = True, group=None,
                         compute: Optional[Callable] = None, maxheight_compute: Optional[Callable] = None,
                         **kw) -> torch.Tensor:
    """WECT of one explicit complex, direction-sharded: rank r computes the rows
    shard_range(D, world, r) with M over ALL directions (reading A2) -- all-reduced from the
    per-shard maxima (global_maxheight) unless the caller fixes `maxheight` -- then all_gather."""
    compute = compute or _lib_complex
    world, rank = _world(group)
    D = int(dirs.shape[0])
    if kw.get("maxheight", 0.0) <= 0.0 and world > 1:
        kw["maxheight"] = global_maxheight(coords, dirs, group=group, compute=maxheight_compute)
    lo, hi = shard_range(D, world, rank)
    if hi > lo:
        local = compute(coords, cells, dirs, T, lo, hi - lo, **kw)
    else:  # more ranks than directions: an empty shard (d_count == 0 would mean "all rows")
        local = None
    if local is None:
        ref = compute(coords, cells, dirs, T, 0, 1, **kw)
        local = ref[:0]
    return gather_rows(local, D, 0, group) if gather else local


def _lib_ecf_images(img, T, **kw):
    from . import ecf_images

    return ecf_images(img, T, **kw)


def ecf_images_sharded(img: torch.Tensor, T: int, *, gather: bool = True, group=None,
                       compute: Optional[Callable] = None, **kw) -> torch.Tensor:
    """Image ECF (ecf_images, NEXT-1) of a batch across ranks: every image is its own complex
    (its own M, or the caller's fixed grid), so rank r computes images shard_range(B, world, r)
    with no exchange; gather=True assembles [B, T] on every rank (all_gather)."""
    compute = compute or _lib_ecf_images
    world, rank = _world(group)
    B = int(img.shape[0])
    lo, hi = shard_range(B, world, rank)
    local = compute(img[lo:hi].contiguous(), T, **kw)
    return gather_rows(local, B, 0, group) if gather else local


def _lib_backward(coords, cells, dirs, T, G_rows, d_begin, d_count, **kw):
    from . import wect_complex_backward

    return wect_complex_backward(coords, cells, dirs, T, G_rows, d_begin=d_begin, d_count=d_count, **kw)


def wect_complex_backward_sharded(coords, cells: Sequence[Tuple], dirs, T: int, G, *, group=None,
                                  compute: Optional[Callable] = None, **kw):
    """Weights gradient (NEXT-3) of one complex, direction-sharded.  dL/dw(s) is a SUM over
    the direction rows p (include/wect.h), so rank r computes the partial gradient of its rows
    shard_range(D, world, r) (M over ALL directions, reading A2) and the partials are
    all-reduced (SUM) -- the one real exchange step of the path.  G: the full [D, T] fp64.
    Returns (grad_vweights, [grad_cells_i]) on every rank.  Exact for integer-valued G; for
    general G the cross-rank sum adds one more reassociation to reading A13."""
    compute = compute or _lib_backward
    world, rank = _world(group)
    D = int(dirs.shape[0])
    lo, hi = shard_range(D, world, rank)
    if hi > lo:
        gv, gc = compute(coords, cells, dirs, T, G[lo:hi].contiguous(), lo, hi - lo, **kw)
    else:  # more ranks than directions: a zero partial
        gv, gc = compute(coords, cells, dirs, T, G[:1].contiguous(), 0, 1, **kw)
        gv = torch.zeros_like(gv)
        gc = [torch.zeros_like(g) for g in gc]
    if world > 1:
        flat = torch.cat([gv.reshape(-1)] + [g.reshape(-1) for g in gc])
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        sizes = [gv.numel()] + [g.numel() for g in gc]
        parts = list(torch.split(flat, sizes))
        gv, gc = parts[0].view_as(gv), [p.view_as(g) for p, g in zip(parts[1:], gc)]
    return gv, gc
