#!/usr/bin/env python
"""bench.py -- WECT throughput of the B200 hot path on BASELINE.json's configs.

Default workload (N = 1 line the driver records): BASELINE.json configs[1], the
MNIST-shaped batch -- 60,000 synthetic 28x28 uint8 images per GPU, D = 64
directions on S^1, T = 128 bins, int32 output [60000, 64, 128].  One step = one
wect_images call over the batch = every row of SURVEY.md section 8(a): grid M
(a2), exact vertex bins + per-direction counting sort (a1, a3), and the sweep
kernel (a0, a4-a7: implicit cells, max rule, signed regrouped accumulation,
cumsum, 1.97 GB output write).

  python bench.py [--gpus N --steps K --warmup W] [--config 1|2|3|4|ecfx|ecfimg|ecfimg1k|bwd3|bwd4|freud] [--impl reference]

Multi-GPU (one rank per GPU; `--gpus N` relaunches itself under torch.distributed.run when
WORLD_SIZE is unset): STRONG scaling over the workload BASELINE.json names -- the one
60,000-image batch is split into contiguous image shards (no data-path collective), a
single volume / mesh is split into direction rows with M all-reduced (MAX) from per-shard
maxima (reading A2), the weights gradient all-reduces (SUM) its partials.  Times are the
max over ranks (all_reduce MAX); the all_gather that would assemble the full output is
timed separately (`gather_ms`).  --impl reference times the CPU oracle (O2) on the host on
a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "WECT complexes/sec and simplex·direction updates/sec; HBM GB/s vs peak"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy, burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# Shared-memory int32 atomic throughput (lane-ops per clock per SM, conflict-free): the
# ALU-side roofline of the histogram kernels (one red.shared per (cell or regrouped vertex,
# direction)).  Read from the committed output of tools/microbench/smem_ubench.cu on a B200
# (profiles/r02_smem_ubench.txt, line "ATOMS conflict-free ... lane-ops/clk/SM").
def smem_atoms_per_clk():
    p = os.path.join(ROOT, "profiles", "r02_smem_ubench.txt")
    try:
        for line in open(p):
            if line.startswith("ATOMS conflict-free"):
                return float(line.split("Gop/s")[1].split()[0]), "profiles/r02_smem_ubench.txt"
    except OSError:
        pass
    raise RuntimeError("profiles/r02_smem_ubench.txt (smem_ubench output) is missing: the alu roofline needs it")


def alu_peak(sm_mhz):
    """Peak shared-atomic updates per second: 148 SMs x measured lane-ops/clk x the max SM clock."""
    return 148 * smem_atoms_per_clk()[0] * sm_mhz * 1e6


def load_traffic(key):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if key in d:
            return d[key].get("dram_bytes_per_launch")
    return None


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML every ~5 ms while running."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples),
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]}


# --------------------------------------------------------------- workloads
def workload(cfg: str, rank: int):
    """Returns a dict describing the per-rank workload (host arrays)."""
    if cfg == "freud":
        # the cfg2 batch as Freudenthal triangulations
        wl = workload("1", rank)
        H, W = wl["img"].shape[1:]
        ncells = H * W + H * (W - 1) + W * (H - 1) + 3 * (H - 1) * (W - 1)
        D = wl["dirs"].shape[0]
        wl.update(kind="images", name="freudenthal_mnist60k", freudenthal=True, updates=wl["B"] * ncells * D,
                  atomics=wl["B"] * H * W * 6 * D,
                  desc=wl["desc"].replace("u8 images", "u8 images as Freudenthal complexes"))
        return wl
    if cfg in ("1", "0", "2"):
        c = int(cfg)
        spec = dict(synth.CONFIGS[c])
        B, dims = spec["B"], spec["dims"]
        seed = synth.S0 + c  # one batch for every rank: ranks take shards of it (strong scaling)
        img = synth.images_u8(B, dims, seed, "uniform" if c != 2 else "uniform")
        n = len(dims)
        dirs = synth.directions_s1(spec["D"]) if n == 2 else synth.directions_sphere(spec["D"], n, synth.S0 + 30)
        nv = int(np.prod(dims))
        ncells = int(np.prod([2 * d - 1 for d in dims]))
        out_dtype = "int32" if 255 * ncells < 2 ** 31 else "int64"
        osz = 4 if out_dtype == "int32" else 8
        return dict(kind="images", name=spec["name"], img=img, dirs=dirs, T=spec["T"], B=B, out_dtype=out_dtype,
                    units=B, updates=B * ncells * spec["D"], atomics=B * nv * spec["D"],
                    alg_bytes=B * nv + B * spec["D"] * spec["T"] * osz,
                    unit="complexes/s", desc=f"{B}x{'x'.join(map(str, dims))} u8 images, D={spec['D']}, T={spec['T']}, {out_dtype} out")
    if cfg in ("ecfimg", "ecfimg1k"):
        # image ECF (Remark "which-ecf" P:273-282; T = 256,
        # one bin per intensity): FMNIST-shaped 60k x 28x28, or 'padded ImageNet' 1000^2
        B, dims, kind, seed = (60000, (28, 28), "fmnist", synth.S0 + 60) if cfg == "ecfimg" else \
            (64, (1000, 1000), "uniform", synth.S0 + 61)
        img = synth.images_u8(B, dims, seed, kind)
        nv = int(np.prod(dims))
        ncells = int(np.prod([2 * d - 1 for d in dims]))
        T = 256
        return dict(kind="ecfimg", name=f"ecf_images_{B}x{'x'.join(map(str, dims))}_T{T}", img=img, T=T, B=B,
                    out_dtype="int32", units=B, updates=B * ncells, atomics=B * ncells,
                    alg_bytes=B * nv + B * T * 4, unit="complexes/s",
                    desc=f"image ECF: {B}x{'x'.join(map(str, dims))} u8 ({kind}), intensity filter, grid [0, 255], "
                         f"T={T}, int32 out")
    if cfg in ("bwd3", "bwd4"):
        # weights gradient through the WECT on the cfg4 / cfg5 complex
        c = 3 if cfg == "bwd3" else 4
        d = synth.make_config(c)
        cx, dirs, T = d["complex"], d["dirs"], d["T"]
        ncells = cx.num_cells()
        D = dirs.shape[0]
        G = synth.rng(synth.S0 + 70 + c).integers(-3, 4, size=(D, T)).astype(np.float64)
        idx_bytes = sum(c_.verts.nbytes for c_ in cx.cells)
        return dict(kind="grad", name=d["name"] + "_backward", cx=cx, dirs=dirs, T=T, G=G, units=1,
                    updates=ncells * D, atomics=ncells * D,
                    alg_bytes=cx.coords.nbytes + idx_bytes + G.nbytes + ncells * 8, unit="complexes/s",
                    desc=f"dL/dweights through the WECT of {cx.k0} V / {ncells} cells, n={cx.n}, D={D}, T={T}")
    if cfg in ("3", "4", "ecfx"):
        c = 3 if cfg in ("3", "ecfx") else 4
        d = synth.make_config(c)
        cx, dirs, T = d["complex"], d["dirs"], d["T"]
        ncells = cx.num_cells()
        idx_bytes = sum(c_.verts.nbytes for c_ in cx.cells)
        w_bytes = (cx.vweights.nbytes if cx.vweights is not None else 0) + sum(
            c_.weights.nbytes for c_ in cx.cells if c_.weights is not None)
        # one filter (ECF m = 1, or the WECT at D = 1): k_vbin1 bins the vertices once and the
        # dominant kernel k_stream reads the index lists, weights and the 2-byte vertex bins
        kbytes_1filter = idx_bytes + w_bytes + cx.k0 * 2 + T * 8
        if cfg == "ecfx":
            f = synth.rng(synth.S0 + 60).uniform(-1, 1, (cx.k0, 1)).astype(np.float32)
            return dict(kind="ecf", name="ecfx_torus10M_m1", cx=cx, fvals=f, T=T, units=1, updates=ncells,
                        alg_bytes=f.nbytes + idx_bytes + w_bytes + T * 8, kernel_bytes=kbytes_1filter,
                        unit="complexes/s",
                        desc=f"ECF of the cfg4 torus mesh ({cx.k0} V, {ncells} cells), m=1 filter, T={T}")
        D = dirs.shape[0]
        return dict(kind="complex", name=d["name"], cx=cx, dirs=dirs, T=T, units=1, updates=ncells * D,
                    kernel_bytes_1filter=kbytes_1filter,
                    atomics=ncells * D,
                    alg_bytes=cx.coords.nbytes + idx_bytes + w_bytes + D * T * 8, unit="complexes/s",
                    desc=f"explicit complex {cx.k0} V / {ncells} cells, n={cx.n}, D={D}, T={T}, "
                         f"{'f32' if cx.is_float else 'i32'} weights")
    raise ValueError(cfg)


# ------------------------------------------------------------- our arm (GPU)
def plan_shard(wl, world, rank):
    """How rank `rank` of `world` shares the workload:
    batch      -- image batches: contiguous image shards, no collective in the data path;
    directions -- one volume / mesh / gradient: contiguous direction rows, M from an
                  all_reduce(MAX) of per-shard maxima (reading A2), gradients all_reduce(SUM);
    replicas   -- one tiny image or one filter (nothing to split): every rank the same call."""
    from paper_2511_03909_b200.dist import shard_range

    if world == 1:
        return dict(mode="single", lo=0, hi=None, scaling="weak", parallelism="single GPU")
    if wl["kind"] in ("images", "ecfimg") and wl["B"] > 1:
        lo, hi = shard_range(wl["B"], world, rank)
        return dict(mode="batch", lo=lo, hi=hi, scaling="strong", parallelism=f"image-batch shards x{world}")
    if wl["kind"] in ("images", "complex", "grad"):
        lo, hi = shard_range(wl["dirs"].shape[0], world, rank)
        return dict(mode="directions", lo=lo, hi=hi, scaling="strong", parallelism=f"direction-row shards x{world}")
    return dict(mode="replicas", lo=0, hi=None, scaling="weak", parallelism=f"replicas x{world}")


def _allreduce(vals, op, dev):
    import torch
    import torch.distributed as dist

    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor(vals, dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=op)
    return [float(x) for x in t.cpu()]


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2511_03909_b200 as w
    from paper_2511_03909_b200 import dist as wdist

    dev = torch.device("cuda", local_rank % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    wl = workload(args.config, rank)
    if args.D and "dirs" in wl and wl["kind"] == "complex":
        wl["dirs"] = np.ascontiguousarray(wl["dirs"][: args.D])
        wl["updates"] = wl["updates"] // synth.CONFIGS[int(args.config)]["D"] * args.D
        wl["atomics"] = wl["updates"]
        wl["alg_bytes"] += (args.D - synth.CONFIGS[int(args.config)]["D"]) * wl["T"] * 8
        wl["name"] += f"_D{args.D}"
    stream = torch.cuda.current_stream(dev)
    sh = plan_shard(wl, world, rank)
    # this rank's share of the work (units, updates, bytes) for the roofline of its kernels
    if sh["mode"] == "batch":
        frac = (sh["hi"] - sh["lo"]) / wl["B"]
    elif sh["mode"] == "directions":
        frac = (sh["hi"] - sh["lo"]) / wl["dirs"].shape[0]
    else:
        frac = 1.0
    rows = None if sh["mode"] != "directions" else (sh["lo"], sh["hi"] - sh["lo"])
    gather = None  # (local output, total rows, dim) for the separately timed all_gather

    if wl["kind"] == "ecfimg":
        lo, hi = (sh["lo"], sh["hi"]) if sh["mode"] == "batch" else (0, wl["B"])
        img_d = torch.from_numpy(wl["img"][lo:hi]).to(dev)
        out_d = torch.empty((hi - lo, wl["T"]), dtype=torch.int32, device=dev)
        gather = (out_d, wl["B"], 0) if sh["mode"] == "batch" else None

        def step(flags=0):
            w.ecf_images(img_d, wl["T"], lo=0.0, hi=255.0, out=out_d, flags=flags)
    elif wl["kind"] == "images":
        lo, hi = (sh["lo"], sh["hi"]) if sh["mode"] == "batch" else (0, wl["B"])
        img_d = torch.from_numpy(wl["img"][lo:hi]).to(dev)
        dirs_d = torch.from_numpy(wl["dirs"]).to(dev)
        nrows = rows[1] if rows else wl["dirs"].shape[0]
        out_d = torch.empty((hi - lo, nrows, wl["T"]), dtype=getattr(torch, wl["out_dtype"]), device=dev)
        if sh["mode"] == "batch":
            gather = (out_d, wl["B"], 0)
        elif sh["mode"] == "directions":
            gather = (out_d, wl["dirs"].shape[0], 1)
        d0, dc = rows if rows else (0, 0)

        def step(flags=0):
            # direction shards pass the FULL direction set + their rows: the grid M is the
            # analytic max over the bounding-box corners and ALL directions (reading A2)
            w.wect_images(img_d, dirs_d, wl["T"], d_begin=d0, d_count=dc, out_dtype=wl["out_dtype"], out=out_d,
                          flags=flags, freudenthal=wl.get("freudenthal", False))
    else:
        cx = wl["cx"]
        cells = [(torch.from_numpy(c.verts).to(dev), None if c.weights is None else torch.from_numpy(c.weights).to(dev),
                  c.dim) for c in cx.cells]
        vw = None if cx.vweights is None else torch.from_numpy(cx.vweights).to(dev)
        if wl["kind"] == "grad":
            coords_d = torch.from_numpy(cx.coords).to(dev)
            dirs_d = torch.from_numpy(wl["dirs"]).to(dev)
            G_d = torch.from_numpy(wl["G"]).to(dev)
            out_d = G_d
            grad_group = None

            def step(flags=0):
                if sh["mode"] == "directions":
                    # partial gradients of this rank's rows, all_reduce(SUM) (the path's one exchange)
                    wdist.wect_complex_backward_sharded(coords_d, cells, dirs_d, wl["T"], G_d, flags=flags)
                else:
                    w.wect_complex_backward(coords_d, cells, dirs_d, wl["T"], G_d, flags=flags)
        elif wl["kind"] == "ecf":
            f_d = torch.from_numpy(wl["fvals"]).to(dev)
            out_d = torch.empty((1, wl["T"]), dtype=torch.float64 if cx.is_float else torch.int64, device=dev)

            def step(flags=0):
                w.ecf_complex(f_d, cells, wl["T"], vweights=vw, is_float=cx.is_float, out=out_d, flags=flags)
        else:
            coords_d = torch.from_numpy(cx.coords).to(dev)
            dirs_d = torch.from_numpy(wl["dirs"]).to(dev)
            nrows = rows[1] if rows else wl["dirs"].shape[0]
            out_d = torch.empty((nrows, wl["T"]), dtype=torch.float64 if cx.is_float else torch.int64, device=dev)
            if sh["mode"] == "directions":
                gather = (out_d, wl["dirs"].shape[0], 0)
            d0, dc = rows if rows else (0, 0)

            def step(flags=0):
                if sh["mode"] == "directions":
                    # M over ALL directions from per-shard maxima (reading A2): max is exact
                    M = wdist.global_maxheight(coords_d, dirs_d)
                    w.wect_complex(coords_d, cells, dirs_d, wl["T"], vweights=vw, is_float=cx.is_float, d_begin=d0,
                                   d_count=dc, maxheight=M, out=out_d, flags=flags)
                else:
                    w.wect_complex(coords_d, cells, dirs_d, wl["T"], vweights=vw, is_float=cx.is_float, out=out_d,
                                   flags=flags)

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20), dtype=torch.uint8, device=dev)

    for _ in range(args.warmup):
        flush.zero_()
        step(w.TIME_MAIN)
    torch.cuda.synchronize()
    w.sync_status()
    w.stats(reset=True)
    w.repair_count(reset=True)

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    sampler = ClockSampler(local_rank)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with sampler:
        for i in range(K):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
            step(w.TIME_MAIN)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    w.sync_status()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(step_ms))
    launches, tl, tms = w.stats(reset=True)  # launches inside the timed region only
    repairs = w.repair_count(reset=True)
    # warm-L2 variant (after the timed region) (no flush between steps), a few steps, reported beside the cold number
    kw = min(K, 10)
    evw = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(kw)]
    torch.cuda.synchronize()
    for i in range(kw):
        evw[i][0].record(stream)
        step(0)
        evw[i][1].record(stream)
    torch.cuda.synchronize()
    warm_ms = statistics.median([a.elapsed_time(b) for a, b in evw])

    main_ms = tms / max(tl, 1)
    if world > 1:
        total_ms, main_ms = _allreduce([total_ms, main_ms], torch.distributed.ReduceOp.MAX, dev)
    # the all_gather that would assemble the full output on every rank (NCCL), timed apart
    gather_ms = None
    if world > 1 and gather is not None:
        local, n_total, gdim = gather
        wdist.gather_rows(local, n_total, gdim)  # warm-up (communicator buffers)
        torch.cuda.synchronize()
        torch.distributed.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        full = wdist.gather_rows(local, n_total, gdim)
        g1.record(stream)
        torch.cuda.synchronize()
        gather_ms = _allreduce([g0.elapsed_time(g1)], torch.distributed.ReduceOp.MAX, dev)[0]
        del full

    ms_per_step = total_ms / K
    # strong scaling: the shards add up to ONE workload; replicas: every rank does a whole one
    mult = 1 if sh["scaling"] == "strong" else world
    value = mult * wl["units"] * K / (total_ms / 1e3)
    peak, peak_src = load_peaks()
    per_call_launches = tl / max(K, 1)  # timed (dominant-kernel) launches per step
    D = wl["dirs"].shape[0] if "dirs" in wl else 1
    if wl["kind"] == "ecfimg":
        kname, bound = ("k_ecf_img2d_w4", "hbm") if args.config == "ecfimg" else ("k_ecf_img2d_rows", "alu")
    elif wl["kind"] == "images" and (args.config in ("0", "1") or wl.get("freudenthal")):
        # WECT_IMAGES_MMA=1: the opt-in tensor-core contraction (k_mma.cu) instead of the sweep
        mma = os.environ.get("WECT_IMAGES_MMA") == "1" and not wl.get("freudenthal")
        kname, bound = ("k_mma2d" if mma else "k_sweep2d"), "hbm"
    elif wl["kind"] == "images":
        kname, bound = "k_grid_hist", "alu"
    elif wl["kind"] == "grad":
        kname, bound = "k_grad_cells", "alu"
    elif wl["kind"] == "ecf" or D <= 24:
        kname, bound = "k_stream", "hbm"
    else:
        kname, bound = "k_cells_vb", "alu"
    kbytes = wl["alg_bytes"]
    if "kernel_bytes" in wl:
        kbytes = wl["kernel_bytes"]
    elif wl["kind"] == "complex" and wl["dirs"].shape[0] == 1:
        kbytes = wl["kernel_bytes_1filter"]
    if bound == "hbm":
        achieved = frac * kbytes / per_call_launches / (main_ms / 1e3) / 1e9
        roof = {"kernel": kname, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_src,
                "alg_bytes_per_launch": frac * kbytes / per_call_launches}
    else:
        # algorithmic work = shared-memory histogram updates: (cell, direction) pairs for
        # explicit complexes, regrouped (vertex, direction) pairs for voxel grids
        work = frac * wl["atomics"] / per_call_launches
        apeak = alu_peak(float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0))
                         if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1965.0)
        achieved = work / (main_ms / 1e3) / 1e9
        roof = {"kernel": kname, "bound": "alu", "achieved": achieved, "peak": apeak / 1e9, "unit": "Gupdates/s",
                "frac": achieved * 1e9 / apeak,
                "peak_source": f"148 SMs x {smem_atoms_per_clk()[0]:.2f} shared int32 atomic lane-ops/clk "
                               f"(measured: {smem_atoms_per_clk()[1]}) x sm_max_mhz",
                "work_per_launch": work,
                "hbm_achieved_gbs": frac * wl["alg_bytes"] / per_call_launches / (main_ms / 1e3) / 1e9}
    traffic = load_traffic(f"cfg{args.config}" + (f"_D{args.D}" if args.D else ""))
    res = {
        "metric": METRIC,
        "value": value,
        "unit": wl["unit"],
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": sh["scaling"],
        "vs_baseline": None,
        "dtype": "int32" if wl.get("out_dtype") == "int32" else ("f64" if wl["kind"] == "grad" or ("cx" in wl and wl["cx"].is_float) else "int64"),
        "data": "synthetic (seeded; DESIGN.md input recipe)",
        "config": {"workload": wl["name"], "desc": wl["desc"],
                   "per_gpu_units": wl["units"] * frac if sh["scaling"] == "strong" else wl["units"],
                   "shard": {"mode": sh["mode"], "lo": sh["lo"], "hi": sh["hi"]},
                   "l2": f"flushed between timed steps ({flush.numel() >> 20} MiB write, untimed)",
                   "parallelism": sh["parallelism"]},
        "gather_ms": gather_ms,
        "step_ms_p50": float(np.percentile(step_ms, 50)),
        "step_ms_p99": float(np.percentile(step_ms, 99)),
        "warm_l2_ms_per_step": warm_ms,
        "updates_per_s": mult * wl["updates"] * K / (total_ms / 1e3),
        "hbm_gbs": mult * wl["alg_bytes"] * K / (total_ms / 1e3) / 1e9,
        "roofline": dict(roof, traffic=traffic, kernel_ms=main_ms, launches_per_step=per_call_launches,
                         kernel_share_of_step=main_ms * per_call_launches / ms_per_step),
        "gpu_launches": int(launches),
        "repairs_binary64": int(repairs),
        "clocks": sampler.summary(),
    }
    # end to end through the public API with HOST buffers (H2D + compute + D2H every step),
    # each rank on its own shard, max over ranks
    if not args.no_e2e:
        pin = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        d0, dc = rows if rows else (0, 0)
        if wl["kind"] in ("ecfimg", "images"):
            lo, hi = (sh["lo"], sh["hi"]) if sh["mode"] == "batch" else (0, wl["B"])
            img_h = pin(wl["img"][lo:hi])
            out_h = torch.empty(tuple(out_d.shape), dtype=out_d.dtype).pin_memory()
            if wl["kind"] == "ecfimg":
                h2d = img_h.numel()
                path = "ecf_images(host pinned in, host pinned out): library stages H2D, D2H, syncs"

                def e2e_step():
                    return w.ecf_images(img_h, wl["T"], lo=0.0, hi=255.0, out=out_h)
            else:
                dirs_h = torch.from_numpy(wl["dirs"])
                h2d = img_h.numel() + dirs_h.numel() * 4
                path = "wect_images(host pinned in, host pinned out): library stages H2D, D2H, syncs"

                def e2e_step():
                    return w.wect_images(img_h, dirs_h, wl["T"], d_begin=d0, d_count=dc, out_dtype=wl["out_dtype"],
                                         out=out_h, freudenthal=wl.get("freudenthal", False))
            ke = max(1, min(5, K))
        elif wl["kind"] == "grad":
            cx = wl["cx"]
            cells_h = [(pin(c.verts), None, c.dim) for c in cx.cells]
            coords_h, dirs_h, G_h = pin(cx.coords), pin(wl["dirs"]), pin(wl["G"][d0:d0 + dc] if rows else wl["G"])
            h2d = cx.coords.nbytes + sum(c.verts.nbytes for c in cx.cells) + G_h.numel() * 8
            path = "wect_complex_backward(host pinned in, host out) per rank's rows"

            def e2e_step():
                gv, gc = w.wect_complex_backward(coords_h, cells_h, dirs_h, wl["T"], G_h, d_begin=d0, d_count=dc)
                return torch.cat([gv] + list(gc))
            ke = 2
        else:
            cx = wl["cx"]
            cells_h = [(pin(c.verts), pin(c.weights), c.dim) for c in cx.cells]
            vw_h, coords_h = pin(cx.vweights), pin(cx.coords)
            src_h = pin(wl["fvals"]) if wl["kind"] == "ecf" else pin(wl["dirs"])
            out_h = torch.empty(tuple(out_d.shape), dtype=out_d.dtype).pin_memory()
            h2d = (cx.coords.nbytes if wl["kind"] != "ecf" else wl["fvals"].nbytes) + sum(
                c.verts.nbytes + (c.weights.nbytes if c.weights is not None else 0) for c in cx.cells) + (
                cx.vweights.nbytes if cx.vweights is not None else 0)
            path = "wect_complex / ecf_complex(host pinned in, host pinned out) per rank's rows"

            def e2e_step():
                if wl["kind"] == "ecf":
                    return w.ecf_complex(src_h, cells_h, wl["T"], vweights=vw_h, is_float=cx.is_float, out=out_h)
                M = wdist.global_maxheight(coords_h, src_h) if rows else 0.0
                return w.wect_complex(coords_h, cells_h, src_h, wl["T"], vweights=vw_h, is_float=cx.is_float,
                                      d_begin=d0, d_count=dc, maxheight=M, out=out_h)
            ke = 2
        o = e2e_step()  # warm-up (pool, modules)
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            o = e2e_step()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            e2e_s = _allreduce([e2e_s], torch.distributed.ReduceOp.MAX, dev)[0]
        res["e2e"] = {"value": mult * wl["units"] * ke / e2e_s, "unit": wl["unit"], "h2d_bytes_per_step": int(h2d),
                      "d2h_bytes_per_step": int(o.numel() * o.element_size()), "steps": ke, "path": path}
    # the CPU oracle beside it (rank 0, N = 1 only)
    if rank == 0 and world == 1 and not args.no_cpu:
        res["cpu_baseline"] = cpu_baseline(wl, budget_s=args.cpu_budget)
    return res


# ---------------------------------------------------------- the CPU oracle
def cpu_model():
    """The host CPU's model name (lscpu / /proc/cpuinfo) for the cpu_baseline record."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(wl, budget_s=15.0, max_units=None):
    """Time O2 (oracle/, binary64, OpenMP over directions) on a bounded sample."""
    res = _cpu_baseline(wl, budget_s, max_units)
    res["cpu_model"] = cpu_model()
    return res


def _cpu_baseline(wl, budget_s=15.0, max_units=None):
    import oracle

    cores = oracle.num_threads()
    if wl["kind"] == "ecfimg":
        chunk = 200 if wl["img"].shape[1:] == (28, 28) else 1
        done, t = 0, 0.0
        limit = wl["B"] if max_units is None else min(max_units, wl["B"])
        while done < limit and t < budget_s:
            n = min(chunk, limit - done)
            t0 = time.perf_counter()
            oracle.ecf_images(wl["img"][done:done + n], wl["T"], 0.0, 255.0)
            t += time.perf_counter() - t0
            done += n
        return {"value": done / t, "unit": wl["unit"], "cores": cores, "kind": "oracle",
                "sample": f"O2 (per image, explicit complex) on images [0, {done}) of the {wl['B']}-image workload "
                          f"({t:.1f} s)"}
    if wl["kind"] == "images" and wl["B"] == 1 and wl["img"][0].size > 1 << 20:
        # one large volume: O2 on 8 sampled directions with the full set's M, scaled to D
        dims = wl["img"].shape[1:]
        coords = oracle.grid_coords(dims)
        corners = np.array([[c0, c1, c2] for c0 in (coords[:, 0].min(), coords[:, 0].max())
                            for c1 in (coords[:, 1].min(), coords[:, 1].max())
                            for c2 in (coords[:, 2].min(), coords[:, 2].max())], np.float32)
        M = float(np.abs(oracle.heights(corners, wl["dirs"])).max())
        nd, D = 8, wl["dirs"].shape[0]
        t0 = time.perf_counter()
        oracle.wect_images(wl["img"], wl["dirs"][:nd], wl["T"], maxheight_override=M)
        t = time.perf_counter() - t0
        return {"value": 1.0 / (t * D / nd), "unit": wl["unit"], "cores": cores, "kind": "oracle",
                "sample": f"O2 on {nd} of {D} directions of the volume ({t:.1f} s), scaled by D/{nd}"}
    if wl.get("freudenthal"):
        done, t = 0, 0.0
        while done < wl["B"] and t < budget_s:
            t0 = time.perf_counter()
            oracle.wect_images_freudenthal(wl["img"][done:done + 50], wl["dirs"], wl["T"])
            t += time.perf_counter() - t0
            done += 50
        return {"value": done / t, "unit": wl["unit"], "cores": cores, "kind": "oracle",
                "sample": f"O2 on the explicit Freudenthal complexes of images [0, {done}) ({t:.1f} s)"}
    if wl["kind"] == "images" and wl["img"].shape[1:] == (28, 28):
        # all host cores, then one core (the paper's single-core comparison)
        res = _cpu_baseline(dict(wl, kind="images_batch"), budget_s, max_units)
        oracle.set_num_threads(1)
        try:
            one = _cpu_baseline(dict(wl, kind="images_batch"), min(5.0, budget_s), 200)
        finally:
            oracle.set_num_threads(cores)
        res["value_1core"] = one["value"]
        res["sample_1core"] = one["sample"]
        return res
    if wl["kind"] in ("images", "images_batch"):
        chunk = 500 if wl["img"].shape[1:] == (28, 28) else 1
        if max_units is not None:
            chunk = min(chunk, max_units)
        done, t = 0, 0.0
        limit = wl["B"] if max_units is None else min(max_units, wl["B"])
        while done < limit and t < budget_s:
            n = min(chunk, limit - done)
            t0 = time.perf_counter()
            oracle.wect_images(wl["img"][done:done + n], wl["dirs"], wl["T"])
            t += time.perf_counter() - t0
            done += n
        return {"value": done / t, "unit": wl["unit"], "cores": cores, "kind": "oracle",
                "sample": f"O2 on images [0, {done}) of the {wl['B']}-image workload ({t:.1f} s)"}
    # explicit complexes: a subset of directions, scaled to complexes/s
    import oracle as orc

    cx = wl["cx"]
    if wl["kind"] == "grad":
        # the closed-form oracle gradient on a bounded sample: 2 directions, full complex
        import synth as sy

        nd, per_dim = 2, 4000
        sub = sy.Complex(cx.coords, cx.vweights, [sy.Cells(c.verts[:per_dim], None, c.dim) for c in cx.cells],
                         cx.k0, is_float=False)
        sampled = cx.k0 + sum(min(per_dim, len(c.verts)) for c in cx.cells)
        t0 = time.perf_counter()
        fv = orc.heights(cx.coords, wl["dirs"][:nd])
        M = orc.maxheight(fv)
        orc.wecfs_grad(fv, sub, wl["T"], -M, M, wl["G"][:nd])
        t = time.perf_counter() - t0
        D = wl["dirs"].shape[0]
        scale = (D / nd) * (cx.num_cells() / sampled)
        return {"value": 1.0 / (t * scale), "unit": wl["unit"], "cores": 1, "kind": "oracle",
                "sample": f"closed-form gradient oracle on {nd} of {D} directions, all vertices + the first "
                          f"{per_dim} cells of each dimension ({t:.1f} s), scaled by D/{nd} x cells/sampled"}
    if wl["kind"] == "ecf":
        t0 = time.perf_counter()
        orc.ecf_complex(cx, wl["fvals"], wl["T"])
        t = time.perf_counter() - t0
        return {"value": 1.0 / t, "unit": wl["unit"], "cores": cores, "kind": "oracle",
                "sample": f"O2 ECF on the full mesh ({t:.1f} s)"}
    D = wl["dirs"].shape[0]
    fv_time = 0.0
    nd = 8
    t0 = time.perf_counter()
    orc.wect_complex(cx, wl["dirs"][:nd], wl["T"])
    t = time.perf_counter() - t0
    return {"value": 1.0 / (t * D / nd), "unit": wl["unit"], "cores": cores, "kind": "oracle",
            "sample": f"O2 on {nd} of {D} directions ({t:.1f} s), scaled by D/{nd}"}


def run_reference(args):
    """--impl reference: the oracle as it stands, on the host cores, same metric/config."""
    wl = workload(args.config, 0)
    import oracle

    big_volume = wl["kind"] == "images" and wl["B"] == 1 and wl["img"][0].size > 1 << 20
    if wl["kind"] == "images" and not big_volume:
        per_step = min(50 if wl.get("freudenthal") else 2000, wl["B"])
    elif wl["kind"] == "ecfimg":
        per_step = min(400 if wl["B"] > 64 else 1, wl["B"])
    else:
        per_step = None  # one large complex: the bounded cpu_baseline sample, scaled
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = None
        if per_step is not None and wl["kind"] == "images":
            if wl.get("freudenthal"):
                oracle.wect_images_freudenthal(wl["img"][:per_step], wl["dirs"], wl["T"])
            else:
                oracle.wect_images(wl["img"][:per_step], wl["dirs"], wl["T"])
        elif per_step is not None:
            oracle.ecf_images(wl["img"][:per_step], wl["T"], 0.0, 255.0)
        else:
            r = cpu_baseline(wl)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append((dt, per_step, r))
    if per_step is not None:
        tot = sum(t for t, _, _ in times)
        value = per_step * len(times) / tot
        sample = f"O2 on images [0, {per_step}) of the {wl['B']}-image workload per step"
    else:
        value = statistics.median([r["value"] for _, _, r in times])
        sample = times[0][2]["sample"]
    cores = oracle.num_threads()
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": wl["unit"], "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(t for t, _, _ in times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 bins / int64 sums", "data": "synthetic",
            "config": {"workload": wl["name"], "desc": wl["desc"]},
            "cpu_baseline": {"value": value, "unit": wl["unit"], "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": wl["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def relaunch(n):
    """`bench.py --gpus N` without a launcher: run N ranks under torch.distributed.run on this
    node (127.0.0.1); rank 0 prints the JSON line.  Returns the launcher's exit code."""
    import socket
    import subprocess

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="1", help="BASELINE configs index (0-4), ecfx, ecfimg, ecfimg1k, bwd3, bwd4 or freud")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--D", type=int, default=0, help="override the direction count (D-sweep of configs 3/4)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    if world > 1:
        import torch

        dev = torch.device("cuda", local_rank % max(1, torch.cuda.device_count()))
        torch.cuda.set_device(dev)
        if torch.cuda.device_count() >= world:
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init log (NVLS / P2P / rings) to stderr
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.distributed.init_process_group("nccl", device_id=dev)
        else:  # more ranks than GPUs (a logic check on a small box): gloo for the host-side collectives
            print(f"bench: {world} ranks on {torch.cuda.device_count()} GPU(s): gloo, ranks share devices",
                  file=sys.stderr)
            torch.distributed.init_process_group("gloo")
    res = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
