"""Timing experiment: the cfg2 image batch with int32 vs int64 output (same sweep work, 2x the
output bytes): is k_sweep2d output-bound?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2511_03909_b200 as w
c = synth.make_config(1)
img = torch.from_numpy(c["img"]).cuda(); dirs = torch.from_numpy(c["dirs"]).cuda()
for dt in ("int32", "int64", "int32", "int64"):
    out = torch.empty((img.shape[0], dirs.shape[0], c["T"]), dtype=getattr(torch, dt), device="cuda")
    for _ in range(3):
        w.wect_images(img, dirs, c["T"], out_dtype=dt, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        w.wect_images(img, dirs, c["T"], out_dtype=dt, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(dt, "ms/call %.4f" % ms, "GB/s %.0f" % (out.numel() * out.element_size() / ms / 1e6))
