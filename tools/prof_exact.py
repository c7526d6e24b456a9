#!/usr/bin/env python
"""Profiling driver for the exact-local-solver kernel (ncu -k exact_patch): one AVS step with A_v^{-1} on a
2D / 3D level.   python tools/prof_exact.py --dim 2 --degree 4 --level 8"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_05082_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=2)
ap.add_argument("--degree", type=int, default=4)
ap.add_argument("--level", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
ctx = api.Context(a.dim, a.degree, a.level)
ctx.set_local_solver(True)
n = ctx.n_dofs(a.level)
g = torch.Generator(device="cpu").manual_seed(20241205)
x = (torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1).cuda()
b = (torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1).cuda()
om = 0.25 if a.dim == 2 else 0.1
ctx.smooth(a.level, "avs_atomic", 1, om, b, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    ctx.smooth(a.level, "avs_atomic", 1, om, b, x)
e1.record()
torch.cuda.synchronize()
print(f"exact AVS step {a.dim}D k={a.degree} L={a.level}: {n} DoFs, {e0.elapsed_time(e1) / a.reps:.3f} ms "
      f"({n / (e0.elapsed_time(e1) / a.reps * 1e-3) / 1e9:.3f} GDoF/s)")
