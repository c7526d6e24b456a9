#!/usr/bin/env python
"""Profiling driver: a few smoothing steps / matvecs on one large level (for ncu -k <kernel>).

usage: python tools/prof_step.py --dim 2 --degree 4 [--sm avs|mvs] [--dtype f64|f32] [--reps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from c0ip_inputs import CFG2_CELLS, CFG4_CELLS, random_xb  # noqa: E402
from paper_2412_05082_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=2)
ap.add_argument("--degree", type=int, default=4)
ap.add_argument("--sm", default="avs")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cells", type=int, default=0)
a = ap.parse_args()
k, d = a.degree, a.dim
N = a.cells or (CFG2_CELLS[k] if d == 2 else CFG4_CELLS[k])
dt = torch.float64 if a.dtype == "f64" else torch.float32
ctx = api.Context(d, k, 3, cells_override=N)
x0, b0 = random_xb(k, d, N)
x = torch.tensor(x0, device="cuda", dtype=dt)
b = torch.tensor(b0, device="cuda", dtype=dt)
om = (0.25 if d == 2 else 0.1) if a.sm.startswith("avs") else (1.0 if d == 2 else 0.7)
for _ in range(a.reps):
    if a.sm == "apply":
        ctx.apply(3, x, b)
    else:
        ctx.smooth(3, a.sm, 1, om, b, x)
torch.cuda.synchronize()
print("done", N, ctx.n_dofs(3))
