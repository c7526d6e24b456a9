#!/usr/bin/env python
"""compute-sanitizer driver: every kernel family of libc0ip.so once, at small sizes that still reach
the fused tile kernels (2D N >= 8, 3D N >= 8) and their boundary branches.

usage (on a GPU box):
  compute-sanitizer --tool memcheck  --error-exitcode 1 python tools/sanitize.py
  compute-sanitizer --tool racecheck --error-exitcode 1 python tools/sanitize.py --quick
  compute-sanitizer --tool synccheck --error-exitcode 1 python tools/sanitize.py --quick
  compute-sanitizer --tool initcheck --error-exitcode 1 python tools/sanitize.py --quick
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_05082_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true", help="one degree per dimension (racecheck is slow)")
a = ap.parse_args()

dev = torch.device("cuda", 0)
rng = np.random.default_rng(7)


def rand(n, dt):
    return torch.tensor(rng.uniform(-1, 1, n), device=dev, dtype=dt)


def smoothers(ctx, lv, d):
    for dt in (torch.float64, torch.float32):
        n = ctx.n_dofs(lv)
        x, b = rand(n, dt), rand(n, dt)
        ctx.apply(lv, x)
        ctx.residual(lv, b, x)
        om = 0.25 if d == 2 else 0.1
        for sm in ("avs_atomic", "avs_det", "avs_colored"):
            ctx.smooth(lv, sm, 1, om, b, x.clone())
        for rev in (False, True):
            ctx.smooth(lv, "mvs", 1, 0.8, b, x.clone(), reverse=rev)
        if lv >= 2:
            c = ctx.restrict(lv, x)
            ctx.prolongate_add(lv, c, x)


degs2 = (4,) if a.quick else (2, 3, 4, 5, 6, 7)
degs3 = (3,) if a.quick else (2, 3, 4, 5)
for k in degs2:
    ctx = api.Context(2, k, 3, cells_override=12)    # fused tile kernels, boundary + interior tiles
    smoothers(ctx, 3, 2)
    ctx.close()
    print("2D k", k, "ok", flush=True)
for k in degs3:
    ctx = api.Context(3, k, 3, cells_override=10)
    smoothers(ctx, 3, 3)
    ctx.close()
    print("3D k", k, "ok", flush=True)

# solvers: V-cycle graph, PCG, GMRES, FP32 cycle, exact local solvers
ctx = api.Context(2, 4, 4)
b = ctx.rhs(4)
for sm, om, sym in (("avs", 0.25, True), ("mvs", 0.8, True)):
    for cdt in (torch.float64, torch.float32):
        ctx.pcg(api.MG(sm, 2 if sm == "avs" else 1, om, sym, cdt), b, max_iter=30)
ctx.gmres(api.MG("mvs", 1, 0.8, False), b, max_iter=30, restart=10)
ctx.set_local_solver(True)
ctx.pcg(api.MG("avs", 2, 0.25, True), b, max_iter=30)
ctx.smooth(4, "mvs", 1, 1.0, b, torch.zeros_like(b))
ctx.close()
print("solvers ok", flush=True)

# graded mesh (generic per-axis kernels) and the Poisson SIPG workload
t = np.linspace(0, 1, 9)
nodes = [t + 0.5 * t * (1 - t), t - 0.4 * t * (1 - t)]
ctx = api.Context(2, 3, 3, nodes=nodes)
b = ctx.rhs(3)
ctx.pcg(api.MG("avs", 2, 0.25, True), b, max_iter=20)
ctx.close()
ctx = api.Context(2, 3, 4, sipg=True)
b = ctx.rhs(4)
ctx.pcg(api.MG("avs", 2, 0.25, True), b, max_iter=20)
ctx.close()
torch.cuda.synchronize()
print("sanitize run complete", flush=True)
