#!/usr/bin/env python
"""Diagnostic: FP32 vs FP64 V-cycle output (relative difference and the residual b - A z it leaves) and
GMRES convergence with each cycle, on a few nested levels (DESIGN.md §8 mixed precision).
usage: python tools/vc_check.py"""
import torch, sys
sys.path.insert(0, '.')
from paper_2412_05082_b200 import api
for (d, k, L, om) in [(3, 3, 7, 0.7), (3, 2, 6, 0.7), (2, 4, 8, 1.0)]:
    ctx = api.Context(d, k, L)
    b = ctx.rhs(L)
    for sym in (True, False):
        z64 = ctx.vcycle(api.MG("mvs", 1, om, symmetric=sym, cycle_dtype=torch.float64), b)
        z32 = ctx.vcycle(api.MG("mvs", 1, om, symmetric=sym, cycle_dtype=torch.float32), b)
        rel = (z64 - z32).norm() / z64.norm()
        # residual reduction of one preconditioned step: ||b - A z|| / ||b||
        r64 = ctx.residual(L, b, z64).norm() / b.norm()
        r32 = ctx.residual(L, b, z32).norm() / b.norm()
        print(d, k, L, "sym" if sym else "same", f"rel(z32,z64)={rel:.3e}  ||b-Az||/||b||: fp64 {r64:.3e} fp32 {r32:.3e}")
    x, rep, h = ctx.gmres(api.MG("mvs", 1, om, symmetric=False, cycle_dtype=torch.float32), b, max_iter=20, restart=20)
    print("gmres fp32", rep["iterations"], rep["converged"], h[:6])
    x, rep, h = ctx.gmres(api.MG("mvs", 1, om, symmetric=False, cycle_dtype=torch.float64), b, max_iter=20, restart=20)
    print("gmres fp64", rep["iterations"], rep["converged"], h[:6])
    ctx.close()
