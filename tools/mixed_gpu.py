"""FP64 vs FP32 V-cycle inside the FP64 outer Krylov solver on the GPU, as the level grows (
DESIGN.md §8).  Paper protocol: AVS-2 + CG (omega 1/4 | 0.1), MVS-1 + GMRES same-order cycle (omega 0.8 | 0.7),
F = c0ip_rhs (paper load + boundary data), rtol 1e-8.
  python tools/mixed_gpu.py --dim 2 --degree 4 --levels 5,6,7,8,9,10,11"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2412_05082_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--degree", type=int, default=4)
    ap.add_argument("--levels", default="5,6,7")
    ap.add_argument("--smoothers", default="avs,mvs")
    a = ap.parse_args()
    d, k = a.dim, a.degree
    for L in map(int, a.levels.split(",")):
        ctx = api.Context(d, k, L)
        b = ctx.rhs(L)
        row = {"dim": d, "degree": k, "level": L, "dofs": ctx.n_dofs(L)}
        for sm in a.smoothers.split(","):
            for name, cdt in (("fp64", torch.float64), ("fp32", torch.float32)):
                if sm == "avs":
                    mg = api.MG("avs", 2, 0.25 if d == 2 else 0.1, cycle_dtype=cdt)
                    ctx.pcg(mg, b, max_iter=2)
                    torch.cuda.synchronize()
                    _, rep, hist = ctx.pcg(mg, b, max_iter=80)
                else:
                    mg = api.MG("mvs", 1, 0.8 if d == 2 else 0.7, symmetric=False, cycle_dtype=cdt)
                    ctx.gmres(mg, b, max_iter=2, restart=30)
                    torch.cuda.synchronize()
                    _, rep, hist = ctx.gmres(mg, b, max_iter=60, restart=30)
                row[f"{sm}_{name}"] = {"it": rep["iterations"], "nu": round(rep["nu"], 2), "conv": rep["converged"],
                                       "s": round(rep["seconds"], 4)}
        print(json.dumps(row), flush=True)
        ctx.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
