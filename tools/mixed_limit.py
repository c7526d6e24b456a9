"""Oracle evidence for the size limit of the FP32 V-cycle: nu of the
paper protocol with the FP64 and the FP32 cycle (every table rounded, reading Q21) as the level grows.
Test infrastructure: calls oracle/ only.   python tools/mixed_limit.py --dim 2 --degree 4 --levels 4,5,6,7"""
import argparse
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def job(a):
    from oracle.multigrid import solve_paper
    d, k, L, kind, steps, dt = a
    n, nu, h = solve_paper(d, k, L, kind, steps, cycle_dtype=dt)
    A = h.A[L]
    import scipy.sparse.linalg as spla
    lmax = spla.eigsh(A, 1, which="LA", return_eigenvectors=False)[0]
    lmin = spla.eigsh(A, 1, sigma=0, which="LM", return_eigenvectors=False)[0]
    return a, n, nu, lmax / lmin


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--degree", type=int, default=4)
    ap.add_argument("--levels", default="4,5,6")
    ap.add_argument("--jobs", type=int, default=8)
    a = ap.parse_args()
    jobs = [(a.dim, a.degree, int(L), kind, steps, dt) for L in a.levels.split(",")
            for kind, steps in (("avs", 2), ("mvs", 1)) for dt in (np.float64, np.float32)]
    with ProcessPoolExecutor(a.jobs) as ex:
        for (d, k, L, kind, steps, dt), n, nu, kap in ex.map(job, jobs):
            print(f"{d}D k={k} L={L} {kind}-{steps} {np.dtype(dt).name}: n={n} nu={nu:.2f} "
                  f"kappa(A)={kap:.2e} u32*kappa={kap * 2 ** -24:.2e}", flush=True)


if __name__ == "__main__":
    main()
