"""Oracle fractional iteration counts nu for PAPER.md Tables 1-3 (test infrastructure: calls oracle/ only).

  python tools/paper_tables.py --dim 2 --table 2 --levels 6,7 --degrees 2,3,4 [--jobs 8]

Protocol (readings Q8b, Q11, Q27, Q28 in DESIGN.md §2): x0 = 0,
F = paper_rhs (f = Delta^2 u* plus the Nitsche boundary data of u* = prod sin(pi x_a)), rtol 1e-8 on
||r_n||/||r_0||, nu = -8/log10(rbar).  AVS: CG, symmetric cycle, omega 1/4 (2D) / 0.1 (3D), `steps`
pre- and post-smoothing steps.  MVS: GMRES (FGMRES(50)), same-order cycle, omega 1 (exact) / 0.8 (2D
inexact) / 0.7 (3D).  Exact local solvers (Table 1): A_v = R_v A R_v^T.
"""
import argparse
import itertools
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PAPER = {  # (dim, table, smoother, steps) -> {(L, k): nu}
    (2, 1, "avs", 2): {(6, 4): 10.3, (6, 5): 10.1, (6, 6): 10.4, (6, 7): 10.9, (7, 2): 21.9, (7, 3): 11.7,
                       (7, 4): 9.9, (7, 5): 9.5, (7, 6): 10.2, (7, 7): 10.9, (8, 2): 22.8, (8, 3): 11.7},
    (2, 1, "mvs", 1): {(6, 4): 2.9, (6, 5): 2.6, (6, 6): 2.5, (6, 7): 2.3, (7, 2): 8.8, (7, 3): 4.4,
                       (7, 4): 2.9, (8, 2): 8.9, (8, 3): 4.4},
    (2, 2, "avs", 2): {(6, 4): 9.2, (6, 5): 9.9, (6, 6): 10.3, (6, 7): 10.8, (7, 2): 19.2, (7, 3): 10.4,
                       (7, 4): 9.0, (7, 5): 9.3, (8, 2): 19.6, (8, 3): 10.3},
    (2, 2, "mvs", 1): {(6, 4): 4.2, (6, 5): 4.5, (6, 6): 5.2, (6, 7): 5.8, (7, 2): 9.2, (7, 3): 4.8,
                       (7, 4): 4.2, (8, 2): 9.4, (8, 3): 4.8},
    (3, 3, "avs", 1): {(4, 4): 20.6, (4, 5): 20.5, (5, 2): 29.8, (5, 3): 23.6, (5, 4): 22.3},
    (3, 3, "avs", 2): {(4, 4): 14.0, (4, 5): 14.1, (5, 2): 17.9, (5, 3): 16.1, (5, 4): 15.1},
    (3, 3, "mvs", 1): {(4, 4): 5.4, (4, 5): 5.9, (5, 2): 9.1, (5, 3): 4.9, (5, 4): 4.6},
    (3, 3, "mvs", 2): {(4, 4): 3.2, (4, 5): 3.6, (5, 2): 7.2, (5, 3): 4.0, (5, 4): 3.3},
}


def solve_nu(d, k, L, kind, steps, exact=False, omega=None):
    from oracle.multigrid import solve_paper
    n, nu, _ = solve_paper(d, k, L, kind, steps, exact, omega)
    return n, nu


def _job(a):
    t = time.time()
    n, nu = solve_nu(*a)
    return a, n, nu, time.time() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--table", type=int, default=2)
    ap.add_argument("--smoothers", default="avs:2,mvs:1")
    ap.add_argument("--levels", default="6")
    ap.add_argument("--degrees", default="2,3,4")
    ap.add_argument("--jobs", type=int, default=4)
    a = ap.parse_args()
    exact = a.table == 1
    jobs = []
    for sm, L, k in itertools.product(a.smoothers.split(","), a.levels.split(","), a.degrees.split(",")):
        kind, steps = sm.split(":")
        jobs.append((a.dim, int(k), int(L), kind, int(steps), exact))
    with ProcessPoolExecutor(a.jobs) as ex:
        for (d, k, L, kind, steps, ex_), n, nu, sec in ex.map(_job, jobs):
            ref = PAPER.get((d, a.table, kind, steps), {}).get((L, k))
            print(f"{d}D table{a.table} {kind}-{steps} k={k} L={L}: n={n} nu={nu:.2f} paper={ref} ({sec:.0f}s)",
                  flush=True)


if __name__ == "__main__":
    main()
