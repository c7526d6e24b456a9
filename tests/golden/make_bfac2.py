"""Writes k2_N2_sigma6_bfac2_1d.txt: exact 1D M, L, B for k=2, N=2 (h=1/2), sigma=6, boundary-facet
penalty 2 sigma/h (reading Q27), boundary nodes eliminated.  Sympy only (no oracle/):
Lagrange basis on the Gauss-Lobatto nodes 0, 1/2, 1; cell integrals PAPER.md:323-332 (Eq. matrix1d);
face terms (sigma_f/h)[phi'][phi'] - {phi''}[phi'] - [phi']{phi''} (Eqs. ev/eh)
with the jump/mean of PAPER.md:87-106 (one-sided on the two boundary facets)."""
import os
import sympy as sy

t = sy.symbols("t")
k, N, sigma, bfac = 2, 2, sy.Integer(6), 2
nodes = [sy.Integer(0), sy.Rational(1, 2), sy.Integer(1)]
ell = []
for i, ti in enumerate(nodes):
    p = sy.Integer(1)
    for j, tj in enumerate(nodes):
        if j != i:
            p = p * (t - tj) / (ti - tj)
    ell.append(sy.expand(p))
h = sy.Rational(1, N)
nn = k * N + 1
M = sy.zeros(nn, nn); L = sy.zeros(nn, nn); B = sy.zeros(nn, nn)
for c in range(N):
    for m in range(k + 1):
        for q in range(k + 1):
            M[c * k + m, c * k + q] += h * sy.integrate(ell[m] * ell[q], (t, 0, 1))
            L[c * k + m, c * k + q] += sy.integrate(sy.diff(ell[m], t) * sy.diff(ell[q], t), (t, 0, 1)) / h
            B[c * k + m, c * k + q] += sy.integrate(sy.diff(ell[m], t, 2) * sy.diff(ell[q], t, 2), (t, 0, 1)) / h ** 3
for f in range(N + 1):
    a, b = {}, {}
    if f > 0:       # cell on the left of node f*k, outward normal +e at t=1
        for m in range(k + 1):
            g = (f - 1) * k + m
            a[g] = a.get(g, 0) + sy.diff(ell[m], t).subs(t, 1) / h
            b[g] = b.get(g, 0) + sy.diff(ell[m], t, 2).subs(t, 1) / h ** 2 / (1 if f == N else 2)
    if f < N:       # cell on the right, outward normal -e at t=0
        for m in range(k + 1):
            g = f * k + m
            a[g] = a.get(g, 0) - sy.diff(ell[m], t).subs(t, 0) / h
            b[g] = b.get(g, 0) + sy.diff(ell[m], t, 2).subs(t, 0) / h ** 2 / (1 if f == 0 else 2)
    sf = sigma * (bfac if f in (0, N) else 1)
    for i in a:
        for j in a:
            B[i, j] += sf / h * a[i] * a[j] - a[i] * b[j] - b[i] * a[j]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "k2_N2_sigma6_bfac2_1d.txt")
with open(out, "w") as fh:
    fh.write(__doc__.replace("Writes ", "# Written by tests/golden/make_bfac2.py: ").replace("\n", "\n# ").rstrip("# ") + "\n")
    for name, X in (("M", M), ("L", L), ("B", B)):
        fh.write(f"{name} {nn - 2} {nn - 2}\n")
        for i in range(1, nn - 1):
            fh.write(" ".join(str(sy.nsimplify(X[i, j])) for j in range(1, nn - 1)) + "\n")
