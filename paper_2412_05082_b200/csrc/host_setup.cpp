// Host-side setup tables; see host_setup.hpp.  Citations are to /root/reference/PAPER.md.
#include "host_setup.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>

namespace c0ip {

// ----------------------------------------------------------------------------- quadrature / basis
static void legendre_p(int n, double x, double& p, double& dp) {
  // P_n(x) and P_n'(x) on [-1,1] by the three-term recurrence
  double p0 = 1.0, p1 = x;
  if (n == 0) { p = 1.0; dp = 0.0; return; }
  for (int m = 2; m <= n; ++m) {
    double p2 = ((2.0 * m - 1.0) * x * p1 - (m - 1.0) * p0) / m;
    p0 = p1; p1 = p2;
  }
  p = p1;
  dp = (std::fabs(1.0 - x * x) < 1e-300) ? 0.0 : n * (x * p1 - p0) / (x * x - 1.0);
}

void gauss_legendre(int nq, std::vector<double>& x, std::vector<double>& w) {
  x.assign(nq, 0.0); w.assign(nq, 0.0);
  for (int i = 0; i < nq; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (nq + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre_p(nq, z, p, dp);
      double dz = p / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    double p, dp;
    legendre_p(nq, z, p, dp);
    x[nq - 1 - i] = 0.5 * (z + 1.0);
    w[nq - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);     // 2/((1-z^2)P'^2) on [-1,1], halved
  }
}

Basis1D make_basis(int k) {
  // Gauss-Lobatto points: 0, 1 and the roots of P_k'(2t-1) (reading Q18: deal.II FE_Q default)
  Basis1D b;
  b.k = k;
  b.pts.assign(k + 1, 0.0);
  b.pts[0] = 0.0; b.pts[k] = 1.0;
  for (int i = 1; i < k; ++i) {
    double z = -std::cos(M_PI * i / k);
    for (int it = 0; it < 200; ++it) {
      double p, dp;
      legendre_p(k, z, p, dp);
      double d2p = (2.0 * z * dp - k * (k + 1.0) * p) / (1.0 - z * z);    // Legendre ODE
      double dz = dp / d2p;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    b.pts[i] = 0.5 * (z + 1.0);
  }
  std::sort(b.pts.begin(), b.pts.end());
  return b;
}

void Basis1D::eval(double t, double* v, double* d1, double* d2) const {
  // l_m(t) = prod_{j!=m} (t - t_j)/(t_m - t_j), differentiated by truncated Taylor arithmetic
  for (int m = 0; m <= k; ++m) {
    double c0 = 1.0, c1 = 0.0, c2 = 0.0;   // coefficients of eps^0, eps^1, eps^2
    for (int j = 0; j <= k; ++j) {
      if (j == m) continue;
      double den = pts[m] - pts[j];
      double a0 = (t - pts[j]) / den, a1 = 1.0 / den;
      double n0 = c0 * a0, n1 = c0 * a1 + c1 * a0, n2 = c1 * a1 + c2 * a0;
      c0 = n0; c1 = n1; c2 = n2;
    }
    if (v) v[m] = c0;
    if (d1) d1[m] = c1;
    if (d2) d2[m] = 2.0 * c2;
  }
}

// ----------------------------------------------------------------------------- reference data
RefData make_ref(int k, double sigma) {
  // Eq. matrix1d on the unit cell; face terms per Eqs. ev/eh
  RefData r;
  r.k = k;
  r.sigma = sigma;
  r.sigma_b = kBoundaryPenalty * sigma;
  Basis1D b = make_basis(k);
  const int n1 = k + 1;
  std::vector<double> qx, qw;
  gauss_legendre(k + 2, qx, qw);
  r.Mc.assign(n1 * n1, 0.0); r.Lc.assign(n1 * n1, 0.0); r.Bc.assign(n1 * n1, 0.0);
  std::vector<double> v(n1), d1(n1), d2(n1);
  for (size_t q = 0; q < qx.size(); ++q) {
    b.eval(qx[q], v.data(), d1.data(), d2.data());
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) {
        r.Mc[i * n1 + j] += qw[q] * v[i] * v[j];
        r.Lc[i * n1 + j] += qw[q] * d1[i] * d1[j];
        r.Bc[i * n1 + j] += qw[q] * d2[i] * d2[j];
      }
  }
  std::vector<double> v0(n1), a0(n1), b0(n1), v1(n1), a1(n1), b1(n1);
  b.eval(0.0, v0.data(), a0.data(), b0.data());
  b.eval(1.0, v1.data(), a1.data(), b1.data());
  // interior face: [phi'] = phi'(x^-) - phi'(x^+) (sum of outward normal derivatives),
  // {phi''} = (phi''(x^-) + phi''(x^+))/2; left cell nodes 0..k, right cell nodes k..2k
  r.fa.assign(2 * k + 1, 0.0); r.fb.assign(2 * k + 1, 0.0);
  for (int m = 0; m < n1; ++m) {
    r.fa[m] += a1[m];       r.fb[m] += 0.5 * b1[m];
    r.fa[k + m] -= a0[m];   r.fb[k + m] += 0.5 * b0[m];
  }
  // boundary facets (reading Q26): one-sided, outward normal -e at 0, +e at 1
  r.la.resize(n1); r.lb.resize(n1); r.ua.resize(n1); r.ub.resize(n1);
  for (int m = 0; m < n1; ++m) {
    r.la[m] = -a0[m]; r.lb[m] = b0[m];
    r.ua[m] = a1[m];  r.ub[m] = b1[m];
  }
  return r;
}

void global_bands(const RefData& rd, int64_t N, Band& M, Band& L, Band& B, bool eliminate) {
  const int k = rd.k, n1 = k + 1, hw = 2 * k, W = 2 * hw + 1;
  const int64_t nn = k * N + 1;           // full nodes
  std::vector<double> fm(nn * W, 0.0), fl(nn * W, 0.0), fbm(nn * W, 0.0);
  auto add = [&](std::vector<double>& X, int64_t i, int64_t j, double val) {
    X[i * W + (j - i + hw)] += val;
  };
  for (int64_t c = 0; c < N; ++c)
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) {
        add(fm, c * k + i, c * k + j, rd.Mc[i * n1 + j]);
        add(fl, c * k + i, c * k + j, rd.Lc[i * n1 + j]);
        add(fbm, c * k + i, c * k + j, rd.Bc[i * n1 + j]);
      }
  // face f at node f*k: (sigma_f/h_f) a a^T - a b^T - b a^T, h_f = h (reference: h = 1); boundary
  // facets carry sigma_b (reading Q27)
  for (int64_t f = 0; f <= N; ++f) {
    const double *a, *b;
    int len;
    int64_t g0;
    double sf = rd.sigma_b;
    if (f == 0) { a = rd.la.data(); b = rd.lb.data(); len = n1; g0 = 0; }
    else if (f == N) { a = rd.ua.data(); b = rd.ub.data(); len = n1; g0 = (N - 1) * k; }
    else { a = rd.fa.data(); b = rd.fb.data(); len = 2 * k + 1; g0 = (f - 1) * k; sf = rd.sigma; }
    for (int i = 0; i < len; ++i)
      for (int j = 0; j < len; ++j)
        add(fbm, g0 + i, g0 + j, sf * a[i] * a[j] - a[i] * b[j] - b[i] * a[j]);
  }
  if (!eliminate) {
    for (Band* X : {&M, &L, &B}) { X->n = nn; X->hw = hw; }
    M.v = fm; L.v = fl; B.v = fbm;
    return;
  }
  const int64_t n = nn - 2;                // eliminate nodes 0 and kN (u = 0 strongly)
  for (Band* X : {&M, &L, &B}) { X->n = n; X->hw = hw; X->v.assign(n * W, 0.0); }
  for (int64_t i = 0; i < n; ++i)
    for (int q = 0; q < W; ++q) {
      int64_t j = i + q - hw;
      if (j < 0 || j >= n) continue;
      M.v[i * W + q] = fm[(i + 1) * W + q];
      L.v[i * W + q] = fl[(i + 1) * W + q];
      B.v[i * W + q] = fbm[(i + 1) * W + q];
    }
}

bool band_is_spd(const Band& B) {
  // banded Cholesky (lower), returns false on a non-positive pivot
  const int64_t n = B.n;
  const int hw = B.hw;
  std::vector<double> Lw(n * (hw + 1), 0.0);     // L[i][i-p] at Lw[i*(hw+1)+p]
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = std::max<int64_t>(0, i - hw); j <= i; ++j) {
      double s = B.at(i, j);
      for (int64_t m = std::max<int64_t>(0, i - hw); m < j; ++m) {
        if (j - m > hw) continue;
        s -= Lw[i * (hw + 1) + (i - m)] * Lw[j * (hw + 1) + (j - m)];
      }
      if (i == j) {
        if (!(s > 0.0)) return false;
        Lw[i * (hw + 1)] = std::sqrt(s);
      } else {
        Lw[i * (hw + 1) + (i - j)] = s / Lw[j * (hw + 1)];
      }
    }
  }
  return true;
}

void jacobi_eigen(int n, std::vector<double> A, std::vector<double>& w, std::vector<double>& V) {
  V.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += A[i * n + j] * A[i * n + j];
        if (i != j) off += A[i * n + j] * A[i * n + j];
      }
    if (off <= 1e-32 * tot) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        double apq = A[p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        double theta = (A[q * n + q] - A[p * n + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int r = 0; r < n; ++r) {          // A <- A J
          double arp = A[r * n + p], arq = A[r * n + q];
          A[r * n + p] = c * arp - s * arq;
          A[r * n + q] = s * arp + c * arq;
        }
        for (int r = 0; r < n; ++r) {          // A <- J^T A
          double apr = A[p * n + r], aqr = A[q * n + r];
          A[p * n + r] = c * apr - s * aqr;
          A[q * n + r] = s * apr + c * aqr;
        }
        for (int r = 0; r < n; ++r) {          // V <- V J
          double vrp = V[r * n + p], vrq = V[r * n + q];
          V[r * n + p] = c * vrp - s * vrq;
          V[r * n + q] = s * vrp + c * vrq;
        }
      }
  }
  w.resize(n);
  for (int i = 0; i < n; ++i) w[i] = A[i * n + i];
}

static bool cholesky(int n, const std::vector<double>& A, std::vector<double>& C) {
  C.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = A[i * n + j];
      for (int m = 0; m < j; ++m) s -= C[i * n + m] * C[j * n + m];
      if (i == j) {
        if (!(s > 0.0)) return false;
        C[i * n + i] = std::sqrt(s);
      } else {
        C[i * n + j] = s / C[j * n + j];
      }
    }
  return true;
}

bool gen_eig(int np, const std::vector<double>& Mv, const std::vector<double>& Bv, std::vector<double>& Sout,
             std::vector<double>& lam, std::string& err) {
  // Generalized eigenproblem B_v S = M_v S Lambda with S^T M_v S = I (reading Q6), by Cholesky M_v = C C^T and
  // cyclic Jacobi on C^{-1} B_v C^{-T}.
  std::vector<double> C;
  if (!cholesky(np, Mv, C)) { err = "patch mass block not SPD"; return false; }
  // K = C^{-1} B C^{-T}: solve C Y = B, then C K^T = Y^T
  std::vector<double> Y(np * np), K(np * np);
  for (int col = 0; col < np; ++col)
    for (int i = 0; i < np; ++i) {
      double s = Bv[i * np + col];
      for (int m = 0; m < i; ++m) s -= C[i * np + m] * Y[m * np + col];
      Y[i * np + col] = s / C[i * np + i];
    }
  for (int row = 0; row < np; ++row)          // K[row][:] solves C K[row]^T = Y[row]^T ... use symmetry
    for (int i = 0; i < np; ++i) {
      double s = Y[row * np + i];
      for (int m = 0; m < i; ++m) s -= C[i * np + m] * K[row * np + m];
      K[row * np + i] = s / C[i * np + i];
    }
  for (int i = 0; i < np; ++i)                 // symmetrize rounding
    for (int j = 0; j < i; ++j) {
      double a = 0.5 * (K[i * np + j] + K[j * np + i]);
      K[i * np + j] = K[j * np + i] = a;
    }
  std::vector<double> w, Q;
  jacobi_eigen(np, K, w, Q);
  // S = C^{-T} Q  (back substitution with C^T)
  std::vector<double> S(np * np);
  for (int col = 0; col < np; ++col)
    for (int i = np - 1; i >= 0; --i) {
      double s = Q[i * np + col];
      for (int m = i + 1; m < np; ++m) s -= C[m * np + i] * S[m * np + col];
      S[i * np + col] = s / C[i * np + i];
    }
  // sort ascending, sign: largest-magnitude component positive
  std::vector<int> idx(np);
  for (int i = 0; i < np; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return w[a] < w[b]; });
  Sout.assign(np * np, 0.0);
  lam.assign(np, 0.0);
  for (int c = 0; c < np; ++c) {
    int src = idx[c];
    if (!(w[src] > 0.0)) { err = "patch B block not positive definite (penalty too small)"; return false; }
    int imax = 0;
    for (int i = 1; i < np; ++i)
      if (std::fabs(S[i * np + src]) > std::fabs(S[imax * np + src])) imax = i;
    double sg = S[imax * np + src] < 0 ? -1.0 : 1.0;
    for (int i = 0; i < np; ++i) Sout[i * np + c] = sg * S[i * np + src];
    lam[c] = w[src];
  }
  return true;
}

static void patch_blocks(const Band& M, const Band& L, const Band& B, int k, int64_t v, std::vector<double>& Mv,
                         std::vector<double>& Lv, std::vector<double>& Bv) {
  const int np = 2 * k - 1;
  const int64_t base = (v - 1) * k;
  Mv.assign(np * np, 0.0); Lv.assign(np * np, 0.0); Bv.assign(np * np, 0.0);
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j) {
      Mv[i * np + j] = M.at(base + i, base + j);
      Bv[i * np + j] = B.at(base + i, base + j);
      Lv[i * np + j] = L.at(base + i, base + j);
    }
}

bool make_fdm(const RefData& rd, int64_t N, const Band& M, const Band& L, const Band& B, Fdm& out,
              std::string& err) {
  // per axis variant (translation invariance of the uniform mesh)
  const int k = rd.k, np = 2 * k - 1;
  out.np = np;
  int64_t vs[4] = {1, 2, N - 1, 1};
  bool pres[4];
  if (N == 2) { pres[0] = pres[1] = pres[2] = false; pres[3] = true; }
  else { pres[0] = pres[2] = true; pres[1] = (N >= 4); pres[3] = false; }
  for (int var = 0; var < 4; ++var) {
    out.present[var] = pres[var];
    if (!pres[var]) continue;
    std::vector<double> Mv, Lv, Bv;
    patch_blocks(M, L, B, k, vs[var], Mv, Lv, Bv);
    if (!gen_eig(np, Mv, Bv, out.S[var], out.lam[var], err)) return false;
    out.Mv[var] = Mv; out.Bv[var] = Bv; out.Lv[var] = Lv;
  }
  return true;
}

bool make_fdm_vertices(int k, int64_t N, const Band& M, const Band& L, const Band& B, std::vector<double>& S,
                       std::vector<double>& lam, std::string& err) {
  // graded meshes: every vertex has its own patch blocks (no translation invariance), v = 1 .. N-1
  const int np = 2 * k - 1;
  S.assign(size_t(N - 1) * np * np, 0.0);
  lam.assign(size_t(N - 1) * np, 0.0);
  for (int64_t v = 1; v <= N - 1; ++v) {
    std::vector<double> Mv, Lv, Bv, Sv, lv;
    patch_blocks(M, L, B, k, v, Mv, Lv, Bv);
    if (!gen_eig(np, Mv, Bv, Sv, lv, err)) return false;
    std::copy(Sv.begin(), Sv.end(), S.begin() + (v - 1) * np * np);
    std::copy(lv.begin(), lv.end(), lam.begin() + (v - 1) * np);
  }
  return true;
}

void global_bands_graded(const RefData& rd, const std::vector<double>& X, Band& M, Band& L, Band& B) {
  // per-cell widths h_c = X[c+1] - X[c] (physical scale): M = sum h_c M^, L = sum L^ / h_c,
  // B = sum B^ / h_c^3 + facets with the cells' own derivative scalings, interior penalty sigma / h_e with h_e the
  // harmonic mean of the adjacent widths, boundary sigma_b / h_c (reading Q27)
  const int k = rd.k, n1 = k + 1, hw = 2 * k, W = 2 * hw + 1;
  const int64_t N = int64_t(X.size()) - 1, nn = k * N + 1;
  std::vector<double> fm(nn * W, 0.0), fl(nn * W, 0.0), fbm(nn * W, 0.0);
  auto add = [&](std::vector<double>& Xv, int64_t i, int64_t j, double val) { Xv[i * W + (j - i + hw)] += val; };
  std::vector<double> h(N);
  for (int64_t c = 0; c < N; ++c) h[c] = X[c + 1] - X[c];
  for (int64_t c = 0; c < N; ++c)
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) {
        add(fm, c * k + i, c * k + j, h[c] * rd.Mc[i * n1 + j]);
        add(fl, c * k + i, c * k + j, rd.Lc[i * n1 + j] / h[c]);
        add(fbm, c * k + i, c * k + j, rd.Bc[i * n1 + j] / (h[c] * h[c] * h[c]));
      }
  for (int64_t f = 0; f <= N; ++f) {
    std::vector<double> a, bb;
    int64_t g0;
    double pen;
    if (f == 0) {
      for (int m = 0; m < n1; ++m) { a.push_back(rd.la[m] / h[0]); bb.push_back(rd.lb[m] / (h[0] * h[0])); }
      g0 = 0; pen = rd.sigma_b / h[0];
    } else if (f == N) {
      const double hc = h[N - 1];
      for (int m = 0; m < n1; ++m) { a.push_back(rd.ua[m] / hc); bb.push_back(rd.ub[m] / (hc * hc)); }
      g0 = (N - 1) * k; pen = rd.sigma_b / hc;
    } else {
      const double hl = h[f - 1], hr = h[f];
      a.assign(2 * k + 1, 0.0); bb.assign(2 * k + 1, 0.0);
      for (int m = 0; m < n1; ++m) {
        a[m] += rd.ua[m] / hl;          bb[m] += 0.5 * rd.ub[m] / (hl * hl);
        a[k + m] += rd.la[m] / hr;      bb[k + m] += 0.5 * rd.lb[m] / (hr * hr);
      }
      g0 = (f - 1) * k; pen = rd.sigma * (hl + hr) / (2.0 * hl * hr);
    }
    const int len = int(a.size());
    for (int i = 0; i < len; ++i)
      for (int j = 0; j < len; ++j) add(fbm, g0 + i, g0 + j, pen * a[i] * a[j] - a[i] * bb[j] - bb[i] * a[j]);
  }
  const int64_t n = nn - 2;                // eliminate nodes 0 and kN (u = 0 strongly)
  for (Band* Xb : {&M, &L, &B}) { Xb->n = n; Xb->hw = hw; Xb->v.assign(n * W, 0.0); }
  for (int64_t i = 0; i < n; ++i)
    for (int qq = 0; qq < W; ++qq) {
      int64_t j = i + qq - hw;
      if (j < 0 || j >= n) continue;
      M.v[i * W + qq] = fm[(i + 1) * W + qq];
      L.v[i * W + qq] = fl[(i + 1) * W + qq];
      B.v[i * W + qq] = fbm[(i + 1) * W + qq];
    }
}

RectBand embedding_graded(int k, const std::vector<double>& Xf) {
  // E_ij = phi^coarse_j(x^fine_i) on nested graded meshes (coarse boundaries = every second fine one)
  Basis1D b = make_basis(k);
  const int64_t Nf = int64_t(Xf.size()) - 1, Nc = Nf / 2;
  const int64_t nf = k * Nf - 1, nc = k * Nc - 1;
  RectBand E;
  E.rows = nf; E.cols = nc; E.width = k + 1;
  E.lo.assign(nf, 0);
  E.v.assign(nf * (k + 1), 0.0);
  std::vector<double> val(k + 1);
  for (int64_t i = 0; i < nf; ++i) {
    const int64_t jf = i + 1;
    int64_t cf = jf / k, p = jf % k;
    if (cf == Nf) { cf -= 1; p = k; }
    const double x = Xf[cf] + b.pts[p] * (Xf[cf + 1] - Xf[cf]);
    const int64_t cc = cf / 2;
    const double tl = (x - Xf[2 * cc]) / (Xf[2 * cc + 2] - Xf[2 * cc]);
    b.eval(tl, val.data(), nullptr, nullptr);
    const int64_t lo = cc * k - 1;
    int64_t lo_c = std::max<int64_t>(0, lo);
    lo_c = std::min<int64_t>(lo_c, nc - (k + 1) < 0 ? 0 : nc - (k + 1));
    E.lo[i] = lo_c;
    for (int m = 0; m <= k; ++m) {
      const int64_t col = lo + m;
      if (col < 0 || col >= nc) continue;
      double xv = val[m];
      if (std::fabs(xv) < 1e-15) xv = 0.0;
      const int64_t q = col - lo_c;
      if (q >= 0 && q <= k) E.v[i * (k + 1) + q] += xv;
    }
  }
  return E;
}

std::vector<double> sine_load_1d_graded(int k, const std::vector<double>& X) {
  // f1_i = int sin(pi x) phi_i(x) dx on the graded cells, Gauss k+3 points per cell
  Basis1D b = make_basis(k);
  std::vector<double> qx, qw;
  gauss_legendre(k + 3, qx, qw);
  const int64_t N = int64_t(X.size()) - 1;
  std::vector<double> full(k * N + 1, 0.0), v(k + 1);
  for (int64_t c = 0; c < N; ++c) {
    const double h = X[c + 1] - X[c];
    for (size_t q = 0; q < qx.size(); ++q) {
      const double x = X[c] + qx[q] * h;
      b.eval(qx[q], v.data(), nullptr, nullptr);
      for (int m = 0; m <= k; ++m) full[c * k + m] += h * qw[q] * std::sin(M_PI * x) * v[m];
    }
  }
  return std::vector<double>(full.begin() + 1, full.end() - 1);
}

std::vector<double> boundary_normal_1d_graded(const RefData& rd, const std::vector<double>& X) {
  const int k = rd.k;
  const int64_t N = int64_t(X.size()) - 1;
  const double h0 = X[1] - X[0], h1 = X[N] - X[N - 1];
  std::vector<double> full(k * N + 1, 0.0);
  for (int m = 0; m <= k; ++m) {
    full[m] += (rd.sigma_b / h0) * (rd.la[m] / h0) - rd.lb[m] / (h0 * h0);
    full[(N - 1) * k + m] += (rd.sigma_b / h1) * (rd.ua[m] / h1) - rd.ub[m] / (h1 * h1);
  }
  return std::vector<double>(full.begin() + 1, full.end() - 1);
}

RectBand embedding(int k, int64_t Nc) {
  // E_ij = phi^coarse_j(x^fine_i) over interior nodes (natural embedding)
  Basis1D b = make_basis(k);
  const int64_t nf = 2 * k * Nc - 1, nc = k * Nc - 1;
  RectBand E;
  E.rows = nf; E.cols = nc; E.width = k + 1;
  E.lo.assign(nf, 0);
  E.v.assign(nf * (k + 1), 0.0);
  std::vector<double> val(k + 1);
  for (int64_t i = 0; i < nf; ++i) {
    int64_t jf = i + 1;
    int64_t cf = jf / k, p = jf % k;
    if (cf == 2 * Nc) { cf -= 1; p = k; }       // not reached for interior nodes
    int64_t cc = cf / 2;
    double tl = (double(cf % 2) + b.pts[p]) * 0.5;
    b.eval(tl, val.data(), nullptr, nullptr);
    // coarse nodes cc*k + m, interior column index jc - 1
    int64_t lo = cc * k - 1;
    int64_t lo_c = std::max<int64_t>(0, lo);
    lo_c = std::min<int64_t>(lo_c, nc - (k + 1) < 0 ? 0 : nc - (k + 1));
    E.lo[i] = lo_c;
    for (int m = 0; m <= k; ++m) {
      int64_t col = lo + m;
      if (col < 0 || col >= nc) continue;
      double x = val[m];
      if (std::fabs(x) < 1e-15) x = 0.0;
      int64_t q = col - lo_c;
      if (q >= 0 && q <= k) E.v[i * (k + 1) + q] += x;
    }
  }
  return E;
}

RectBand transpose(const RectBand& E) {
  RectBand T;
  T.rows = E.cols; T.cols = E.rows;
  std::vector<int64_t> lo(T.rows, INT64_MAX), hi(T.rows, -1);
  for (int64_t i = 0; i < E.rows; ++i)
    for (int q = 0; q < E.width; ++q) {
      if (E.v[i * E.width + q] == 0.0) continue;
      int64_t c = E.lo[i] + q;
      lo[c] = std::min(lo[c], i); hi[c] = std::max(hi[c], i);
    }
  int w = 1;
  for (int64_t c = 0; c < T.rows; ++c) if (hi[c] >= 0) w = std::max<int>(w, int(hi[c] - lo[c] + 1));
  T.width = w;
  T.lo.assign(T.rows, 0);
  T.v.assign(T.rows * w, 0.0);
  for (int64_t c = 0; c < T.rows; ++c) {
    int64_t l = hi[c] >= 0 ? lo[c] : 0;
    l = std::min<int64_t>(l, std::max<int64_t>(0, T.cols - w));
    T.lo[c] = l;
  }
  for (int64_t i = 0; i < E.rows; ++i)
    for (int q = 0; q < E.width; ++q) {
      double x = E.v[i * E.width + q];
      if (x == 0.0) continue;
      int64_t c = E.lo[i] + q;
      T.v[c * w + (i - T.lo[c])] = x;
    }
  return T;
}

std::vector<double> sine_load_1d(int k, int64_t N) {
  // f1_i = int_0^1 sin(pi x) phi_i dx, Gauss with k+3 points per cell
  Basis1D b = make_basis(k);
  std::vector<double> qx, qw;
  gauss_legendre(k + 3, qx, qw);
  const double h = 1.0 / double(N);
  std::vector<double> full(k * N + 1, 0.0), v(k + 1);
  for (int64_t c = 0; c < N; ++c)
    for (size_t q = 0; q < qx.size(); ++q) {
      double x = (double(c) + qx[q]) * h;
      double fx = std::sin(M_PI * x);
      b.eval(qx[q], v.data(), nullptr, nullptr);
      for (int m = 0; m <= k; ++m) full[c * k + m] += h * qw[q] * fx * v[m];
    }
  return std::vector<double>(full.begin() + 1, full.end() - 1);
}

std::vector<double> boundary_normal_1d(const RefData& rd, int64_t N) {
  // facet x=0: outward normal -e, d_n phi = -phi'(0)/h, d_n^2 phi = phi''(0)/h^2 (first cell's nodes);
  // facet x=1: +e on the last cell.  la/ua hold d_n phi, lb/ub d_n^2 phi at h = 1.
  const int k = rd.k;
  const double h = 1.0 / double(N);
  std::vector<double> full(k * N + 1, 0.0);
  for (int m = 0; m <= k; ++m) {
    full[m] += (rd.sigma_b / h) * (rd.la[m] / h) - rd.lb[m] / (h * h);
    full[(N - 1) * k + m] += (rd.sigma_b / h) * (rd.ua[m] / h) - rd.ub[m] / (h * h);
  }
  return std::vector<double>(full.begin() + 1, full.end() - 1);
}

// ---- Poisson SIPG comparison workload (reading Q30) ---------------------------
void sipg_bands(const RefData& rd, int64_t N, double sigma, Band& M, Band& L) {
  // discontinuous Q_k, cell c owns nodes c (k+1) + m; h = 1/N (physical scale): M = h M^ per cell,
  // L = L^ / h per cell + facets (sigma_f / h) [u][v] - {u'}[v] - [u]{v'} with [u] = u^- - u^+ (normal +e of the
  // left cell), {u'} = (u'^- + u'^+) / 2; boundary facets one-sided with penalty 2 sigma (reading Q27 convention)
  const int k = rd.k, n1 = k + 1, hw = 2 * k + 1, W = 2 * hw + 1;
  const int64_t n = N * n1;
  const double h = 1.0 / double(N);
  Basis1D b = make_basis(k);
  std::vector<double> v0(n1), a0(n1), v1(n1), a1(n1);
  b.eval(0.0, v0.data(), a0.data(), nullptr);
  b.eval(1.0, v1.data(), a1.data(), nullptr);
  for (Band* X : {&M, &L}) { X->n = n; X->hw = hw; X->v.assign(n * W, 0.0); }
  auto add = [&](Band& X, int64_t i, int64_t j, double val) { X.v[i * W + (j - i + hw)] += val; };
  for (int64_t c = 0; c < N; ++c)
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n1; ++j) {
        add(M, c * n1 + i, c * n1 + j, h * rd.Mc[i * n1 + j]);
        add(L, c * n1 + i, c * n1 + j, rd.Lc[i * n1 + j] / h);
      }
  for (int64_t f = 0; f <= N; ++f) {
    std::vector<double> J, D;
    int64_t g0;
    double pen;
    if (f == 0) {
      for (int m = 0; m < n1; ++m) { J.push_back(v0[m]); D.push_back(-a0[m] / h); }
      g0 = 0; pen = 2.0 * sigma / h;
    } else if (f == N) {
      for (int m = 0; m < n1; ++m) { J.push_back(v1[m]); D.push_back(a1[m] / h); }
      g0 = (N - 1) * n1; pen = 2.0 * sigma / h;
    } else {
      J.assign(2 * n1, 0.0); D.assign(2 * n1, 0.0);
      for (int m = 0; m < n1; ++m) {
        J[m] = v1[m];        D[m] = 0.5 * a1[m] / h;
        J[n1 + m] = -v0[m];  D[n1 + m] = 0.5 * a0[m] / h;
      }
      g0 = (f - 1) * n1; pen = sigma / h;
    }
    const int len = int(J.size());
    for (int i = 0; i < len; ++i)
      for (int j = 0; j < len; ++j) add(L, g0 + i, g0 + j, pen * J[i] * J[j] - J[i] * D[j] - D[i] * J[j]);
  }
}

bool make_fdm_sipg(int k, int64_t N, const Band& M, const Band& L, Fdm& out, std::string& err) {
  // SIPG patches hold the (2k+2) DoFs of their 2 cells per axis; the patch operator is exactly L_v (x) M_v +
  // M_v (x) L_v, so L_v S = M_v S Lambda gives the exact FDM
  const int np = 2 * k + 2;
  out.np = np;
  int64_t vs[4] = {1, 2, N - 1, 1};
  bool pres[4];
  if (N == 2) { pres[0] = pres[1] = pres[2] = false; pres[3] = true; }
  else { pres[0] = pres[2] = true; pres[1] = (N >= 4); pres[3] = false; }
  for (int var = 0; var < 4; ++var) {
    out.present[var] = pres[var];
    if (!pres[var]) continue;
    const int64_t base = (vs[var] - 1) * (k + 1);
    std::vector<double> Mv(np * np), Lv(np * np);
    for (int i = 0; i < np; ++i)
      for (int j = 0; j < np; ++j) { Mv[i * np + j] = M.at(base + i, base + j); Lv[i * np + j] = L.at(base + i, base + j); }
    if (!gen_eig(np, Mv, Lv, out.S[var], out.lam[var], err)) return false;
    out.Mv[var] = Mv; out.Bv[var] = Lv; out.Lv[var] = Lv;
  }
  return true;
}

RectBand embedding_dg(int k, int64_t Nc) {
  // coarse cell polynomials at the nodes of its two fine cells (block structure, width k+1)
  Basis1D b = make_basis(k);
  const int n1 = k + 1;
  RectBand E;
  E.rows = 2 * Nc * n1; E.cols = Nc * n1; E.width = n1;
  E.lo.assign(E.rows, 0);
  E.v.assign(E.rows * n1, 0.0);
  std::vector<double> val(n1);
  for (int64_t cf = 0; cf < 2 * Nc; ++cf)
    for (int m = 0; m < n1; ++m) {
      const int64_t i = cf * n1 + m;
      b.eval((double(cf % 2) + b.pts[m]) * 0.5, val.data(), nullptr, nullptr);
      E.lo[i] = (cf / 2) * n1;
      for (int q = 0; q < n1; ++q) E.v[i * n1 + q] = std::fabs(val[q]) < 1e-15 ? 0.0 : val[q];
    }
  return E;
}

std::vector<double> sine_load_1d_dg(int k, int64_t N) {
  Basis1D b = make_basis(k);
  std::vector<double> qx, qw;
  gauss_legendre(k + 3, qx, qw);
  const double h = 1.0 / double(N);
  std::vector<double> out(N * (k + 1), 0.0), v(k + 1);
  for (int64_t c = 0; c < N; ++c)
    for (size_t q = 0; q < qx.size(); ++q) {
      b.eval(qx[q], v.data(), nullptr, nullptr);
      const double fx = std::sin(M_PI * (double(c) + qx[q]) * h);
      for (int m = 0; m <= k; ++m) out[c * (k + 1) + m] += h * qw[q] * fx * v[m];
    }
  return out;
}

}  // namespace c0ip
