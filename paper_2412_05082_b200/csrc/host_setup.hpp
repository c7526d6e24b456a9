// Host-side setup for the C0IP vertex-patch smoother (arXiv 2412.05082), FP64.
//
// Everything here runs once per context (c0ip_create) and produces small constant tables:
//   * Q_k Lagrange basis on Gauss-Lobatto points (reading Q18),
//   * reference (h = 1) 1D element matrices M^, L^, B^bulk and face jump/mean vectors
//     (PAPER.md:323-332 Eq. matrix1d; Eqs. ev/eh PAPER.md:301-312; jump/mean PAPER.md:87-106),
//   * global banded 1D matrices M, L, B of one level (h = 1/N, boundary nodes eliminated),
//   * patch principal submatrices per axis variant and their generalized eigenpairs
//     B_v S = M_v S Lambda, S^T M_v S = I (PAPER.md:356-365 Eq. inverse, reading Q6),
//   * the 1D embedding E and the separable paper load.
// This file shares no code with oracle/ (the CPU test oracle).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace c0ip {

struct Basis1D {
  int k = 0;
  std::vector<double> pts;                 // k+1 Gauss-Lobatto points on [0,1]
  // value / first / second derivative of l_m at t (m = 0..k)
  void eval(double t, double* v, double* d1, double* d2) const;
};

Basis1D make_basis(int k);
void gauss_legendre(int nq, std::vector<double>& x, std::vector<double>& w);   // on [0,1]

// Reference data for one degree (h = 1).  Global matrices on N cells are
//   M = h * Mhat,  L = Lhat / h,  B = Bhat / h^3   (all face terms included in Bhat).
// Boundary facets: sigma/h_e with h_e = h/2 (reading Q27): the Nitsche penalty of the
// clamped condition is twice the interior-facet penalty.
constexpr double kBoundaryPenalty = 2.0;

struct RefData {
  int k = 0;
  double sigma = 0;                        // interior facets (reading Q4)
  double sigma_b = 0;                      // boundary facets = kBoundaryPenalty * sigma (reading Q27)
  std::vector<double> Mc, Lc, Bc;          // (k+1)^2 cell matrices, row-major
  std::vector<double> fa, fb;              // interior face: a, b over 2k+1 nodes
  std::vector<double> la, lb, ua, ub;      // boundary faces (x=0: lower, x=1: upper), k+1 nodes
};
RefData make_ref(int k, double sigma);

// Banded square matrix: row i has entries at columns i-hw .. i+hw (hw = 2k), zero outside [0,n).
struct Band {
  int64_t n = 0;
  int hw = 0;
  std::vector<double> v;                   // n * (2 hw + 1)
  double at(int64_t i, int64_t j) const {
    int64_t q = j - i + hw;
    return (q < 0 || q > 2 * hw) ? 0.0 : v[i * (2 * hw + 1) + q];
  }
};

// Reference-scaled global 1D matrices of the interior nodes of an N-cell mesh (h factor NOT applied):
// Mhat_glob, Lhat_glob, Bhat_glob (so that M = h*Mhat_glob etc.).
void global_bands(const RefData& rd, int64_t N, Band& M, Band& L, Band& B, bool eliminate = true);
// (eliminate = false: all kN+1 nodes, row/column j = node index)

// Rectangular band: row i has `width` entries starting at column lo[i].
struct RectBand {
  int64_t rows = 0, cols = 0;
  int width = 0;
  std::vector<int64_t> lo;
  std::vector<double> v;                   // rows * width
};
RectBand embedding(int k, int64_t Nc);     // E: fine interior (2Nc cells) x coarse interior
RectBand transpose(const RectBand& E);     // E^T as a rectangular band

// Patch 1D blocks and FDM factors per axis variant (reference scaling, h = 1):
//   variant 0 = left (v=1), 1 = interior (v=2..N-2), 2 = right (v=N-1), 3 = both (N=2).
struct Fdm {
  int np = 0;                              // 2k-1
  bool present[4] = {false, false, false, false};
  std::vector<double> S[4], lam[4];        // S: np x np row-major (S[l][i] = l-th entry of i-th eigvec)
  std::vector<double> Mv[4], Bv[4], Lv[4]; // patch principal submatrices (np x np)
};
// Returns false (and a message) if a patch B block / M block is not SPD (coercivity).
bool make_fdm(const RefData& rd, int64_t N, const Band& M, const Band& L, const Band& B, Fdm& out,
              std::string& err);
bool band_is_spd(const Band& B);
// B_v S = M_v S Lambda, S^T M_v S = I for one patch block (ascending, sign convention of SPEC.md:320)
bool gen_eig(int np, const std::vector<double>& Mv, const std::vector<double>& Bv, std::vector<double>& S,
             std::vector<double>& lam, std::string& err);

// ---- graded / anisotropic Cartesian meshes: X = cell boundaries of one axis (N+1 values)
// physical-scale eliminated bands with per-cell widths and harmonic-mean facet widths
void global_bands_graded(const RefData& rd, const std::vector<double>& X, Band& M, Band& L, Band& B);
// per-vertex FDM factors: S[(v-1) np^2 + l np + i], lam[(v-1) np + i], v = 1 .. N-1
bool make_fdm_vertices(int k, int64_t N, const Band& M, const Band& L, const Band& B, std::vector<double>& S,
                       std::vector<double>& lam, std::string& err);
RectBand embedding_graded(int k, const std::vector<double>& Xf);
std::vector<double> sine_load_1d_graded(int k, const std::vector<double>& X);
std::vector<double> boundary_normal_1d_graded(const RefData& rd, const std::vector<double>& X);

// ---- Poisson SIPG comparison workload (reading Q30): DG mass / SIPG stiffness bands (hw 2k+1,
// physical scale), exact FDM per axis variant (patches of 2k+2 DoFs per axis), DG embedding, DG sine load
void sipg_bands(const RefData& rd, int64_t N, double sigma, Band& M, Band& L);
bool make_fdm_sipg(int k, int64_t N, const Band& M, const Band& L, Fdm& out, std::string& err);
RectBand embedding_dg(int k, int64_t Nc);
std::vector<double> sine_load_1d_dg(int k, int64_t N);

// 1D load f1_i = int sin(pi x) phi_i(x) dx (reference scaling: includes h), Gauss k+3 pts/cell.
std::vector<double> sine_load_1d(int k, int64_t N);
// 1D boundary-facet factor of the Nitsche boundary data (reading Q8b): over the interior nodes,
// g1_i = sum_{facets x=0, x=1} ( (sigma_b/h) d_n phi_i - d_n^2 phi_i ) at the facet (physical h = 1/N).
std::vector<double> boundary_normal_1d(const RefData& rd, int64_t N);

// Cyclic Jacobi eigen-solver for a symmetric n x n matrix (row-major). Eigenvectors in columns of V.
void jacobi_eigen(int n, std::vector<double> A, std::vector<double>& w, std::vector<double>& V);

}  // namespace c0ip
