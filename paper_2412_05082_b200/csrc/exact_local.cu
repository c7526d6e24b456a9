// Exact local solvers A_v^{-1} (Table 1): the vertex-patch
// smoothers with the *exact* patch matrix A_v = R_v A_l R_v^T instead of the separable surrogate.
//
// A_v is the principal submatrix of the Kronecker form of A_l (Eqs. c0iptensorvp /
// c0iptensorvp3D) on the patch's (2k-1)^d interior DoFs, so it depends only on the patch's axis-variant
// tuple (left / interior / right / both per axis).  The host builds A_v from the 1D patch blocks of the
// level's banded M, L, B, inverts it densely in FP64 (Cholesky), and uploads A_v^{-1} per variant tuple.
//
// Application: for a list of patches of one variant tuple, U = A_v^{-1} R where the columns of R are the
// gathered patch residuals R_v r -- a dense GEMM (M = K = (2k-1)^d, N = #patches) with the gather fused
// into the B-operand staging and the scatter-add x += omega R_v^T u fused into the epilogue
// (red.global.add; patches of one MVS colour are disjoint, AVS overlaps resolve in L2 like the paper's
// "atomic AVS").  FP64 runs on the FP64 tensor cores (mma.sync.m8n8k4.f64, SASS DMMA), FP32
// on FFMA with the same tiling.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <type_traits>

#include "exact_local.hpp"

namespace c0ip {

namespace {

constexpr int TM = 64, TN = 64, TK = 16;     // CTA tile: 64 local rows x 64 patches, K chunks of 16
constexpr int SA = TK + 1;                   // smem row pitch of the A chunk (doubles)
constexpr int SB = TN + 2;                   // smem row pitch of the B chunk

__device__ __forceinline__ void dmma_exact(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__device__ __forceinline__ void red_add(double* p, double v) { atomicAdd(p, v); }
__device__ __forceinline__ void red_add(float* p, float v) { atomicAdd(p, v); }

// patch origin: global id of local DoF (0,..,0) = sum_a (v_a - 1) k n^a, v_a = 1 + (p / (N-1)^a) % (N-1)
__device__ __forceinline__ int64_t patch_origin(int64_t p, int d, int k, int64_t N, int64_t n) {
  int64_t o = 0, s = 1;
  for (int a = 0; a < d; ++a) {
    const int64_t va = 1 + p % (N - 1);
    p /= (N - 1);
    o += (va - 1) * k * s;
    s *= n;
  }
  return o;
}

template <typename T>
__global__ void __launch_bounds__(256) exact_patch_kernel(ExactArgs<T> a) {
  __shared__ T sA[2][TM * SA];
  __shared__ T sB[2][TK * SB];
  __shared__ int64_t org[TN];
  const int tid = threadIdx.x;
  const int64_t p0 = int64_t(blockIdx.x) * TN;
  const int row0 = blockIdx.y * TM;
  if (tid < TN) {
    const int64_t pi = p0 + tid;
    org[tid] = pi < a.count ? patch_origin(a.list[pi], a.d, a.k, a.N, a.n) : int64_t(-1);
  }
  __syncthreads();
  const int nk = (a.nloc + TK - 1) / TK;

  auto stage = [&](int kc, int buf) {
    const int k0 = kc * TK;
    // A chunk: rows row0..row0+63, cols k0..k0+15 of A_v^{-1} (row-major, nloc x nloc); 1024 elements
    for (int e = tid; e < TM * TK; e += 256) {
      const int i = e / TK, j = e % TK;
      const int gr = row0 + i, gc = k0 + j;
      sA[buf][i * SA + j] = (gr < a.nloc && gc < a.nloc) ? a.Ainv[int64_t(gr) * a.nloc + gc] : T(0);
    }
    // B chunk: gathered residuals r[origin(p) + off[k0 + i]] (patch-local row k0+i of patch column j)
    for (int e = tid; e < TK * TN; e += 256) {
      const int i = e / TN, j = e % TN;
      const int gk = k0 + i;
      const int64_t o = org[j];
      sB[buf][i * SB + j] = (gk < a.nloc && o >= 0) ? a.r[o + a.off[gk]] : T(0);
    }
  };

  const int warp = tid >> 5, lane = tid & 31;
  if constexpr (std::is_same<T, double>::value) {
    // 8 warps: 4 along M (16 rows each) x 2 along N (32 patches each); per warp 2 x 4 m8n8 blocks
    const int wm = warp & 3, wn = warp >> 2;
    const int g = lane >> 2, q = lane & 3;
    double acc[2][4][2] = {};
    stage(0, 0);
    __syncthreads();
    for (int kc = 0; kc < nk; ++kc) {
      const int buf = kc & 1;
      if (kc + 1 < nk) stage(kc + 1, buf ^ 1);
#pragma unroll
      for (int ks = 0; ks < TK / 4; ++ks) {
        double af[2], bf[4];
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) af[mb] = sA[buf][(wm * 16 + mb * 8 + g) * SA + ks * 4 + q];
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) bf[nb] = sB[buf][(ks * 4 + q) * SB + wn * 32 + nb * 8 + g];
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) dmma_exact(acc[mb][nb][0], acc[mb][nb][1], af[mb], bf[nb]);
      }
      __syncthreads();
    }
    // epilogue: x[origin(p) + off[row]] += omega * u
#pragma unroll
    for (int mb = 0; mb < 2; ++mb) {
      const int row = row0 + wm * 16 + mb * 8 + g;
      if (row >= a.nloc) continue;
      const int64_t orow = a.off[row];
#pragma unroll
      for (int nb = 0; nb < 4; ++nb)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int col = wn * 32 + nb * 8 + 2 * q + c;
          const int64_t o = org[col];
          if (o >= 0) red_add(a.x + o + orow, a.omega * acc[mb][nb][c]);
        }
    }
  } else {
    // FP32: each thread a 4 x 4 micro-tile (rows ty + 16 i, patches tx + 16 j)
    const int ty = tid / 16, tx = tid % 16;
    float acc[4][4] = {};
    stage(0, 0);
    __syncthreads();
    for (int kc = 0; kc < nk; ++kc) {
      const int buf = kc & 1;
      if (kc + 1 < nk) stage(kc + 1, buf ^ 1);
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = sA[buf][(ty + 16 * i) * SA + kk];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = sB[buf][kk * SB + tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = row0 + ty + 16 * i;
      if (row >= a.nloc) continue;
      const int64_t orow = a.off[row];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t o = org[tx + 16 * j];
        if (o >= 0) red_add(a.x + o + orow, a.omega * acc[i][j]);
      }
    }
  }
}

}  // namespace

template <typename T>
void launch_exact_patches(const ExactArgs<T>& a, cudaStream_t st) {
  if (a.count <= 0) return;
  dim3 grid((unsigned)((a.count + TN - 1) / TN), (unsigned)((a.nloc + TM - 1) / TM));
  exact_patch_kernel<T><<<grid, 256, 0, st>>>(a);
}

template void launch_exact_patches<double>(const ExactArgs<double>&, cudaStream_t);
template void launch_exact_patches<float>(const ExactArgs<float>&, cudaStream_t);

}  // namespace c0ip

// ------------------------------------------------------------------------------------------ host tables
namespace c0ip {

namespace {

// representative vertex of an axis variant: 0 left (v = 1), 1 interior (v = 2), 2 right (v = N-1), 3 both
int64_t rep_vertex(int var, int64_t N) { return var == 0 || var == 3 ? 1 : (var == 1 ? 2 : N - 1); }

int axis_variant(int64_t v, int64_t N) {
  if (N == 2) return 3;
  if (v == 1) return 0;
  if (v == N - 1) return 2;
  return 1;
}

std::vector<double> block1d(const Band& X, int k, int64_t v) {
  const int np = 2 * k - 1;
  const int64_t r0 = (v - 1) * k;
  std::vector<double> out(np * np);
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j) out[i * np + j] = X.at(r0 + i, r0 + j);
  return out;
}

// dense SPD inverse by Cholesky: A = L L^T, A^{-1} = L^{-T} L^{-1}
bool spd_inverse(int n, std::vector<double>& A) {
  std::vector<double> L(size_t(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double s = A[size_t(j) * n + j];
    const double* Lj = &L[size_t(j) * n];
    for (int m = 0; m < j; ++m) s -= Lj[m] * Lj[m];
    if (!(s > 0.0)) return false;
    const double ljj = std::sqrt(s);
    L[size_t(j) * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      const double* Li = &L[size_t(i) * n];
      double t = A[size_t(i) * n + j];
      for (int m = 0; m < j; ++m) t -= Li[m] * Lj[m];
      L[size_t(i) * n + j] = t / ljj;
    }
  }
  // W = L^{-1} (lower triangular), column by column of the identity
  std::vector<double> W(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i) {
    const double* Li = &L[size_t(i) * n];
    double* Wi = &W[size_t(i) * n];
    Wi[i] = 1.0 / Li[i];
    for (int j = 0; j < i; ++j) {
      double t = 0.0;
      for (int m = j; m < i; ++m) t += Li[m] * W[size_t(m) * n + j];
      Wi[j] = -t / Li[i];
    }
  }
  // A^{-1} = W^T W
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double t = 0.0;
      for (int m = i; m < n; ++m) t += W[size_t(m) * n + i] * W[size_t(m) * n + j];
      A[size_t(i) * n + j] = A[size_t(j) * n + i] = t;
    }
  return true;
}

}  // namespace

bool build_exact_host(int d, int k, int64_t N, const Band& M, const Band& L, const Band& B,
                      const std::vector<int32_t>& colour_of_patch, int ncolours, ExactHost& out,
                      std::string& err) {
  const int np = 2 * k - 1;
  int nloc = 1;
  for (int a = 0; a < d; ++a) nloc *= np;
  out = ExactHost();
  out.nloc = nloc;
  const int64_t n = k * N - 1;
  out.off.resize(nloc);
  for (int e = 0; e < nloc; ++e) {
    int64_t o = 0, s = 1;
    int q = e;
    for (int a = 0; a < d; ++a) { o += int64_t(q % np) * s; q /= np; s *= n; }
    out.off[e] = o;
  }
  // group patches by variant tuple
  int64_t npatch = 1;
  for (int a = 0; a < d; ++a) npatch *= (N - 1);
  std::vector<int> tuple_of(npatch);
  std::vector<int> slot(64, -1);
  for (int64_t p = 0; p < npatch; ++p) {
    int64_t q = p;
    int t = 0;
    for (int a = 0, m = 1; a < d; ++a, m *= 4) { t += axis_variant(1 + q % (N - 1), N) * m; q /= (N - 1); }
    tuple_of[p] = t;
    if (slot[t] < 0) { slot[t] = (int)out.tuples.size(); out.tuples.push_back(t); }
  }
  const int nt = (int)out.tuples.size();
  out.all.assign(nt, {});
  out.by_color.assign(ncolours, std::vector<std::vector<int32_t>>(nt));
  for (int64_t p = 0; p < npatch; ++p) {
    out.all[slot[tuple_of[p]]].push_back((int32_t)p);
    out.by_color[colour_of_patch[p]][slot[tuple_of[p]]].push_back((int32_t)p);
  }
  // dense A_v = sum of Kronecker terms of the 1D patch blocks, inverted per tuple.
  out.inv.assign(nt, {});
  for (int ti = 0; ti < nt; ++ti) {
    const int t = out.tuples[ti];
    std::vector<double> Mb[3], Lb[3], Bb[3];
    for (int a = 0; a < d; ++a) {
      const int var = (t >> (2 * a)) & 3;
      const int64_t v = rep_vertex(var, N);
      Mb[a] = block1d(M, k, v); Lb[a] = block1d(L, k, v); Bb[a] = block1d(B, k, v);
    }
    std::vector<double> A(size_t(nloc) * nloc, 0.0);
    for (int e = 0; e < nloc; ++e)
      for (int f = 0; f < nloc; ++f) {
        int ie[3] = {e % np, (e / np) % np, e / (np * np)}, jf[3] = {f % np, (f / np) % np, f / (np * np)};
        auto m = [&](const std::vector<double>* X, int a) { return X[a][ie[a] * np + jf[a]]; };
        double val;
        if (d == 2) {
          val = m(Mb, 1) * m(Bb, 0) + 2.0 * m(Lb, 1) * m(Lb, 0) + m(Bb, 1) * m(Mb, 0);
        } else {
          val = m(Mb, 2) * m(Mb, 1) * m(Bb, 0) + m(Mb, 2) * m(Bb, 1) * m(Mb, 0) + m(Bb, 2) * m(Mb, 1) * m(Mb, 0) +
                2.0 * (m(Mb, 2) * m(Lb, 1) * m(Lb, 0) + m(Lb, 2) * m(Lb, 1) * m(Mb, 0) + m(Lb, 2) * m(Mb, 1) * m(Lb, 0));
        }
        A[size_t(e) * nloc + f] = val;
      }
    if (!spd_inverse(nloc, A)) {
      err = "exact patch matrix A_v not positive definite";
      return false;
    }
    out.inv[ti] = std::move(A);
  }
  return true;
}

}  // namespace c0ip
