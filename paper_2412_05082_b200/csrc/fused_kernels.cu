// Fused tile kernels for large 2D levels (sm_100a, FP64 and FP32).
//
// Two kernels make one additive smoothing step:
//   apply2d  : r = b - A x  (or y = A x) for a tile of C x C cells, all 1D contractions of the
//              Kronecker sum A = h^-2 (M^_y B^_x + 2 L^_y L^_x + B^_y M^_x) done
//              in shared memory on a halo'd box of x;
//   fdm2d    : x += omega h^2 sum_v R_v^T A^~_v^{-1} R_v r for the same tile,
//              written as a GATHER: the patch-eigenbasis transform S^T R_v is shared by all
//              patches of a patch row, every owned DoF sums its <= 4 patch corrections in a
//              fixed order (deterministic, no atomics), and the result is stored once.
// Work is organised so that every lane of a warp applies the *same* coefficients (same class
// p = j mod k of the output node, or same patch axis variant): the coefficients live in the
// kernel parameter bank (__grid_constant__) and feed DFMA/FFMA as constant-bank operands.
// Tiles touching the domain boundary take a uniform per-warp branch to the one-sided face rows
// and the left/right patch variants.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <vector>

#include <type_traits>

#include "fused_dispatch.hpp"

namespace c0ip {

// ----------------------------------------------------------------------------- constants
template <typename T, int K>
struct Coef2 {
  static constexpr int NP = 2 * K - 1;
  T BI[K][4 * K + 1];       // interior class p: B row, column offsets -2K..2K
  T MI[K][2 * K + 1];       // offsets -K..K
  T LI[K][2 * K + 1];
  T BS[2 * K][4 * K + 1];   // special rows: [0,K) nodes j=1..K ; [K,2K) nodes j=KN-K..KN-1
  T MS[2 * K][4 * K + 1];   // (offsets -2K..2K, zero padded)
  T LS[2 * K][4 * K + 1];
  T S[3][NP * NP];          // patch eigenvectors, variants 0 left / 1 interior / 2 right: S[l*NP+i]
  T lam[3][NP];
};

template <typename T, int K>
struct ApplyP {
  Coef2<T, K> c;
  const T* x;
  const T* b;               // nullptr: y = A x
  T* y;
  int64_t N, n;             // cells, 1D interior dofs (n = KN-1)
  T scale;                  // h^-2
};

template <typename T, int K>
struct FdmP {
  Coef2<T, K> c;
  const T* r;
  T* x;
  int64_t N, n;
  T factor;                 // omega * h^2
};

template <int K>
struct Tile {
  // cells per tile edge: ~32 owned nodes per axis
  static constexpr int C = (K == 2) ? 16 : (K == 3) ? 10 : (K == 4) ? 8 : (K == 5) ? 6 : (K == 6) ? 5 : 4;
  static constexpr int O = C * K;
};

__host__ __device__ constexpr int odd(int v) { return v | 1; }

// ----------------------------------------------------------------------------- banded rows
// B row of an output node of class P (j = cK + P): w[0] <-> node (c-2)K, columns j-2K..j+2K.
// Structural zeros (column outside the support of row P) are skipped at compile time.
template <typename T, int K, int P, typename F>
__device__ __forceinline__ T rowB(F coef, const T* w) {
  T s = 0;
#pragma unroll
  for (int q = 0; q <= 4 * K; ++q)
    if (P == 0 || (q >= K - P && q <= 4 * K - P)) s = fma(coef(q), w[P + q], s);
  return s;
}
// M or L row (bandwidth K): w2[0] <-> node (c-1)K, coefficient index q <-> column j - K + q.
template <typename T, int K, int P, typename F>
__device__ __forceinline__ T rowML(F coef, const T* w2) {
  T s = 0;
#pragma unroll
  for (int q = 0; q <= 2 * K; ++q)
    if (P == 0 || (q >= K - P && q <= 2 * K - P)) s = fma(coef(q), w2[P + q], s);
  return s;
}

// x-stage of one output node: (B^ x, L^ x, M^ x) for class P, interior (s < 0) or special row s
template <typename T, int K, int P>
__device__ __forceinline__ void stage_x_node(const Coef2<T, K>& c, int s, const T* w, T& b, T& l, T& m) {
  if (s < 0) {
    b = rowB<T, K, P>([&](int q) { return c.BI[P][q]; }, w);
    l = rowML<T, K, P>([&](int q) { return c.LI[P][q]; }, w + K);
    m = rowML<T, K, P>([&](int q) { return c.MI[P][q]; }, w + K);
  } else {
    b = rowB<T, K, P>([&](int q) { return c.BS[s][q]; }, w);
    l = rowML<T, K, P>([&](int q) { return c.LS[s][q + K]; }, w + K);
    m = rowML<T, K, P>([&](int q) { return c.MS[s][q + K]; }, w + K);
  }
}

// y-stage of one output node: B^(wM) + M^(wB) + 2 L^(wL)   (wB2/wL2: base (c-1)K)
template <typename T, int K, int P>
__device__ __forceinline__ T stage_y_node(const Coef2<T, K>& c, int s, const T* wM, const T* wB2, const T* wL2) {
  if (s < 0)
    return rowB<T, K, P>([&](int q) { return c.BI[P][q]; }, wM) +
           rowML<T, K, P>([&](int q) { return c.MI[P][q]; }, wB2) +
           T(2) * rowML<T, K, P>([&](int q) { return c.LI[P][q]; }, wL2);
  return rowB<T, K, P>([&](int q) { return c.BS[s][q]; }, wM) +
         rowML<T, K, P>([&](int q) { return c.MS[s][q + K]; }, wB2) +
         T(2) * rowML<T, K, P>([&](int q) { return c.LS[s][q + K]; }, wL2);
}

// compile-time dispatch of a runtime-unrolled class index p (p is a constant after unrolling)
template <int K, typename F>
__device__ __forceinline__ void with_p(int p, F f) {
  switch (p) {
    case 0: if constexpr (0 < K) f(std::integral_constant<int, 0>{}); break;
    case 1: if constexpr (1 < K) f(std::integral_constant<int, 1>{}); break;
    case 2: if constexpr (2 < K) f(std::integral_constant<int, 2>{}); break;
    case 3: if constexpr (3 < K) f(std::integral_constant<int, 3>{}); break;
    case 4: if constexpr (4 < K) f(std::integral_constant<int, 4>{}); break;
    case 5: if constexpr (5 < K) f(std::integral_constant<int, 5>{}); break;
    case 6: if constexpr (6 < K) f(std::integral_constant<int, 6>{}); break;
  }
}

// special-row index of node j, or -1 for an interior-class row
template <int K>
__device__ __forceinline__ int special_row(int64_t j, int64_t N) {
  if (j <= K) return int(j - 1);
  if (j >= K * N - K) return int(K + (j - (K * N - K)));
  return -1;
}

// ----------------------------------------------------------------------------- apply2d
template <typename T, int K>
__global__ void __launch_bounds__(256) apply2d_kernel(const __grid_constant__ ApplyP<T, K> P) {
  constexpr int C = Tile<K>::C, O = Tile<K>::O;
  constexpr int BW = (C + 3) * K + 1;       // box: nodes [(c0-2)K, (c0+C+1)K]
  constexpr int PX = odd(BW), PO = odd(O);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* xb = reinterpret_cast<T*>(smem_raw);
  T* sB = xb + BW * PX;
  T* sL = sB + BW * PO;
  T* sM = sL + BW * PO;
  const int64_t N = P.N, n = P.n, KN = K * N;
  const int64_t cx0 = (int64_t)blockIdx.x * C, cy0 = (int64_t)blockIdx.y * C;
  const int64_t X0 = (cx0 - 2) * K, Y0 = (cy0 - 2) * K;
  const int tid = threadIdx.x;

  for (int e = tid; e < BW * BW; e += blockDim.x) {
    const int r = e / BW, cc = e % BW;
    const int64_t jy = Y0 + r, jx = X0 + cc;
    T v = 0;
    if (jx >= 1 && jx <= KN - 1 && jy >= 1 && jy <= KN - 1) v = P.x[(jy - 1) * n + (jx - 1)];
    xb[r * PX + cc] = v;
  }
  __syncthreads();

  // x-stage: B^_x x, L^_x x, M^_x x on all box rows, owned columns.  lanes <-> rows.
  for (int u = tid; u < BW * C; u += blockDim.x) {
    const int r = u % BW, ci = u / BW;
    const int64_t cx = cx0 + ci;
    if (cx >= N) continue;
    T w[4 * K + 1];
#pragma unroll
    for (int q = 0; q <= 4 * K; ++q) w[q] = xb[r * PX + ci * K + q];
    T ob[K], ol[K], om[K];
    const bool inner = (cx >= 2 && cx <= N - 2);
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const int s = inner ? -1 : special_row<K>(cx * K + p, N);
      with_p<K>(p, [&](auto PC) {
        constexpr int PP = decltype(PC)::value;
        stage_x_node<T, K, PP>(P.c, s, w, ob[PP], ol[PP], om[PP]);
      });
    }
#pragma unroll
    for (int p = 0; p < K; ++p) {
      sB[r * PO + ci * K + p] = ob[p];
      sL[r * PO + ci * K + p] = ol[p];
      sM[r * PO + ci * K + p] = om[p];
    }
  }
  __syncthreads();

  // y-stage: y = h^-2 (M^_y (B^_x x) + 2 L^_y (L^_x x) + B^_y (M^_x x)).  lanes <-> columns.
  for (int u = tid; u < O * C; u += blockDim.x) {
    const int col = u % O, ci = u / O;
    const int64_t cy = cy0 + ci;
    const int64_t jx = cx0 * K + col;
    if (cy >= N || jx < 1 || jx > KN - 1) continue;
    T wM[4 * K + 1], wB[2 * K + 1], wL[2 * K + 1];
#pragma unroll
    for (int q = 0; q <= 4 * K; ++q) wM[q] = sM[(ci * K + q) * PO + col];
#pragma unroll
    for (int q = 0; q <= 2 * K; ++q) {
      wB[q] = sB[(ci * K + K + q) * PO + col];
      wL[q] = sL[(ci * K + K + q) * PO + col];
    }
    const bool inner = (cy >= 2 && cy <= N - 2);
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const int64_t j = cy * K + p;
      if (j < 1 || j > KN - 1) continue;
      const int s = inner ? -1 : special_row<K>(j, N);
      T v = 0;
      with_p<K>(p, [&](auto PC) {
        constexpr int PP = decltype(PC)::value;
        v = stage_y_node<T, K, PP>(P.c, s, wM, wB, wL);
      });
      const int64_t g = (j - 1) * n + (jx - 1);
      v *= P.scale;
      P.y[g] = P.b ? P.b[g] - v : v;
    }
  }
}

// ----------------------------------------------------------------------------- fdm2d
__device__ __forceinline__ int variant_of(int64_t v, int64_t N) { return v == 1 ? 0 : (v == N - 1 ? 2 : 1); }

// z[i] = sum_l S[l][i] w[l]   (S^T w)
template <typename T, int K, int V>
__device__ __forceinline__ void s_t(const Coef2<T, K>& c, const T* w, T* z) {
  constexpr int NP = 2 * K - 1;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    T s = 0;
#pragma unroll
    for (int l = 0; l < NP; ++l) s = fma(c.S[V][l * NP + i], w[l], s);
    z[i] = s;
  }
}

// acc[l] += sum_i S[l][i] z[i]   (S z)
template <typename T, int K, int V>
__device__ __forceinline__ void s_n(const Coef2<T, K>& c, const T* z, T* acc) {
  constexpr int NP = 2 * K - 1;
#pragma unroll
  for (int l = 0; l < NP; ++l) {
    T s = acc[l];
#pragma unroll
    for (int i = 0; i < NP; ++i) s = fma(c.S[V][l * NP + i], z[i], s);
    acc[l] = s;
  }
}

// out[p] += sum_i S[OFF + p][i] z[i] for p in [P0, K)  (rows OFF+p of patch-local index)
template <typename T, int K, int V, int OFF, int P0>
__device__ __forceinline__ void s_rows(const Coef2<T, K>& c, const T* z, T* out) {
  constexpr int NP = 2 * K - 1;
#pragma unroll
  for (int p = P0; p < K; ++p) {
    T s = out[p];
#pragma unroll
    for (int i = 0; i < NP; ++i) s = fma(c.S[V][(OFF + p) * NP + i], z[i], s);
    out[p] = s;
  }
}

template <typename T, int K>
__global__ void __launch_bounds__(256) fdm2d_kernel(const __grid_constant__ FdmP<T, K> P) {
  constexpr int C = Tile<K>::C, O = Tile<K>::O, NP = 2 * K - 1;
  constexpr int RN = (C + 2) * K - 1;          // residual box: nodes [(c0-1)K+1, (c0+C+1)K-1]
  constexpr int E = (C + 1) * NP;              // patch-eigen columns: patches c0 .. c0+C
  constexpr int PR = odd(RN), PE = odd(E), PS = odd(O);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* rb = reinterpret_cast<T*>(smem_raw);      // [RN][PR]   (later: out staging [O][PS])
  T* z1 = rb + RN * PR;                        // [RN][PE]
  T* z3 = z1 + RN * PE;                        // [O][PE]
  const int64_t N = P.N, n = P.n, KN = K * N;
  const int64_t cx0 = (int64_t)blockIdx.x * C, cy0 = (int64_t)blockIdx.y * C;
  const int64_t X0 = (cx0 - 1) * K + 1, Y0 = (cy0 - 1) * K + 1;
  const int tid = threadIdx.x;

  for (int e = tid; e < RN * RN; e += blockDim.x) {
    const int r = e / RN, cc = e % RN;
    const int64_t jy = Y0 + r, jx = X0 + cc;
    T v = 0;
    if (jx >= 1 && jx <= KN - 1 && jy >= 1 && jy <= KN - 1) v = P.r[(jy - 1) * n + (jx - 1)];
    rb[r * PR + cc] = v;
  }
  __syncthreads();

  // FX: Z1[y][v_x, i] = sum_l S_vx[l][i] r[y][(vx-1)K+1+l]   lanes <-> rows, same patch
  for (int u = tid; u < RN * (C + 1); u += blockDim.x) {
    const int r = u % RN, pi = u / RN;
    const int64_t vx = cx0 + pi;
    T z[NP];
    if (vx >= 1 && vx <= N - 1) {
      T w[NP];
#pragma unroll
      for (int l = 0; l < NP; ++l) w[l] = rb[r * PR + pi * K + l];
      const int var = variant_of(vx, N);
      if (var == 1) s_t<T, K, 1>(P.c, w, z);
      else if (var == 0) s_t<T, K, 0>(P.c, w, z);
      else s_t<T, K, 2>(P.c, w, z);
    } else {
#pragma unroll
      for (int i = 0; i < NP; ++i) z[i] = 0;
    }
#pragma unroll
    for (int i = 0; i < NP; ++i) z1[r * PE + pi * NP + i] = z[i];
  }
  __syncthreads();

  // FY: per column (vx, i_x): march over patch rows vy = cy0..cy0+C: gather S_vy^T, divide by
  // lambda_vy + lambda_vx, scatter S_vy into row accumulators; emit completed owned rows.
  for (int col = tid; col < E; col += blockDim.x) {
    const int pi = col / NP, ix = col % NP;
    const int64_t vx = cx0 + pi;
    const bool vx_ok = (vx >= 1 && vx <= N - 1);
    const int varx = vx_ok ? variant_of(vx, N) : 1;
    const T lx = P.c.lam[varx][ix];
    T inv1[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) inv1[i] = T(1) / (P.c.lam[1][i] + lx);
    T acc[NP];
#pragma unroll
    for (int l = 0; l < NP; ++l) acc[l] = 0;
    for (int qi = 0; qi <= C; ++qi) {
      const int64_t vy = cy0 + qi;
      if (vx_ok && vy >= 1 && vy <= N - 1) {
        T w[NP], z[NP];
#pragma unroll
        for (int l = 0; l < NP; ++l) w[l] = z1[(qi * K + l) * PE + col];
        const int vary = variant_of(vy, N);
        if (vary == 1) {
          s_t<T, K, 1>(P.c, w, z);
#pragma unroll
          for (int i = 0; i < NP; ++i) z[i] *= inv1[i];
          s_n<T, K, 1>(P.c, z, acc);
        } else if (vary == 0) {
          s_t<T, K, 0>(P.c, w, z);
#pragma unroll
          for (int i = 0; i < NP; ++i) z[i] /= (P.c.lam[0][i] + lx);
          s_n<T, K, 0>(P.c, z, acc);
        } else {
          s_t<T, K, 2>(P.c, w, z);
#pragma unroll
          for (int i = 0; i < NP; ++i) z[i] /= (P.c.lam[2][i] + lx);
          s_n<T, K, 2>(P.c, z, acc);
        }
      }
      // rows (vy-1)K+1 .. vy K are complete: emit the owned ones, then shift by K
#pragma unroll
      for (int l = 0; l < K; ++l) {
        const int64_t ny = (vy - 1) * K + 1 + l;
        const int64_t o = ny - cy0 * K;
        if (o >= 0 && o < O) z3[o * PE + col] = acc[l];
      }
#pragma unroll
      for (int l = 0; l < NP; ++l) acc[l] = (l + K < NP) ? acc[l + K] : T(0);
    }
  }
  __syncthreads();

  // FS: out[y][cx K + p] = sum_i S_cx[K-1+p][i] Z3[y][cx][i] + sum_i S_{cx+1}[p-1][i] Z3[y][cx+1][i]
  T* outs = rb;                                  // [O][PS] staging (rb is dead)
  for (int u = tid; u < O * C; u += blockDim.x) {
    const int oy = u % O, ci = u / O;
    const int64_t cx = cx0 + ci;
    T out[K];
#pragma unroll
    for (int p = 0; p < K; ++p) out[p] = 0;
    if (cx < N) {
      T z0[NP], z1v[NP];
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        z0[i] = z3[oy * PE + ci * NP + i];
        z1v[i] = z3[oy * PE + (ci + 1) * NP + i];
      }
      if (cx >= 1) {                       // patch cx: local rows K-1 .. 2K-2
        const int v0 = variant_of(cx, N);
        if (v0 == 1) s_rows<T, K, 1, K - 1, 0>(P.c, z0, out);
        else if (v0 == 0) s_rows<T, K, 0, K - 1, 0>(P.c, z0, out);
        else s_rows<T, K, 2, K - 1, 0>(P.c, z0, out);
      }
      if (cx + 1 <= N - 1) {               // patch cx+1: local rows p-1 for p >= 1
        const int v1 = variant_of(cx + 1, N);
        if (v1 == 1) s_rows<T, K, 1, -1, 1>(P.c, z1v, out);
        else if (v1 == 0) s_rows<T, K, 0, -1, 1>(P.c, z1v, out);
        else s_rows<T, K, 2, -1, 1>(P.c, z1v, out);
      }
    }
#pragma unroll
    for (int p = 0; p < K; ++p) outs[oy * PS + ci * K + p] = out[p];
  }
  __syncthreads();

  for (int e = tid; e < O * O; e += blockDim.x) {
    const int oy = e / O, ox = e % O;
    const int64_t jy = cy0 * K + oy, jx = cx0 * K + ox;
    if (jx < 1 || jx > KN - 1 || jy < 1 || jy > KN - 1) continue;
    const int64_t g = (jy - 1) * n + (jx - 1);
    P.x[g] = fma(P.factor, outs[oy * PS + ox], P.x[g]);
  }
}

// ----------------------------------------------------------------------------- host side
struct FusedLevel {
  int d = 0, k = 0;
  int64_t N = 0, n = 0;
  double h = 0;
  std::vector<double> c64;   // serialized Coef2<double,K> (reference scale)
  std::vector<float> c32;
};

void FusedLevelDeleter::operator()(FusedLevel* p) const { delete p; }

template <typename T, int K>
static void fill_coef(const FusedLevel& F, const RefData& ref, Coef2<T, K>& c) {
  Band M, L, B, Mf, Lf, Bf;
  global_bands(ref, F.N, M, L, B);            // reference scale (h = 1), eliminated (for the FDM)
  global_bands(ref, F.N, Mf, Lf, Bf, false);  // all nodes: rows indexed by node j
  std::memset(&c, 0, sizeof(c));
  const int hw = 2 * K;
  for (int p = 0; p < K; ++p) {
    const int64_t i = 2 * K + p;              // node j = 2K + p (class p): faces 1..3 interior, N >= 4
    for (int q = 0; q <= 4 * K; ++q) c.BI[p][q] = (T)Bf.at(i, i + q - hw);
    for (int q = 0; q <= 2 * K; ++q) {
      c.MI[p][q] = (T)Mf.at(i, i + q - K);
      c.LI[p][q] = (T)Lf.at(i, i + q - K);
    }
  }
  const int64_t KN = K * F.N;
  for (int s = 0; s < 2 * K; ++s) {
    const int64_t j = (s < K) ? (s + 1) : (KN - K + (s - K));   // node index = full-band row
    for (int q = 0; q <= 4 * K; ++q) {
      c.BS[s][q] = (T)Bf.at(j, j + q - hw);
      c.MS[s][q] = (T)Mf.at(j, j + q - hw);
      c.LS[s][q] = (T)Lf.at(j, j + q - hw);
    }
  }
  Fdm fr;
  std::string err;
  if (!make_fdm(ref, F.N, M, L, B, fr, err)) throw std::runtime_error("coercivity: " + err);
  constexpr int NP = 2 * K - 1;
  for (int v = 0; v < 3; ++v)
    for (int i = 0; i < NP * NP; ++i) c.S[v][i] = (T)fr.S[v][i];
  for (int v = 0; v < 3; ++v)
    for (int i = 0; i < NP; ++i) c.lam[v][i] = (T)fr.lam[v][i];
}

template <int K>
static void build_coefs(FusedLevel& F, const RefData& ref) {
  Coef2<double, K> c64;
  Coef2<float, K> c32;
  fill_coef<double, K>(F, ref, c64);
  fill_coef<float, K>(F, ref, c32);
  F.c64.assign(reinterpret_cast<const double*>(&c64), reinterpret_cast<const double*>(&c64) + sizeof(c64) / sizeof(double));
  F.c32.assign(reinterpret_cast<const float*>(&c32), reinterpret_cast<const float*>(&c32) + sizeof(c32) / sizeof(float));
}

std::unique_ptr<FusedLevel, FusedLevelDeleter> make_fused_level_impl(int d, int k, int64_t N, const RefData& ref,
                                                                     const Fdm&, double h) {
  if (d != 2 || N < 8 || k < 2 || k > 7) return nullptr;
  if (std::getenv("C0IP_DISABLE_FUSED")) return nullptr;
  std::unique_ptr<FusedLevel, FusedLevelDeleter> F(new FusedLevel());
  F->d = d; F->k = k; F->N = N; F->n = k * N - 1; F->h = h;
  switch (k) {
    case 2: build_coefs<2>(*F, ref); break;
    case 3: build_coefs<3>(*F, ref); break;
    case 4: build_coefs<4>(*F, ref); break;
    case 5: build_coefs<5>(*F, ref); break;
    case 6: build_coefs<6>(*F, ref); break;
    case 7: build_coefs<7>(*F, ref); break;
  }
  return F;
}

template <typename T>
static const std::vector<T>& coef_of(const FusedLevel& F);
template <>
const std::vector<double>& coef_of<double>(const FusedLevel& F) { return F.c64; }
template <>
const std::vector<float>& coef_of<float>(const FusedLevel& F) { return F.c32; }

template <typename T, int K>
static void launch_apply(const FusedLevel& F, const T* x, const T* b, T* y, cudaStream_t st) {
  constexpr int C = Tile<K>::C, O = Tile<K>::O;
  constexpr int BW = (C + 3) * K + 1;
  const size_t smem = sizeof(T) * (size_t(BW) * odd(BW) + 3 * size_t(BW) * odd(O));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(apply2d_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  ApplyP<T, K> p;
  std::memcpy(&p.c, coef_of<T>(F).data(), sizeof(p.c));
  p.x = x; p.b = b; p.y = y; p.N = F.N; p.n = F.n;
  p.scale = T(1.0 / (F.h * F.h));
  const unsigned g = unsigned((F.N + C - 1) / C);
  apply2d_kernel<T, K><<<dim3(g, g), 256, smem, st>>>(p);
}

template <typename T, int K>
static void launch_fdm(const FusedLevel& F, T omega, const T* r, T* x, cudaStream_t st) {
  constexpr int C = Tile<K>::C, O = Tile<K>::O, NP = 2 * K - 1;
  constexpr int RN = (C + 2) * K - 1, E = (C + 1) * NP;
  const size_t smem = sizeof(T) * (size_t(RN) * odd(RN) + size_t(RN) * odd(E) + size_t(O) * odd(E));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fdm2d_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  FdmP<T, K> p;
  std::memcpy(&p.c, coef_of<T>(F).data(), sizeof(p.c));
  p.r = r; p.x = x; p.N = F.N; p.n = F.n;
  p.factor = T(double(omega) * F.h * F.h);
  const unsigned g = unsigned((F.N + C - 1) / C);
  fdm2d_kernel<T, K><<<dim3(g, g), 256, smem, st>>>(p);
}

template <typename T>
bool fused_apply(FusedLevel& F, const T* x, const T* b, T* y, cudaStream_t st, int64_t* launches) {
  if (F.d != 2) return false;
  switch (F.k) {
    case 2: launch_apply<T, 2>(F, x, b, y, st); break;
    case 3: launch_apply<T, 3>(F, x, b, y, st); break;
    case 4: launch_apply<T, 4>(F, x, b, y, st); break;
    case 5: launch_apply<T, 5>(F, x, b, y, st); break;
    case 6: launch_apply<T, 6>(F, x, b, y, st); break;
    case 7: launch_apply<T, 7>(F, x, b, y, st); break;
    default: return false;
  }
  (*launches)++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("fused apply2d launch: ") + cudaGetErrorString(e));
  return true;
}

template <typename T>
bool fused_avs(FusedLevel& F, T omega, const T* b, T* x, T* scratch, cudaStream_t st, int64_t* launches) {
  if (F.d != 2) return false;
  fused_apply<T>(F, x, b, scratch, st, launches);             // r = b - A x (one residual per step)
  switch (F.k) {
    case 2: launch_fdm<T, 2>(F, omega, scratch, x, st); break;
    case 3: launch_fdm<T, 3>(F, omega, scratch, x, st); break;
    case 4: launch_fdm<T, 4>(F, omega, scratch, x, st); break;
    case 5: launch_fdm<T, 5>(F, omega, scratch, x, st); break;
    case 6: launch_fdm<T, 6>(F, omega, scratch, x, st); break;
    case 7: launch_fdm<T, 7>(F, omega, scratch, x, st); break;
    default: return false;
  }
  (*launches)++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("fused fdm2d launch: ") + cudaGetErrorString(e));
  return true;
}

template <typename T>
bool fused_mvs_color(FusedLevel&, int, T, const T*, T*, cudaStream_t, int64_t*) { return false; }

template bool fused_apply<double>(FusedLevel&, const double*, const double*, double*, cudaStream_t, int64_t*);
template bool fused_apply<float>(FusedLevel&, const float*, const float*, float*, cudaStream_t, int64_t*);
template bool fused_avs<double>(FusedLevel&, double, const double*, double*, double*, cudaStream_t, int64_t*);
template bool fused_avs<float>(FusedLevel&, float, const float*, float*, float*, cudaStream_t, int64_t*);
template bool fused_mvs_color<double>(FusedLevel&, int, double, const double*, double*, cudaStream_t, int64_t*);
template bool fused_mvs_color<float>(FusedLevel&, int, float, const float*, float*, cudaStream_t, int64_t*);

}  // namespace c0ip
