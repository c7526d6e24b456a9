// Shared device helpers of the fused tile kernels (2D: fused_kernels.cu, 3D: fused3d.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>
#include <vector>

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
  int zero;                 // 0 at run time (opaque to the compiler)
  int64_t row0, lrows;      // slab window: local row 0 = global interior row row0; lrows rows held
  int64_t out_lo, out_hi;   // node rows j (= interior row + 1) to write, [out_lo, out_hi)
  int chunk;                // apply2d: tile rows per column chunk
};

template <typename T, int K>
struct FdmP {
  Coef2<T, K> c;
  const T* r;
  T* x;
  int64_t N, n;
  T factor;                 // omega * h^2
  int zero;
  int64_t row0, lrows;      // slab window (see ApplyP)
  int64_t out_lo, out_hi;
};

template <typename T, int K>
struct MvsP {
  Coef2<T, K> c;
  T* x;
  const T* b;
  const int32_t* list;      // patch ids of the colour
  int64_t count;
  int64_t N, n;
  T scale;                  // h^-2  (A = h^-2 A^)
  T factor;                 // omega h^2 (A~^-1 = h^2 A^~^-1)
  int zero;
};

template <int K>
struct Tile {
  // cells per tile edge: ~32 owned nodes per axis
  static constexpr int C = (K == 2) ? 16 : (K == 3) ? 10 : (K == 4) ? 8 : (K == 5) ? 6 : (K == 6) ? 5 : 4;
  static constexpr int O = C * K;
};

template <typename T, int K>
struct Blk {
  // maximum register-blocking factor (lines per thread sharing one coefficient load)
  static constexpr int RB = (sizeof(T) == 8) ? (K <= 3 ? 3 : (K <= 5 ? 2 : 1)) : (K <= 5 ? 3 : 2);
};

__host__ __device__ constexpr int odd(int v) { return v | 1; }
__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }

template <typename T, int K>
__device__ __forceinline__ const Coef2<T, K>& coef_at(const Coef2<T, K>& c, int off) {
  return *reinterpret_cast<const Coef2<T, K>*>(reinterpret_cast<const char*>(&c) + off);
}

// compile-time dispatch of an unrolled index p (p is a constant after unrolling)
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

__device__ __forceinline__ int variant_of(int64_t v, int64_t N) { return v == 1 ? 0 : (v == N - 1 ? 2 : 1); }

// ----------------------------------------------------------------------------- banded rows (RB lines)
// B row of an output node of class P (j = cK + P): w[r][0] <-> node (c-2)K; columns j-2K..j+2K.
// acc[r] += sum_q coef(q) w[r][P+q]; structural zeros skipped at compile time.
template <typename T, int K, int P, int RB, int W, typename F>
__device__ __forceinline__ void rowB(F coef, const T (&w)[RB][W], int wofs, T (&acc)[RB]) {
#pragma unroll
  for (int q = 0; q <= 4 * K; ++q) {
    if (P == 0 || (q >= K - P && q <= 4 * K - P)) {
      const T cq = coef(q);
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[r] = fma(cq, w[r][wofs + P + q], acc[r]);
    }
  }
}
// M or L row (bandwidth K): w[r][wofs] <-> node (c-1)K; coefficient q <-> column j - K + q.
template <typename T, int K, int P, int RB, int W, typename F>
__device__ __forceinline__ void rowML(F coef, const T (&w)[RB][W], int wofs, T (&acc)[RB]) {
#pragma unroll
  for (int q = 0; q <= 2 * K; ++q) {
    if (P == 0 || (q >= K - P && q <= 2 * K - P)) {
      const T cq = coef(q);
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[r] = fma(cq, w[r][wofs + P + q], acc[r]);
    }
  }
}

// ----------------------------------------------------------------------------- interior rows, all classes
// acc[r] += c * w[r][o] over the RB lines of a thread; FP32 pairs go through the packed FFMA2 (f32x2
// FMA with a scalar uniform operand on sm_100a: two FMAs per issue slot)
template <typename T, int RB, int W>
__device__ __forceinline__ void fma_rb(T c, const T (&w)[RB][W], int o, T (&acc)[RB]) {
  if constexpr (std::is_same<T, float>::value && RB >= 2) {
#pragma unroll
    for (int r = 0; r + 1 < RB; r += 2) {
      const float2 v = __ffma2_rn(make_float2(c, c), make_float2(w[r][o], w[r + 1][o]),
                                  make_float2(acc[r], acc[r + 1]));
      acc[r] = v.x;
      acc[r + 1] = v.y;
    }
    if constexpr (RB % 2 == 1) acc[RB - 1] = fmaf(c, w[RB - 1][o], acc[RB - 1]);
  } else {
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = fma(c, w[r][o], acc[r]);
  }
}

// Interior rows of all K classes of one cell at once, window index outermost so that every DFMA
// of an accumulator is separated by the other 3K*RB (or K*RB) accumulators (ILP), coefficients
// shared by the RB lines.  w[r][o] <-> node (c-2)K + o.
template <typename T, int K, int RB>
__device__ __forceinline__ void x_all_interior(const Coef2<T, K>& c, const T (&w)[RB][4 * K + 1], T (&ob)[K][RB],
                                               T (&ol)[K][RB], T (&om)[K][RB]) {
#pragma unroll
  for (int p = 0; p < K; ++p)
#pragma unroll
    for (int r = 0; r < RB; ++r) ob[p][r] = ol[p][r] = om[p][r] = 0;
#pragma unroll
  for (int o = 0; o <= 4 * K; ++o)
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const int q = o - p;                           // B coefficient index (offset q - 2K)
      if (q >= 0 && q <= 4 * K && (p == 0 || (q >= K - p && q <= 4 * K - p))) {
        fma_rb<T, RB>(c.BI[p][q], w, o, ob[p]);
      }
      const int qm = o - p - K;                      // M/L coefficient index (offset qm - K)
      if (qm >= 0 && qm <= 2 * K && (p == 0 || (qm >= K - p && qm <= 2 * K - p))) {
        fma_rb<T, RB>(c.LI[p][qm], w, o, ol[p]);
        fma_rb<T, RB>(c.MI[p][qm], w, o, om[p]);
      }
    }
}

// acc[p][r] += sum over the band of class p: WHICH 0 = B (window 4K+1, base (c-2)K), 1 = M, 2 = L
// (window 2K+1, base (c-1)K); window index outermost.
template <typename T, int K, int RB, int WHICH, int W>
__device__ __forceinline__ void y_all_interior(const Coef2<T, K>& c, const T (&w)[RB][W], T (&acc)[K][RB]) {
#pragma unroll
  for (int o = 0; o < W; ++o)
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const int q = o - p;
      const bool ok = (WHICH == 0) ? (q >= 0 && q <= 4 * K && (p == 0 || (q >= K - p && q <= 4 * K - p)))
                                   : (q >= 0 && q <= 2 * K && (p == 0 || (q >= K - p && q <= 2 * K - p)));
      if (ok) {
        fma_rb<T, RB>((WHICH == 0) ? c.BI[p][q] : (WHICH == 1 ? c.MI[p][q] : c.LI[p][q]), w, o, acc[p]);
      }
    }
}

// ----------------------------------------------------------------------------- async copies
// cp.async (LDGSTS) element copies global -> shared with zero fill (src-size 0) for the nodes
// outside the interior (the eliminated clamped-boundary nodes).
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? (int)sizeof(T) : 0;
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// ROWS x COLS box of nodes starting at node (Y0, X0) into smem with row pitch PITCH.  Global node
// rows are held in a slab window: node row jy lives at local interior row jy - 1 - row0, valid for
// local rows [0, lrows); everything else (clamped boundary, outside the window) is zero-filled.
template <typename T, int ROWS, int COLS, int PITCH>
__device__ __forceinline__ void load_box_async(T* dst, const T* src, int64_t n, int64_t KN, int64_t Y0,
                                               int64_t X0, int64_t row0, int64_t lrows) {
  const int64_t ylo = (row0 + 1 > 1) ? row0 + 1 : int64_t(1), yhi = (row0 + lrows < KN - 1) ? row0 + lrows : KN - 1;
  const bool inner = (X0 >= 1 && X0 + COLS - 1 <= KN - 1 && Y0 >= ylo && Y0 + ROWS - 1 <= yhi);
  const T* base = src + (Y0 - 1 - row0) * n + (X0 - 1);
  if (inner) {
    for (int e = threadIdx.x; e < ROWS * COLS; e += blockDim.x) {
      const int r = e / COLS, c = e - (e / COLS) * COLS;
      cp_async_elem(dst + r * PITCH + c, base + (int64_t)r * n + c, true);
    }
  } else {
    for (int e = threadIdx.x; e < ROWS * COLS; e += blockDim.x) {
      const int r = e / COLS, c = e - (e / COLS) * COLS;
      const int64_t jy = Y0 + r, jx = X0 + c;
      const bool ok = (jx >= 1 && jx <= KN - 1 && jy >= ylo && jy <= yhi);
      cp_async_elem(dst + r * PITCH + c, ok ? base + (int64_t)r * n + c : src, ok);
    }
  }
}

template <typename T, int ROWS, int COLS, int PITCH>
__device__ __forceinline__ void load_box_rows_async(T* dst, const T* src, int64_t n, int64_t KN, int64_t Y0,
                                               int64_t X0, int64_t row0, int64_t lrows) {
  // one warp per box row, lanes along the row (no per-element index division)
  const int64_t ylo = (row0 + 1 > 1) ? row0 + 1 : int64_t(1), yhi = (row0 + lrows < KN - 1) ? row0 + lrows : KN - 1;
  const bool xin = (X0 >= 1 && X0 + COLS - 1 <= KN - 1);
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const T* base = src + (Y0 - 1 - row0) * n + (X0 - 1);
  for (int r = threadIdx.x >> 5; r < ROWS; r += nw) {
    const int64_t jy = Y0 + r;
    const bool rok = (jy >= ylo && jy <= yhi);
    const T* rowp = base + (int64_t)r * n;
    T* d = dst + r * PITCH;
    if (rok && xin) {
#pragma unroll
      for (int c = lane; c < COLS; c += 32) cp_async_elem(d + c, rowp + c, true);
    } else {
#pragma unroll
      for (int c = lane; c < COLS; c += 32) {
        const int64_t jx = X0 + c;
        const bool ok = rok && jx >= 1 && jx <= KN - 1;
        cp_async_elem(d + c, ok ? rowp + c : src, ok);
      }
    }
  }
}

// tile rows covering node rows [out_lo, out_hi): ty in [ty0, ty1)
template <int K, int C>
__device__ __forceinline__ void tile_rows(int64_t out_lo, int64_t out_hi, int& ty0, int& ty1) {
  ty0 = int((out_lo / K) / C);
  ty1 = int(((out_hi - 1) / K) / C) + 1;
}

// ----------------------------------------------------------------------------- host-side level data
struct FusedLevel {
  int d = 0, k = 0;
  int64_t N = 0, n = 0;
  double h = 0;
  std::vector<double> c64;   // serialized Coef2<double,K> (reference scale)
  std::vector<float> c32;
};

template <typename T>
inline const std::vector<T>& coef_of(const FusedLevel& F);
template <>
inline const std::vector<double>& coef_of<double>(const FusedLevel& F) { return F.c64; }
template <>
inline const std::vector<float>& coef_of<float>(const FusedLevel& F) { return F.c32; }

}  // namespace c0ip
