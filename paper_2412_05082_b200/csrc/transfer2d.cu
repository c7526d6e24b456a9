// Fused 2D transfer kernels (sm_100a, FP64 / FP32): prolongation-add fine += (E (x) E) coarse and
// restriction coarse = (E^T (x) E^T) fine, with E the natural embedding V_{l-1} -> V_l.
//
// E is translation invariant in the coarse cell: a fine node of class q = j_f mod 2k inside coarse
// cell c takes  E[j_f][c k + m] = pe[q][m]  (m = 0..k, the coarse Lagrange basis at the fine node);
// a coarse node of class pc = j_c mod k gathers  E^T[j_c][2(c-1)k + o] = re[pc][o]  (o = 0..4k)
// from the fine nodes of its support.  The eliminated boundary nodes are zero-filled in the shared
// memory boxes, so no boundary variants exist.  Tiles of C coarse cells per axis, both 1D
// contractions in shared memory, coefficients warp-uniform (lanes <-> lines of the same cell).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "fused_common.cuh"

namespace c0ip {

template <typename T, int K>
struct XferCoef {
  T pe[2 * K][K + 1];
  T re[K][4 * K + 1];
};

template <typename T, int K>
struct XferP {
  XferCoef<T, K> c;
  const T* src;
  T* dst;
  int64_t Nc;               // coarse cells
  int64_t nc, nf;           // interior nodes per axis (coarse, fine)
};

template <int K>
struct XTile {
  static constexpr int C = (K <= 2) ? 8 : (K <= 4 ? 4 : 2);    // coarse cells per tile edge
};

// fine += (E (x) E) coarse on the fine nodes [2 c0 K, 2 (c0 + C) K) per axis
template <typename T, int K>
__global__ void __launch_bounds__(256) prolong2d_kernel(const __grid_constant__ XferP<T, K> P) {
  constexpr int C = XTile<K>::C, CB = C * K + 1, FO = 2 * C * K;
  constexpr int PB = odd(CB), PF = odd(FO);
  __shared__ T cb[CB * PB];          // coarse box: nodes [c0 K, (c0 + C) K]
  __shared__ T tx[CB * PF];          // x-contracted: coarse rows x fine cols
  const int64_t Nc = P.Nc, nc = P.nc, nf = P.nf, KNc = K * Nc, KNf = 2 * KNc;
  const int ntx = int((Nc + C - 1) / C);
  const int64_t cx0 = int64_t(blockIdx.x % ntx) * C, cy0 = int64_t(blockIdx.x / ntx) * C;
  const int tid = threadIdx.x;
  for (int e = tid; e < CB * CB; e += blockDim.x) {
    const int r = e / CB, cc = e - (e / CB) * CB;
    const int64_t jy = cy0 * K + r, jx = cx0 * K + cc;
    cb[r * PB + cc] = (jx >= 1 && jx <= KNc - 1 && jy >= 1 && jy <= KNc - 1) ? P.src[(jy - 1) * nc + (jx - 1)] : T(0);
  }
  __syncthreads();
  // x-stage: unit = (coarse row, coarse cell) -> 2K fine columns
  for (int u = tid; u < CB * C; u += blockDim.x) {
    const int r = u % CB, ci = u / CB;
    T w[K + 1];
#pragma unroll
    for (int m = 0; m <= K; ++m) w[m] = cb[r * PB + ci * K + m];
#pragma unroll
    for (int q = 0; q < 2 * K; ++q) {
      T s = 0;
#pragma unroll
      for (int m = 0; m <= K; ++m) s = fma(P.c.pe[q][m], w[m], s);
      tx[r * PF + ci * 2 * K + q] = s;
    }
  }
  __syncthreads();
  // y-stage: unit = (fine column, coarse cell row) -> 2K fine rows; fine += ...
  for (int u = tid; u < FO * C; u += blockDim.x) {
    const int fc = u % FO, ci = u / FO;
    const int64_t jx = 2 * cx0 * K + fc;
    if (jx < 1 || jx > KNf - 1) continue;
    T w[K + 1];
#pragma unroll
    for (int m = 0; m <= K; ++m) w[m] = tx[(ci * K + m) * PF + fc];
#pragma unroll
    for (int q = 0; q < 2 * K; ++q) {
      const int64_t jy = 2 * (cy0 + ci) * K + q;
      if (jy < 1 || jy > KNf - 1) continue;
      T s = 0;
#pragma unroll
      for (int m = 0; m <= K; ++m) s = fma(P.c.pe[q][m], w[m], s);
      T* d = P.dst + (jy - 1) * nf + (jx - 1);
      *d += s;
    }
  }
}

// coarse = (E^T (x) E^T) fine on the coarse nodes [c0 K, (c0 + C) K) per axis
template <typename T, int K>
__global__ void __launch_bounds__(256) restrict2d_kernel(const __grid_constant__ XferP<T, K> P) {
  constexpr int C = XTile<K>::C, O = C * K, FB = (2 * C + 2) * K + 1;
  constexpr int PB = odd(FB), PO = odd(O);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* fb = reinterpret_cast<T*>(smem_raw);     // fine box: nodes [2(c0-1)K, 2(c0+C)K]
  T* tx = fb + FB * PB;                       // fine rows x coarse cols
  const int64_t Nc = P.Nc, nc = P.nc, nf = P.nf, KNc = K * Nc, KNf = 2 * KNc;
  const int ntx = int((Nc + C - 1) / C);
  const int64_t cx0 = int64_t(blockIdx.x % ntx) * C, cy0 = int64_t(blockIdx.x / ntx) * C;
  const int tid = threadIdx.x;
  const int64_t FX0 = 2 * (cx0 - 1) * K, FY0 = 2 * (cy0 - 1) * K;
  for (int e = tid; e < FB * FB; e += blockDim.x) {
    const int r = e / FB, cc = e - (e / FB) * FB;
    const int64_t jy = FY0 + r, jx = FX0 + cc;
    fb[r * PB + cc] = (jx >= 1 && jx <= KNf - 1 && jy >= 1 && jy <= KNf - 1) ? P.src[(jy - 1) * nf + (jx - 1)] : T(0);
  }
  __syncthreads();
  // x-stage: unit = (fine row, coarse cell) -> K coarse columns (window 4K+1 fine nodes)
  for (int u = tid; u < FB * C; u += blockDim.x) {
    const int r = u % FB, ci = u / FB;
    T w[4 * K + 1];
#pragma unroll
    for (int o = 0; o <= 4 * K; ++o) w[o] = fb[r * PB + 2 * ci * K + o];
#pragma unroll
    for (int pc = 0; pc < K; ++pc) {
      T s = 0;
#pragma unroll
      for (int o = 0; o <= 4 * K; ++o)
        if (pc == 0 || o >= 2 * K) s = fma(P.c.re[pc][o], w[o], s);
      tx[r * PO + ci * K + pc] = s;
    }
  }
  __syncthreads();
  // y-stage: unit = (coarse column, coarse cell row) -> K coarse rows
  for (int u = tid; u < O * C; u += blockDim.x) {
    const int col = u % O, ci = u / O;
    const int64_t jx = cx0 * K + col;
    if (jx < 1 || jx > KNc - 1) continue;
    T w[4 * K + 1];
#pragma unroll
    for (int o = 0; o <= 4 * K; ++o) w[o] = tx[(2 * ci * K + o) * PO + col];
#pragma unroll
    for (int pc = 0; pc < K; ++pc) {
      const int64_t jy = (cy0 + ci) * K + pc;
      if (jy < 1 || jy > KNc - 1) continue;
      T s = 0;
#pragma unroll
      for (int o = 0; o <= 4 * K; ++o)
        if (pc == 0 || o >= 2 * K) s = fma(P.c.re[pc][o], w[o], s);
      P.dst[(jy - 1) * nc + (jx - 1)] = s;
    }
  }
}

// ----------------------------------------------------------------------------- host side
template <typename T, int K>
static void fill_xfer(XferCoef<T, K>& c) {
  // extract the class rows from the embedding of a 4-cell coarse mesh (host_setup.cpp)
  RectBand E = embedding(K, 4);
  auto Eat = [&](int64_t jf, int64_t jc) -> double {       // node indices (1-based interior nodes)
    const int64_t i = jf - 1, col = jc - 1;
    const int64_t q = col - E.lo[i];
    return (q >= 0 && q < E.width) ? E.v[i * E.width + q] : 0.0;
  };
  for (int q = 0; q < 2 * K; ++q)
    for (int m = 0; m <= K; ++m) c.pe[q][m] = (T)Eat(2 * K + q, K + m);           // fine in coarse cell 1
  for (int pc = 0; pc < K; ++pc)
    for (int o = 0; o <= 4 * K; ++o) c.re[pc][o] = (T)Eat(2 * K + o, 2 * K + pc); // coarse cell 2
}

template <typename T, int K>
static void launch_xfer(bool prolong, int64_t Nc, const T* src, T* dst, cudaStream_t st) {
  static XferCoef<T, K> coef;
  static bool have = false;
  if (!have) { fill_xfer<T, K>(coef); have = true; }
  XferP<T, K> p;
  p.c = coef;
  p.src = src; p.dst = dst; p.Nc = Nc; p.nc = K * Nc - 1; p.nf = 2 * K * Nc - 1;
  constexpr int C = XTile<K>::C;
  const int64_t nt = (Nc + C - 1) / C;
  if (prolong) {
    prolong2d_kernel<T, K><<<(unsigned)(nt * nt), 256, 0, st>>>(p);
  } else {
    constexpr int FB = (2 * C + 2) * K + 1, O = C * K;
    const size_t smem = sizeof(T) * (size_t(FB) * odd(FB) + size_t(FB) * odd(O));
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(restrict2d_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    restrict2d_kernel<T, K><<<(unsigned)(nt * nt), 256, smem, st>>>(p);
  }
}

template <typename T>
bool fused_transfer2d(int k, bool prolong, int64_t Nc, const T* src, T* dst, cudaStream_t st, int64_t* launches) {
  if (Nc < 4) return false;
  switch (k) {
    case 2: launch_xfer<T, 2>(prolong, Nc, src, dst, st); break;
    case 3: launch_xfer<T, 3>(prolong, Nc, src, dst, st); break;
    case 4: launch_xfer<T, 4>(prolong, Nc, src, dst, st); break;
    case 5: launch_xfer<T, 5>(prolong, Nc, src, dst, st); break;
    case 6: launch_xfer<T, 6>(prolong, Nc, src, dst, st); break;
    case 7: launch_xfer<T, 7>(prolong, Nc, src, dst, st); break;
    default: return false;
  }
  (*launches)++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("fused transfer2d launch: ") + cudaGetErrorString(e));
  return true;
}

template bool fused_transfer2d<double>(int, bool, int64_t, const double*, double*, cudaStream_t, int64_t*);
template bool fused_transfer2d<float>(int, bool, int64_t, const float*, float*, cudaStream_t, int64_t*);

}  // namespace c0ip
