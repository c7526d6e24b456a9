// Fused tile kernels for large 2D levels (sm_100a, FP64 and FP32).
//
// Two kernels make one additive smoothing step:
//   apply2d  : r = b - A x  (or y = A x) for a tile of C x C cells; all 1D contractions of the
//              Kronecker sum A = h^-2 (M^_y B^_x + 2 L^_y L^_x + B^_y M^_x) in
//              shared memory on a halo'd box of x;
//   fdm2d    : x += omega h^2 sum_v R_v^T A~_v^{-1} R_v r for the same tile,
//              written as a GATHER: the patch-eigenbasis transform S^T R_v is shared by all
//              patches of a patch row, every owned DoF sums its <= 4 patch corrections in a
//              fixed order (deterministic, no atomics) and is stored once.
// Both kernels are persistent: each CTA walks tiles t, t + gridDim.x, ... and prefetches the
// next tile's inputs with cp.async while computing the current one.
//
// Coefficients.  Every lane of a warp applies the *same* coefficients (same class p = j mod k of
// the output node, or same patch axis variant), so they are read from the kernel parameter bank
// (__grid_constant__) as uniform-register operands of DFMA/FFMA (LDCU + DFMA R, R, UR, R).  Each
// loaded coefficient is reused for RB independent lines held by the same thread (register
// blocking), and the coefficient base is offset by an opaque zero per round so that the compiler
// issues the LDCU at the point of use instead of hoisting hundreds of constants into registers.
// Tiles touching the domain boundary take a uniform per-warp branch to the one-sided face rows and
// the left/right patch variants.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "fused_common.cuh"

namespace c0ip {

// register-blocking factor of a stage with `lines` lines per unit column and `mult` unit columns:
// minimise rounds(rb) * rb over 256 threads (the per-thread work of a stage), prefer larger rb on ties
__host__ __device__ constexpr int pick_rb(int lines, int mult, int maxrb, int nt = 256) {
  int best = 1, bestc = 1 << 30;
  for (int rb = 1; rb <= maxrb; ++rb) {
    const int cost = cdiv(cdiv(lines, rb) * mult, nt) * rb;
    if (cost <= bestc) { bestc = cost; best = rb; }
  }
  return best;
}

// ----------------------------------------------------------------------------- apply2d
template <typename T, int K, int NT_>
struct ApplyLayout {
  static constexpr int NT = NT_;                   // threads per CTA
  static constexpr int C = Tile<K>::C, O = Tile<K>::O, RB = Blk<T, K>::RB;
  static constexpr int BW = (C + 3) * K + 1;       // box: nodes [(c0-2)K, (c0+C+1)K]
  static constexpr int PX = odd(BW), PO = odd(O);
  static constexpr int XN = O * PX;                // the O new box rows of a tile below the previous one
  static constexpr int STAGE = BW * PO;            // one of the three x-stage outputs
  // the full box of a chunk's first tile lives in the two new-row buffers (2 O >= BW rows); b is read
  // from global memory in the epilogue (streamed once, issued before the y-stage contractions)
  static_assert(2 * O >= BW, "first box must fit the two new-row buffers");
  static constexpr int TOTAL = 2 * XN + 3 * STAGE;
  // register blocking: the column-walk stages have few units (O rows x C cells); for FP64 k = 4 blocking
  // RB lines per thread (one LDCU per RB DFMA) and 128-thread CTAs (every thread busy, 3 CTAs per SM)
  static constexpr bool FORCE = (K == 4 && sizeof(T) == 8);
  static constexpr int RBX = pick_rb(BW, C, RB, NT), RBY = FORCE ? RB : pick_rb(O, C, RB, NT);
  static constexpr int RBXN = FORCE ? RB : pick_rb(O, C, RB, NT);   // x-stage on the O new rows only
  static_assert(BW - O <= O, "carried rows must not overlap the rows they are copied from");
  static constexpr int GX = cdiv(BW, RBX);         // row groups of the x-stage
  static constexpr int GY = cdiv(O, RBY);          // column groups of the y-stage
  static constexpr int MINB = NT == 128 ? 3 : 2;   // CTAs per SM
};

template <typename T, int K, int NT_>
__global__ void __launch_bounds__(NT_, ApplyLayout<T, K, NT_>::MINB) apply2d_kernel(const __grid_constant__ ApplyP<T, K> P) {
  // Work item = (tile column tx, chunk of CH tile rows): the CTA walks down the chunk.  Consecutive
  // tiles of a column share BW - O box rows; their x-stage outputs are carried over (shifted up in
  // shared memory), so only the O new box rows are loaded and contracted per tile after the first.
  using LY = ApplyLayout<T, K, NT_>;
  constexpr int C = LY::C, O = LY::O, BW = LY::BW, PX = LY::PX, PO = LY::PO;
  const int CH = P.chunk;                        // tiles per column chunk (host: ~8 items per CTA)
  constexpr int GY = LY::GY;
  constexpr int NT = LY::NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* const xnew0 = sm;                           // [2][XN] new rows of a tile; [BW][PX] full box of a chunk's first tile
  T* const xfull = xnew0;
  T* sB = xnew0 + 2 * LY::XN;
  T* sL = sB + LY::STAGE;
  T* sM = sL + LY::STAGE;
  const int64_t N = P.N, n = P.n, KN = K * N;
  const int ntx = int((N + C - 1) / C);
  int ty0, ty1;
  tile_rows<K, C>(P.out_lo, P.out_hi, ty0, ty1);
  const int nch = (ty1 - ty0 + CH - 1) / CH;
  const int nitems = ntx * nch;
  const int tid = threadIdx.x;
  int round = 0;

  auto load_new = [&](int64_t cx0, int64_t cy0, int buf) {   // box rows [BW - O, BW) of tile row cy0
    load_box_async<T, O, BW, PX>(xnew0 + buf * LY::XN, P.x, n, KN, (cy0 - 2) * K + (BW - O), (cx0 - 2) * K,
                                 P.row0, P.lrows);
  };

  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int tx = item % ntx, ch = item / ntx;
    const int tA = ty0 + ch * CH, tB = min(tA + CH, ty1);
    const int64_t cx0 = int64_t(tx) * C;
    // first tile of the chunk: full box (synchronous) in both new-row buffers
    load_box_async<T, BW, BW, PX>(xfull, P.x, n, KN, (int64_t(tA) * C - 2) * K, (cx0 - 2) * K, P.row0, P.lrows);
    cp_async_commit();
    int buf = 0;
    for (int ty = tA; ty < tB; ++ty) {
      const bool first = (ty == tA);
      // prefetch the next tile's new rows into the other buffer (after the first tile: once its x-stage
      // has consumed the box, which occupies both buffers)
      if (!first && ty + 1 < tB) load_new(cx0, int64_t(ty + 1) * C, buf ^ 1);
      cp_async_commit();
      cp_async_wait1();
      if (!first) {                            // carry the x-stage rows shared with the previous tile
        for (int e = tid; e < (BW - O) * O; e += NT) {
          const int r = e / O, cc = e - (e / O) * O;
          const T vb = sB[(r + O) * PO + cc], vl = sL[(r + O) * PO + cc], vm = sM[(r + O) * PO + cc];
          sB[r * PO + cc] = vb;
          sL[r * PO + cc] = vl;
          sM[r * PO + cc] = vm;
        }
      }
      __syncthreads();
      const T* xsrc = first ? xfull : xnew0 + buf * LY::XN;
      const int64_t cy0 = int64_t(ty) * C;
    const bool tin = (cx0 >= 2 && cx0 + C - 1 <= N - 2 && cy0 >= 2 && cy0 + C - 1 <= N - 2);
    auto tile_body = [&](auto INC) {
      constexpr bool IN = decltype(INC)::value;
    // x-stage: B^_x x, L^_x x, M^_x x on box rows [BW - NR, BW), owned columns.  lanes <-> row
    // groups; a thread holds rows g, g + GX, ... (RB rows) of one cell and reuses every coefficient
    // RB times.  x rows come from xsrc (local row = box row - (BW - NR)).
    auto xstage = [&](auto NRC, auto RBC) {
    constexpr int NR = decltype(NRC)::value, RB = decltype(RBC)::value;
    constexpr int GX = cdiv(NR, RB), R0 = BW - NR;
#pragma unroll 1
    for (int it = 0; it < cdiv(GX * C, NT); ++it, ++round) {
      const int u = it * NT + tid;
      if (u >= GX * C) continue;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      const int g = u % GX, ci = u / GX;
      const int64_t cx = cx0 + ci;
      if (!IN && cx >= N) continue;
      T w[RB][4 * K + 1];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int lrow = min(g + r * GX, NR - 1);
#pragma unroll
        for (int q = 0; q <= 4 * K; ++q) w[r][q] = xsrc[lrow * PX + ci * K + q];
      }
      const bool inner = IN || (cx >= 2 && cx <= N - 2);
      if (inner) {
        T ob[K][RB], ol[K][RB], om[K][RB];
        x_all_interior<T, K, RB>(c, w, ob, ol, om);
#pragma unroll
        for (int p = 0; p < K; ++p)
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            const int row = R0 + g + r * GX;
            if (g + r * GX < NR) {
              sB[row * PO + ci * K + p] = ob[p][r];
              sL[row * PO + ci * K + p] = ol[p][r];
              sM[row * PO + ci * K + p] = om[p][r];
            }
          }
        continue;
      }
#pragma unroll
      for (int p = 0; p < K; ++p) {
        T ob[RB], ol[RB], om[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) ob[r] = ol[r] = om[r] = 0;
        const int s = inner ? -1 : special_row<K>(cx * K + p, N);
        with_p<K>(p, [&](auto PC) {
          constexpr int PP = decltype(PC)::value;
          if (s < 0) {
            rowB<T, K, PP>([&](int q) { return c.BI[PP][q]; }, w, 0, ob);
            rowML<T, K, PP>([&](int q) { return c.LI[PP][q]; }, w, K, ol);
            rowML<T, K, PP>([&](int q) { return c.MI[PP][q]; }, w, K, om);
          } else {
            rowB<T, K, PP>([&](int q) { return c.BS[s][q]; }, w, 0, ob);
            rowML<T, K, PP>([&](int q) { return c.LS[s][q + K]; }, w, K, ol);
            rowML<T, K, PP>([&](int q) { return c.MS[s][q + K]; }, w, K, om);
          }
        });
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const int row = R0 + g + r * GX;
          if (g + r * GX < NR) {
            sB[row * PO + ci * K + p] = ob[r];
            sL[row * PO + ci * K + p] = ol[r];
            sM[row * PO + ci * K + p] = om[r];
          }
        }
      }
    }
    };
    if (first) xstage(std::integral_constant<int, BW>{}, std::integral_constant<int, LY::RBX>{});
    else xstage(std::integral_constant<int, O>{}, std::integral_constant<int, LY::RBXN>{});
    __syncthreads();
    if (first && ty + 1 < tB) {                // the box is consumed: prefetch the next tile's new rows
      load_new(cx0, int64_t(ty + 1) * C, 1);
      cp_async_commit();
    }

    // y-stage: y = h^-2 (B^_y (M^_x x) + M^_y (B^_x x) + 2 L^_y (L^_x x)).  lanes <-> column
    // groups; three passes (one window at a time) accumulate K outputs for RB columns.
#pragma unroll 1
    for (int it = 0; it < cdiv(GY * C, NT); ++it, ++round) {
      constexpr int RB = LY::RBY;
      const int u = it * NT + tid;
      if (u >= GY * C) continue;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      const int g = u % GY, ci = u / GY;
      const int64_t cy = cy0 + ci;
      if (!IN && cy >= N) continue;
      const bool inner = IN || (cy >= 2 && cy <= N - 2);
      T acc[K][RB];
#pragma unroll
      for (int p = 0; p < K; ++p)
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[p][r] = 0;
      int col[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) col[r] = min(g + r * GY, O - 1);
      // b of the unit's outputs (read once from global memory; issued before the contractions)
      T bv[K][RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int cc = g + r * GY;
        const int64_t jx = cx0 * K + cc;
        const bool okc = cc < O && (IN || (jx >= 1 && jx <= KN - 1));
#pragma unroll
        for (int p = 0; p < K; ++p) {
          const int64_t j = cy * K + p;
          const bool ok = P.b && okc && j >= P.out_lo && j < P.out_hi;
          bv[p][r] = ok ? P.b[(j - 1 - P.row0) * n + (jx - 1)] : T(0);
        }
      }
      if (inner) {
        T accL[K][RB];
#pragma unroll
        for (int p = 0; p < K; ++p)
#pragma unroll
          for (int r = 0; r < RB; ++r) accL[p][r] = 0;
        {
          T w[RB][4 * K + 1];
#pragma unroll
          for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int q = 0; q <= 4 * K; ++q) w[r][q] = sM[(ci * K + q) * PO + col[r]];
          y_all_interior<T, K, RB, 0, 4 * K + 1>(c, w, acc);
        }
        {
          T w[RB][2 * K + 1];
#pragma unroll
          for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int q = 0; q <= 2 * K; ++q) w[r][q] = sB[(ci * K + K + q) * PO + col[r]];
          y_all_interior<T, K, RB, 1, 2 * K + 1>(c, w, acc);
        }
        {
          T w[RB][2 * K + 1];
#pragma unroll
          for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int q = 0; q <= 2 * K; ++q) w[r][q] = sL[(ci * K + K + q) * PO + col[r]];
          y_all_interior<T, K, RB, 2, 2 * K + 1>(c, w, accL);
        }
#pragma unroll
        for (int p = 0; p < K; ++p)
#pragma unroll
          for (int r = 0; r < RB; ++r) acc[p][r] = fma(T(2), accL[p][r], acc[p][r]);
      } else {
      {
        T w[RB][4 * K + 1];
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int q = 0; q <= 4 * K; ++q) w[r][q] = sM[(ci * K + q) * PO + col[r]];
#pragma unroll
        for (int p = 0; p < K; ++p) {
          const int s = inner ? -1 : special_row<K>(cy * K + p, N);
          with_p<K>(p, [&](auto PC) {
            constexpr int PP = decltype(PC)::value;
            if (s < 0) rowB<T, K, PP>([&](int q) { return c.BI[PP][q]; }, w, 0, acc[PP]);
            else rowB<T, K, PP>([&](int q) { return c.BS[s][q]; }, w, 0, acc[PP]);
          });
        }
      }
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const T* src = pass == 0 ? sB : sL;
        T w[RB][2 * K + 1];
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int q = 0; q <= 2 * K; ++q) w[r][q] = src[(ci * K + K + q) * PO + col[r]];
#pragma unroll
        for (int p = 0; p < K; ++p) {
          const int s = inner ? -1 : special_row<K>(cy * K + p, N);
          T tmp[RB];
#pragma unroll
          for (int r = 0; r < RB; ++r) tmp[r] = 0;
          with_p<K>(p, [&](auto PC) {
            constexpr int PP = decltype(PC)::value;
            if (pass == 0) {
              if (s < 0) rowML<T, K, PP>([&](int q) { return c.MI[PP][q]; }, w, 0, tmp);
              else rowML<T, K, PP>([&](int q) { return c.MS[s][q + K]; }, w, 0, tmp);
            } else {
              if (s < 0) rowML<T, K, PP>([&](int q) { return c.LI[PP][q]; }, w, 0, tmp);
              else rowML<T, K, PP>([&](int q) { return c.LS[s][q + K]; }, w, 0, tmp);
            }
          });
#pragma unroll
          for (int r = 0; r < RB; ++r) acc[p][r] += (pass == 0 ? T(1) : T(2)) * tmp[r];
        }
      }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int cc = g + r * GY;
        const int64_t jx = cx0 * K + cc;
        if (cc >= O || (!IN && (jx < 1 || jx > KN - 1))) continue;
#pragma unroll
        for (int p = 0; p < K; ++p) {
          const int64_t j = cy * K + p;
          if (j < P.out_lo || j >= P.out_hi) continue;   // (slab window; always true for the full domain)
          const T v = P.scale * acc[p][r];
          P.y[(j - 1 - P.row0) * n + (jx - 1)] = P.b ? bv[p][r] - v : v;
        }
      }
    }
    };
    if (tin) tile_body(std::true_type{});
    else tile_body(std::false_type{});
    __syncthreads();
    buf ^= 1;
    }
  }
}

// ----------------------------------------------------------------------------- fdm2d
// z[r][i] = sum_l S[l][i] w[r][l]   (S^T w) for RB lines
template <typename T, int K, int V, int RB>
__device__ __forceinline__ void s_t(const Coef2<T, K>& c, const T (&w)[RB][2 * K - 1], T (&z)[RB][2 * K - 1]) {
  // contraction index outermost: NP * RB independent accumulators between dependent FMAs
  constexpr int NP = 2 * K - 1;
#pragma unroll
  for (int i = 0; i < NP; ++i)
#pragma unroll
    for (int r = 0; r < RB; ++r) z[r][i] = 0;
#pragma unroll
  for (int l = 0; l < NP; ++l)
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const T s = c.S[V][l * NP + i];
      if constexpr (std::is_same<T, float>::value && RB >= 2) {
#pragma unroll
        for (int r = 0; r + 1 < RB; r += 2) {
          const float2 v = __ffma2_rn(make_float2(s, s), make_float2(w[r][l], w[r + 1][l]),
                                      make_float2(z[r][i], z[r + 1][i]));
          z[r][i] = v.x;
          z[r + 1][i] = v.y;
        }
        if constexpr (RB % 2 == 1) z[RB - 1][i] = fmaf(s, w[RB - 1][l], z[RB - 1][i]);
      } else {
#pragma unroll
        for (int r = 0; r < RB; ++r) z[r][i] = fma(s, w[r][l], z[r][i]);
      }
    }
}

// out[r][p] += sum_i S[OFF + p][i] z[r][i] for p in [P0, K)
template <typename T, int K, int V, int OFF, int P0, int RB>
__device__ __forceinline__ void s_rows(const Coef2<T, K>& c, const T (&z)[RB][2 * K - 1], T (&out)[RB][K]) {
  constexpr int NP = 2 * K - 1;
#pragma unroll
  for (int i = 0; i < NP; ++i)
#pragma unroll
    for (int p = P0; p < K; ++p) {
      const T s = c.S[V][(OFF + p) * NP + i];
      if constexpr (std::is_same<T, float>::value && RB >= 2) {
#pragma unroll
        for (int r = 0; r + 1 < RB; r += 2) {
          const float2 v = __ffma2_rn(make_float2(s, s), make_float2(z[r][i], z[r + 1][i]),
                                      make_float2(out[r][p], out[r + 1][p]));
          out[r][p] = v.x;
          out[r + 1][p] = v.y;
        }
        if constexpr (RB % 2 == 1) out[RB - 1][p] = fmaf(s, z[RB - 1][i], out[RB - 1][p]);
      } else {
#pragma unroll
        for (int r = 0; r < RB; ++r) out[r][p] = fma(s, z[r][i], out[r][p]);
      }
    }
}

template <typename T, int K, int V, int RB>
__device__ __forceinline__ void s_t_var(int var, const Coef2<T, K>& c, const T (&w)[RB][2 * K - 1],
                                        T (&z)[RB][2 * K - 1]) {
  if (var == 1) s_t<T, K, 1, RB>(c, w, z);
  else if (var == 0) s_t<T, K, 0, RB>(c, w, z);
  else s_t<T, K, 2, RB>(c, w, z);
}

// out[r][p] (p < K) for the K nodes of cell `cell`: patch cell (local K-1+p), patch cell+1 (local p-1)
template <typename T, int K, int RB>
__device__ __forceinline__ void cell_from_patches(const Coef2<T, K>& c, int64_t cell, int64_t N,
                                                  const T (&z0)[RB][2 * K - 1], const T (&z1)[RB][2 * K - 1],
                                                  T (&out)[RB][K]) {
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int p = 0; p < K; ++p) out[r][p] = 0;
  if (cell >= 1 && cell <= N - 1) {
    const int v0 = variant_of(cell, N);
    if (v0 == 1) s_rows<T, K, 1, K - 1, 0, RB>(c, z0, out);
    else if (v0 == 0) s_rows<T, K, 0, K - 1, 0, RB>(c, z0, out);
    else s_rows<T, K, 2, K - 1, 0, RB>(c, z0, out);
  }
  if (cell + 1 >= 1 && cell + 1 <= N - 1) {
    const int v1 = variant_of(cell + 1, N);
    if (v1 == 1) s_rows<T, K, 1, -1, 1, RB>(c, z1, out);
    else if (v1 == 0) s_rows<T, K, 0, -1, 1, RB>(c, z1, out);
    else s_rows<T, K, 2, -1, 1, RB>(c, z1, out);
  }
}

template <typename T, int K>
struct FdmLayout {
  static constexpr int C = Tile<K>::C, O = Tile<K>::O, NP = 2 * K - 1, RB = Blk<T, K>::RB;
  static constexpr int RN = (C + 2) * K - 1;       // residual box: nodes [(c0-1)K+1, (c0+C+1)K-1]
  static constexpr int E = (C + 1) * NP;           // patch-eigen columns: patches c0 .. c0+C
  static constexpr int PR = odd(RN), PE = odd(E), PS = odd(O);
  static constexpr int RB_ = RN * PR, XT = O * PS; // r box, x tile (prefetched, double buffered)
  static constexpr int Z1 = RN * PE;               // Z1 [RN][E]; later Z3 [O][E]
  static constexpr int Z2 = (C + 1) * NP * PE;     // Z2 [vy][iy][E]; later out staging [O][PS]
  static constexpr int TOTAL = 2 * (RB_ + XT) + Z1 + Z2 + NP * NP;
  static constexpr int RB_FX = pick_rb(RN, C + 1, RB), RB_G = pick_rb(E, C + 1, RB);
  static constexpr int RB_S = pick_rb(E, C, RB), RB_O = pick_rb(O, C, RB);
  static constexpr int GR = cdiv(RN, RB_FX);       // FX row groups
  static constexpr int GEG = cdiv(E, RB_G);        // FYg column groups
  static constexpr int GES = cdiv(E, RB_S);        // FYs column groups
  static constexpr int GO = cdiv(O, RB_O);         // FS row groups
};

// x += omega h^2 sum_v R_v^T A~_v^{-1} R_v r on the tile (gather form, see file header):
//   FX  (row, vx)  Z1[y][vx,i]    = sum_l S_vx[l][i] r[y][(vx-1)K+1+l]
//   FYg (col, vy)  Z2[vy][i][col] = (sum_l S_vy[l][i] Z1[(vy-1)K+1+l][col]) / (lam_vy,i + lam_vx,ix)
//   FYs (col, cy)  Z3[y][col]     = sum over the <= 2 patches of row y of S_vy[y-..][i] Z2[vy][i][col]
//   FS  (row, cx)  out[y][x]      = sum over the <= 2 patches of column x of S_vx[x-..][i] Z3[y][vx,i]
template <typename T, int K>
__global__ void __launch_bounds__(256, 2) fdm2d_kernel(const __grid_constant__ FdmP<T, K> P) {
  using LY = FdmLayout<T, K>;
  constexpr int C = LY::C, O = LY::O, NP = LY::NP, RN = LY::RN, E = LY::E;
  constexpr int PR = LY::PR, PE = LY::PE, PS = LY::PS, GR = LY::GR, GO = LY::GO;
  constexpr int NT = 256;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* const rbuf0 = sm;                           // [2][RB_]
  T* const xbuf0 = sm + 2 * LY::RB_;             // [2][XT]
  T* z1 = sm + 2 * (LY::RB_ + LY::XT);
  T* z3 = z1;                                    // Z1 is dead after FYg
  T* z2 = z1 + LY::Z1;
  T* outs = z2;                                  // Z2 is dead after FYs
  T* invd = z2 + LY::Z2;                         // 1/(lam_int[i] + lam_int[j])
  static_assert(RN >= O && LY::Z2 >= O * PS, "Z3 / staging do not fit");
  const int64_t N = P.N, n = P.n, KN = K * N;
  const int ntx = int((N + C - 1) / C);
  int ty0, ty1;
  tile_rows<K, C>(P.out_lo, P.out_hi, ty0, ty1);
  const int ntiles = ntx * (ty1 - ty0);
  const int tid = threadIdx.x;

  for (int e = tid; e < NP * NP; e += blockDim.x)
    invd[e] = T(1) / (P.c.lam[1][e / NP] + P.c.lam[1][e % NP]);

  auto issue = [&](int t, int buf) {
    const int64_t cx0 = int64_t(t % ntx) * C, cy0 = int64_t(ty0 + t / ntx) * C;
    load_box_async<T, RN, RN, PR>(rbuf0 + buf * LY::RB_, P.r, n, KN, (cy0 - 1) * K + 1, (cx0 - 1) * K + 1,
                                  P.row0, P.lrows);
    load_box_async<T, O, O, PS>(xbuf0 + buf * LY::XT, P.x, n, KN, cy0 * K, cx0 * K, P.row0, P.lrows);
  };

  int buf = 0, round = 0;
  if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
  cp_async_commit();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (t + (int)gridDim.x < ntiles) issue(t + gridDim.x, buf ^ 1);
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    const T* rb = rbuf0 + buf * LY::RB_;
    const T* xt = xbuf0 + buf * LY::XT;
    const int64_t cx0 = int64_t(t % ntx) * C, cy0 = int64_t(ty0 + t / ntx) * C;

    // interior tiles (every patch of the tile has the interior variant on both axes) take a
    // specialised path without variant / range checks
    const bool tin = (cx0 >= 2 && cx0 + C <= N - 2 && cy0 >= 2 && cy0 + C <= N - 2);
    auto tile_body = [&](auto INC) {
      constexpr bool IN = decltype(INC)::value;
    // FX: lanes <-> row groups, one patch vx per unit (uniform variant)
#pragma unroll 1
    for (int it = 0; it < cdiv(GR * (C + 1), NT); ++it, ++round) {
      constexpr int RB = LY::RB_FX;
      const int u = it * NT + tid;
      if (u >= GR * (C + 1)) continue;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      const int g = u % GR, pi = u / GR;
      const int64_t vx = cx0 + pi;
      T z[RB][NP];
      if (IN || (vx >= 1 && vx <= N - 1)) {
        T w[RB][NP];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const int row = min(g + r * GR, RN - 1);
#pragma unroll
          for (int l = 0; l < NP; ++l) w[r][l] = rb[row * PR + pi * K + l];
        }
        if constexpr (IN) s_t<T, K, 1, RB>(c, w, z);
        else s_t_var<T, K, 1, RB>(variant_of(vx, N), c, w, z);
      } else {
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int i = 0; i < NP; ++i) z[r][i] = 0;
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int row = g + r * GR;
        if (row < RN)
#pragma unroll
          for (int i = 0; i < NP; ++i) z1[row * PE + pi * NP + i] = z[r][i];
      }
    }
    __syncthreads();

    // FYg: lanes <-> column groups, one patch row vy per unit
#pragma unroll 1
    for (int it = 0; it < cdiv(LY::GEG * (C + 1), NT); ++it, ++round) {
      constexpr int RB = LY::RB_G, GE = LY::GEG;
      const int u = it * NT + tid;
      if (u >= GE * (C + 1)) continue;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      const int g = u % GE, qi = u / GE;
      const int64_t vy = cy0 + qi;
      int col[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) col[r] = min(g + r * GE, E - 1);
      T z[RB][NP];
      if (IN || (vy >= 1 && vy <= N - 1)) {
        T w[RB][NP];
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int l = 0; l < NP; ++l) w[r][l] = z1[(qi * K + l) * PE + col[r]];
        const int vary = IN ? 1 : variant_of(vy, N);
        if constexpr (IN) s_t<T, K, 1, RB>(c, w, z);
        else s_t_var<T, K, 1, RB>(vary, c, w, z);
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          if constexpr (IN) {
            const int ix = col[r] - (col[r] / NP) * NP;
#pragma unroll
            for (int i = 0; i < NP; ++i) z[r][i] *= invd[i * NP + ix];
            continue;
          }
          const int pi = col[r] / NP, ix = col[r] - (col[r] / NP) * NP;
          const int64_t vx = cx0 + pi;
          if (vx < 1 || vx > N - 1) {
#pragma unroll
            for (int i = 0; i < NP; ++i) z[r][i] = 0;
          } else if (vary == 1 && variant_of(vx, N) == 1) {
#pragma unroll
            for (int i = 0; i < NP; ++i) z[r][i] *= invd[i * NP + ix];
          } else {
            const T lx = P.c.lam[variant_of(vx, N)][ix];
#pragma unroll
            for (int i = 0; i < NP; ++i) z[r][i] /= (P.c.lam[vary][i] + lx);
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int i = 0; i < NP; ++i) z[r][i] = 0;
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int cc = g + r * GE;
        if (cc < E)
#pragma unroll
          for (int i = 0; i < NP; ++i) z2[(qi * NP + i) * PE + cc] = z[r][i];
      }
    }
    __syncthreads();

    // FYs: lanes <-> column groups, one cell row cy per unit: rows cyK .. cyK+K-1
#pragma unroll 1
    for (int it = 0; it < cdiv(LY::GES * C, NT); ++it, ++round) {
      constexpr int RB = LY::RB_S, GE = LY::GES;
      const int u = it * NT + tid;
      if (u >= GE * C) continue;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      const int g = u % GE, ci = u / GE;
      T a0[RB][NP], a1[RB][NP], out[RB][K];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int cc = min(g + r * GE, E - 1);
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          a0[r][i] = z2[(ci * NP + i) * PE + cc];
          a1[r][i] = z2[((ci + 1) * NP + i) * PE + cc];
        }
      }
      if constexpr (IN) {
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int p = 0; p < K; ++p) out[r][p] = 0;
        s_rows<T, K, 1, K - 1, 0, RB>(c, a0, out);
        s_rows<T, K, 1, -1, 1, RB>(c, a1, out);
      } else {
        cell_from_patches<T, K, RB>(c, cy0 + ci, N, a0, a1, out);
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int cc = g + r * GE;
        if (cc < E)
#pragma unroll
          for (int p = 0; p < K; ++p) z3[(ci * K + p) * PE + cc] = out[r][p];
      }
    }
    __syncthreads();

    // FS: lanes <-> row groups, one cell column cx per unit
#pragma unroll 1
    for (int it = 0; it < cdiv(GO * C, NT); ++it, ++round) {
      constexpr int RB = LY::RB_O;
      const int u = it * NT + tid;
      if (u >= GO * C) continue;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      const int g = u % GO, ci = u / GO;
      T a0[RB][NP], a1[RB][NP], out[RB][K];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int oy = min(g + r * GO, O - 1);
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          a0[r][i] = z3[oy * PE + ci * NP + i];
          a1[r][i] = z3[oy * PE + (ci + 1) * NP + i];
        }
      }
      if constexpr (IN) {
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int p = 0; p < K; ++p) out[r][p] = 0;
        s_rows<T, K, 1, K - 1, 0, RB>(c, a0, out);
        s_rows<T, K, 1, -1, 1, RB>(c, a1, out);
      } else {
        cell_from_patches<T, K, RB>(c, cx0 + ci, N, a0, a1, out);
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int oy = g + r * GO;
        if (oy < O)
#pragma unroll
          for (int p = 0; p < K; ++p) outs[oy * PS + ci * K + p] = out[r][p];
      }
    }
    __syncthreads();

    };
    if (tin) tile_body(std::true_type{});
    else tile_body(std::false_type{});

    for (int e = tid; e < O * O; e += NT) {
      const int oy = e / O, ox = e - (e / O) * O;
      const int64_t jy = cy0 * K + oy, jx = cx0 * K + ox;
      if (jx < 1 || jx > KN - 1 || jy < P.out_lo || jy >= P.out_hi) continue;
      P.x[(jy - 1 - P.row0) * n + (jx - 1)] = fma(P.factor, outs[oy * PS + ox], xt[oy * PS + ox]);
    }
    __syncthreads();
    buf ^= 1;
  }
}

// ----------------------------------------------------------------------------- mvs2d
// One colour of the coloured multiplicative smoother, patch-parallel and fused:
// for every patch v of the colour (a batch of PB patches per CTA):
//   r_v = (b - A x) on the (2k-1)^2 patch nodes, from the x box [(v-2)k, (v+2)k]^2 (the residual
//         footprint: patch cells plus their face neighbours; identical to the global
//         residual recomputed per colour because same-colour patches never touch each other's footprint),
//   u_v = A~_v^{-1} r_v by FDM (S^T along x and y, divide by lambda_x + lambda_y, S along y and x),
//   x  += omega u_v on the patch nodes (disjoint within a colour, plain stores).
template <typename T, int K>
struct MvsLayout {
  static constexpr int NP = 2 * K - 1, BX = 4 * K + 1;
  static constexpr int PER = BX * BX + 3 * BX * NP + 2 * NP * NP;   // per patch
  static constexpr int PB = (K <= 2) ? 32 : (K == 3) ? 16 : (K == 4) ? 12 : (K == 5) ? 8 : (K == 6) ? 6 : 4;
  static constexpr int TOTAL = PB * PER;
};

template <typename T, int K>
__global__ void __launch_bounds__(256, 2) mvs2d_kernel(const __grid_constant__ MvsP<T, K> P) {
  using LY = MvsLayout<T, K>;
  constexpr int NP = LY::NP, BX = LY::BX, PB = LY::PB, PER = LY::PER;
  constexpr int NT = 256;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int64_t N = P.N, n = P.n, KN = K * N;
  const int tid = threadIdx.x;
  const int64_t first = (int64_t)blockIdx.x * PB;
  int round = 0;
  // per patch: xb [BX][BX] | sB, sL, sM [BX][NP] ; later rr [NP][NP] and z [NP][NP] alias xb
  auto xb = [&](int p) { return sm + p * PER; };
  auto sX = [&](int p, int which) { return sm + p * PER + BX * BX + which * BX * NP; };
  auto rr = [&](int p) { return sm + p * PER + BX * BX + 3 * BX * NP; };
  auto zz = [&](int p) { return rr(p) + NP * NP; };
  __shared__ int pv[PB][2];            // patch vertices (0 = no patch)
  if (tid < PB) {
    const int64_t q = first + tid;
    if (q < P.count) {
      const int pid = P.list[q], Nm1 = (int)(N - 1);
      pv[tid][0] = 1 + pid % Nm1;
      pv[tid][1] = 1 + pid / Nm1;
    } else {
      pv[tid][0] = pv[tid][1] = 0;
    }
  }
  __syncthreads();
  auto vert = [&](int p, int64_t& vx, int64_t& vy) -> bool {
    vx = pv[p][0];
    vy = pv[p][1];
    return vx != 0;
  };

  // 0. x boxes [(v-2)K, (v+2)K]^2 and b on the patch nodes
  for (int e = tid; e < PB * BX * BX; e += NT) {
    const int p = e / (BX * BX), rem = e - p * (BX * BX), r = rem / BX, cc = rem - (rem / BX) * BX;
    int64_t vx, vy;
    T v = 0;
    if (vert(p, vx, vy)) {
      const int64_t jy = (vy - 2) * K + r, jx = (vx - 2) * K + cc;
      if (jx >= 1 && jx <= KN - 1 && jy >= 1 && jy <= KN - 1) v = P.x[(jy - 1) * n + (jx - 1)];
    }
    xb(p)[r * BX + cc] = v;
  }
  for (int e = tid; e < PB * NP * NP; e += NT) {
    const int p = e / (NP * NP), rem = e - p * (NP * NP), r = rem / NP, cc = rem - (rem / NP) * NP;
    int64_t vx, vy;
    T v = 0;
    if (vert(p, vx, vy)) v = P.b[((vy - 1) * K + r) * n + ((vx - 1) * K + cc)];
    rr(p)[r * NP + cc] = v;
  }
  __syncthreads();

  // 1. x-stage on every box row, patch columns only: B^_x, L^_x, M^_x.  unit = (patch, box row).
#pragma unroll 1
  for (int it = 0; it < cdiv(PB * BX, NT); ++it, ++round) {
    const int u = it * NT + tid;
    if (u >= PB * BX) continue;
    const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
    const int p = u / BX, r = u - (u / BX) * BX;
    int64_t vx, vy;
    if (!vert(p, vx, vy)) continue;
    T w[BX];
#pragma unroll
    for (int q = 0; q < BX; ++q) w[q] = xb(p)[r * BX + q];
    const bool edge = (vx == 1 || vx == N - 1);
#pragma unroll
    for (int l = 0; l < NP; ++l) {
      // output node jx = (vx-1)K + 1 + l at box column K + 1 + l, class (1 + l) mod K
      const int cb = K + 1 + l;
      const int64_t jx = (vx - 1) * K + 1 + l;
      const int s = edge ? special_row<K>(jx, N) : -1;
      T ob = 0, ol = 0, om = 0;
      with_p<K>((1 + l) % K, [&](auto PC) {
        constexpr int PP = decltype(PC)::value;
        auto body = [&](auto fb, auto fl, auto fm) {
#pragma unroll
          for (int q = 0; q <= 4 * K; ++q) {
            const int col = cb + q - 2 * K;
            if (col < 0 || col >= BX) continue;
            if (!(PP == 0 || (q >= K - PP && q <= 4 * K - PP))) continue;
            ob = fma(fb(q), w[col], ob);
            if (q >= K && q <= 3 * K && (PP == 0 || (q - K >= K - PP && q - K <= 2 * K - PP))) {
              ol = fma(fl(q), w[col], ol);
              om = fma(fm(q), w[col], om);
            }
          }
        };
        if (s < 0)
          body([&](int q) { return c.BI[PP][q]; }, [&](int q) { return c.LI[PP][q - K]; },
               [&](int q) { return c.MI[PP][q - K]; });
        else
          body([&](int q) { return c.BS[s][q]; }, [&](int q) { return c.LS[s][q]; },
               [&](int q) { return c.MS[s][q]; });
      });
      sX(p, 0)[r * NP + l] = ob;
      sX(p, 1)[r * NP + l] = ol;
      sX(p, 2)[r * NP + l] = om;
    }
  }
  __syncthreads();

  // 2. y-stage: r = b - h^-2 (B^_y(M^x) + M^_y(B^x) + 2 L^_y(L^x)) on the patch rows.  unit = (patch, col).
#pragma unroll 1
  for (int it = 0; it < cdiv(PB * NP, NT); ++it, ++round) {
    const int u = it * NT + tid;
    if (u >= PB * NP) continue;
    const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
    const int p = u / NP, l = u - (u / NP) * NP;
    int64_t vx, vy;
    if (!vert(p, vx, vy)) continue;
    T wM[BX], wB[BX], wL[BX];
#pragma unroll
    for (int q = 0; q < BX; ++q) {
      wM[q] = sX(p, 2)[q * NP + l];
      wB[q] = sX(p, 0)[q * NP + l];
      wL[q] = sX(p, 1)[q * NP + l];
    }
    const bool edge = (vy == 1 || vy == N - 1);
#pragma unroll
    for (int m = 0; m < NP; ++m) {
      const int cb = K + 1 + m;
      const int64_t jy = (vy - 1) * K + 1 + m;
      const int s = edge ? special_row<K>(jy, N) : -1;
      T v = 0;
      with_p<K>((1 + m) % K, [&](auto PC) {
        constexpr int PP = decltype(PC)::value;
        auto body = [&](auto fb, auto fl, auto fm) {
#pragma unroll
          for (int q = 0; q <= 4 * K; ++q) {
            const int row = cb + q - 2 * K;
            if (row < 0 || row >= BX) continue;
            if (!(PP == 0 || (q >= K - PP && q <= 4 * K - PP))) continue;
            v = fma(fb(q), wM[row], v);
            if (q >= K && q <= 3 * K && (PP == 0 || (q - K >= K - PP && q - K <= 2 * K - PP))) {
              v = fma(fm(q), wB[row], v);
              v = fma(T(2) * fl(q), wL[row], v);
            }
          }
        };
        if (s < 0)
          body([&](int q) { return c.BI[PP][q]; }, [&](int q) { return c.LI[PP][q - K]; },
               [&](int q) { return c.MI[PP][q - K]; });
        else
          body([&](int q) { return c.BS[s][q]; }, [&](int q) { return c.LS[s][q]; },
               [&](int q) { return c.MS[s][q]; });
      });
      rr(p)[m * NP + l] = rr(p)[m * NP + l] - P.scale * v;
    }
  }
  __syncthreads();

  // 3. FDM: FX rows (S_vx^T), FY columns (S_vy^T, divide, S_vy), FS rows (S_vx) + update.
#pragma unroll 1
  for (int it = 0; it < cdiv(PB * NP, NT); ++it, ++round) {
    const int u = it * NT + tid;
    if (u >= PB * NP) continue;
    const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
    const int p = u / NP, i = u - (u / NP) * NP;
    int64_t vx, vy;
    if (!vert(p, vx, vy)) continue;
    T w[1][NP], z[1][NP];
#pragma unroll
    for (int l = 0; l < NP; ++l) w[0][l] = rr(p)[i * NP + l];
    s_t_var<T, K, 1, 1>(variant_of(vx, N), c, w, z);
#pragma unroll
    for (int l = 0; l < NP; ++l) zz(p)[i * NP + l] = z[0][l];
  }
  __syncthreads();
#pragma unroll 1
  for (int it = 0; it < cdiv(PB * NP, NT); ++it, ++round) {
    const int u = it * NT + tid;
    if (u >= PB * NP) continue;
    const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
    const int p = u / NP, j = u - (u / NP) * NP;
    int64_t vx, vy;
    if (!vert(p, vx, vy)) continue;
    T w[1][NP], z[1][NP];
#pragma unroll
    for (int l = 0; l < NP; ++l) w[0][l] = zz(p)[l * NP + j];
    const int vary = variant_of(vy, N), varx = variant_of(vx, N);
    s_t_var<T, K, 1, 1>(vary, c, w, z);
    const T lx = P.c.lam[varx][j];
#pragma unroll
    for (int i = 0; i < NP; ++i) z[0][i] /= (P.c.lam[vary][i] + lx);
    // S_vy z  -> column j
#pragma unroll
    for (int l = 0; l < NP; ++l) {
      T s = 0;
      if (vary == 1) {
#pragma unroll
        for (int i = 0; i < NP; ++i) s = fma(c.S[1][l * NP + i], z[0][i], s);
      } else if (vary == 0) {
#pragma unroll
        for (int i = 0; i < NP; ++i) s = fma(c.S[0][l * NP + i], z[0][i], s);
      } else {
#pragma unroll
        for (int i = 0; i < NP; ++i) s = fma(c.S[2][l * NP + i], z[0][i], s);
      }
      rr(p)[l * NP + j] = s;
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int it = 0; it < cdiv(PB * NP, NT); ++it, ++round) {
    const int u = it * NT + tid;
    if (u >= PB * NP) continue;
    const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
    const int p = u / NP, i = u - (u / NP) * NP;
    int64_t vx, vy;
    if (!vert(p, vx, vy)) continue;
    T z[NP];
#pragma unroll
    for (int l = 0; l < NP; ++l) z[l] = rr(p)[i * NP + l];
    const int varx = variant_of(vx, N);
    const int64_t row = ((vy - 1) * K + i) * n + (vx - 1) * K;
#pragma unroll
    for (int l = 0; l < NP; ++l) {
      T s = 0;
      if (varx == 1) {
#pragma unroll
        for (int m = 0; m < NP; ++m) s = fma(c.S[1][l * NP + m], z[m], s);
      } else if (varx == 0) {
#pragma unroll
        for (int m = 0; m < NP; ++m) s = fma(c.S[0][l * NP + m], z[m], s);
      } else {
#pragma unroll
        for (int m = 0; m < NP; ++m) s = fma(c.S[2][l * NP + m], z[m], s);
      }
      P.x[row + l] = fma(P.factor, s, P.x[row + l]);
    }
  }
}

// ----------------------------------------------------------------------------- host side


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
  if (N < 8 || k < 2 || k > 7 || (d == 3 && k > 5)) return nullptr;
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



template <typename KernelT>
static int persistent_grid(KernelT kern, size_t smem, int ntiles, int nt = 256) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, nt, smem);
  return std::max(1, std::min(ntiles, sms * std::max(per, 1)));
}

template <typename T, int K, int NT>
static void launch_apply_nt(const FusedLevel& F, const T* x, const T* b, T* y, const SlabWindow& w, cudaStream_t st) {
  using LY = ApplyLayout<T, K, NT>;
  const size_t smem = sizeof(T) * size_t(LY::TOTAL);
  static int grid_cache = -1;
  if (grid_cache < 0) {
    cudaFuncSetAttribute(apply2d_kernel<T, K, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(apply2d_kernel<T, K, NT>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    grid_cache = persistent_grid(apply2d_kernel<T, K, NT>, smem, 1 << 30, NT);
  }
  ApplyP<T, K> p;
  std::memcpy(&p.c, coef_of<T>(F).data(), sizeof(p.c));
  p.x = x; p.b = b; p.y = y; p.N = F.N; p.n = F.n;
  p.scale = T(1.0 / (F.h * F.h));
  p.zero = 0;
  p.row0 = w.row0; p.lrows = w.lrows; p.out_lo = w.out_lo; p.out_hi = w.out_hi;
  const int64_t ntx = (F.N + LY::C - 1) / LY::C;
  const int64_t nty = ((w.out_hi - 1) / K) / LY::C - (w.out_lo / K) / LY::C + 1;
  // ~8 column chunks per CTA (static balance), each as tall as possible
  const int64_t want = std::max<int64_t>(1, (8 * int64_t(grid_cache) + ntx - 1) / ntx);
  p.chunk = int(std::max<int64_t>(1, (nty + want - 1) / want));
  const int64_t nch = (nty + p.chunk - 1) / p.chunk;
  const int grid = (int)std::min<int64_t>(grid_cache, ntx * nch);
  apply2d_kernel<T, K, NT><<<grid, NT, smem, st>>>(p);
}

// CTA size: 128 threads for FP64 (the column-walk stages have ~128 register-blocked units at k = 4; measured
// residual k = 2..7 0.158/0.206/0.162/0.242/0.332/0.364 ms vs 0.158/0.214/0.192/0.280/0.315/0.423 ms with
// 256 threads), except k = 6; 256 for FP32; C0IP_APPLY_NT overrides (measurement knob)
template <typename T, int K>
static void launch_apply(const FusedLevel& F, const T* x, const T* b, T* y, const SlabWindow& w, cudaStream_t st) {
  static const int nt = [] {
    const char* e = std::getenv("C0IP_APPLY_NT");
    if (e) return std::atoi(e) == 128 ? 128 : 256;
    return (sizeof(T) == 8 && K != 6) ? 128 : 256;
  }();
  if (nt == 128) launch_apply_nt<T, K, 128>(F, x, b, y, w, st);
  else launch_apply_nt<T, K, 256>(F, x, b, y, w, st);
}

template <typename T, int K>
static void launch_fdm(const FusedLevel& F, T omega, const T* r, T* x, const SlabWindow& w, cudaStream_t st) {
  using LY = FdmLayout<T, K>;
  const size_t smem = sizeof(T) * size_t(LY::TOTAL);
  static int grid_cache = -1;
  if (grid_cache < 0) {
    cudaFuncSetAttribute(fdm2d_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(fdm2d_kernel<T, K>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    grid_cache = persistent_grid(fdm2d_kernel<T, K>, smem, 1 << 30);
  }
  FdmP<T, K> p;
  std::memcpy(&p.c, coef_of<T>(F).data(), sizeof(p.c));
  p.r = r; p.x = x; p.N = F.N; p.n = F.n;
  p.factor = T(double(omega) * F.h * F.h);
  p.zero = 0;
  p.row0 = w.row0; p.lrows = w.lrows; p.out_lo = w.out_lo; p.out_hi = w.out_hi;
  const int64_t ntx = (F.N + LY::C - 1) / LY::C;
  const int64_t nty = ((w.out_hi - 1) / K) / LY::C - (w.out_lo / K) / LY::C + 1;
  const int grid = (int)std::min<int64_t>(grid_cache, ntx * nty);
  fdm2d_kernel<T, K><<<grid, 256, smem, st>>>(p);
}

static SlabWindow full_window(const FusedLevel& F) { return SlabWindow{0, F.n, 1, int64_t(F.k) * F.N}; }

static void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
bool fused_apply(FusedLevel& F, const T* x, const T* b, T* y, cudaStream_t st, int64_t* launches,
                 const SlabWindow* win) {
  if (F.d != 2) return false;
  const SlabWindow w = win ? *win : full_window(F);
  if (w.out_hi <= w.out_lo) return true;
  switch (F.k) {
    case 2: launch_apply<T, 2>(F, x, b, y, w, st); break;
    case 3: launch_apply<T, 3>(F, x, b, y, w, st); break;
    case 4: launch_apply<T, 4>(F, x, b, y, w, st); break;
    case 5: launch_apply<T, 5>(F, x, b, y, w, st); break;
    case 6: launch_apply<T, 6>(F, x, b, y, w, st); break;
    case 7: launch_apply<T, 7>(F, x, b, y, w, st); break;
    default: return false;
  }
  (*launches)++;
  check_launch("fused apply2d launch");
  return true;
}

template <typename T>
bool fused_fdm(FusedLevel& F, T omega, const T* r, T* x, cudaStream_t st, int64_t* launches, const SlabWindow* win) {
  if (F.d != 2) return false;
  const SlabWindow w = win ? *win : full_window(F);
  if (w.out_hi <= w.out_lo) return true;
  if constexpr (std::is_same<T, double>::value) {
    if (mma_fdm2d(F, double(omega), r, x, w, st)) {
      (*launches)++;
      check_launch("fdm2d_mma launch");
      return true;
    }
  }
  switch (F.k) {
    case 2: launch_fdm<T, 2>(F, omega, r, x, w, st); break;
    case 3: launch_fdm<T, 3>(F, omega, r, x, w, st); break;
    case 4: launch_fdm<T, 4>(F, omega, r, x, w, st); break;
    case 5: launch_fdm<T, 5>(F, omega, r, x, w, st); break;
    case 6: launch_fdm<T, 6>(F, omega, r, x, w, st); break;
    case 7: launch_fdm<T, 7>(F, omega, r, x, w, st); break;
    default: return false;
  }
  (*launches)++;
  check_launch("fused fdm2d launch");
  return true;
}

template <typename T>
bool fused_avs(FusedLevel& F, T omega, const T* b, T* x, T* scratch, cudaStream_t st, int64_t* launches) {
  if (F.d != 2) return false;
  fused_apply<T>(F, x, b, scratch, st, launches, nullptr);       // r = b - A x (one residual per step)
  return fused_fdm<T>(F, omega, scratch, x, st, launches, nullptr);
}

template <typename T, int K>
static void launch_mvs(const FusedLevel& F, const int32_t* list, int64_t count, T omega, const T* b, T* x,
                       cudaStream_t st) {
  using LY = MvsLayout<T, K>;
  const size_t smem = sizeof(T) * size_t(LY::TOTAL);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(mvs2d_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(mvs2d_kernel<T, K>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  MvsP<T, K> p;
  std::memcpy(&p.c, coef_of<T>(F).data(), sizeof(p.c));
  p.x = x; p.b = b; p.list = list; p.count = count; p.N = F.N; p.n = F.n;
  p.scale = T(1.0 / (F.h * F.h));
  p.factor = T(double(omega) * F.h * F.h);
  p.zero = 0;
  const int64_t grid = (count + LY::PB - 1) / LY::PB;
  mvs2d_kernel<T, K><<<(unsigned)grid, 256, smem, st>>>(p);
}

// ----------------------------------------------------------------------------- patch_list2d
// x += omega h^2 A~_v^{-1} R_v r over a list of mutually disjoint patches (one MVS colour after a full
// residual): NP = 2K - 1 lanes per patch, PW = 32 / NP patches per warp; lane
// (p, j) loads row j of patch p and contracts it with S_x^T in registers, one transpose through a per-warp
// shared buffer gives lane (p, i) the column i for S_y^T, the scaling 1 / (lam_x,i + lam_y,j) and S_y, a
// second transpose returns the rows for S_x and the update (plain read-modify-write: the patches of the
// list are disjoint).  Each lane holds the row of G = 2 patches (two groups per warp iteration) so that a
// coefficient load serves two lines.  Warps whose patches are all interior take S as warp-uniform
// kernel-parameter operands, the others read the per-lane variants from a shared copy.  Used for the 2D MVS at k >= 5,
// where the fused per-patch footprint residual (mvs2d_kernel) costs more than one residual per colour.
template <typename T, int K>
struct PatchListP {
  Coef2<T, K> c;
  const T* r;
  T* x;
  const int32_t* list;
  int64_t count;
  int64_t N, n;
  T factor;                 // omega h^2
  int zero;
};

template <typename T, int K>
struct List2Layout {
  static constexpr int NP = 2 * K - 1, NP2 = NP * NP, PW = 32 / NP, LANES = PW * NP;
  static constexpr int G = 2;                      // patch groups per warp iteration (coefficient reuse)
  static constexpr int PR = NP | 1;                // odd row pitch
  static constexpr int GB = PW * NP * PR;          // one group's buffer
  static constexpr int WB = G * GB;                // per-warp buffer
  static constexpr int TOTAL = 8 * WB + NP2 + 3 * NP2 + 3 * NP;   // | interior 1/(lx+ly) | S[3] | lam[3]
};

template <typename T, int K>
__global__ void __launch_bounds__(256) patch_list2d_kernel(const __grid_constant__ PatchListP<T, K> P) {
  using LY = List2Layout<T, K>;
  constexpr int NP = LY::NP, NP2 = LY::NP2, PW = LY::PW, PR = LY::PR, G = LY::G;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* const sm = reinterpret_cast<T*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* const buf = sm + warp * LY::WB;
  T* const tab = sm + 8 * LY::WB;                  // [i][j] interior 1 / (lam_i + lam_j)
  T* const sS = tab + NP2;
  T* const sL = sS + 3 * NP2;
  for (int e = tid; e < NP2; e += 256) tab[e] = T(1) / (P.c.lam[1][e / NP] + P.c.lam[1][e % NP]);
  for (int e = tid; e < 3 * NP2; e += 256) sS[e] = P.c.S[e / NP2][e % NP2];
  for (int e = tid; e < 3 * NP; e += 256) sL[e] = P.c.lam[e / NP][e % NP];
  __syncthreads();
  const int64_t N = P.N, n = P.n;
  const int Nm1 = int(N - 1);
  const int p = lane / NP, j = lane - (lane / NP) * NP;
  const bool act = lane < LY::LANES;
  const int64_t ngroups = (P.count + G * PW - 1) / (G * PW), gstride = int64_t(gridDim.x) * 8;
  int round = 0;
#pragma unroll 1
  for (int64_t g = int64_t(blockIdx.x) * 8 + warp; g < ngroups; g += gstride, ++round) {
    // lane (p, j) holds row j of patch p of each of the G groups
    bool live[G];
    int varx[G], vary[G];
    int64_t g0[G];
    bool allin = true;
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const int64_t q = (g * G + h) * PW + p;
      live[h] = act && q < P.count;
      int vx = 1, vy = 1;
      if (live[h]) {
        const int pid = P.list[q];
        vy = 1 + pid / Nm1;
        vx = 1 + (pid - (vy - 1) * Nm1);
      }
      varx[h] = variant_of(vx, N);
      vary[h] = variant_of(vy, N);
      allin = allin && (!live[h] || (varx[h] == 1 && vary[h] == 1));
      // row j of the patch: nodes ((vx-1)K + 1 + i, (vy-1)K + 1 + j), interior index (jy - 1) n + (jx - 1)
      g0[h] = (int64_t(vy - 1) * K + j) * n + int64_t(vx - 1) * K;
    }
    const bool inner = __all_sync(0xffffffffu, allin);
    // the lines live in the per-warp buffer; each contraction walks its input index l at run time (one
    // buffer load per group and NP coefficient loads per l, shared by the G groups on interior warps), so
    // only the G x NP accumulators are live
    T* row[G];
    T* col[G];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      row[h] = buf + h * LY::GB + (p * NP + j) * PR;        // row j of patch p
      col[h] = buf + h * LY::GB + p * NP * PR + j;          // column i = j of patch p (stride PR)
      if (act) {
#pragma unroll
        for (int i = 0; i < NP; ++i) row[h][i] = live[h] ? P.r[g0[h] + i] : T(0);
      }
    }
    T o[G][NP];
    auto body = [&](auto INC) {
      constexpr bool IN = decltype(INC)::value;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      auto contract = [&](T* const* line, int stride, auto SEL, bool tr) {
        // o[h][a] = sum_l S_h[l NP + a] line_h[l stride] (tr) or S_h[a NP + l] line_h[l stride]
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
          for (int a2 = 0; a2 < NP; ++a2) o[h][a2] = 0;
#pragma unroll 1
        for (int l = 0; l < NP; ++l) {
          T wl[G];
#pragma unroll
          for (int h = 0; h < G; ++h) wl[h] = act ? line[h][l * stride] : T(0);
          if (IN) {
#pragma unroll
            for (int a2 = 0; a2 < NP; ++a2) {
              const T cf = c.S[1][tr ? l * NP + a2 : a2 * NP + l];
#pragma unroll
              for (int h = 0; h < G; ++h) o[h][a2] = fma(cf, wl[h], o[h][a2]);
            }
          } else {
#pragma unroll
            for (int h = 0; h < G; ++h) {
              const T* S = sS + SEL(h) * NP2;
#pragma unroll
              for (int a2 = 0; a2 < NP; ++a2) o[h][a2] = fma(S[tr ? l * NP + a2 : a2 * NP + l], wl[h], o[h][a2]);
            }
          }
        }
      };
      auto selx = [&](int h) { return varx[h]; };
      auto sely = [&](int h) { return vary[h]; };
      // S_x^T on row j
      contract(row, 1, selx, true);
      if (act) {
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
          for (int i = 0; i < NP; ++i) row[h][i] = o[h][i];
      }
      __syncwarp();
      // lane (p, j) now owns column i = j: S_y^T, scale 1 / (lam_x,i + lam_y,jj), S_y
      contract(col, PR, sely, true);
#pragma unroll
      for (int h = 0; h < G; ++h) {
        // interior patches multiply by the tabulated reciprocal on either path (a patch gives the same bits
        // whichever warp it lands in: the slab MVS colour lists group patches differently)
        if (IN || (varx[h] == 1 && vary[h] == 1)) {
#pragma unroll
          for (int jj = 0; jj < NP; ++jj) o[h][jj] *= tab[j * NP + jj];
        } else {
          const T lx = sL[varx[h] * NP + j];
#pragma unroll
          for (int jj = 0; jj < NP; ++jj) o[h][jj] *= T(1) / (lx + sL[vary[h] * NP + jj]);
        }
        if (act) {                                   // the column is this lane's own: no sync needed
#pragma unroll
          for (int jj = 0; jj < NP; ++jj) col[h][jj * PR] = o[h][jj];
        }
      }
      contract(col, PR, sely, false);
      if (act) {
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
          for (int jj = 0; jj < NP; ++jj) col[h][jj * PR] = o[h][jj];
      }
      __syncwarp();
      // S_x on row j
      contract(row, 1, selx, false);
      __syncwarp();                                  // the buffer is rewritten by the next iteration
    };
    if (inner) body(std::true_type{});
    else body(std::false_type{});
#pragma unroll
    for (int h = 0; h < G; ++h)
      if (live[h]) {
#pragma unroll
        for (int i = 0; i < NP; ++i) P.x[g0[h] + i] = fma(P.factor, o[h][i], P.x[g0[h] + i]);
      }
  }
}

template <typename T, int K>
static void launch_list2d(const FusedLevel& F, T omega, const T* r, T* x, const int32_t* list, int64_t count,
                          cudaStream_t st) {
  using LY = List2Layout<T, K>;
  const size_t smem = sizeof(T) * size_t(LY::TOTAL);
  static int grid_cache = -1;
  if (grid_cache < 0) {
    cudaFuncSetAttribute(patch_list2d_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    grid_cache = persistent_grid(patch_list2d_kernel<T, K>, smem, 1 << 30);
  }
  PatchListP<T, K> p;
  std::memcpy(&p.c, coef_of<T>(F).data(), sizeof(p.c));
  p.r = r; p.x = x; p.list = list; p.count = count; p.N = F.N; p.n = F.n;
  p.factor = T(double(omega) * F.h * F.h);
  p.zero = 0;
  const int64_t groups = (count + LY::G * LY::PW - 1) / (LY::G * LY::PW);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(grid_cache, (groups + 7) / 8));
  patch_list2d_kernel<T, K><<<(unsigned)grid, 256, smem, st>>>(p);
}

// whether the 2D MVS colour runs as residual + patch_list2d instead of the fused per-patch kernels:
// k = 2 and k >= 5 (measured MVS step: k = 2 9.9 vs 7.8 GDoF/s for mvs2d_mma, whose 8x8 fragments pad the
// 3-point patch lines; k = 3, 4: 7.7 / 8.7 vs 13.6 / 14.4); C0IP_MVS2D_SPLIT_K = m splits exactly k >= m
// (measurement knob)
static bool mvs2d_split(int k) {
  static const int m = [] {
    const char* e = std::getenv("C0IP_MVS2D_SPLIT_K");
    return e ? std::atoi(e) : 0;
  }();
  return m > 0 ? k >= m : (k == 2 || k >= 5);
}

template <typename T>
bool fused2_patch_list(FusedLevel& F, T omega, const T* r, T* x, const int32_t* list, int64_t count,
                       cudaStream_t st, int64_t* launches) {
  if (F.d != 2) return false;
  if (count == 0) return true;
  switch (F.k) {
    case 2: launch_list2d<T, 2>(F, omega, r, x, list, count, st); break;
    case 3: launch_list2d<T, 3>(F, omega, r, x, list, count, st); break;
    case 4: launch_list2d<T, 4>(F, omega, r, x, list, count, st); break;
    case 5: launch_list2d<T, 5>(F, omega, r, x, list, count, st); break;
    case 6: launch_list2d<T, 6>(F, omega, r, x, list, count, st); break;
    case 7: launch_list2d<T, 7>(F, omega, r, x, list, count, st); break;
    default: return false;
  }
  (*launches)++;
  check_launch("patch_list2d launch");
  return true;
}

template <typename T>
bool fused_mvs_color(FusedLevel& F, const int32_t* list, int64_t count, T omega, const T* b, T* x, cudaStream_t st,
                     int64_t* launches) {
  if (F.d != 2) return false;
  if (count == 0) return true;
  if (mvs2d_split(F.k)) return false;          // caller: residual + fused2_patch_list per colour
  if constexpr (std::is_same<T, double>::value) {
    if (mma_mvs2d(F, list, count, double(omega), b, x, st)) {
      (*launches)++;
      check_launch("mvs2d_mma launch");
      return true;
    }
  }
  switch (F.k) {
    case 2: launch_mvs<T, 2>(F, list, count, omega, b, x, st); break;
    case 3: launch_mvs<T, 3>(F, list, count, omega, b, x, st); break;
    case 4: launch_mvs<T, 4>(F, list, count, omega, b, x, st); break;
    case 5: launch_mvs<T, 5>(F, list, count, omega, b, x, st); break;
    case 6: launch_mvs<T, 6>(F, list, count, omega, b, x, st); break;
    case 7: launch_mvs<T, 7>(F, list, count, omega, b, x, st); break;
    default: return false;
  }
  (*launches)++;
  check_launch("fused mvs2d launch");
  return true;
}

bool fused_supports_slab(const FusedLevel& F) { return F.d == 2 || (F.d == 3 && F.k <= 5); }
int fused_dim(const FusedLevel& F) { return F.d; }

#define C0IP_INST(T)                                                                                       \
  template bool fused_apply<T>(FusedLevel&, const T*, const T*, T*, cudaStream_t, int64_t*, const SlabWindow*); \
  template bool fused_fdm<T>(FusedLevel&, T, const T*, T*, cudaStream_t, int64_t*, const SlabWindow*);        \
  template bool fused_avs<T>(FusedLevel&, T, const T*, T*, T*, cudaStream_t, int64_t*);                        \
  template bool fused_mvs_color<T>(FusedLevel&, const int32_t*, int64_t, T, const T*, T*, cudaStream_t, int64_t*); \
  template bool fused2_patch_list<T>(FusedLevel&, T, const T*, T*, const int32_t*, int64_t, cudaStream_t, int64_t*);
C0IP_INST(double)
C0IP_INST(float)
#undef C0IP_INST

}  // namespace c0ip
