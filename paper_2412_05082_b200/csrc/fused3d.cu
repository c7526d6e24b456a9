// Fused kernels for large 3D levels (sm_100a, FP64 and FP32), k = 2..5.
//
//   apply3d      : r = b - A x (or y = A x) with A = h^-1 (B^M^M^ + M^B^M^ + M^M^B^ + 2(L^L^M^ + M^L^L^ +
//                  L^M^L^)) (Eq. c0iptensorvp3D).  A CTA owns a C x C in-plane tile
//                  and a chunk of CZ cell layers along z and streams through z: per cell layer it
//                  builds, for K new node planes, the in-plane results
//                    P = B^_y M^_x + M^_y B^_x + 2 L^_y L^_x,  Q = L^_y M^_x + M^_y L^_x,  R = M^_y M^_x
//                  (x- and y-stages in shared memory); each thread, owning one in-plane node, adds
//                  every arriving plane of P, Q, R into the 4K + 1 pending outputs of its z column
//                    y = M^_z P + 2 L^_z Q + B^_z R
//                  (scatter form of the banded z rows, uniform coefficients) and emits the finished
//                  cell layer.
//   patch_fdm3d  : x += omega h A~_v^{-1} R_v r for a list of patches: per patch the
//                  six 1D contractions (S^T along x, y, z; divide by lambda_x + lambda_y + lambda_z; S
//                  along z, y, x) with one thread per patch line and register-blocked lines.  Launched
//                  per parity class (2^d non-overlapping classes, plain stores: deterministic) for the
//                  additive smoother and per colour for the multiplicative one.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "fused_common.cuh"

namespace c0ip {

template <int K>
struct Tile3 {
  static constexpr int C = (K == 2) ? 8 : (K == 3) ? 5 : (K == 4) ? 4 : 3;   // in-plane cells
  static constexpr int O = C * K;                                            // owned nodes per axis (<= 16)
  static constexpr int CZ = 32;                                              // cell layers per chunk
};

template <typename T, int K>
struct Apply3P {
  Coef2<T, K> c;
  const T* x;
  const T* b;
  T* y;
  int64_t N, n;
  int64_t row0, lrows;      // slab window along z (see SlabWindow); the full domain: 0, n
  int64_t out_lo, out_hi;   // node planes written
  int64_t cz_lo, cz_hi;     // cell layers covering [out_lo, out_hi)
  T scale;                  // h^-1
  int zero;
};

template <typename T, int K>
struct Apply3Layout {
  static constexpr int C = Tile3<K>::C, O = Tile3<K>::O;
  static constexpr int BW = (C + 3) * K + 1;      // in-plane box [(c0-2)K, (c0+C+1)K]
  // x-stage output pitch odd and >= O + 1: with the y-stage columns padded to OP = 16 lanes per cell row (O = 15
  // at k = 3, 5) the two half-warps cover every bank pair once (PO = 15 gave 3-way conflicts on the column loads)
  static constexpr int PX = odd(BW), PO = odd(O + 1), OP = (O == 15) ? 16 : O;
  static constexpr int XB = K * BW * PX;          // K planes of the box (double buffered)
  static constexpr int SX = K * 3 * BW * PO;      // x-stage outputs (B, L, M) of K planes
  static constexpr int PQR = K * 3 * O * O;       // in-plane results of K planes
  static constexpr int TOTAL = 2 * XB + SX + PQR;
  static constexpr int MINB = (K <= 3) ? 2 : 1;   // CTAs per SM (registers / shared memory)
};

// banded row of class PP applied to a window w (w index o <-> offset o - 2K around the output node)
template <typename T, int K, int PP, int W, typename F>
__device__ __forceinline__ T row_band(F coef, const T* w, int base) {
  T s = 0;
#pragma unroll
  for (int q = 0; q <= W - 1; ++q) {
    const bool nz = (W == 4 * K + 1) ? (PP == 0 || (q >= K - PP && q <= 4 * K - PP))
                                     : (PP == 0 || (q >= K - PP && q <= 2 * K - PP));
    if (nz) s = fma(coef(q), w[base + PP + q], s);
  }
  return s;
}

// K node planes z0 .. z0+K-1 of the in-plane box into smem (cp.async, zero fill outside the domain)
// (node plane jz lives at local plane jz - 1 - row0, valid for local planes [0, lrows)).  Thread t copies
// the in-plane positions t, t + 256, ... of the BW x BW box for all K planes: one split of the position
// by a compile-time constant per position, the 64-bit base address formed once per call, so a box inside
// the domain (every CTA but the boundary ones) costs a few integer instructions per element.
template <typename T, int K, int BW, int PX>
__device__ __forceinline__ void load_planes_async(T* dst, const T* src, int64_t n, int64_t KN, int64_t z0,
                                                  int64_t Y0, int64_t X0, int64_t row0, int64_t lrows) {
  constexpr int TOT2 = BW * BW;
  const int64_t zlo = (row0 + 1 > 1) ? row0 + 1 : int64_t(1), zhi = (row0 + lrows < KN - 1) ? row0 + lrows : KN - 1;
  const bool inner = (X0 >= 1 && X0 + BW - 1 <= KN - 1 && Y0 >= 1 && Y0 + BW - 1 <= KN - 1 && z0 >= zlo &&
                      z0 + K - 1 <= zhi);
  const T* base = src + ((z0 - 1 - row0) * n + (Y0 - 1)) * n + (X0 - 1);
  const int64_t pstride = n * n;
  for (int rc = threadIdx.x; rc < TOT2; rc += 256) {
    const int r = rc / BW, cc = rc - r * BW;
    T* const d = dst + r * PX + cc;
    const T* const s0 = base + int64_t(r) * n + cc;
    if (inner) {
#pragma unroll
      for (int pz = 0; pz < K; ++pz) cp_async_elem(d + pz * (BW * PX), s0 + pz * pstride, true);
    } else {
      const int64_t jy = Y0 + r, jx = X0 + cc;
      const bool xy = jy >= 1 && jy <= KN - 1 && jx >= 1 && jx <= KN - 1;
#pragma unroll
      for (int pz = 0; pz < K; ++pz) {
        const bool ok = xy && z0 + pz >= zlo && z0 + pz <= zhi;
        cp_async_elem(d + pz * (BW * PX), ok ? s0 + pz * pstride : src, ok);
      }
    }
  }
}

template <typename T, int K>
__global__ void __launch_bounds__(256, Apply3Layout<T, K>::MINB) apply3d_kernel(const __grid_constant__ Apply3P<T, K> P) {
  using LY = Apply3Layout<T, K>;
  constexpr int C = LY::C, O = LY::O, BW = LY::BW, PX = LY::PX, PO = LY::PO, CZ = Tile3<K>::CZ;
  constexpr int NT = 256;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* const xb0 = sm;              // [2][K][BW][PX]
  T* sx = xb0 + 2 * LY::XB;       // [K][3][BW][PO]  (0: B^x, 1: L^x, 2: M^x)
  T* pqr = sx + LY::SX;           // [K][3][O][O]    (0: P, 1: Q, 2: R)
  const int64_t N = P.N, n = P.n, KN = K * N;
  const int ntx = int((N + C - 1) / C);
  const int tile = blockIdx.x % (ntx * ntx), chunk = blockIdx.x / (ntx * ntx);
  const int64_t cx0 = int64_t(tile % ntx) * C, cy0 = int64_t(tile / ntx) * C, cz0 = P.cz_lo + int64_t(chunk) * CZ;
  const int tid = threadIdx.x;
  // tiles whose cells are all interior along x / y take the all-classes interior rows (CTA-uniform)
  const bool tinx = (cx0 >= 2 && cx0 + C - 1 <= N - 2), tiny = (cy0 >= 2 && cy0 + C - 1 <= N - 2);
  const int oy = tid / O, ox = tid - (tid / O) * O;       // z-stage ownership (tid < O*O)
  const bool zown = tid < O * O;
  // z-stage, two forms (measured per degree):
  //  * scatter (k = 3): acc[i] <-> output node plane (cn - 2) K + i, i in [0, 4K], where cn is the cell
  //    layer whose K node planes ((cn-1)K, cnK] arrive at this step; every arriving plane adds its P, Q, R
  //    values to the outputs within the band (M^_z, 2 L^_z, B^_z), and layer cn - 2 is complete.  4K + 1
  //    live registers instead of 10K + 3 (frees the registers for XR = 2 in the x-stage at 2 CTAs/SM);
  //  * windows (k = 2, 4, 5): sliding register windows of P, Q, R along z, output-centric banded rows.
  constexpr bool SCAT = (K == 3);
  T acc[SCAT ? 4 * K + 1 : 1];
#pragma unroll
  for (int i = 0; i < (SCAT ? 4 * K + 1 : 1); ++i) acc[i] = 0;
  T wR[SCAT ? 1 : 4 * K + 1], wP[SCAT ? 1 : 3 * K + 1], wQ[SCAT ? 1 : 3 * K + 1];
#pragma unroll
  for (int i = 0; i < (SCAT ? 1 : 4 * K + 1); ++i) wR[i] = 0;
#pragma unroll
  for (int i = 0; i < (SCAT ? 1 : 3 * K + 1); ++i) wP[i] = wQ[i] = 0;
  int round = 0;
  const int nsteps = int(std::min<int64_t>(CZ, P.cz_hi - cz0)) + 4;

  // prefetch pipeline: the K planes of step s + 1 load while step s computes
  load_planes_async<T, K, BW, PX>(xb0, P.x, n, KN, (cz0 - 3) * K + 1, (cy0 - 2) * K, (cx0 - 2) * K, P.row0, P.lrows);
  cp_async_commit();
  for (int s = 0; s < nsteps; ++s) {
    // node planes of this step: (cz0 - 3 + s) K + 1 + pz, pz < K
    if (s + 1 < nsteps)
      load_planes_async<T, K, BW, PX>(xb0 + ((s + 1) & 1) * LY::XB, P.x, n, KN, (cz0 - 2 + s) * K + 1,
                                      (cy0 - 2) * K, (cx0 - 2) * K, P.row0, P.lrows);
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    const T* xb = xb0 + (s & 1) * LY::XB;

    // x-stage: unit = (plane, box row group, cell) -> B^ L^ M^ along x for the K nodes of the cell;
    // rows hr, hr + HB, ... (XR rows) share every coefficient load (register blocking; fits the 2-CTA
    // register budget at every degree since the z-stage holds 4K + 1 accumulators instead of windows)
    {
      constexpr int XR = (K == 3 && sizeof(T) == 8 && !SCAT) ? 1 : 2;
      constexpr int HB = cdiv(BW, XR);
#pragma unroll 1
      for (int it = 0; it < cdiv(K * HB * C, NT); ++it, ++round) {
        const int u = it * NT + tid;
        const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
        if (u >= K * HB * C) continue;
        const int hr = u % HB, rest = u / HB, ci = rest % C, pz = rest / C;
        const int64_t cx = cx0 + ci;
        if (cx >= N) continue;
        int rr[XR];
#pragma unroll
        for (int j = 0; j < XR; ++j) rr[j] = min(hr + j * HB, BW - 1);
        T w[XR][4 * K + 1];
#pragma unroll
        for (int j = 0; j < XR; ++j)
#pragma unroll
          for (int q = 0; q <= 4 * K; ++q) w[j][q] = xb[(pz * BW + rr[j]) * PX + ci * K + q];
        if (tinx) {                 // every cell of the tile interior along x: all K classes at once
          T ob[K][XR], ol[K][XR], om[K][XR];
          x_all_interior<T, K, XR>(c, w, ob, ol, om);
#pragma unroll
          for (int p = 0; p < K; ++p)
#pragma unroll
            for (int j = 0; j < XR; ++j) {
              if (hr + j * HB >= BW) continue;
              const int r = rr[j];
              sx[((pz * 3 + 0) * BW + r) * PO + ci * K + p] = ob[p][j];
              sx[((pz * 3 + 1) * BW + r) * PO + ci * K + p] = ol[p][j];
              sx[((pz * 3 + 2) * BW + r) * PO + ci * K + p] = om[p][j];
            }
          continue;
        }
        const bool inner = (cx >= 2 && cx <= N - 2);
#pragma unroll
        for (int p = 0; p < K; ++p) {
          T ob[XR], ol[XR], om[XR];
#pragma unroll
          for (int j = 0; j < XR; ++j) ob[j] = ol[j] = om[j] = T(0);
          const int sp = inner ? -1 : special_row<K>(cx * K + p, N);
          with_p<K>(p, [&](auto PC) {
            constexpr int PP = decltype(PC)::value;
            if (sp < 0) {
              rowB<T, K, PP>([&](int q) { return c.BI[PP][q]; }, w, 0, ob);
              rowML<T, K, PP>([&](int q) { return c.LI[PP][q]; }, w, K, ol);
              rowML<T, K, PP>([&](int q) { return c.MI[PP][q]; }, w, K, om);
            } else {
              rowB<T, K, PP>([&](int q) { return c.BS[sp][q]; }, w, 0, ob);
              rowML<T, K, PP>([&](int q) { return c.LS[sp][q + K]; }, w, K, ol);
              rowML<T, K, PP>([&](int q) { return c.MS[sp][q + K]; }, w, K, om);
            }
          });
#pragma unroll
          for (int j = 0; j < XR; ++j) {
            if (hr + j * HB >= BW) continue;
            const int r = rr[j];
            sx[((pz * 3 + 0) * BW + r) * PO + ci * K + p] = ob[j];
            sx[((pz * 3 + 1) * BW + r) * PO + ci * K + p] = ol[j];
            sx[((pz * 3 + 2) * BW + r) * PO + ci * K + p] = om[j];
          }
        }
      }
    }
    __syncthreads();

    // y-stage: unit = (plane, owned column, cell row) -> P, Q, R for the K nodes of the cell row
#pragma unroll 1
    for (int it = 0; it < cdiv(K * LY::OP * C, NT); ++it, ++round) {
      const int u = it * NT + tid;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      if (u >= K * LY::OP * C) continue;
      const int col = u % LY::OP, rest = u / LY::OP, ci = rest % C, pz = rest / C;
      if (col >= O) continue;
      const int64_t cy = cy0 + ci;
      if (cy >= N) continue;
      const T* sB = sx + (pz * 3 + 0) * BW * PO;
      const T* sL = sx + (pz * 3 + 1) * BW * PO;
      const T* sM = sx + (pz * 3 + 2) * BW * PO;
      T wM[4 * K + 1], wB[2 * K + 1], wL[2 * K + 1];
#pragma unroll
      for (int q = 0; q <= 4 * K; ++q) wM[q] = sM[(ci * K + q) * PO + col];
#pragma unroll
      for (int q = 0; q <= 2 * K; ++q) {
        wB[q] = sB[(ci * K + K + q) * PO + col];
        wL[q] = sL[(ci * K + K + q) * PO + col];
      }
      if (tiny) {                   // every cell row of the tile interior along y: all K classes at once
        T w1[1][4 * K + 1], wb[1][2 * K + 1], wl[1][2 * K + 1], wmk[1][2 * K + 1];
#pragma unroll
        for (int q = 0; q <= 4 * K; ++q) w1[0][q] = wM[q];
#pragma unroll
        for (int q = 0; q <= 2 * K; ++q) { wb[0][q] = wB[q]; wl[0][q] = wL[q]; wmk[0][q] = wM[K + q]; }
        T aP[K][1], aL[K][1], aQ[K][1], aR[K][1];
#pragma unroll
        for (int p = 0; p < K; ++p) aP[p][0] = aL[p][0] = aQ[p][0] = aR[p][0] = T(0);
        y_all_interior<T, K, 1, 0, 4 * K + 1>(c, w1, aP);     // B^_y (M^_x x)
        y_all_interior<T, K, 1, 1, 2 * K + 1>(c, wb, aP);     // M^_y (B^_x x)
        y_all_interior<T, K, 1, 2, 2 * K + 1>(c, wl, aL);     // L^_y (L^_x x)
        y_all_interior<T, K, 1, 2, 2 * K + 1>(c, wmk, aQ);    // L^_y (M^_x x)
        y_all_interior<T, K, 1, 1, 2 * K + 1>(c, wl, aQ);     // M^_y (L^_x x)
        y_all_interior<T, K, 1, 1, 2 * K + 1>(c, wmk, aR);    // M^_y (M^_x x)
#pragma unroll
        for (int p = 0; p < K; ++p) {
          const int orow = ci * K + p;
          pqr[((pz * 3 + 0) * O + orow) * O + col] = fma(T(2), aL[p][0], aP[p][0]);
          pqr[((pz * 3 + 1) * O + orow) * O + col] = aQ[p][0];
          pqr[((pz * 3 + 2) * O + orow) * O + col] = aR[p][0];
        }
        continue;
      }
      const bool inner = (cy >= 2 && cy <= N - 2);
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const int sp = inner ? -1 : special_row<K>(cy * K + p, N);
        T vP = 0, vQ = 0, vR = 0;
        with_p<K>(p, [&](auto PC) {
          constexpr int PP = decltype(PC)::value;
          if (sp < 0) {
            vP = row_band<T, K, PP, 4 * K + 1>([&](int q) { return c.BI[PP][q]; }, wM, 0) +
                 row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.MI[PP][q]; }, wB, 0) +
                 T(2) * row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.LI[PP][q]; }, wL, 0);
            vQ = row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.LI[PP][q]; }, wM, K) +
                 row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.MI[PP][q]; }, wL, 0);
            vR = row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.MI[PP][q]; }, wM, K);
          } else {
            vP = row_band<T, K, PP, 4 * K + 1>([&](int q) { return c.BS[sp][q]; }, wM, 0) +
                 row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.MS[sp][q + K]; }, wB, 0) +
                 T(2) * row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.LS[sp][q + K]; }, wL, 0);
            vQ = row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.LS[sp][q + K]; }, wM, K) +
                 row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.MS[sp][q + K]; }, wL, 0);
            vR = row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.MS[sp][q + K]; }, wM, K);
          }
        });
        const int orow = ci * K + p;
        pqr[((pz * 3 + 0) * O + orow) * O + col] = vP;
        pqr[((pz * 3 + 1) * O + orow) * O + col] = vQ;
        pqr[((pz * 3 + 2) * O + orow) * O + col] = vR;
      }
    }
    __syncthreads();

    if constexpr (SCAT) {
      // z-stage (scatter form, see acc above): the K planes appended now are (cn-1)K + 1 + pz, cn = cz0 - 2 + s
      const int64_t cn = cz0 - 2 + s, cz = cn - 2;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      if (zown) {
        // every output node of the pending range is an interior-class row unless the range meets the
        // boundary rows j <= K or j >= KN - K (uniform over the CTA)
        const bool zin = (cn - 2) * K > K && (cn + 2) * K < KN - K;
#pragma unroll
        for (int pz = 0; pz < K; ++pz) {
          const T vP = pqr[((pz * 3 + 0) * O + oy) * O + ox];
          const T vQ = T(2) * pqr[((pz * 3 + 1) * O + oy) * O + ox];
          const T vR = pqr[((pz * 3 + 2) * O + oy) * O + ox];
#pragma unroll
          for (int i = 0; i <= 4 * K; ++i) {
            const int d = K + 1 + pz - i;              // input plane - output plane
            const int po = i % K;                      // class of the output node
            const int qb = d + 2 * K, qm = d + K;      // B index (offsets -2K..2K), M/L index (-K..K)
            const bool nzb = qb >= 0 && qb <= 4 * K && (po == 0 || (qb >= K - po && qb <= 4 * K - po));
            const bool nzm = qm >= 0 && qm <= 2 * K && (po == 0 || (qm >= K - po && qm <= 2 * K - po));
            if (!nzb && !nzm) continue;
            if (zin) {
              if (nzb) acc[i] = fma(c.BI[po][nzb ? qb : 0], vR, acc[i]);
              if (nzm) {
                acc[i] = fma(c.MI[po][nzm ? qm : 0], vP, acc[i]);
                acc[i] = fma(c.LI[po][nzm ? qm : 0], vQ, acc[i]);
              }
            } else {
              const int sp = special_row<K>((cn - 2) * K + i, N);
              if (sp < 0) {
                if (nzb) acc[i] = fma(c.BI[po][nzb ? qb : 0], vR, acc[i]);
                if (nzm) {
                  acc[i] = fma(c.MI[po][nzm ? qm : 0], vP, acc[i]);
                  acc[i] = fma(c.LI[po][nzm ? qm : 0], vQ, acc[i]);
                }
              } else if (qb >= 0 && qb <= 4 * K) {       // special rows: offsets -2K..2K, zero padded
                acc[i] = fma(c.BS[sp][qb], vR, acc[i]);
                acc[i] = fma(c.MS[sp][qb], vP, acc[i]);
                acc[i] = fma(c.LS[sp][qb], vQ, acc[i]);
              }
            }
          }
        }
      }
      // layer cz = cn - 2 is complete (emitted for cz >= cz0, i.e. s >= 4)
      if (s >= 4 && zown) {
        const int64_t jx = cx0 * K + ox, jy = cy0 * K + oy;
        if (jx >= 1 && jx <= KN - 1 && jy >= 1 && jy <= KN - 1) {
#pragma unroll
          for (int p = 0; p < K; ++p) {
            const int64_t jz = cz * K + p;
            if (jz < P.out_lo || jz >= P.out_hi) continue;
            const int64_t g = ((jz - 1 - P.row0) * n + (jy - 1)) * n + (jx - 1);
            const T v = acc[p] * P.scale;
            P.y[g] = P.b ? P.b[g] - v : v;
          }
        }
      }
      // shift the pending outputs by one cell layer
#pragma unroll
      for (int i = 0; i <= 3 * K; ++i) acc[i] = acc[i + K];
#pragma unroll
      for (int i = 3 * K + 1; i <= 4 * K; ++i) acc[i] = 0;
    } else {
      // z-stage: shift the windows by K planes, append the new ones, emit the finished cell layer
      if (zown) {
#pragma unroll
        for (int i = 0; i <= 3 * K; ++i) wR[i] = wR[i + K];
#pragma unroll
        for (int i = 0; i <= 2 * K; ++i) { wP[i] = wP[i + K]; wQ[i] = wQ[i + K]; }
#pragma unroll
        for (int pz = 0; pz < K; ++pz) {
          wP[2 * K + 1 + pz] = pqr[((pz * 3 + 0) * O + oy) * O + ox];
          wQ[2 * K + 1 + pz] = pqr[((pz * 3 + 1) * O + oy) * O + ox];
          wR[3 * K + 1 + pz] = pqr[((pz * 3 + 2) * O + oy) * O + ox];
        }
      }
      // after this step the newest plane is (cz0 - 2 + s) K: layer cz = cz0 + s - 4 is complete
      const int64_t cz = cz0 + s - 4;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      if (s >= 4 && zown) {
        const int64_t jx = cx0 * K + ox, jy = cy0 * K + oy;
        if (jx >= 1 && jx <= KN - 1 && jy >= 1 && jy <= KN - 1) {
          const bool inner = (cz >= 2 && cz <= N - 2);
#pragma unroll
          for (int p = 0; p < K; ++p) {
            const int64_t jz = cz * K + p;
            if (jz < P.out_lo || jz >= P.out_hi) continue;
            const int sp = inner ? -1 : special_row<K>(jz, N);
            T v = 0;
            // windows: wR[i] <-> plane (cz-2)K + i ; wP/wQ[i] <-> plane (cz-1)K + i
            with_p<K>(p, [&](auto PC) {
              constexpr int PP = decltype(PC)::value;
              if (sp < 0)
                v = row_band<T, K, PP, 4 * K + 1>([&](int q) { return c.BI[PP][q]; }, wR, 0) +
                    row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.MI[PP][q]; }, wP, 0) +
                    T(2) * row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.LI[PP][q]; }, wQ, 0);
              else
                v = row_band<T, K, PP, 4 * K + 1>([&](int q) { return c.BS[sp][q]; }, wR, 0) +
                    row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.MS[sp][q + K]; }, wP, 0) +
                    T(2) * row_band<T, K, PP, 2 * K + 1>([&](int q) { return c.LS[sp][q + K]; }, wQ, 0);
            });
            const int64_t g = ((jz - 1 - P.row0) * n + (jy - 1)) * n + (jx - 1);
            v *= P.scale;
            P.y[g] = P.b ? P.b[g] - v : v;
          }
        }
      }
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------- patch_fdm3d
template <typename T, int K>
struct Fdm3P {
  Coef2<T, K> c;
  const T* r;
  T* x;
  const int32_t* list;      // patch ids, or nullptr: the box of vertices vlo + vstr * i, i < vcnt (per axis)
  int64_t count;
  int vlo[3], vcnt[3], vstr;
  unsigned mag[2];          // floor((2^32 - 1) / d) for d = vcnt[0], vcnt[1] (list mode: N - 1, (N - 1)^2)
  int zc, zpar;             // zrun: patches per z chunk, parity of the chunks of this launch
  int64_t N, n;
  int64_t row0, lrows;      // slab window along z (see SlabWindow); the full domain: 0, n
  int64_t out_lo, out_hi;   // node planes written
  T factor;                 // omega h (A~^-1 = h A^~^-1 in 3D)
  int zero;
  int atomic;               // 1: overlapping patches (atomic AVS, red.global.add), 0: disjoint list
};

// CTA-cooperative variant (PB patches per CTA, one thread per patch line, smem gather/scatter): faster
// than the warp-per-patch kernel for the disjoint parity-class / colour lists (plain stores)
template <typename T, int K>
struct Fdm3CtaLayout {
  static constexpr int NP = 2 * K - 1, NL = NP * NP * NP;
  static constexpr int PB = cdiv(256, NP * NP);   // patches per CTA so that one stage ~ 256 lines
  static constexpr int TOTAL = 2 * PB * NL;
};

// one 1D contraction along axis AX of every patch line: out = S^T in (TR) or S in (!TR)
template <typename T, int K, int AX, bool TR>
__device__ __forceinline__ void contract3(const Coef2<T, K>& c, int var, const T* in, T* out) {
  constexpr int NP = 2 * K - 1;
  constexpr int ST = AX == 0 ? 1 : (AX == 1 ? NP : NP * NP);
  T w[NP];
#pragma unroll
  for (int l = 0; l < NP; ++l) w[l] = in[l * ST];
  auto body = [&](auto VC) {
    constexpr int V = decltype(VC)::value;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      T s = 0;
#pragma unroll
      for (int l = 0; l < NP; ++l) s = fma(TR ? c.S[V][l * NP + i] : c.S[V][i * NP + l], w[l], s);
      out[i * ST] = s;
    }
  };
  if (var == 1) body(std::integral_constant<int, 1>{});
  else if (var == 0) body(std::integral_constant<int, 0>{});
  else body(std::integral_constant<int, 2>{});
}

template <typename T, int K>
__global__ void __launch_bounds__(256, 2) patch_fdm3d_cta_kernel(const __grid_constant__ Fdm3P<T, K> P) {
  using LY = Fdm3CtaLayout<T, K>;
  constexpr int NP = LY::NP, NL = LY::NL, PB = LY::PB;
  constexpr int NT = 256;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* buf0 = reinterpret_cast<T*>(smem_raw);
  T* buf1 = buf0 + PB * NL;
  __shared__ int64_t gbase[PB];       // global index of the patch's first DoF (or -1)
  __shared__ int8_t pvar[PB][3];      // axis variants
  __shared__ int pjz[PB];             // node plane of the patch's first DoF plane
  const int64_t N = P.N, n = P.n;
  const int tid = threadIdx.x;
  int round = 0;
  if (tid < PB) {
    const int64_t q = (int64_t)blockIdx.x * PB + tid;
    if (q < P.count) {
      int vx, vy, vz;
      if (P.list) {
        const int pid = P.list[q], Nm1 = (int)(N - 1);
        vx = 1 + pid % Nm1; vy = 1 + (pid / Nm1) % Nm1; vz = 1 + pid / (Nm1 * Nm1);
      } else {
        const int iq = (int)q, ix = iq % P.vcnt[0], rest = iq / P.vcnt[0];
        vx = P.vlo[0] + P.vstr * ix;
        vy = P.vlo[1] + P.vstr * (rest % P.vcnt[1]);
        vz = P.vlo[2] + P.vstr * (rest / P.vcnt[1]);
      }
      gbase[tid] = (((int64_t)(vz - 1) * K - P.row0) * n + (int64_t)(vy - 1) * K) * n + (int64_t)(vx - 1) * K;
      pjz[tid] = (vz - 1) * K + 1;
      pvar[tid][0] = (int8_t)variant_of(vx, N);
      pvar[tid][1] = (int8_t)variant_of(vy, N);
      pvar[tid][2] = (int8_t)variant_of(vz, N);
    } else {
      gbase[tid] = -1;
    }
  }
  __syncthreads();
  // gather R_v r (every plane of a patch touching the owned planes lies inside the slab window)
  for (int e = tid; e < PB * NL; e += NT) {
    const int p = e / NL, l = e - p * NL;
    const int lx = l % NP, ly = (l / NP) % NP, lz = l / (NP * NP);
    const int64_t g0 = gbase[p];
    buf0[e] = g0 >= 0 ? P.r[g0 + ((int64_t)lz * n + ly) * n + lx] : T(0);
  }
  __syncthreads();
  T* in = buf0;
  T* out = buf1;
  // S^T along x, y, z; divide; S along z, y, x  (one thread per patch line; units = (patch, line))
#pragma unroll
  for (int stage = 0; stage < 6; ++stage) {
    const int ax = stage < 3 ? stage : 5 - stage;
#pragma unroll 1
    for (int it = 0; it < cdiv(PB * NP * NP, NT); ++it, ++round) {
      const int u = it * NT + tid;
      if (u >= PB * NP * NP) continue;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      const int p = u / (NP * NP), li = u - p * (NP * NP);
      if (gbase[p] < 0) continue;
      const int var = pvar[p][ax];
      int base;
      if (ax == 0) base = li * NP;                                   // line (ly, lz)
      else if (ax == 1) base = (li / NP) * NP * NP + (li % NP);      // line (lx, lz)
      else base = li;                                                // line (lx, ly)
      T* o = out + p * NL + base;
      const T* ii = in + p * NL + base;
      if (ax == 0) { if (stage < 3) contract3<T, K, 0, true>(c, var, ii, o); else contract3<T, K, 0, false>(c, var, ii, o); }
      else if (ax == 1) { if (stage < 3) contract3<T, K, 1, true>(c, var, ii, o); else contract3<T, K, 1, false>(c, var, ii, o); }
      else { if (stage < 3) contract3<T, K, 2, true>(c, var, ii, o); else contract3<T, K, 2, false>(c, var, ii, o); }
    }
    __syncthreads();
    T* t = in; in = out; out = t;
    if (stage == 2) {
      for (int e = tid; e < PB * NL; e += NT) {
        const int p = e / NL, l = e - p * NL;
        if (gbase[p] < 0) continue;
        const int lx = l % NP, ly = (l / NP) % NP, lz = l / (NP * NP);
        in[e] /= (P.c.lam[pvar[p][0]][lx] + P.c.lam[pvar[p][1]][ly] + P.c.lam[pvar[p][2]][lz]);
      }
      __syncthreads();
    }
  }
  // scatter: x += omega h u  (disjoint patches within one launch: plain read-modify-write), owned planes only
  for (int e = tid; e < PB * NL; e += NT) {
    const int p = e / NL, l = e - p * NL;
    const int64_t g0 = gbase[p];
    if (g0 < 0) continue;
    const int lx = l % NP, ly = (l / NP) % NP, lz = l / (NP * NP);
    const int64_t g = g0 + ((int64_t)lz * n + ly) * n + lx;
    const int64_t jz = pjz[p] + lz;
    if (jz < P.out_lo || jz >= P.out_hi) continue;
    if (P.atomic) atomicAdd(P.x + g, P.factor * in[e]);
    else P.x[g] = fma(P.factor, in[e], P.x[g]);
  }
}

template <typename T, int K>
struct Fdm3Layout {
  static constexpr int NP = 2 * K - 1, NL = NP * NP * NP, NL2 = NP * NP;
  static constexpr int LPL = cdiv(NL2, 32);        // patch lines per lane
  static constexpr int WB = NL + (NL % 2 == 0 ? 1 : 0);   // per-warp buffer (odd pitch)
  static constexpr int TOTAL = 8 * WB + NL;        // 8 warp buffers | interior 1/(lx+ly+lz) table
};

// out[i] = sum_l S_V[l][i] w[l] (TR: S^T w) or sum_l S_V[i][l] w[l]; coefficients are warp-uniform
// kernel-parameter operands
template <typename T, int K, int V, bool TR>
__device__ __forceinline__ void sdot(const Coef2<T, K>& c, const T (&w)[2 * K - 1], T (&o)[2 * K - 1]) {
  constexpr int NP = 2 * K - 1;
#pragma unroll
  for (int i = 0; i < NP; ++i) o[i] = 0;
#pragma unroll
  for (int l = 0; l < NP; ++l)
#pragma unroll
    for (int i = 0; i < NP; ++i) o[i] = fma(TR ? c.S[V][l * NP + i] : c.S[V][i * NP + l], w[l], o[i]);
}
// same with the interior S held in registers (Sr[l * NP + i] = S_1[l][i])
template <typename T, int K, bool TR, int M>
__device__ __forceinline__ void sdot_reg(const T (&Sr)[M], const T (&w)[2 * K - 1], T (&o)[2 * K - 1]) {
  constexpr int NP = 2 * K - 1;
  static_assert(M == NP * NP, "register S");
#pragma unroll
  for (int i = 0; i < NP; ++i) o[i] = 0;
#pragma unroll
  for (int l = 0; l < NP; ++l)
#pragma unroll
    for (int i = 0; i < NP; ++i) o[i] = fma(TR ? Sr[l * NP + i] : Sr[i * NP + l], w[l], o[i]);
}
template <typename T, int K, bool TR>
__device__ __forceinline__ void sdot_var(const Coef2<T, K>& c, int var, const T (&w)[2 * K - 1], T (&o)[2 * K - 1]) {
  if (var == 1) sdot<T, K, 1, TR>(c, w, o);
  else if (var == 0) sdot<T, K, 0, TR>(c, w, o);
  else sdot<T, K, 2, TR>(c, w, o);
}

// x += omega h A~_v^{-1} R_v r, one warp per patch: lanes own patch lines; the six
// contractions (S^T along x, y, z; scale by 1/(lam_x + lam_y + lam_z); S along z, y, x) run on
// register lines with warp-uniform coefficients, the line transposes between axes go through a
// per-warp shared-memory buffer (__syncwarp only).  The z stage does S_z^T, the scaling and S_z in
// registers.  r lines are read from global memory, the x update is a read-modify-write (disjoint
// patch list) or red.global.add (atomic AVS) restricted to the owned node planes.
template <typename T, int K>
__global__ void __launch_bounds__(256, (K == 3 && sizeof(T) == 8) ? 3 : 4) patch_fdm3d_kernel(const __grid_constant__ Fdm3P<T, K> P) {
  using LY = Fdm3Layout<T, K>;
  constexpr int NP = LY::NP, NL2 = LY::NL2, LPL = LY::LPL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* const tab = reinterpret_cast<T*>(smem_raw) + 8 * LY::WB;    // interior variant 1/(lx + ly + lz)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* const buf = reinterpret_cast<T*>(smem_raw) + warp * LY::WB;
  for (int e = tid; e < LY::NL; e += 256) {
    const int i = e % NP, j = (e / NP) % NP, m = e / NL2;
    tab[e] = T(1) / (P.c.lam[1][i] + P.c.lam[1][j] + P.c.lam[1][m]);
  }
  __syncthreads();
  const int64_t N = P.N, n = P.n;
  const int Nm1 = int(N - 1);
  // interior-variant S in registers for k <= 3 (every contraction of an interior patch then runs on
  // register operands only)
  constexpr bool REGS = K <= 3;
  T Sr[REGS ? NP * NP : 1];
#pragma unroll
  for (int e = 0; e < (REGS ? NP * NP : 1); ++e) Sr[e] = P.c.S[1][e];
  // uniform trip count over the CTA (the coefficient offsets below must be provably uniform)
  const int64_t stride = int64_t(gridDim.x) * 8, first = int64_t(blockIdx.x) * 8;
  const int iters = P.count > first ? int((P.count - first + stride - 1) / stride) : 0;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const int64_t q = first + warp + int64_t(it) * stride;
    if (q >= P.count) continue;
    // divisions by the (runtime) box extents through multiply-high, corrected by at most one
    auto udiv = [](unsigned a, unsigned d, unsigned m) {
      unsigned qq = __umulhi(a, m);
      if (a - qq * d >= d) ++qq;
      return qq;
    };
    int vx, vy, vz;
    if (P.list) {
      const unsigned pid = unsigned(P.list[q]);
      const unsigned t = udiv(pid, unsigned(Nm1), P.mag[0]), zz = udiv(pid, unsigned(Nm1 * Nm1), P.mag[1]);
      vx = 1 + int(pid - t * unsigned(Nm1)); vy = 1 + int(t - zz * unsigned(Nm1)); vz = 1 + int(zz);
    } else {
      const unsigned iq = unsigned(q), rest = udiv(iq, unsigned(P.vcnt[0]), P.mag[0]);
      const unsigned iz = udiv(rest, unsigned(P.vcnt[1]), P.mag[1]);
      vx = P.vlo[0] + P.vstr * int(iq - rest * unsigned(P.vcnt[0]));
      vy = P.vlo[1] + P.vstr * int(rest - iz * unsigned(P.vcnt[1]));
      vz = P.vlo[2] + P.vstr * int(iz);
    }
    const int varx = variant_of(vx, N), vary = variant_of(vy, N), varz = variant_of(vz, N);
    const int64_t g0 = ((int64_t(vz - 1) * K - P.row0) * n + int64_t(vy - 1) * K) * n + int64_t(vx - 1) * K;
    const int64_t jz0 = int64_t(vz - 1) * K + 1;
    const bool inner = (varx == 1 && vary == 1 && varz == 1);
    auto patch = [&](auto INC) {
      constexpr bool INNER = decltype(INC)::value;
    T w[NP], o[NP], xl[NP];
    // coefficients through an opaque zero offset per stage: loaded (LDCU) at the point of use as
    // uniform operands instead of being hoisted into registers (one R2UR per DFMA otherwise)
    // S_x^T on x lines (y, z) = (a, b), straight from global memory
    const Coef2<T, K>& c0 = coef_at(P.c, (it * 8 + 0) * P.zero);
#pragma unroll 1
    for (int s = 0; s < LPL; ++s) {
      const int ll = lane + 32 * s, la = ll % NP, lb = ll / NP;
      if (ll >= NL2) continue;
      const T* rp = P.r + g0 + (int64_t(lb) * n + la) * n;
#pragma unroll
      for (int l = 0; l < NP; ++l) w[l] = rp[l];
      if (!P.atomic && LPL == 1) {      // the x line of the final stage is this lane's line: load it now
        const T* xq = P.x + g0 + (int64_t(lb) * n + la) * n;
#pragma unroll
        for (int l = 0; l < NP; ++l) xl[l] = xq[l];
      }
      if constexpr (INNER && REGS) sdot_reg<T, K, true>(Sr, w, o); else sdot_var<T, K, true>(c0, varx, w, o);
#pragma unroll
      for (int i = 0; i < NP; ++i) buf[(lb * NP + la) * NP + i] = o[i];
    }
    __syncwarp();
    // S_y^T on y lines (i, z) = (a, b)
    const Coef2<T, K>& c1 = coef_at(P.c, (it * 8 + 1) * P.zero);
#pragma unroll 1
    for (int s = 0; s < LPL; ++s) {
      const int ll = lane + 32 * s, la = ll % NP, lb = ll / NP;
      if (ll >= NL2) continue;
#pragma unroll
      for (int l = 0; l < NP; ++l) w[l] = buf[(lb * NP + l) * NP + la];
      if constexpr (INNER && REGS) sdot_reg<T, K, true>(Sr, w, o); else sdot_var<T, K, true>(c1, vary, w, o);
#pragma unroll
      for (int j = 0; j < NP; ++j) buf[(lb * NP + j) * NP + la] = o[j];
    }
    __syncwarp();
    // S_z^T, 1 / (lam_x + lam_y + lam_z), S_z on z lines (i, j) = (a, b)
    const Coef2<T, K>& c2 = coef_at(P.c, (it * 8 + 2) * P.zero);
#pragma unroll 1
    for (int s = 0; s < LPL; ++s) {
      const int ll = lane + 32 * s, la = ll % NP, lb = ll / NP;
      if (ll >= NL2) continue;
#pragma unroll
      for (int l = 0; l < NP; ++l) w[l] = buf[(l * NP + lb) * NP + la];
      if constexpr (INNER && REGS) sdot_reg<T, K, true>(Sr, w, o); else sdot_var<T, K, true>(c2, varz, w, o);
      if (INNER) {
#pragma unroll
        for (int m = 0; m < NP; ++m) o[m] *= tab[(m * NP + lb) * NP + la];
      } else {
        const T lxy = P.c.lam[varx][la] + P.c.lam[vary][lb];
#pragma unroll
        for (int m = 0; m < NP; ++m) o[m] /= (lxy + P.c.lam[varz][m]);
      }
      if constexpr (INNER && REGS) sdot_reg<T, K, false>(Sr, o, w); else sdot_var<T, K, false>(c2, varz, o, w);
#pragma unroll
      for (int m = 0; m < NP; ++m) buf[(m * NP + lb) * NP + la] = w[m];
    }
    __syncwarp();
    // S_y on y lines (i, z)
    const Coef2<T, K>& c3 = coef_at(P.c, (it * 8 + 3) * P.zero);
#pragma unroll 1
    for (int s = 0; s < LPL; ++s) {
      const int ll = lane + 32 * s, la = ll % NP, lb = ll / NP;
      if (ll >= NL2) continue;
#pragma unroll
      for (int l = 0; l < NP; ++l) w[l] = buf[(lb * NP + l) * NP + la];
      if constexpr (INNER && REGS) sdot_reg<T, K, false>(Sr, w, o); else sdot_var<T, K, false>(c3, vary, w, o);
#pragma unroll
      for (int j = 0; j < NP; ++j) buf[(lb * NP + j) * NP + la] = o[j];
    }
    __syncwarp();
    // S_x on x lines (y, z), x += omega h u on the owned planes
    const Coef2<T, K>& c4 = coef_at(P.c, (it * 8 + 4) * P.zero);
#pragma unroll 1
    for (int s = 0; s < LPL; ++s) {
      const int ll = lane + 32 * s, la = ll % NP, lb = ll / NP;
      if (ll >= NL2) continue;
#pragma unroll
      for (int l = 0; l < NP; ++l) w[l] = buf[(lb * NP + la) * NP + l];
      if constexpr (INNER && REGS) sdot_reg<T, K, false>(Sr, w, o); else sdot_var<T, K, false>(c4, varx, w, o);
      const int64_t jz = jz0 + lb;
      if (jz < P.out_lo || jz >= P.out_hi) continue;
      T* xp = P.x + g0 + (int64_t(lb) * n + la) * n;
      if (P.atomic) {
#pragma unroll
        for (int i = 0; i < NP; ++i) atomicAdd(xp + i, P.factor * o[i]);
      } else if (LPL == 1) {
#pragma unroll
        for (int i = 0; i < NP; ++i) xp[i] = fma(P.factor, o[i], xl[i]);
      } else {
#pragma unroll
        for (int i = 0; i < NP; ++i) xp[i] = fma(P.factor, o[i], xp[i]);
      }
    }
    __syncwarp();
    };
    if (inner) patch(std::true_type{});
    else patch(std::false_type{});
  }
}

// ----------------------------------------------------------------------------- patch_fdm3d_run
// Atomic AVS patch solves x += omega h A~_v^{-1} R_v r for runs of PW consecutive
// patches along x (same vy, vz): NP = 2K - 1 lanes per patch, PW = 32 / NP patches per warp; lane (p, m)
// holds the node plane z = m of patch p (NP x NP values in registers).  S_x^T and S_y^T (and S_y, S_x on the
// way back) contract the lane's plane in registers; the z stage (S_z^T, 1 / (lam_x + lam_y + lam_z), S_z)
// runs after one transpose through a per-warp shared buffer, lane m then holding the z lines
// t = m, m + NP, ... of its patch.  Consecutive patches of a run overlap in K - 1 node columns: lane
// (p + 1, m) hands those columns to lane (p, m) (warp shuffles), which adds them before its red.global.add,
// so the run updates every node column once per plane ((2k-1)/k instead of ((2k-1)/k)^3 atomics per DoF
// along x).  Interior runs take coefficients as warp-uniform kernel-parameter operands; runs touching the
// boundary read per-lane variants from a shared copy.  Used for k <= 3 (2 CTAs per SM); at k = 4 the 49
// plane values per lane leave 1 CTA per SM and the kernel measured no faster than patch_fdm3d_kernel.
template <typename T, int K>
struct Fdm3RunLayout {
  static constexpr int NP = 2 * K - 1, NP2 = NP * NP, PW = 32 / NP, LANES = PW * NP;
  static constexpr int PL = NP2 | 1;               // odd plane pitch (conflict-free plane stores)
  static constexpr int WB = LANES * PL;            // per-warp transpose buffer
  static constexpr int TAB = NP2 * NP;             // interior 1 / (lx + ly + lz), index (m NP + j) NP + i
  static constexpr int TOTAL = 8 * WB + TAB + 3 * NP2 + 3 * NP;
};

// out = S^T w (TR) or S w (!TR) of one line, coefficients from coef(idx) with idx = l NP + i
template <int NP, bool TR, typename T, typename F>
__device__ __forceinline__ void line_mul(F coef, const T (&w)[NP], T (&o)[NP]) {
#pragma unroll
  for (int i = 0; i < NP; ++i) o[i] = 0;
#pragma unroll
  for (int l = 0; l < NP; ++l)
#pragma unroll
    for (int i = 0; i < NP; ++i) o[i] = fma(coef(TR ? l * NP + i : i * NP + l), w[l], o[i]);
}

template <typename T, int K>
__global__ void __launch_bounds__(256, K <= 3 ? 2 : 1) patch_fdm3d_run_kernel(const __grid_constant__ Fdm3P<T, K> P) {
  using LY = Fdm3RunLayout<T, K>;
  constexpr int NP = LY::NP, NP2 = LY::NP2, PW = LY::PW, PL = LY::PL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* const sm = reinterpret_cast<T*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* const buf = sm + warp * LY::WB;
  T* const tab = sm + 8 * LY::WB;
  T* const sS = tab + LY::TAB;                     // [3][NP2] S of the variants
  T* const sL = sS + 3 * NP2;                      // [3][NP]  lambda of the variants
  for (int e = tid; e < LY::TAB; e += 256) {
    const int i = e % NP, j = (e / NP) % NP, m = e / NP2;
    tab[e] = T(1) / (P.c.lam[1][i] + P.c.lam[1][j] + P.c.lam[1][m]);
  }
  for (int e = tid; e < 3 * NP2; e += 256) sS[e] = P.c.S[e / NP2][e % NP2];
  for (int e = tid; e < 3 * NP; e += 256) sL[e] = P.c.lam[e / NP][e % NP];
  __syncthreads();
  const int64_t N = P.N, n = P.n;
  const int nvx = P.vcnt[0], nvy = P.vcnt[1], nvz = P.vcnt[2];
  const int runs_x = (nvx + PW - 1) / PW;
  const int64_t nruns = int64_t(runs_x) * nvy * nvz;
  const int p = lane / NP, m = lane - (lane / NP) * NP;
  const int64_t wstride = int64_t(gridDim.x) * 8;
  int round = 0;
#pragma unroll 1
  for (int64_t run = int64_t(blockIdx.x) * 8 + warp; run < nruns; run += wstride, ++round) {
    const int64_t rz = run / (int64_t(runs_x) * nvy), rest = run - rz * (int64_t(runs_x) * nvy);
    const int ry = int(rest / runs_x), rx = int(rest - int64_t(ry) * runs_x);
    const int vx0 = P.vlo[0] + rx * PW, vy = P.vlo[1] + ry, vz = P.vlo[2] + int(rz);
    const int npat = min(PW, P.vlo[0] + nvx - vx0);
    const int vx = vx0 + p;
    const bool live = lane < LY::LANES && p < npat;
    const int varx = variant_of(vx, N), vary = variant_of(vy, N), varz = variant_of(vz, N);
    const bool inner = vary == 1 && varz == 1 && vx0 > 1 && vx0 + npat - 1 < N - 1;   // uniform over the warp
    const int64_t g0 = ((int64_t(vz - 1) * K + m - P.row0) * n + int64_t(vy - 1) * K) * n + int64_t(vx - 1) * K;
    T pl[NP][NP];                                  // [y row j][x column i] of plane m
#pragma unroll
    for (int j = 0; j < NP; ++j)
#pragma unroll
      for (int i = 0; i < NP; ++i) pl[j][i] = live ? P.r[g0 + int64_t(j) * n + i] : T(0);
    auto body = [&](auto INC) {
      constexpr bool IN = decltype(INC)::value;
      const Coef2<T, K>& c = coef_at(P.c, round * P.zero);
      auto Sx = [&](int idx) { return IN ? c.S[1][idx] : sS[varx * NP2 + idx]; };
      auto Sy = [&](int idx) { return IN ? c.S[1][idx] : sS[vary * NP2 + idx]; };
      auto Sz = [&](int idx) { return IN ? c.S[1][idx] : sS[varz * NP2 + idx]; };
      T w[NP], o[NP];
      // S_x^T along the rows, S_y^T along the columns (registers)
#pragma unroll
      for (int j = 0; j < NP; ++j) {
#pragma unroll
        for (int i = 0; i < NP; ++i) w[i] = pl[j][i];
        line_mul<NP, true>(Sx, w, o);
#pragma unroll
        for (int i = 0; i < NP; ++i) pl[j][i] = o[i];
      }
#pragma unroll
      for (int i = 0; i < NP; ++i) {
#pragma unroll
        for (int j = 0; j < NP; ++j) w[j] = pl[j][i];
        line_mul<NP, true>(Sy, w, o);
#pragma unroll
        for (int j = 0; j < NP; ++j) pl[j][i] = o[j];
      }
      // transpose: lane (p, m) now takes the z lines q = m + NP t of patch p (lanes >= LANES hold no plane)
      if (lane < LY::LANES) {
#pragma unroll
        for (int j = 0; j < NP; ++j)
#pragma unroll
          for (int i = 0; i < NP; ++i) buf[lane * PL + j * NP + i] = pl[j][i];
      }
      __syncwarp();
      if (lane < LY::LANES) {
#pragma unroll
        for (int t = 0; t < NP; ++t) {
          const int q = m + NP * t;                 // line (j, i) = (q / NP, q % NP)
#pragma unroll
          for (int mm = 0; mm < NP; ++mm) w[mm] = buf[(p * NP + mm) * PL + q];
          line_mul<NP, true>(Sz, w, o);
          if (IN) {
#pragma unroll
            for (int mm = 0; mm < NP; ++mm) o[mm] *= tab[mm * NP2 + q];
          } else {
            const int qj = q / NP, qi = q - qj * NP;
            const T lxy = sL[varx * NP + qi] + sL[vary * NP + qj];
#pragma unroll
            for (int mm = 0; mm < NP; ++mm) o[mm] /= (lxy + sL[varz * NP + mm]);
          }
          line_mul<NP, false>(Sz, o, w);
#pragma unroll
          for (int mm = 0; mm < NP; ++mm) buf[(p * NP + mm) * PL + q] = w[mm];
        }
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < NP; ++j)
#pragma unroll
        for (int i = 0; i < NP; ++i) pl[j][i] = lane < LY::LANES ? buf[lane * PL + j * NP + i] : T(0);
      __syncwarp();                                 // the buffer is rewritten by the next run
      // S_y along the columns, S_x along the rows
#pragma unroll
      for (int i = 0; i < NP; ++i) {
#pragma unroll
        for (int j = 0; j < NP; ++j) w[j] = pl[j][i];
        line_mul<NP, false>(Sy, w, o);
#pragma unroll
        for (int j = 0; j < NP; ++j) pl[j][i] = o[j];
      }
#pragma unroll
      for (int j = 0; j < NP; ++j) {
#pragma unroll
        for (int i = 0; i < NP; ++i) w[i] = pl[j][i];
        line_mul<NP, false>(Sx, w, o);
#pragma unroll
        for (int i = 0; i < NP; ++i) pl[j][i] = o[i];
      }
    };
    if (inner) body(std::true_type{});
    else body(std::false_type{});
    // run merge: columns [0, K-1) of patch p + 1 are columns [K, 2K-1) of patch p
#pragma unroll
    for (int cc = 0; cc < K - 1; ++cc)
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const T v = __shfl_down_sync(0xffffffffu, pl[j][cc], NP);
        if (p + 1 < npat) pl[j][K + cc] += v;
      }
    const int64_t jz = int64_t(vz - 1) * K + 1 + m;
    if (live && jz >= P.out_lo && jz < P.out_hi) {
      const int c0 = p > 0 ? K - 1 : 0;
#pragma unroll
      for (int j = 0; j < NP; ++j)
#pragma unroll
        for (int i = 0; i < NP; ++i)
          if (i >= c0) atomicAdd(P.x + g0 + int64_t(j) * n + i, P.factor * pl[j][i]);
    }
  }
}

// ----------------------------------------------------------------------------- patch_fdm3d_zrun
// Deterministic additive FDM update without atomics: one warp per patch column (vx, vy) of one x-y
// parity class (columns of a class are disjoint in x and y), walking the patches of the column along
// z.  Consecutive patches of a column overlap in k - 1 node planes: each patch's correction is added
// to a per-warp ring of node planes in shared memory, and the k planes no later patch touches are
// flushed to x with a plain read-modify-write (owned planes only).  Every DoF is written once per
// class launch (4 launches per AVS step instead of 8 parity classes).
template <typename T, int K>
__global__ void __launch_bounds__(256, 3) patch_fdm3d_zrun_kernel(const __grid_constant__ Fdm3P<T, K> P) {
  using LY = Fdm3Layout<T, K>;
  constexpr int NP = LY::NP, NL2 = LY::NL2, LPL = LY::LPL;
  constexpr int RING = 2 * K;                         // node planes held per warp (>= NP)
  constexpr int WB = LY::WB + RING * NL2;             // FDM buffer | plane ring [RING][NP][NP]
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* const tab = reinterpret_cast<T*>(smem_raw) + 8 * WB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* const buf = reinterpret_cast<T*>(smem_raw) + warp * WB;
  T* const ring = buf + LY::WB;
  for (int e = tid; e < LY::NL; e += 256) {
    const int i = e % NP, j = (e / NP) % NP, m = e / NL2;
    tab[e] = T(1) / (P.c.lam[1][i] + P.c.lam[1][j] + P.c.lam[1][m]);
  }
  for (int e = lane; e < RING * NL2; e += 32) ring[e] = T(0);
  __syncthreads();
  const int64_t N = P.N, n = P.n;
  constexpr bool REGS = K <= 3;
  T Sr[REGS ? NP * NP : 1];
#pragma unroll
  for (int e = 0; e < (REGS ? NP * NP : 1); ++e) Sr[e] = P.c.S[1][e];
  // work item = (column of the class, z chunk of this launch's parity); chunks of one launch are
  // separated by a chunk of the other parity, so their planes never overlap
  // chunks are aligned to absolute vertex planes (chunk k: vz in [1 + k zc, 1 + (k+1) zc)), so a slab
  // run splits its columns exactly where the full-domain run does (bitwise-equal owned planes)
  const int ncol = P.vcnt[0] * P.vcnt[1];
  const int zlo = P.vlo[2], zhi = P.vlo[2] + P.vcnt[2] - 1;
  const int k0 = (zlo - 1) / P.zc, k1 = (zhi - 1) / P.zc;
  const int kf = k0 + ((k0 & 1) != P.zpar ? 1 : 0);  // first chunk of parity zpar
  const int nck = kf > k1 ? 0 : (k1 - kf) / 2 + 1;
  const int nitem = ncol * nck;
  const int stride = int(gridDim.x) * 8, first = int(blockIdx.x) * 8;
  const int iters = nitem > first ? (nitem - first + stride - 1) / stride : 0;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const int item = first + warp + it * stride;
    if (item >= nitem) continue;
    const int col = item % ncol, ck = kf + 2 * (item / ncol);
    const int vz_a = max(1 + ck * P.zc, zlo), vz_b = min(1 + (ck + 1) * P.zc, zhi + 1);
    const int vx = P.vlo[0] + P.vstr * (col % P.vcnt[0]), vy = P.vlo[1] + P.vstr * (col / P.vcnt[0]);
    const int varx = variant_of(vx, N), vary = variant_of(vy, N);
    const int64_t gxy = int64_t(vy - 1) * K * n + int64_t(vx - 1) * K;   // in-plane offset of the patch corner
    auto flush = [&](int64_t jz, int slot) {          // node plane jz from ring slot: x += omega h acc
      const bool own = jz >= P.out_lo && jz < P.out_hi;
      T* xs = P.x + (jz - 1 - P.row0) * n * n + gxy;
#pragma unroll 1
      for (int e = lane; e < NL2; e += 32) {
        const int xi = e % NP, yi = e / NP;
        T* xp = xs + int64_t(yi) * n + xi;
        T& a = ring[slot * NL2 + e];
        if (own) *xp = fma(P.factor, a, *xp);
        a = T(0);
      }
    };
#pragma unroll 1
    for (int vz = vz_a; vz < vz_b; ++vz) {
      const int varz = variant_of(vz, N);
      const int64_t g0 = (int64_t(vz - 1) * K - P.row0) * n * n + gxy;
      const int64_t jz0 = int64_t(vz - 1) * K + 1;
      T w[NP], o[NP];
      const bool inner = (varx == 1 && vary == 1 && varz == 1);
      auto patch = [&](auto INC) {
        constexpr bool INNER = decltype(INC)::value;
        const Coef2<T, K>& c0 = coef_at(P.c, (it * 8 + 0) * P.zero);
#pragma unroll 1
        for (int s = 0; s < LPL; ++s) {
          const int ll = lane + 32 * s, la = ll % NP, lb = ll / NP;
          if (ll >= NL2) continue;
          const T* rp = P.r + g0 + (int64_t(lb) * n + la) * n;
#pragma unroll
          for (int l = 0; l < NP; ++l) w[l] = rp[l];
          if constexpr (INNER && REGS) sdot_reg<T, K, true>(Sr, w, o); else sdot_var<T, K, true>(c0, varx, w, o);
#pragma unroll
          for (int i = 0; i < NP; ++i) buf[(lb * NP + la) * NP + i] = o[i];
        }
        __syncwarp();
        const Coef2<T, K>& c1 = coef_at(P.c, (it * 8 + 1) * P.zero);
#pragma unroll 1
        for (int s = 0; s < LPL; ++s) {
          const int ll = lane + 32 * s, la = ll % NP, lb = ll / NP;
          if (ll >= NL2) continue;
#pragma unroll
          for (int l = 0; l < NP; ++l) w[l] = buf[(lb * NP + l) * NP + la];
          if constexpr (INNER && REGS) sdot_reg<T, K, true>(Sr, w, o); else sdot_var<T, K, true>(c1, vary, w, o);
#pragma unroll
          for (int j = 0; j < NP; ++j) buf[(lb * NP + j) * NP + la] = o[j];
        }
        __syncwarp();
        const Coef2<T, K>& c2 = coef_at(P.c, (it * 8 + 2) * P.zero);
#pragma unroll 1
        for (int s = 0; s < LPL; ++s) {
          const int ll = lane + 32 * s, la = ll % NP, lb = ll / NP;
          if (ll >= NL2) continue;
#pragma unroll
          for (int l = 0; l < NP; ++l) w[l] = buf[(l * NP + lb) * NP + la];
          if constexpr (INNER && REGS) sdot_reg<T, K, true>(Sr, w, o); else sdot_var<T, K, true>(c2, varz, w, o);
          if (INNER) {
#pragma unroll
            for (int m = 0; m < NP; ++m) o[m] *= tab[(m * NP + lb) * NP + la];
          } else {
            const T lxy = P.c.lam[varx][la] + P.c.lam[vary][lb];
#pragma unroll
            for (int m = 0; m < NP; ++m) o[m] /= (lxy + P.c.lam[varz][m]);
          }
          if constexpr (INNER && REGS) sdot_reg<T, K, false>(Sr, o, w); else sdot_var<T, K, false>(c2, varz, o, w);
#pragma unroll
          for (int m = 0; m < NP; ++m) buf[(m * NP + lb) * NP + la] = w[m];
        }
        __syncwarp();
        const Coef2<T, K>& c3 = coef_at(P.c, (it * 8 + 3) * P.zero);
#pragma unroll 1
        for (int s = 0; s < LPL; ++s) {
          const int ll = lane + 32 * s, la = ll % NP, lb = ll / NP;
          if (ll >= NL2) continue;
#pragma unroll
          for (int l = 0; l < NP; ++l) w[l] = buf[(lb * NP + l) * NP + la];
          if constexpr (INNER && REGS) sdot_reg<T, K, false>(Sr, w, o); else sdot_var<T, K, false>(c3, vary, w, o);
#pragma unroll
          for (int j = 0; j < NP; ++j) buf[(lb * NP + j) * NP + la] = o[j];
        }
        __syncwarp();
        // S_x on x lines (y, z), accumulated into the plane ring
        const Coef2<T, K>& c4 = coef_at(P.c, (it * 8 + 4) * P.zero);
#pragma unroll 1
        for (int s = 0; s < LPL; ++s) {
          const int ll = lane + 32 * s, la = ll % NP, lb = ll / NP;
          if (ll >= NL2) continue;
#pragma unroll
          for (int l = 0; l < NP; ++l) w[l] = buf[(lb * NP + la) * NP + l];
          if constexpr (INNER && REGS) sdot_reg<T, K, false>(Sr, w, o); else sdot_var<T, K, false>(c4, varx, w, o);
          T* rg = ring + int((jz0 + lb) % RING) * NL2 + la * NP;
#pragma unroll
          for (int i = 0; i < NP; ++i) rg[i] += o[i];
        }
        __syncwarp();
      };
      if (inner) patch(std::true_type{});
      else patch(std::false_type{});
      // planes jz0 .. jz0 + K - 1 are final (the next patch of the column starts at jz0 + K)
#pragma unroll 1
      for (int pz = 0; pz < K; ++pz) flush(jz0 + pz, int((jz0 + pz) % RING));
      __syncwarp();
    }
    // the chunk's last patch's remaining NP - K planes (the next chunk, in the other launch, adds to
    // them afterwards)
    const int64_t jzl = int64_t(vz_b - 2) * K + 1 + K;
#pragma unroll 1
    for (int pz = 0; pz < NP - K; ++pz) flush(jzl + pz, int((jzl + pz) % RING));
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------- mvs3d
// One colour of the coloured multiplicative smoother in 3D, fused per patch, one
// warp per patch (k <= 3): the residual r_v = b - A x on the np^3 patch nodes is evaluated from x on
// the patch footprint (patch cells plus their face neighbours; same-colour patches never
// write it, so the in-place update is race-free) by sum factorisation of the six Kronecker terms of
// Eq. c0iptensorvp3D, per axis with F = [(v-2)k, (v+2)k] (4k+1 nodes), W =
// [(v-1)k, (v+1)k] (2k+1) and the patch nodes P ((v-1)k+1 .. (v+1)k-1, np):
//   x stage (lanes <-> rows (y, z) of the cross F x W u W x F):  Xm = M^_x x on every cross row,
//            Xb = B^_x x and Xl = L^_x x on the W x W rows (x in F, resp. W)
//   y stage (lanes <-> lines (x, z)):  G1 = M^_y Xb + B^_y Xm + 2 L^_y Xl  (z in W)
//                                      G2 = M^_y Xm                       (z in F)
//                                      G3 = 2 M^_y Xl + 2 L^_y Xm          (z in W)
//   z stage (lanes <-> lines (x, y)):  A x = M^_z G1 + B^_z G2 + L^_z G3 on P,  r = b - h^-1 A x
// followed by the FDM solve on the same lines (S_z^T in registers, S_y^T, S_x^T / scale / S_x, S_y
// through a per-warp buffer, S_z) and x += omega h u on the patch nodes.
// acc[j] += c * w[j] for RB lines sharing the coefficient c; FP32 pairs go through the packed
// FFMA2 (f32x2 FMA with a scalar operand, sm_100a): two FMAs per issue slot
template <typename T, int RB>
__device__ __forceinline__ void fma_lines(T c, const T (&w)[RB], T (&acc)[RB]) {
  if constexpr (std::is_same<T, float>::value) {
#pragma unroll
    for (int j = 0; j + 1 < RB; j += 2) {
      const float2 r = __ffma2_rn(make_float2(c, c), make_float2(w[j], w[j + 1]), make_float2(acc[j], acc[j + 1]));
      acc[j] = r.x;
      acc[j + 1] = r.y;
    }
    if constexpr (RB % 2 == 1) acc[RB - 1] = fmaf(c, w[RB - 1], acc[RB - 1]);
  } else {
#pragma unroll
    for (int j = 0; j < RB; ++j) acc[j] = fma(c, w[j], acc[j]);
  }
}

template <typename T, int K>
struct Mvs3Layout {
  static constexpr int NP = 2 * K - 1, W = 2 * K + 1, F = 4 * K + 1;
  static constexpr int XM = F * F * NP;           // Xm[z][y][p] (full F x F index, cross rows filled)
  static constexpr int XB = W * W * NP;           // Xb[z - K][y - K][p], Xl likewise
  static constexpr int G1 = W * NP * NP, G2 = F * NP * NP, G3 = W * NP * NP;   // G[z][y'][x']
  static constexpr int WARP = XM + 2 * XB + G1 + G2 + G3;                   // per warp (FDM buffer aliases Xm)
  static constexpr int NW = 4;                    // warps per CTA
  // coefficient tables per axis variant v: Bt[v][p][f] (P x F), Mt[v][p][w], Lt[v][p][w] (P x W),
  // S[v][l][i], lam[v][i]
  static constexpr int TAB = 3 * (NP * F + 2 * NP * W + NP * NP + NP);
  static constexpr int TOTAL = NW * WARP + TAB;
};

// kernel parameters: MvsP plus the interior-variant (v = 1) rows of the per-variant tables, so that interior
// patches (every axis variant 1, warp-uniform: one warp per patch) read their coefficients as uniform
// kernel-parameter operands instead of one shared-memory load per FMA
template <typename T, int K>
struct Mvs3P {
  MvsP<T, K> m;
  T tB[2 * K - 1][4 * K + 1];
  T tM[2 * K - 1][2 * K + 1];
  T tL[2 * K - 1][2 * K + 1];
};

template <typename T, int K>
__global__ void __launch_bounds__(128) mvs3d_kernel(const __grid_constant__ Mvs3P<T, K> PP) {
  const MvsP<T, K>& P = PP.m;
  using LY = Mvs3Layout<T, K>;
  constexpr int NP = LY::NP, W = LY::W, F = LY::F, NW = LY::NW;
  constexpr int TB = NP * F, TM = NP * W, TS = NP * NP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* const tabs = reinterpret_cast<T*>(smem_raw) + NW * LY::WARP;
  T* const Bt = tabs;                         // [3][NP][F]
  T* const Mt = Bt + 3 * TB;                  // [3][NP][W]
  T* const Lt = Mt + 3 * TM;                  // [3][NP][W]
  T* const St = Lt + 3 * TM;                  // [3][NP][NP]  S[l][i]
  T* const Lam = St + 3 * TS;                 // [3][NP]
  const int64_t N = P.N, n = P.n, KN = K * N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // tables of the three axis variants (representative vertices 1, N/2, N-1; see mvs2d_mma)
  for (int e = tid; e < 3 * (TB + 2 * TM); e += blockDim.x) {
    int v, p, c, which;
    if (e < 3 * TB) { v = e / TB; p = (e % TB) / F; c = e % F; which = 0; }
    else if (e < 3 * (TB + TM)) { const int r = e - 3 * TB; v = r / TM; p = (r % TM) / W; c = r % W; which = 1; }
    else { const int r = e - 3 * (TB + TM); v = r / TM; p = (r % TM) / W; c = r % W; which = 2; }
    const int64_t vr = v == 0 ? 1 : (v == 1 ? N / 2 : N - 1);
    const int64_t jo = (vr - 1) * K + 1 + p;
    const int64_t ji = which == 0 ? (vr - 2) * K + c : (vr - 1) * K + c;
    // op1d of mma2d.cu, inlined: full-band 1D coefficient
    T val = 0;
    const int64_t off = ji - jo;
    if (ji >= 1 && ji <= KN - 1) {
      const int sp = special_row<K>(jo, N);
      if (which == 0) {
        if (off >= -2 * K && off <= 2 * K) val = sp >= 0 ? P.c.BS[sp][off + 2 * K] : P.c.BI[jo % K][off + 2 * K];
      } else if (sp >= 0) {
        if (off >= -2 * K && off <= 2 * K) val = which == 1 ? P.c.MS[sp][off + 2 * K] : P.c.LS[sp][off + 2 * K];
      } else if (off >= -K && off <= K) {
        val = which == 1 ? P.c.MI[jo % K][off + K] : P.c.LI[jo % K][off + K];
      }
    }
    tabs[e] = val;
  }
  for (int e = tid; e < 3 * TS; e += blockDim.x) St[e] = P.c.S[e / TS][e % TS];
  for (int e = tid; e < 3 * NP; e += blockDim.x) Lam[e] = P.c.lam[e / NP][e % NP];
  __syncthreads();

  T* const xm = reinterpret_cast<T*>(smem_raw) + warp * LY::WARP;
  T* const xb = xm + LY::XM;
  T* const xl = xb + LY::XB;
  T* const g1 = xl + LY::XB;
  T* const g2 = g1 + LY::G1;
  T* const g3 = g2 + LY::G2;
  T* const buf = xm;                          // FDM transposes (np^3), Xm is dead by then
  const int Nm1 = int(N - 1);
  const T* __restrict__ X = P.x;
  // uniform trip count over the CTA (the coefficient offsets of the interior path must be provably uniform)
  const int64_t pstride = int64_t(gridDim.x) * NW, pfirst = int64_t(blockIdx.x) * NW;
  const int iters = P.count > pfirst ? int((P.count - pfirst + pstride - 1) / pstride) : 0;

#pragma unroll 1
  for (int round = 0; round < iters; ++round) {
    const int64_t pi = pfirst + warp + int64_t(round) * pstride;
    if (pi >= P.count) continue;
    const int pid = P.list[pi];
    const int vx = 1 + pid % Nm1, vy = 1 + (pid / Nm1) % Nm1, vz = 1 + pid / (Nm1 * Nm1);
    const int varx = variant_of(vx, N), vary = variant_of(vy, N), varz = variant_of(vz, N);
    const int64_t jx0 = int64_t(vx - 2) * K, jy0 = int64_t(vy - 2) * K, jz0 = int64_t(vz - 2) * K;   // F origin
    const bool inner = jx0 >= 1 && jx0 + F - 1 <= KN - 1 && jy0 >= 1 && jy0 + F - 1 <= KN - 1 && jz0 >= 1 &&
                       jz0 + F - 1 <= KN - 1;
    auto ldx = [&](int z, int y, int xx) -> T {            // x at F-local (xx, y, z)
      const int64_t gz = jz0 + z, gy = jy0 + y, gx = jx0 + xx;
      if (!inner && (gx < 1 || gx > KN - 1 || gy < 1 || gy > KN - 1 || gz < 1 || gz > KN - 1)) return T(0);
      return __ldg(X + ((gz - 1) * n + (gy - 1)) * n + (gx - 1));
    };
    auto body = [&](auto INC) {
    constexpr bool IN = decltype(INC)::value;
    // coefficient tables: interior patches from the kernel parameters (opaque zero offset per patch: loaded at
    // the point of use as uniform operands), the others from the shared per-variant copies
    const Mvs3P<T, K>& Q = *reinterpret_cast<const Mvs3P<T, K>*>(reinterpret_cast<const char*>(&PP) + round * P.zero);
    const T* bx = Bt + varx * TB; const T* mx = Mt + varx * TM; const T* lx = Lt + varx * TM;
    const T* by = Bt + vary * TB; const T* my = Mt + vary * TM; const T* ly = Lt + vary * TM;
    const T* bz = Bt + varz * TB; const T* mz = Mt + varz * TM; const T* lz = Lt + varz * TM;
    const T* sx = St + varx * TS; const T* sy = St + vary * TS; const T* sz = St + varz * TS;
    auto bx_ = [&](int i) { return IN ? (&Q.tB[0][0])[i] : bx[i]; };
    constexpr bool INYZ = IN && K == 2;            // k = 3: y / z stages keep the shared tables (registers)
    auto by_ = [&](int i) { return INYZ ? (&Q.tB[0][0])[i] : by[i]; };
    auto bz_ = [&](int i) { return INYZ ? (&Q.tB[0][0])[i] : bz[i]; };
    auto mx_ = [&](int i) { return IN ? (&Q.tM[0][0])[i] : mx[i]; };
    auto my_ = [&](int i) { return INYZ ? (&Q.tM[0][0])[i] : my[i]; };
    auto mz_ = [&](int i) { return INYZ ? (&Q.tM[0][0])[i] : mz[i]; };
    auto lx_ = [&](int i) { return IN ? (&Q.tL[0][0])[i] : lx[i]; };
    auto ly_ = [&](int i) { return INYZ ? (&Q.tL[0][0])[i] : ly[i]; };
    auto lz_ = [&](int i) { return INYZ ? (&Q.tL[0][0])[i] : lz[i]; };
    auto sx_ = [&](int i) { return IN ? Q.m.c.S[1][i] : sx[i]; };
    auto sy_ = [&](int i) { return IN ? Q.m.c.S[1][i] : sy[i]; };
    auto sz_ = [&](int i) { return IN ? Q.m.c.S[1][i] : sz[i]; };
    // ---- x stage: W x W rows (Xm, Xb, Xl); RB1 rows per lane share every coefficient load
    {
      constexpr int RB1 = cdiv(W * W, 32), L1 = cdiv(W * W, RB1);
      if (lane < L1) {
        T w[F][RB1];
        int ry[RB1], rzz[RB1];
        bool ok[RB1];
#pragma unroll
        for (int j = 0; j < RB1; ++j) {
          const int r = lane + j * L1;
          ok[j] = r < W * W;
          const int rc = ok[j] ? r : 0;
          ry[j] = K + rc % W;
          rzz[j] = K + rc / W;
#pragma unroll
          for (int f = 0; f < F; ++f) w[f][j] = ldx(rzz[j], ry[j], f);
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          T ab[RB1], am[RB1], al[RB1];
#pragma unroll
          for (int j = 0; j < RB1; ++j) ab[j] = am[j] = al[j] = 0;
#pragma unroll
          for (int f = 0; f < F; ++f) fma_lines<T, RB1>(bx_(p * F + f), w[f], ab);
#pragma unroll
          for (int c = 0; c < W; ++c) {
            fma_lines<T, RB1>(mx_(p * W + c), w[K + c], am);
            fma_lines<T, RB1>(lx_(p * W + c), w[K + c], al);
          }
#pragma unroll
          for (int j = 0; j < RB1; ++j) {
            if (!ok[j]) continue;
            const int y = ry[j], z = rzz[j];
            xm[(z * F + y) * NP + p] = am[j];
            xb[((z - K) * W + (y - K)) * NP + p] = ab[j];
            xl[((z - K) * W + (y - K)) * NP + p] = al[j];
          }
        }
      }
    }
    // ---- x stage: the other cross rows (y in F \ W, z in W) and (y in W, z in F \ W): Xm only
    {
      constexpr int NR2 = 4 * K * W, RB2 = cdiv(NR2, 32), L2 = cdiv(NR2, RB2);
      if (lane < L2) {
        T w[W][RB2];
        int ry[RB2], rzz[RB2];
        bool ok[RB2];
#pragma unroll
        for (int j = 0; j < RB2; ++j) {
          const int r0 = lane + j * L2;
          ok[j] = r0 < NR2;
          const int r = ok[j] ? r0 : 0;
          const int h = r / (2 * K * W), rr = r % (2 * K * W), o = rr % (2 * K), t = rr / (2 * K);
          const int fo = o < K ? o : o + W;             // F \ W index
          if (h == 0) { ry[j] = fo; rzz[j] = K + t; } else { ry[j] = K + t; rzz[j] = fo; }
#pragma unroll
          for (int c = 0; c < W; ++c) w[c][j] = ldx(rzz[j], ry[j], K + c);
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          T am[RB2];
#pragma unroll
          for (int j = 0; j < RB2; ++j) am[j] = 0;
#pragma unroll
          for (int c = 0; c < W; ++c) fma_lines<T, RB2>(mx_(p * W + c), w[c], am);
#pragma unroll
          for (int j = 0; j < RB2; ++j)
            if (ok[j]) xm[(rzz[j] * F + ry[j]) * NP + p] = am[j];
        }
      }
    }
    __syncwarp();
    // ---- y stage
#pragma unroll 1
    for (int l = lane; l < (2 * W + F) * NP; l += 32) {
      const int xq = l % NP, zl = l / NP;
      if (zl < W) {                                   // G1 on z = K + zl
        const int z = K + zl;
        T wb[W], wl[W], wm[F];
#pragma unroll
        for (int c = 0; c < W; ++c) {
          wb[c] = xb[(zl * W + c) * NP + xq];
          wl[c] = xl[(zl * W + c) * NP + xq];
        }
#pragma unroll
        for (int f = 0; f < F; ++f) wm[f] = xm[(z * F + f) * NP + xq];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          T a = 0;
#pragma unroll
          for (int c = 0; c < W; ++c) a = fma(my_(p * W + c), wb[c], fma(T(2) * ly_(p * W + c), wl[c], a));
#pragma unroll
          for (int f = 0; f < F; ++f) a = fma(by_(p * F + f), wm[f], a);
          g1[(zl * NP + p) * NP + xq] = a;
        }
      } else if (zl < 2 * W) {                        // G3 on z = K + (zl - W)
        const int z3 = zl - W, z = K + z3;
        T wl[W], wm[W];
#pragma unroll
        for (int c = 0; c < W; ++c) {
          wl[c] = xl[(z3 * W + c) * NP + xq];
          wm[c] = xm[(z * F + K + c) * NP + xq];
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          T a = 0;
#pragma unroll
          for (int c = 0; c < W; ++c) a = fma(my_(p * W + c), wl[c], fma(ly_(p * W + c), wm[c], a));
          g3[(z3 * NP + p) * NP + xq] = T(2) * a;
        }
      } else {                                        // G2 on z = zl - 2W in F
        const int z = zl - 2 * W;
        T wm[W];
#pragma unroll
        for (int c = 0; c < W; ++c) wm[c] = xm[(z * F + K + c) * NP + xq];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          T a = 0;
#pragma unroll
          for (int c = 0; c < W; ++c) a = fma(my_(p * W + c), wm[c], a);
          g2[(z * NP + p) * NP + xq] = a;
        }
      }
    }
    __syncwarp();
    // ---- z stage + residual + S_z^T (lanes <-> (x', y') lines)
    const bool act = lane < NP * NP;
    const int xq = lane % NP, yq = lane / NP;
    const int64_t gx = jx0 + K + 1 + xq, gy = jy0 + K + 1 + yq;     // patch node (global node index)
    T rz[NP];
    if (act) {
      T w1[W], w2[F], w3[W];
#pragma unroll
      for (int c = 0; c < W; ++c) {
        w1[c] = g1[(c * NP + yq) * NP + xq];
        w3[c] = g3[(c * NP + yq) * NP + xq];
      }
#pragma unroll
      for (int f = 0; f < F; ++f) w2[f] = g2[(f * NP + yq) * NP + xq];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        T a = 0;
#pragma unroll
        for (int c = 0; c < W; ++c) a = fma(mz_(p * W + c), w1[c], fma(lz_(p * W + c), w3[c], a));
#pragma unroll
        for (int f = 0; f < F; ++f) a = fma(bz_(p * F + f), w2[f], a);
        const int64_t gz = jz0 + K + 1 + p;
        rz[p] = fma(-P.scale, a, P.b[((gz - 1) * n + (gy - 1)) * n + (gx - 1)]);
      }
      // S_z^T on the z line
      T o[NP];
#pragma unroll
      for (int i = 0; i < NP; ++i) o[i] = 0;
#pragma unroll
      for (int l = 0; l < NP; ++l)
#pragma unroll
        for (int i = 0; i < NP; ++i) o[i] = fma(sz_(l * NP + i), rz[l], o[i]);
#pragma unroll
      for (int i = 0; i < NP; ++i) buf[(i * NP + yq) * NP + xq] = o[i];    // buf[z'][y][x]
    }
    __syncwarp();
    // S_y^T on y lines (x, z')
    if (act) {
      const int xa = lane % NP, zb = lane / NP;
      T w[NP], o[NP];
#pragma unroll
      for (int l = 0; l < NP; ++l) w[l] = buf[(zb * NP + l) * NP + xa];
#pragma unroll
      for (int i = 0; i < NP; ++i) o[i] = 0;
#pragma unroll
      for (int l = 0; l < NP; ++l)
#pragma unroll
        for (int i = 0; i < NP; ++i) o[i] = fma(sy_(l * NP + i), w[l], o[i]);
#pragma unroll
      for (int i = 0; i < NP; ++i) buf[(zb * NP + i) * NP + xa] = o[i];
    }
    __syncwarp();
    // S_x^T, scale by omega h / (lam_x + lam_y + lam_z), S_x on x lines (y', z')
    if (act) {
      const int ya = lane % NP, zb = lane / NP;
      T w[NP], o[NP];
#pragma unroll
      for (int l = 0; l < NP; ++l) w[l] = buf[(zb * NP + ya) * NP + l];
#pragma unroll
      for (int i = 0; i < NP; ++i) o[i] = 0;
#pragma unroll
      for (int l = 0; l < NP; ++l)
#pragma unroll
        for (int i = 0; i < NP; ++i) o[i] = fma(sx_(l * NP + i), w[l], o[i]);
      const T lyz = Lam[vary * NP + ya] + Lam[varz * NP + zb];
#pragma unroll
      for (int i = 0; i < NP; ++i) o[i] = P.factor * o[i] / (Lam[varx * NP + i] + lyz);
#pragma unroll
      for (int l = 0; l < NP; ++l) w[l] = 0;
#pragma unroll
      for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int l = 0; l < NP; ++l) w[l] = fma(sx_(l * NP + i), o[i], w[l]);
#pragma unroll
      for (int l = 0; l < NP; ++l) buf[(zb * NP + ya) * NP + l] = w[l];
    }
    __syncwarp();
    // S_y on y lines (x, z')
    if (act) {
      const int xa = lane % NP, zb = lane / NP;
      T w[NP], o[NP];
#pragma unroll
      for (int i = 0; i < NP; ++i) w[i] = buf[(zb * NP + i) * NP + xa];
#pragma unroll
      for (int l = 0; l < NP; ++l) o[l] = 0;
#pragma unroll
      for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int l = 0; l < NP; ++l) o[l] = fma(sy_(l * NP + i), w[i], o[l]);
#pragma unroll
      for (int l = 0; l < NP; ++l) buf[(zb * NP + l) * NP + xa] = o[l];
    }
    __syncwarp();
    // S_z on z lines (x, y), x += u on the patch nodes (disjoint within the colour)
    if (act) {
      T w[NP], o[NP];
#pragma unroll
      for (int i = 0; i < NP; ++i) w[i] = buf[(i * NP + yq) * NP + xq];
#pragma unroll
      for (int l = 0; l < NP; ++l) o[l] = 0;
#pragma unroll
      for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int l = 0; l < NP; ++l) o[l] = fma(sz_(l * NP + i), w[i], o[l]);
#pragma unroll
      for (int l = 0; l < NP; ++l) {
        const int64_t gz = jz0 + K + 1 + l;
        T* xp = P.x + ((gz - 1) * n + (gy - 1)) * n + (gx - 1);
        *xp += o[l];
      }
    }
    __syncwarp();
    };
    // measured MVS step: k = 2 2.53 -> 3.17 GDoF/s with the parameter-space coefficients in every stage; k = 3
    // 2.37 -> 2.22 with them in every stage (158 registers), 2.52 with them in the x-stage and the S contractions
    // only (INYZ)
    if (varx == 1 && vary == 1 && varz == 1) body(std::true_type{});
    else body(std::false_type{});
  }
}

template <typename T, int K>
static void launch_mvs3(const FusedLevel& F, const int32_t* list, int64_t count, T omega, const T* b, T* x,
                        cudaStream_t st) {
  using LY = Mvs3Layout<T, K>;
  const size_t smem = sizeof(T) * size_t(LY::TOTAL);
  static int grid_cache = -1;
  if (grid_cache < 0) {
    cudaFuncSetAttribute(mvs3d_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(mvs3d_kernel<T, K>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mvs3d_kernel<T, K>, 128, smem);
    grid_cache = sms * std::max(per, 1);
  }
  Mvs3P<T, K> pp;
  MvsP<T, K>& p = pp.m;
  std::memcpy(&p.c, coef_of<T>(F).data(), sizeof(p.c));
  p.x = x; p.b = b; p.list = list; p.count = count; p.N = F.N; p.n = F.n;
  p.scale = T(1.0 / F.h);                  // 3D: A = h^-1 A^
  p.factor = T(double(omega) * F.h);       //     A~^-1 = h A^~^-1
  p.zero = 0;
  {   // interior-variant table rows (the kernel's Bt/Mt/Lt[1], representative vertex N/2)
    constexpr int NP = 2 * K - 1;
    const int64_t vr = F.N / 2;
    for (int q = 0; q < NP; ++q) {
      const int64_t jo = (vr - 1) * K + 1 + q;
      const int cls = int(jo % K);
      for (int c = 0; c <= 4 * K; ++c) {
        const int64_t off = (vr - 2) * K + c - jo;
        pp.tB[q][c] = (off >= -2 * K && off <= 2 * K) ? p.c.BI[cls][off + 2 * K] : T(0);
      }
      for (int c = 0; c <= 2 * K; ++c) {
        const int64_t off = (vr - 1) * K + c - jo;
        pp.tM[q][c] = (off >= -K && off <= K) ? p.c.MI[cls][off + K] : T(0);
        pp.tL[q][c] = (off >= -K && off <= K) ? p.c.LI[cls][off + K] : T(0);
      }
    }
  }
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid_cache, (count + LY::NW - 1) / LY::NW));
  mvs3d_kernel<T, K><<<grid, 128, smem, st>>>(pp);
}

template <typename T>
bool fused3_mvs_color(FusedLevel& F, const int32_t* list, int64_t count, T omega, const T* b, T* x, cudaStream_t st,
                      int64_t* launches) {
  if (F.d != 3 || count == 0) return count == 0 && F.d == 3;
  if (std::getenv("C0IP_NO_MVS3")) return false;
  switch (F.k) {
    case 2: launch_mvs3<T, 2>(F, list, count, omega, b, x, st); break;
    case 3: launch_mvs3<T, 3>(F, list, count, omega, b, x, st); break;
    default: return false;
  }
  (*launches)++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("fused mvs3d launch: ") + cudaGetErrorString(e));
  return true;
}

// ----------------------------------------------------------------------------- host side
static SlabWindow full_window3(const FusedLevel& F) { return SlabWindow{0, F.n, 1, int64_t(F.k) * F.N}; }

template <typename T, int K>
static void launch_apply3(const FusedLevel& F, const T* x, const T* b, T* y, const SlabWindow& w, cudaStream_t st) {
  using LY = Apply3Layout<T, K>;
  const size_t smem = sizeof(T) * size_t(LY::TOTAL);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(apply3d_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(apply3d_kernel<T, K>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  Apply3P<T, K> p;
  std::memcpy(&p.c, coef_of<T>(F).data(), sizeof(p.c));
  p.x = x; p.b = b; p.y = y; p.N = F.N; p.n = F.n;
  p.row0 = w.row0; p.lrows = w.lrows; p.out_lo = w.out_lo; p.out_hi = w.out_hi;
  p.cz_lo = w.out_lo / K;
  p.cz_hi = (w.out_hi - 1) / K + 1;
  p.scale = T(1.0 / F.h);
  p.zero = 0;
  const int64_t ntx = (F.N + LY::C - 1) / LY::C, nch = (p.cz_hi - p.cz_lo + Tile3<K>::CZ - 1) / Tile3<K>::CZ;
  apply3d_kernel<T, K><<<(unsigned)(ntx * ntx * nch), 256, smem, st>>>(p);
}

// patch set of one launch: a device list, or an arithmetic box of vertices (vlo + vstr i per axis)
struct PatchSet3 {
  const int32_t* list = nullptr;
  int64_t count = 0;
  int vlo[3] = {1, 1, 1}, vcnt[3] = {0, 0, 0}, vstr = 1;
};

template <typename T, int K>
static void launch_fdm3_cta(const Fdm3P<T, K>& p, int64_t count, cudaStream_t st) {
  using LY = Fdm3CtaLayout<T, K>;
  const size_t smem = sizeof(T) * size_t(LY::TOTAL);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(patch_fdm3d_cta_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(patch_fdm3d_cta_kernel<T, K>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  const int64_t grid = (count + LY::PB - 1) / LY::PB;
  patch_fdm3d_cta_kernel<T, K><<<(unsigned)grid, 256, smem, st>>>(p);
}

template <typename T, int K>
static void launch_fdm3(const FusedLevel& F, T omega, const T* r, T* x, const PatchSet3& ps, int atomic,
                        const SlabWindow& w, cudaStream_t st) {
  using LY = Fdm3Layout<T, K>;
  const size_t smem = sizeof(T) * size_t(LY::TOTAL);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(patch_fdm3d_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(patch_fdm3d_kernel<T, K>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  Fdm3P<T, K> p;
  std::memcpy(&p.c, coef_of<T>(F).data(), sizeof(p.c));
  p.r = r; p.x = x; p.list = ps.list; p.count = ps.count; p.N = F.N; p.n = F.n;
  for (int a = 0; a < 3; ++a) { p.vlo[a] = ps.vlo[a]; p.vcnt[a] = ps.vcnt[a]; }
  p.vstr = ps.vstr;
  {
    const unsigned Nm1 = unsigned(F.N - 1);
    const unsigned d0 = ps.list ? Nm1 : unsigned(std::max(1, ps.vcnt[0]));
    const unsigned d1 = ps.list ? Nm1 * Nm1 : unsigned(std::max(1, ps.vcnt[1]));
    p.mag[0] = unsigned(0xFFFFFFFFull / d0);
    p.mag[1] = unsigned(0xFFFFFFFFull / d1);
  }
  p.row0 = w.row0; p.lrows = w.lrows; p.out_lo = w.out_lo; p.out_hi = w.out_hi;
  p.factor = T(double(omega) * F.h);
  p.zero = 0;
  p.atomic = atomic;
  if (!atomic) {                 // disjoint list: CTA-cooperative kernel (measured faster)
    launch_fdm3_cta<T, K>(p, ps.count, st);
    return;
  }
  if constexpr (K <= 3) {   // k = 4: 3.35 vs 3.26 ms for the warp-per-patch kernel (1 CTA/SM at 253 registers)
    // atomic AVS over a box of vertices: runs of patches along x (patch_fdm3d_run_kernel)
    if (!ps.list && ps.vstr == 1 && !std::getenv("C0IP_FDM3_NORUN")) {
      using RL = Fdm3RunLayout<T, K>;
      const size_t rsm = sizeof(T) * size_t(RL::TOTAL);
      static int rgrid = -1;
      if (rgrid < 0) {
        cudaFuncSetAttribute(patch_fdm3d_run_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
        cudaFuncSetAttribute(patch_fdm3d_run_kernel<T, K>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        int dev = 0, sms = 148, per = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, patch_fdm3d_run_kernel<T, K>, 256, rsm);
        rgrid = sms * std::max(per, 1);
      }
      const int64_t runs = int64_t((ps.vcnt[0] + RL::PW - 1) / RL::PW) * ps.vcnt[1] * ps.vcnt[2];
      const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(rgrid, (runs + 7) / 8));
      patch_fdm3d_run_kernel<T, K><<<(unsigned)grid, 256, rsm, st>>>(p);
      return;
    }
  }
  static int grid_cache = -1;
  if (grid_cache < 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, patch_fdm3d_kernel<T, K>, 256, smem);
    grid_cache = sms * std::max(per, 1);
  }
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(grid_cache, (ps.count + 7) / 8));
  patch_fdm3d_kernel<T, K><<<(unsigned)grid, 256, smem, st>>>(p);
}

static void check3(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
bool fused3_apply(FusedLevel& F, const T* x, const T* b, T* y, cudaStream_t st, int64_t* launches,
                  const SlabWindow* win) {
  if (F.d != 3) return false;
  const SlabWindow w = win ? *win : full_window3(F);
  if (w.out_hi <= w.out_lo) return true;
  switch (F.k) {
    case 2: launch_apply3<T, 2>(F, x, b, y, w, st); break;
    case 3: launch_apply3<T, 3>(F, x, b, y, w, st); break;
    case 4: launch_apply3<T, 4>(F, x, b, y, w, st); break;
    case 5: launch_apply3<T, 5>(F, x, b, y, w, st); break;
    default: return false;
  }
  (*launches)++;
  check3("fused apply3d launch");
  return true;
}

template <typename T>
static bool fdm3_dispatch(FusedLevel& F, T omega, const T* r, T* x, const PatchSet3& ps, int atomic,
                          const SlabWindow& w, cudaStream_t st, int64_t* launches) {
  if (ps.count == 0) return true;
  switch (F.k) {
    case 2: launch_fdm3<T, 2>(F, omega, r, x, ps, atomic, w, st); break;
    case 3: launch_fdm3<T, 3>(F, omega, r, x, ps, atomic, w, st); break;
    case 4: launch_fdm3<T, 4>(F, omega, r, x, ps, atomic, w, st); break;
    case 5: launch_fdm3<T, 5>(F, omega, r, x, ps, atomic, w, st); break;
    default: return false;
  }
  (*launches)++;
  check3("fused patch_fdm3d launch");
  return true;
}

template <typename T>
bool fused3_patch_fdm(FusedLevel& F, T omega, const T* r, T* x, const int32_t* list, int64_t count,
                      cudaStream_t st, int64_t* launches, int atomic) {
  if (F.d != 3 || F.k < 2 || F.k > 5) return false;
  PatchSet3 ps;
  if (list) {
    ps.list = list;
    ps.count = count;
  } else {                                   // all patches 0..count-1 (count = (N-1)^3)
    for (int a = 0; a < 3; ++a) ps.vcnt[a] = int(F.N - 1);
    ps.count = count;
  }
  return fdm3_dispatch<T>(F, omega, r, x, ps, atomic, full_window3(F), st, launches);
}

template <typename T, int K>
static void launch_fdm3_zrun(const FusedLevel& F, T omega, const T* r, T* x, const PatchSet3& ps, const SlabWindow& w,
                             int zc, int zpar, cudaStream_t st) {
  using LY = Fdm3Layout<T, K>;
  const size_t smem = sizeof(T) * size_t(8 * (LY::WB + 2 * K * LY::NL2) + LY::NL);
  static int grid_cache = -1;
  if (grid_cache < 0) {
    cudaFuncSetAttribute(patch_fdm3d_zrun_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, patch_fdm3d_zrun_kernel<T, K>, 256, smem);
    grid_cache = sms * std::max(per, 1);
  }
  Fdm3P<T, K> p;
  std::memcpy(&p.c, coef_of<T>(F).data(), sizeof(p.c));
  p.r = r; p.x = x; p.list = nullptr; p.count = 0; p.N = F.N; p.n = F.n;
  for (int a = 0; a < 3; ++a) { p.vlo[a] = ps.vlo[a]; p.vcnt[a] = ps.vcnt[a]; }
  p.vstr = ps.vstr;
  p.mag[0] = p.mag[1] = 0;
  p.row0 = w.row0; p.lrows = w.lrows; p.out_lo = w.out_lo; p.out_hi = w.out_hi;
  p.factor = T(double(omega) * F.h);
  p.zero = 0;
  p.atomic = 0;
  p.zc = zc;
  p.zpar = zpar;
  const int64_t cols = int64_t(ps.vcnt[0]) * ps.vcnt[1];
  const int zlo = ps.vlo[2], zhi = ps.vlo[2] + ps.vcnt[2] - 1, k0 = (zlo - 1) / zc, k1 = (zhi - 1) / zc;
  const int kf = k0 + ((k0 & 1) != zpar ? 1 : 0);
  const int64_t nck = kf > k1 ? 0 : (k1 - kf) / 2 + 1;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid_cache, (cols * nck + 7) / 8));
  if (cols * nck > 0) patch_fdm3d_zrun_kernel<T, K><<<grid, 256, smem, st>>>(p);
}

template <typename T>
bool fused3_fdm_window(FusedLevel& F, T omega, const T* r, T* x, bool atomic, cudaStream_t st, int64_t* launches,
                       const SlabWindow* win) {
  if (F.d != 3 || F.k < 2 || F.k > 5) return false;
  const SlabWindow w = win ? *win : full_window3(F);
  if (w.out_hi <= w.out_lo) return true;
  const int K = F.k, Nm1 = int(F.N - 1);
  // patches touching node planes [out_lo, out_hi): (v+1)K - 1 >= out_lo and (v-1)K + 1 <= out_hi - 1
  const int vz_lo = std::max<int>(1, int((w.out_lo + 1) / K) - 1 + ((w.out_lo + 1) % K ? 1 : 0));
  const int vz_hi = std::min<int>(Nm1, int((w.out_hi - 2) / K) + 1);
  if (vz_hi < vz_lo) return true;
  if (atomic) {
    PatchSet3 ps;
    ps.vcnt[0] = ps.vcnt[1] = Nm1;
    ps.vlo[2] = vz_lo;
    ps.vcnt[2] = vz_hi - vz_lo + 1;
    ps.count = int64_t(Nm1) * Nm1 * ps.vcnt[2];
    return fdm3_dispatch<T>(F, omega, r, x, ps, 1, w, st, launches);
  }
  // deterministic: 4 x-y parity classes of patch columns, each column walked along z (zrun kernel)
  if (K <= 5 && !std::getenv("C0IP_NO_ZRUN")) {
    for (int c = 0; c < 4; ++c) {
      PatchSet3 ps;
      ps.vstr = 2;
      int cnt = 1;
      for (int a = 0; a < 2; ++a) {
        const int par = (c >> a) & 1;
        const int v0 = 1 + ((1 & 1) != par ? 1 : 0);
        ps.vlo[a] = v0;
        ps.vcnt[a] = v0 > Nm1 ? 0 : (Nm1 - v0) / 2 + 1;
        cnt *= ps.vcnt[a];
      }
      ps.vlo[2] = vz_lo;
      ps.vcnt[2] = vz_hi - vz_lo + 1;
      if (cnt == 0) continue;
      // z chunks of ZC patches, even and odd chunks in two launches (~8 warp waves per launch)
      constexpr int ZC = 8;
      for (int zpar = 0; zpar < 2; ++zpar) {
        switch (K) {
          case 2: launch_fdm3_zrun<T, 2>(F, omega, r, x, ps, w, ZC, zpar, st); break;
          case 3: launch_fdm3_zrun<T, 3>(F, omega, r, x, ps, w, ZC, zpar, st); break;
          case 4: launch_fdm3_zrun<T, 4>(F, omega, r, x, ps, w, ZC, zpar, st); break;
          case 5: launch_fdm3_zrun<T, 5>(F, omega, r, x, ps, w, ZC, zpar, st); break;
        }
        (*launches)++;
        check3("fused patch_fdm3d_zrun launch");
      }
    }
    return true;
  }
  // 2^3 parity classes (v_a mod 2), mutually disjoint patches: deterministic plain stores
  for (int c = 0; c < 8; ++c) {
    PatchSet3 ps;
    ps.vstr = 2;
    const int lo[3] = {1, 1, vz_lo}, hi[3] = {Nm1, Nm1, vz_hi};
    int64_t cnt = 1;
    for (int a = 0; a < 3; ++a) {
      const int par = (c >> a) & 1;
      int v0 = lo[a] + ((lo[a] & 1) != par ? 1 : 0);
      ps.vlo[a] = v0;
      ps.vcnt[a] = v0 > hi[a] ? 0 : (hi[a] - v0) / 2 + 1;
      cnt *= ps.vcnt[a];
    }
    ps.count = cnt;
    if (!fdm3_dispatch<T>(F, omega, r, x, ps, 0, w, st, launches)) return false;
  }
  return true;
}

template bool fused3_mvs_color<double>(FusedLevel&, const int32_t*, int64_t, double, const double*, double*,
                                       cudaStream_t, int64_t*);
template bool fused3_mvs_color<float>(FusedLevel&, const int32_t*, int64_t, float, const float*, float*, cudaStream_t,
                                      int64_t*);
template bool fused3_apply<double>(FusedLevel&, const double*, const double*, double*, cudaStream_t, int64_t*,
                                   const SlabWindow*);
template bool fused3_apply<float>(FusedLevel&, const float*, const float*, float*, cudaStream_t, int64_t*,
                                  const SlabWindow*);
template bool fused3_patch_fdm<double>(FusedLevel&, double, const double*, double*, const int32_t*, int64_t,
                                       cudaStream_t, int64_t*, int);
template bool fused3_patch_fdm<float>(FusedLevel&, float, const float*, float*, const int32_t*, int64_t,
                                      cudaStream_t, int64_t*, int);
template bool fused3_fdm_window<double>(FusedLevel&, double, const double*, double*, bool, cudaStream_t, int64_t*,
                                        const SlabWindow*);
template bool fused3_fdm_window<float>(FusedLevel&, float, const float*, float*, bool, cudaStream_t, int64_t*,
                                       const SlabWindow*);

}  // namespace c0ip
