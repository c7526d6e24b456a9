// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) kernels for large 2D levels, degrees k = 3, 4
// (patch width np = 2k - 1 <= 8, padded to 8).
//
// fdm2d_mma: the additive FDM update  x += omega h^2 sum_v R_v^T A~_v^{-1} R_v r  (PAPER.md:206-213,
// 356-384).  Every patch solve is a chain of four 8x8x8 contractions,
//     D1 = S_x^T R^T        (contract x)        D1[i][y]
//     D2 = D1 S_y           (contract y)        D2[i][j]   then  D2[i][j] /= (lam_x,i + lam_y,j)
//     D3 = S_y D2^T         (contract j)        D3[y][i]
//     D4 = D3 S_x^T         (contract i)        D4[y][x]   = (A~_v^{-1} r_v)[y][x]
// each two m8n8k4 DMMAs.  The contraction index of every stage is the k index of the MMA, and the
// k slots are permuted (slot q of chunk c <-> index 2q + c) so that the accumulator fragment of a
// stage (thread: row lane/4, columns 2(lane%4) + {0,1}) *is* the A or B fragment of the next one:
// a patch solve never leaves registers (8 DMMA + 2 fragment loads + 1 read-modify-write per patch
// per warp).  The constant operands (S of the three axis variants) are per-lane
// fragments in registers (interior variant) or shared memory (boundary variants).
//
// Tiling, slab windows and the gather ownership are those of fdm2d_kernel (fused_kernels.cu): a CTA
// owns the nodes of a tile of C x C cells and solves the (C+1)^2 patches touching them (one halo patch
// row / column), each into its own shared-memory slot (no write conflicts, no barriers between
// patches); every owned DoF then sums its <= 4 patch contributions in a fixed order (deterministic,
// no atomics) and is written once.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "fused_common.cuh"

namespace c0ip {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// per-lane constant fragments of one axis variant: F1[c] = S[2q+c][g], F2[c] = S[g][2q+c]
// (g = lane/4, q = lane%4, zero outside np)
struct Frag {
  double f1[2], f2[2];
};

template <int K>
struct MmaFdmLayout {
  static constexpr int C = 8;                       // cells per tile edge
  static constexpr int O = C * K;                   // owned nodes per axis
  static constexpr int NP = 2 * K - 1;
  static constexpr int RN = (C + 2) * K - 1;        // residual box [(c0-1)K+1, (c0+C+1)K-1]
  static constexpr int RR = C * K + 8;              // rows / cols touched by padded 8x8 patches
  static constexpr int PR = RR;                     // pitch (even: 16-byte pairs when x0 even)
  static constexpr int RBOX = RR * PR;
  static constexpr int NPT = (C + 1) * (C + 1);     // patches per tile (one halo row / column)
  static constexpr int SL = 64;                     // patch slot (8x8), rotated by 4p within the slot
                                                    // (no bank conflicts in the gather)
  static constexpr int OPT = (O * O + 255) / 256;   // owned nodes per thread
  // smem: 2 x r box | patch slots | fragments (3 variants x 32 lanes) | inv scale 9 x 32 x 2
  static constexpr int TOTAL = 2 * RBOX + NPT * SL + 3 * 32 * 4 + 9 * 32 * 2;
  static_assert(RR >= RN && 2 * K <= 8, "layout");
};

// one patch solve: r fragment (b0, b1) -> (e0, e1) = rows g, columns 2q + {0,1} of A~_v^{-1} r_v
__device__ __forceinline__ void patch_solve(const Frag& fx, const Frag& fy, double2 sc, double b0, double b1,
                                            double& e0, double& e1) {
  double d0, d1;
  dmma(d0, d1, fx.f1[0], b0, 0.0, 0.0);          // D1[i][y] = sum_x S_x[x][i] r[y][x]
  dmma(d0, d1, fx.f1[1], b1, d0, d1);
  dmma(e0, e1, d0, fy.f1[0], 0.0, 0.0);          // D2[i][j] = sum_y D1[i][y] S_y[y][j]
  dmma(e0, e1, d1, fy.f1[1], e0, e1);
  e0 *= sc.x;                                    // / (lam_x,i + lam_y,j), times omega h^2
  e1 *= sc.y;
  dmma(d0, d1, fy.f2[0], e0, 0.0, 0.0);          // D3[y][i] = sum_j S_y[y][j] D2[i][j]
  dmma(d0, d1, fy.f2[1], e1, d0, d1);
  dmma(e0, e1, d0, fx.f2[0], 0.0, 0.0);          // D4[y][x] = sum_i D3[y][i] S_x[x][i]
  dmma(e0, e1, d1, fx.f2[1], e0, e1);
}

template <int K>
__device__ __forceinline__ void load_frag(const double* rb, int off, double& b0, double& b1) {
  if constexpr (K % 2 == 0) {
    const double2 bb = *reinterpret_cast<const double2*>(rb + off);
    b0 = bb.x;
    b1 = bb.y;
  } else {
    b0 = rb[off];
    b1 = rb[off + 1];
  }
}

template <int K>
__global__ void __launch_bounds__(256, 3) fdm2d_mma_kernel(const __grid_constant__ FdmP<double, K> P) {
  using LY = MmaFdmLayout<K>;
  constexpr int C = LY::C, O = LY::O, NP = LY::NP, RN = LY::RN, PR = LY::PR, SL = LY::SL, NPT = LY::NPT;
  constexpr int NT = 256, OPT = LY::OPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  double* const rbuf0 = sm;                        // [2][RBOX]
  double* const slot = sm + 2 * LY::RBOX;          // [NPT][SL]: D4 of patch (px, py), row-major 8x8
  Frag* const frag = reinterpret_cast<Frag*>(slot + NPT * SL);         // [3][32]
  double2* const invs = reinterpret_cast<double2*>(frag + 3 * 32);     // [vx*3+vy][32]
  const int64_t N = P.N, n = P.n, KN = K * N;
  const int Ni = int(N);
  const int ntx = int((N + C - 1) / C);
  int ty0, ty1;
  tile_rows<K, C>(P.out_lo, P.out_hi, ty0, ty1);
  const int ntiles = ntx * (ty1 - ty0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;

  // constant fragments; the FDM factor omega h^2 is folded into the inverse eigenvalue sums
  if (tid < 3 * 32) {
    const int v = tid >> 5;
    const int gg = (tid & 31) >> 2, qq = tid & 3;
    Frag f;
    for (int c = 0; c < 2; ++c) {
      const int a = 2 * qq + c;
      f.f1[c] = (a < NP && gg < NP) ? P.c.S[v][a * NP + gg] : 0.0;
      f.f2[c] = (a < NP && gg < NP) ? P.c.S[v][gg * NP + a] : 0.0;
    }
    frag[tid] = f;
  }
  for (int e = tid; e < 9 * 32; e += NT) {
    const int vx = e / 96, vy = (e / 32) % 3, l = e & 31;
    const int i = l >> 2, j0 = 2 * (l & 3);
    double2 s;
    s.x = (i < NP && j0 < NP) ? P.factor / (P.c.lam[vx][i] + P.c.lam[vy][j0]) : 0.0;
    s.y = (i < NP && j0 + 1 < NP) ? P.factor / (P.c.lam[vx][i] + P.c.lam[vy][j0 + 1]) : 0.0;
    invs[e] = s;
  }
  // the padded rows / columns of the r boxes (beyond RN) are never written by the loads: zero once
  for (int e = tid; e < 2 * LY::RBOX; e += NT) {
    const int rem = e % LY::RBOX, r = rem / PR, c = rem % PR;
    if (r >= RN || c >= RN) rbuf0[e] = 0.0;
  }
  __syncthreads();
  const Frag fi = frag[32 + lane];                 // interior variant in registers
  const double2 si = invs[(1 * 3 + 1) * 32 + lane];

  auto issue = [&](int t, int buf) {
    const int64_t cx0 = int64_t(t % ntx) * C, cy0 = int64_t(ty0 + t / ntx) * C;
    load_box_async<double, RN, RN, PR>(rbuf0 + buf * LY::RBOX, P.r, n, KN, (cy0 - 1) * K + 1,
                                       (cx0 - 1) * K + 1, P.row0, P.lrows);
  };

  int buf = 0;
  if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
  cp_async_commit();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (t + (int)gridDim.x < ntiles) issue(t + gridDim.x, buf ^ 1);
    cp_async_commit();
    const int tyy = ty0 + t / ntx;
    const int cx = (t - (t / ntx) * ntx) * C, cy = tyy * C;
    // owned x values into registers now; used after the patch solves (latency hidden)
    double xo[OPT];
#pragma unroll
    for (int u = 0; u < OPT; ++u) {
      const int e = u * NT + tid, oy = e / O, ox = e - (e / O) * O;
      const int64_t jy = int64_t(cy) * K + oy, jx = int64_t(cx) * K + ox;
      xo[u] = (e < O * O && jx >= 1 && jx <= KN - 1 && jy >= P.out_lo && jy < P.out_hi) ? P.x[(jy - 1 - P.row0) * n + (jx - 1)] : 0.0;
    }
    cp_async_wait1();
    __syncthreads();
    const double* rb = rbuf0 + buf * LY::RBOX;
    const bool tin = (cx >= 2 && cx + C <= Ni - 2 && cy >= 2 && cy + C <= Ni - 2);

    // every patch (px, py), px, py in [0, C], solved into its own slot: no write conflicts, two
    // independent DMMA chains per warp
    if (tin) {
#pragma unroll 1
      for (int p0 = warp; p0 < NPT; p0 += 2 * (NT / 32)) {
        const int p1 = p0 + NT / 32;
        const bool two = p1 < NPT;
        const int py0 = p0 / (C + 1), px0 = p0 - py0 * (C + 1);
        const int py1 = p1 / (C + 1), px1 = p1 - py1 * (C + 1);
        double a0, a1, b0 = 0.0, b1 = 0.0, e0, e1, f0, f1;
        load_frag<K>(rb, (py0 * K + g) * PR + px0 * K + 2 * q, a0, a1);
        if (two) load_frag<K>(rb, (py1 * K + g) * PR + px1 * K + 2 * q, b0, b1);
        patch_solve(fi, fi, si, a0, a1, e0, e1);
        patch_solve(fi, fi, si, b0, b1, f0, f1);
        *reinterpret_cast<double2*>(slot + p0 * SL + ((2 * lane + 4 * p0) & 63)) = make_double2(e0, e1);
        if (two) *reinterpret_cast<double2*>(slot + p1 * SL + ((2 * lane + 4 * p1) & 63)) = make_double2(f0, f1);
      }
    } else {
#pragma unroll 1
      for (int p = warp; p < NPT; p += NT / 32) {
        const int py = p / (C + 1), px = p - py * (C + 1);
        const int vx = cx + px, vy = cy + py;
        double e0 = 0.0, e1 = 0.0;
        if (vx >= 1 && vx <= Ni - 1 && vy >= 1 && vy <= Ni - 1) {          // warp-uniform
          const int varx = vx == 1 ? 0 : (vx == Ni - 1 ? 2 : 1), vary = vy == 1 ? 0 : (vy == Ni - 1 ? 2 : 1);
          const Frag fx = frag[varx * 32 + lane], fy = frag[vary * 32 + lane];
          const double2 sc = invs[(varx * 3 + vary) * 32 + lane];
          double a0, a1;
          load_frag<K>(rb, (py * K + g) * PR + px * K + 2 * q, a0, a1);
          patch_solve(fx, fy, sc, a0, a1, e0, e1);
        }
        *reinterpret_cast<double2*>(slot + p * SL + ((2 * lane + 4 * p) & 63)) = make_double2(e0, e1);
      }
    }
    __syncthreads();

    // gather: owned node (oy, ox) = box node (Y, X) = (oy + K - 1, ox + K - 1) receives patches
    // px in {X/K - 1, X/K} (local column X - px K <= 2K - 1 <= 7; the padding of D4 is exactly zero)
    // and likewise in y, summed in a fixed order
#pragma unroll
    for (int u = 0; u < OPT; ++u) {
      const int e = u * NT + tid, oy = e / O, ox = e - (e / O) * O;
      if (O * O % NT != 0 && e >= O * O) break;
      const int64_t jy = int64_t(cy) * K + oy, jx = int64_t(cx) * K + ox;
      const int Y = oy + K - 1, X = ox + K - 1;
      const int my = Y / K, mx = X / K, sy = Y - my * K, sx = X - mx * K;
      auto at = [&](int p, int l) { return slot[p * SL + ((l + 4 * p) & 63)]; };
      const int p = my * (C + 1) + mx;
      double s = at(p, sy * 8 + sx);
      if (mx >= 1) s += at(p - 1, sy * 8 + sx + K);
      if (my >= 1) {
        s += at(p - (C + 1), (sy + K) * 8 + sx);
        if (mx >= 1) s += at(p - (C + 1) - 1, (sy + K) * 8 + sx + K);
      }
      if (jx >= 1 && jx <= KN - 1 && jy >= P.out_lo && jy < P.out_hi) P.x[(jy - 1 - P.row0) * n + (jx - 1)] = xo[u] + s;
    }
    __syncthreads();
    buf ^= 1;
  }
}

template <int K>
static void launch_fdm_mma(const FusedLevel& F, double omega, const double* r, double* x, const SlabWindow& w,
                           cudaStream_t st) {
  using LY = MmaFdmLayout<K>;
  const size_t smem = sizeof(double) * size_t(LY::TOTAL);
  static int grid_cache = -1;
  if (grid_cache < 0) {
    cudaFuncSetAttribute(fdm2d_mma_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(fdm2d_mma_kernel<K>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fdm2d_mma_kernel<K>, 256, smem);
    grid_cache = sms * std::max(per, 1);
  }
  FdmP<double, K> p;
  std::memcpy(&p.c, F.c64.data(), sizeof(p.c));
  p.r = r; p.x = x; p.N = F.N; p.n = F.n;
  p.factor = omega * F.h * F.h;
  p.zero = 0;
  p.row0 = w.row0; p.lrows = w.lrows; p.out_lo = w.out_lo; p.out_hi = w.out_hi;
  const int64_t ntx = (F.N + LY::C - 1) / LY::C;
  const int64_t nty = ((w.out_hi - 1) / K) / LY::C - (w.out_lo / K) / LY::C + 1;
  const int grid = (int)std::min<int64_t>(grid_cache, ntx * nty);
  fdm2d_mma_kernel<K><<<grid, 256, smem, st>>>(p);
}

// ----------------------------------------------------------------------------- mvs2d_mma
// One colour of the coloured multiplicative smoother on the tensor cores, one
// patch per warp: for every patch v of the colour
//   r_v = (b - A x) on the np x np patch nodes, from x on the residual footprint (patch cells plus
//         their face neighbours; identical to the global residual recomputed per colour)
//         as two chained contraction stages of the Kronecker sum A = h^-2 (M^_y B^_x + 2 L^_y L^_x +
//         B^_y M^_x):
//           stage Y (x as the B operand, k = y_in in contiguous chunks of 4, n = 8-column blocks of
//                    x_in):  D_M = M^_y x, D_L = L^_y x, D_B = B^_y x       -> [y_out = g][x_in]
//           stage X (chained A operand, k slot (q, c) <-> x_in = block + 2q + c):
//                    acc = D_M B^_x^T + 2 D_L L^_x^T + D_B M^_x^T           -> [y_out = g][x_out = 2q+s]
//   u_v = A~_v^{-1} r_v by the FDM chain of fdm2d_mma (its input fragment layout is exactly acc's),
//   x  += omega h^2 u_v on the patch nodes (disjoint within a colour: plain stores).
template <int K>
struct MvsMma {
  static constexpr int NP = 2 * K - 1;
  static constexpr int CML = (2 * K + 1 + 3) / 4;   // y_in chunks of M^_y, L^_y: rows [jy0-1, jy0+2K-1]
  static constexpr int CB = (4 * K + 1 + 3) / 4;    // y_in chunks of B^_y: rows [jy0-K-1, jy0+3K-1]
  // x_in blocks: block b (b = 0, 1, 2) covers columns [jx0 - 9 + 8b, jx0 - 2 + 8b]
  __host__ __device__ static constexpr bool need(int lo, int hi, int b) {   // band [jx0+lo, jx0+hi]
    return lo <= -2 + 8 * b && hi >= -9 + 8 * b;
  }
  __host__ __device__ static constexpr bool bm(int b) { return need(-K - 1, 3 * K - 1, b); }   // B^_x band
  __host__ __device__ static constexpr bool bl(int b) { return need(-1, 2 * K - 1, b); }       // L^_x, M^_x band
  // rows of x loaded: [jy0 - K - 1, jy0 - K - 1 + RL); M^/L^ chunk c starts at row offset K + 4c
  static constexpr int RL = (K + 4 * CML > 4 * CB) ? K + 4 * CML : 4 * CB;
  // per-variant constant fragments, structure of arrays over the 32 lanes (conflict-free LDS):
  //   Y[v][f][lane], f = c (M^_y chunk c), CML + c (L^_y), 2 CML + c (B^_y):  Op_y[jy0 + g][row + q]
  //   X[v][f][lane] (double2 over c = 0, 1), f = 3 op + block, op 0 B^_x, 1 2 L^_x, 2 M^_x:
  //                                                                          Op_x[jx0 + g][block + 2q + c]
  static constexpr int NY = 2 * CML + CB, NX = 9;
};

// full-band 1D operator coefficient (reference scale) between nodes jo (row) and ji (column):
// which 0 = B^, 1 = M^, 2 = L^ (fused_common.cuh Coef2 tables)
template <int K>
__device__ double op1d(const Coef2<double, K>& c, int which, int64_t jo, int64_t ji, int64_t N) {
  const int64_t KN = K * N, off = ji - jo;
  if (ji < 1 || ji > KN - 1 || jo < 1 || jo > KN - 1) return 0.0;
  const int s = special_row<K>(jo, N);
  if (which == 0) {
    if (off < -2 * K || off > 2 * K) return 0.0;
    return s >= 0 ? c.BS[s][off + 2 * K] : c.BI[jo % K][off + 2 * K];
  }
  if (s >= 0) {
    if (off < -2 * K || off > 2 * K) return 0.0;
    return which == 1 ? c.MS[s][off + 2 * K] : c.LS[s][off + 2 * K];
  }
  if (off < -K || off > K) return 0.0;
  return which == 1 ? c.MI[jo % K][off + K] : c.LI[jo % K][off + K];
}

template <int K>
__global__ void __launch_bounds__(256, 4) mvs2d_mma_kernel(const __grid_constant__ MvsP<double, K> P) {
  using MV = MvsMma<K>;
  constexpr int NP = MV::NP, CML = MV::CML, CB = MV::CB, NY = MV::NY, NX = MV::NX;
  constexpr int NT = 256;
  __shared__ double ys[3][NY][32];
  __shared__ double2 xs[3][NX][32];
  __shared__ Frag ffs[3][32];
  __shared__ double2 sfs[9][32];
  const int64_t N = P.N, n = P.n, KN = K * N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;

  // constant fragments of the three axis variants (left / interior / right: representative vertex
  // v = 1, N/2, N - 1 -- the interior representative's whole band lies inside the domain)
  if (tid < 96) {
    const int v = tid >> 5, gg = (tid & 31) >> 2, qq = tid & 3, l = tid & 31;
    const int64_t vr = v == 0 ? 1 : (v == 1 ? N / 2 : N - 1);
    const int64_t j0 = (vr - 1) * K + 1;                 // first patch node
    const int64_t jo = gg < NP ? j0 + gg : -1;           // padding row: zero fragments
    for (int c = 0; c < CML; ++c) {
      ys[v][c][l] = op1d<K>(P.c, 1, jo, j0 - 1 + 4 * c + qq, N);
      ys[v][CML + c][l] = op1d<K>(P.c, 2, jo, j0 - 1 + 4 * c + qq, N);
    }
    for (int c = 0; c < CB; ++c) ys[v][2 * CML + c][l] = op1d<K>(P.c, 0, jo, j0 - K - 1 + 4 * c + qq, N);
    for (int bb = 0; bb < 3; ++bb) {
      const int64_t ji = j0 - 9 + 8 * bb + 2 * qq;
      xs[v][bb][l] = make_double2(op1d<K>(P.c, 0, jo, ji, N), op1d<K>(P.c, 0, jo, ji + 1, N));
      xs[v][3 + bb][l] = make_double2(2.0 * op1d<K>(P.c, 2, jo, ji, N), 2.0 * op1d<K>(P.c, 2, jo, ji + 1, N));
      xs[v][6 + bb][l] = make_double2(op1d<K>(P.c, 1, jo, ji, N), op1d<K>(P.c, 1, jo, ji + 1, N));
    }
    Frag f;
    for (int c = 0; c < 2; ++c) {
      const int a = 2 * qq + c;
      f.f1[c] = (a < NP && gg < NP) ? P.c.S[v][a * NP + gg] : 0.0;
      f.f2[c] = (a < NP && gg < NP) ? P.c.S[v][gg * NP + a] : 0.0;
    }
    ffs[v][l] = f;
  }
  for (int e = tid; e < 9 * 32; e += NT) {
    const int vx = e / 96, vy = (e / 32) % 3, l = e & 31;
    const int i = l >> 2, j0 = 2 * (l & 3);
    double2 sc;
    sc.x = (i < NP && j0 < NP) ? P.factor / (P.c.lam[vx][i] + P.c.lam[vy][j0]) : 0.0;
    sc.y = (i < NP && j0 + 1 < NP) ? P.factor / (P.c.lam[vx][i] + P.c.lam[vy][j0 + 1]) : 0.0;
    sfs[vx * 3 + vy][l] = sc;
  }
  __syncthreads();
  const int Nm1 = int(N - 1), KNi = int(KN), ni = int(n);
  const unsigned magic = unsigned(0xFFFFFFFFull / unsigned(Nm1));
  const double* __restrict__ X = P.x;

  // one patch: x rows [jy0 - K - 1, + RL), column blocks [jx0 - 9 + 8b, + 8) (lane: row q + 4c, column g)
  auto body = [&](int vx, int vy, bool edge) {
    const int jx0 = (vx - 1) * K + 1, jy0 = (vy - 1) * K + 1;
    const int vary = edge ? (vy == 1 ? 0 : (vy == Nm1 ? 2 : 1)) : 1;
    const int varx = edge ? (vx == 1 ? 0 : (vx == Nm1 ? 2 : 1)) : 1;
    const double* base = X + int64_t(jy0 - K - 2) * n + (jx0 - 10);   // node (jy0 - K - 1, jx0 - 9)
    auto ld = [&](int r, int col) -> double {                          // r, col relative to that node
      if (edge) {
        const int jy = jy0 - K - 1 + r, jx = jx0 - 9 + col;
        if (jx < 1 || jx > KNi - 1 || jy < 1 || jy > KNi - 1) return 0.0;
      }
      return __ldg(base + (r * ni + col));
    };
    double xm[3][CML], xb[3][CB];
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) {
      if (MV::bl(bb)) {
#pragma unroll
        for (int c = 0; c < CB; ++c) xb[bb][c] = ld(4 * c + q, 8 * bb + g);
      }
      if (MV::bm(bb) || MV::bl(bb)) {
#pragma unroll
        for (int c = 0; c < CML; ++c) {
          // M^/L^ rows start K rows below the B^ rows: for K = 4 they are chunks of the B^ load
          if (K % 4 == 0 && MV::bl(bb) && c + K / 4 < CB) xm[bb][c] = xb[bb][c + K / 4];
          else xm[bb][c] = ld(K + 4 * c + q, 8 * bb + g);
        }
      }
    }
    const int jy = jy0 + g, jx = jx0 + 2 * q;
    const bool r0 = g < NP && 2 * q < NP, r1 = g < NP && 2 * q + 1 < NP;
    const int64_t po = int64_t(jy - 1) * n + (jx - 1);
    const double bv0 = r0 ? __ldg(P.b + po) : 0.0;
    const double bv1 = r1 ? __ldg(P.b + po + 1) : 0.0;
    // stage Y then stage X, accumulated into (a0, a1) = [y_out = g][x_out = 2q + s]
    const double* yv = &ys[vary][0][lane];
    const double2* xv = &xs[varx][0][lane];
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) {
      if (MV::bm(bb)) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int c = 0; c < CML; ++c) dmma(d0, d1, yv[c * 32], xm[bb][c], d0, d1);
        const double2 f = xv[bb * 32];
        dmma(a0, a1, d0, f.x, a0, a1);
        dmma(a0, a1, d1, f.y, a0, a1);
      }
      if (MV::bl(bb)) {
        double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int c = 0; c < CML; ++c) dmma(d0, d1, yv[(CML + c) * 32], xm[bb][c], d0, d1);
#pragma unroll
        for (int c = 0; c < CB; ++c) dmma(e0, e1, yv[(2 * CML + c) * 32], xb[bb][c], e0, e1);
        const double2 fl = xv[(3 + bb) * 32], fm = xv[(6 + bb) * 32];
        dmma(a0, a1, d0, fl.x, a0, a1);
        dmma(a0, a1, d1, fl.y, a0, a1);
        dmma(a0, a1, e0, fm.x, a0, a1);
        dmma(a0, a1, e1, fm.y, a0, a1);
      }
    }
    const double rr0 = fma(-P.scale, a0, bv0), rr1 = fma(-P.scale, a1, bv1);
    double u0, u1;
    patch_solve(ffs[varx][lane], ffs[vary][lane], sfs[varx * 3 + vary][lane], rr0, rr1, u0, u1);
    double* xp = P.x + po;
    if (r0) xp[0] += u0;
    if (r1) xp[1] += u1;
  };

  constexpr int YTOP = MV::RL - K - 2;   // last loaded row relative to jy0
#pragma unroll 1
  for (int64_t pi = int64_t(blockIdx.x) * (NT / 32) + warp; pi < P.count; pi += int64_t(gridDim.x) * (NT / 32)) {
    const int pid = P.list[pi];
    int qy = int(__umulhi(unsigned(pid), magic));        // pid / (N - 1), at most one short
    if (pid - qy * Nm1 >= Nm1) ++qy;
    const int vy = 1 + qy, vx = 1 + pid - qy * Nm1;
    const int jx0 = (vx - 1) * K + 1, jy0 = (vy - 1) * K + 1;
    // fast path: interior variants on both axes and every loaded node inside the interior
    const bool fast = vx >= 2 && vx <= Nm1 - 1 && vy >= 2 && vy <= Nm1 - 1 && jx0 - 9 >= 1 && jx0 + 14 <= KNi - 1 &&
                      jy0 - K - 1 >= 1 && jy0 + YTOP <= KNi - 1;
    if (fast) body(vx, vy, false);
    else body(vx, vy, true);
  }
}

template <int K>
static void launch_mvs_mma(const FusedLevel& F, const int32_t* list, int64_t count, double omega, const double* b,
                           double* x, cudaStream_t st) {
  static int grid_cache = -1;
  if (grid_cache < 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mvs2d_mma_kernel<K>, 256, 0);
    grid_cache = sms * std::max(per, 1);
  }
  MvsP<double, K> p;
  std::memcpy(&p.c, F.c64.data(), sizeof(p.c));
  p.x = x; p.b = b; p.list = list; p.count = count; p.N = F.N; p.n = F.n;
  p.scale = 1.0 / (F.h * F.h);
  p.factor = omega * F.h * F.h;
  p.zero = 0;
  const int64_t want = (count + 7) / 8;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid_cache, want));
  mvs2d_mma_kernel<K><<<grid, 256, 0, st>>>(p);
}

bool mma_mvs2d(const FusedLevel& F, const int32_t* list, int64_t count, double omega, const double* b, double* x,
               cudaStream_t st) {
  if (!mma_enabled() || F.d != 2) return false;
  switch (F.k) {
    case 2: launch_mvs_mma<2>(F, list, count, omega, b, x, st); return true;
    case 3: launch_mvs_mma<3>(F, list, count, omega, b, x, st); return true;
    case 4: launch_mvs_mma<4>(F, list, count, omega, b, x, st); return true;
    default: return false;
  }
}

// ----------------------------------------------------------------------------- patch_fdm2d_mma
// x += omega h^2 R_v^T A~_v^{-1} R_v r for a list of patches (nullptr: every patch), one patch per warp:
// the paper's atomic AVS (fire-and-forget red.global.add.f64) or, for mutually disjoint
// patches (a parity class: coloured AVS), plain read-modify-write.
template <int K>
__global__ void __launch_bounds__(256, 4) patch_fdm2d_mma_kernel(const __grid_constant__ MvsP<double, K> P,
                                                                 const double* __restrict__ r, int atomic) {
  constexpr int NP = 2 * K - 1, NT = 256;
  __shared__ Frag ffs[3][32];
  __shared__ double2 sfs[9][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  if (tid < 96) {
    const int v = tid >> 5, gg = (tid & 31) >> 2, qq = tid & 3;
    Frag f;
    for (int c = 0; c < 2; ++c) {
      const int a = 2 * qq + c;
      f.f1[c] = (a < NP && gg < NP) ? P.c.S[v][a * NP + gg] : 0.0;
      f.f2[c] = (a < NP && gg < NP) ? P.c.S[v][gg * NP + a] : 0.0;
    }
    ffs[v][tid & 31] = f;
  }
  for (int e = tid; e < 9 * 32; e += NT) {
    const int vx = e / 96, vy = (e / 32) % 3, l = e & 31;
    const int i = l >> 2, j0 = 2 * (l & 3);
    double2 sc;
    sc.x = (i < NP && j0 < NP) ? P.factor / (P.c.lam[vx][i] + P.c.lam[vy][j0]) : 0.0;
    sc.y = (i < NP && j0 + 1 < NP) ? P.factor / (P.c.lam[vx][i] + P.c.lam[vy][j0 + 1]) : 0.0;
    sfs[vx * 3 + vy][l] = sc;
  }
  __syncthreads();
  const int Nm1 = int(P.N - 1);
  const unsigned magic = unsigned(0xFFFFFFFFull / unsigned(Nm1));
  const int64_t n = P.n;
  const bool r0 = g < NP && 2 * q < NP, r1 = g < NP && 2 * q + 1 < NP;
  if (!P.list && atomic) {
    // every patch (atomic AVS): warp tasks are runs of RUN consecutive patches along x of one patch
    // row, so the patch origin advances by K nodes per patch (no index division), the interior
    // patches use the register fragments, and the next patch's r fragment is loaded while the current
    // chain runs
    constexpr int RUN = 32;
    const int nrun = (Nm1 + RUN - 1) / RUN;
    const int64_t ntask = int64_t(nrun) * Nm1;
    const Frag fi = ffs[1][lane];
    const double2 si = sfs[4][lane];
#pragma unroll 1
    for (int64_t task = int64_t(blockIdx.x) * (NT / 32) + warp; task < ntask; task += int64_t(gridDim.x) * (NT / 32)) {
      const int vy = 1 + int(task / nrun), vx0 = 1 + int(task % nrun) * RUN;
      const int vx1 = min(vx0 + RUN, Nm1 + 1);
      const int vary = vy == 1 ? 0 : (vy == Nm1 ? 2 : 1);
      int64_t po = int64_t((vy - 1) * K + g) * n + (vx0 - 1) * K + 2 * q;
      double b0 = r0 ? __ldg(r + po) : 0.0, b1 = r1 ? __ldg(r + po + 1) : 0.0;
      double h0 = 0.0, h1 = 0.0;                         // this lane's columns held for the next patch
#pragma unroll 1
      for (int vx = vx0; vx < vx1; ++vx) {
        double nb0 = 0.0, nb1 = 0.0;
        if (vx + 1 < vx1) {
          nb0 = r0 ? __ldg(r + po + K) : 0.0;
          nb1 = r1 ? __ldg(r + po + K + 1) : 0.0;
        }
        double u0, u1;
        if (vary == 1 && vx != 1 && vx != Nm1) {
          patch_solve(fi, fi, si, b0, b1, u0, u1);
        } else {
          const int varx = vx == 1 ? 0 : (vx == Nm1 ? 2 : 1);
          patch_solve(ffs[varx][lane], ffs[vary][lane], sfs[varx * 3 + vary][lane], b0, b1, u0, u1);
        }
        double* xp = P.x + po;
        if constexpr (K % 2 == 0) {
          // consecutive patches of the run overlap in K - 1 columns: the previous patch's columns >= K (lanes
          // q >= S) are this patch's columns < K (lanes q - S) -- merge them in registers and issue one atomic
          // per node row and column of the overlap instead of two ((2k-1)/k instead of ((2k-1)/k)^2 atomics
          // per DoF along x)
          constexpr int S = K / 2;
          const double s0 = __shfl_down_sync(0xffffffffu, h0, S), s1 = __shfl_down_sync(0xffffffffu, h1, S);
          if (q + S <= 3) { u0 += s0; u1 += s1; }
          if (q < S || vx + 1 == vx1) {                  // columns no later patch of the run touches
            if (r0) asm volatile("red.global.add.f64 [%0], %1;" ::"l"(xp), "d"(u0) : "memory");
            if (r1) asm volatile("red.global.add.f64 [%0], %1;" ::"l"(xp + 1), "d"(u1) : "memory");
            h0 = 0.0;
            h1 = 0.0;
          } else {
            h0 = u0;
            h1 = u1;
          }
        } else {
          if (r0) asm volatile("red.global.add.f64 [%0], %1;" ::"l"(xp), "d"(u0) : "memory");
          if (r1) asm volatile("red.global.add.f64 [%0], %1;" ::"l"(xp + 1), "d"(u1) : "memory");
        }
        po += K;
        b0 = nb0;
        b1 = nb1;
      }
    }
    return;
  }
  // software pipeline: the next patch's coordinates and r fragment are loaded before this patch's
  // DMMA chain runs (the r loads are the latency the warps otherwise wait on)
  struct Item {
    int varx, vary;
    int64_t po;
    double b0, b1;
  };
  auto fetch = [&](int64_t pi, Item& it) {
    const int pid = P.list ? P.list[pi] : int(pi);
    int qy = int(__umulhi(unsigned(pid), magic));        // pid / (N - 1), at most one short
    if (pid - qy * Nm1 >= Nm1) ++qy;
    const int vy = 1 + qy, vx = 1 + pid - qy * Nm1;
    it.varx = vx == 1 ? 0 : (vx == Nm1 ? 2 : 1);
    it.vary = vy == 1 ? 0 : (vy == Nm1 ? 2 : 1);
    it.po = int64_t((vy - 1) * K + g) * n + (vx - 1) * K + 2 * q;   // node (jy0 + g, jx0 + 2q)
    it.b0 = r0 ? __ldg(r + it.po) : 0.0;
    it.b1 = r1 ? __ldg(r + it.po + 1) : 0.0;
  };
  const int64_t stride = int64_t(gridDim.x) * (NT / 32);
  int64_t pi = int64_t(blockIdx.x) * (NT / 32) + warp;
  Item cur;
  if (pi < P.count) fetch(pi, cur);
#pragma unroll 1
  for (; pi < P.count; pi += stride) {
    Item nxt;
    if (pi + stride < P.count) fetch(pi + stride, nxt);
    double u0, u1;
    patch_solve(ffs[cur.varx][lane], ffs[cur.vary][lane], sfs[cur.varx * 3 + cur.vary][lane], cur.b0, cur.b1, u0, u1);
    double* xp = P.x + cur.po;
    if (atomic) {
      if (r0) asm volatile("red.global.add.f64 [%0], %1;" ::"l"(xp), "d"(u0) : "memory");
      if (r1) asm volatile("red.global.add.f64 [%0], %1;" ::"l"(xp + 1), "d"(u1) : "memory");
    } else {
      if (r0) xp[0] += u0;
      if (r1) xp[1] += u1;
    }
    cur = nxt;
  }
}

template <int K>
static void launch_patch_fdm_mma(const FusedLevel& F, double omega, const double* r, double* x, const int32_t* list,
                                 int64_t count, int atomic, cudaStream_t st) {
  static int grid_cache = -1;
  if (grid_cache < 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, patch_fdm2d_mma_kernel<K>, 256, 0);
    grid_cache = sms * std::max(per, 1);
  }
  MvsP<double, K> p;
  std::memcpy(&p.c, F.c64.data(), sizeof(p.c));
  p.x = x; p.b = nullptr; p.list = list; p.count = count; p.N = F.N; p.n = F.n;
  p.scale = 1.0 / (F.h * F.h);
  p.factor = omega * F.h * F.h;
  p.zero = 0;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid_cache, (count + 7) / 8));
  patch_fdm2d_mma_kernel<K><<<grid, 256, 0, st>>>(p, r, atomic);
}

bool mma_patch_fdm2d(const FusedLevel& F, double omega, const double* r, double* x, const int32_t* list,
                     int64_t count, int atomic, cudaStream_t st) {
  if (!mma_enabled() || F.d != 2 || count <= 0) return false;
  switch (F.k) {
    case 2: launch_patch_fdm_mma<2>(F, omega, r, x, list, count, atomic, st); return true;
    case 3: launch_patch_fdm_mma<3>(F, omega, r, x, list, count, atomic, st); return true;
    case 4: launch_patch_fdm_mma<4>(F, omega, r, x, list, count, atomic, st); return true;
    default: return false;
  }
}

bool mma_enabled() {
  static const bool on = (std::getenv("C0IP_NO_MMA") == nullptr);
  return on;
}

bool mma_fdm2d(const FusedLevel& F, double omega, const double* r, double* x, const SlabWindow& w, cudaStream_t st) {
  if (!mma_enabled() || F.d != 2) return false;
  // k = 4 only: at k = 3 the 5 -> 8 padding makes the DMMA solve slower than fdm2d_kernel (measured
  // 0.43 vs 0.28 ms at 16.7M DoFs)
  switch (F.k) {
    case 4: launch_fdm_mma<4>(F, omega, r, x, w, st); return true;
    default: return false;
  }
}

}  // namespace c0ip
