// C ABI implementation: context, setup upload, operator / smoother / transfer dispatch,
// V-cycle (Algorithm 1) and MG-preconditioned CG.  See include/c0ip.h for the contract.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <new>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/c0ip.h"
#include "generic_kernels.cuh"
#include "fused_dispatch.hpp"
#include "host_setup.hpp"
#include "exact_local.hpp"

namespace {
thread_local std::string g_err;

c0ip_status fail(c0ip_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

struct CudaError {
  cudaError_t e;
  const char* where;
};

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) throw CudaError{e_, #call};                                   \
  } while (0)

template <typename T>
struct DevArr {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    if (p && n >= count) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (count == 0) return;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      throw CudaError{e, "cudaMalloc"};
    }
    n = count;
  }
  void upload(const std::vector<T>& h) {
    alloc(h.size());
    if (!h.empty()) CK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

template <typename T>
std::vector<T> cast_vec(const std::vector<double>& v) {
  return std::vector<T>(v.begin(), v.end());
}

template <typename T>
struct Tables {
  DevArr<T> M, L, B;                  // square bands (scaled to h), n x (4k+1)
  DevArr<T> E, Et;                    // transfer bands (this level = fine)
  DevArr<T> S[4], lam[4];
  DevArr<T> Ma[3], La[3], Ba[3], Ea[3], Eta[3], Sv[3], lamv[3];   // graded levels: per-axis tables (f4)
  // per-dtype workspaces
  DevArr<T> tmp[6];
  DevArr<T> sres;                     // smoother residual
  DevArr<T> vx, vb, vr;               // V-cycle vectors
};

struct WinLists {                     // slab: patches whose DoF rows meet the owned node rows, per colour
  std::vector<std::vector<int32_t>> h;
  std::vector<DevArr<int32_t>> dev;
  ~WinLists() { for (auto& a : dev) a.free(); }
};

struct ExactDev {                     // exact local solvers of one level
  c0ip::ExactHost host;
  std::vector<DevArr<double>> inv64;
  std::vector<DevArr<float>> inv32;
  DevArr<int64_t> off;
  std::vector<DevArr<int32_t>> all;                 // per tuple
  std::vector<std::vector<DevArr<int32_t>>> by_color;   // [colour][tuple]
  ~ExactDev() {
    for (auto& a : inv64) a.free();
    for (auto& a : inv32) a.free();
    off.free();
    for (auto& a : all) a.free();
    for (auto& c : by_color)
      for (auto& a : c) a.free();
  }
};

struct Level {
  int l = 0;
  int64_t N = 0, n = 0, ndofs = 0, npatch = 0;
  double h = 0;
  c0ip::Band M, L, B;                 // host, scaled to h
  c0ip::Fdm fdm;                      // host, scaled
  c0ip::RectBand E, Et;               // transfer from level l-1 (host)
  DevArr<int64_t> Elo, Etlo;
  Tables<double> t64;
  Tables<float> t32;
  std::vector<int32_t> colors_h;      // concatenated colour lists
  std::vector<int64_t> color_off;     // n_colors + 1
  std::vector<int32_t> parity_h;      // concatenated parity-class lists (2^d)
  std::vector<int64_t> parity_off;
  DevArr<int32_t> colors_d, parity_d;
  std::unique_ptr<c0ip::FusedLevel, c0ip::FusedLevelDeleter> fused;
  std::unique_ptr<ExactDev> exact;    // built on first use of the exact local solver
  bool sipg = false;                  // Poisson SIPG level: DG numbering, A = L (x) M + M (x) L
  // graded / anisotropic Cartesian meshes: per-axis cell boundaries, bands, transfers
  bool graded = false;
  std::vector<double> nodes[3];
  c0ip::Band Ma[3], La[3], Ba[3];
  c0ip::RectBand Ea[3], Eta[3];
  DevArr<int64_t> Ealo[3], Etalo[3];
};

}  // namespace

struct c0ip_ctx_s {
  c0ip_config cfg{};
  int d = 2, k = 2;
  double sigma = 0;
  int lmin = 1, lmax = 1;
  c0ip_path path = C0IP_PATH_AUTO;
  c0ip_local_solver local = C0IP_LOCAL_FDM;
  bool graded = false;
  std::vector<double> nodes[3];                    // finest-level cell boundaries per axis (graded meshes)
  bool sipg = false;                               // Poisson SIPG comparison workload
  std::map<std::tuple<int, int64_t, int64_t>, std::unique_ptr<WinLists>> wins;   // slab MVS patch lists
  c0ip::RefData ref;
  std::vector<Level> levels;          // index = level number (entries < lmin unused)
  int64_t launches = 0;
  DevArr<double> pcg_r, pcg_z, pcg_p, pcg_Ap, dot_part, dot_out;
  DevArr<double> gm_V, gm_Z, gm_w, gm_h;           // GMRES: Krylov basis, preconditioned basis, work, projections
  const double* vc_r = nullptr;                    // buffers the captured V-cycle graph reads / writes
  double* vc_z = nullptr;
  double* dot_host = nullptr;
  // captured V-cycle (CUDA graph) for the PCG loop: key = mg config; replayed on the caller's stream
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t vc_exec = nullptr;
  c0ip_mg_config vc_key{};
  int64_t vc_nodes = 0;
  ~c0ip_ctx_s() {
    if (vc_exec) cudaGraphExecDestroy(vc_exec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (auto& L : levels) {
      for (auto* t : {&L.t64.M, &L.t64.L, &L.t64.B, &L.t64.E, &L.t64.Et, &L.t64.sres, &L.t64.vx,
                      &L.t64.vb, &L.t64.vr})
        t->free();
      for (auto* t : {&L.t32.M, &L.t32.L, &L.t32.B, &L.t32.E, &L.t32.Et, &L.t32.sres, &L.t32.vx,
                      &L.t32.vb, &L.t32.vr})
        t->free();
      for (int i = 0; i < 6; ++i) { L.t64.tmp[i].free(); L.t32.tmp[i].free(); }
      for (int i = 0; i < 4; ++i) { L.t64.S[i].free(); L.t64.lam[i].free(); L.t32.S[i].free(); L.t32.lam[i].free(); }
      for (int a = 0; a < 3; ++a) {
        for (auto* t : {&L.t64.Ma[a], &L.t64.La[a], &L.t64.Ba[a], &L.t64.Ea[a], &L.t64.Eta[a], &L.t64.Sv[a],
                        &L.t64.lamv[a]}) t->free();
        for (auto* t : {&L.t32.Ma[a], &L.t32.La[a], &L.t32.Ba[a], &L.t32.Ea[a], &L.t32.Eta[a], &L.t32.Sv[a],
                        &L.t32.lamv[a]}) t->free();
        L.Ealo[a].free(); L.Etalo[a].free();
      }
      L.Elo.free(); L.Etlo.free(); L.colors_d.free(); L.parity_d.free();
      L.fused.reset();
      L.exact.reset();
    }
    pcg_r.free(); pcg_z.free(); pcg_p.free(); pcg_Ap.free(); dot_part.free(); dot_out.free();
    gm_V.free(); gm_Z.free(); gm_w.free(); gm_h.free();
    if (dot_host) cudaFreeHost(dot_host);
  }
};

namespace {

int ipow(int b, int e) {
  int r = 1;
  while (e--) r *= b;
  return r;
}

int color_of(const int64_t* v, int d) {
  // reading C3: 2 * parity class + red-black key
  int parity = 0;
  int64_t rb = 0;
  for (int a = 0; a < d; ++a) {
    parity |= int(v[a] % 2) << a;
    rb += v[a] / 2;
  }
  return 2 * parity + int(rb % 2);
}

template <typename T>
Tables<T>& tab(Level& L);
template <>
Tables<double>& tab<double>(Level& L) { return L.t64; }
template <>
Tables<float>& tab<float>(Level& L) { return L.t32; }

dim3 grid_for(int64_t total, int block = 256) {
  int64_t g = (total + block - 1) / block;
  g = std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
  return dim3((unsigned)g);
}

template <typename T>
c0ip::LineOp<T> square_op(const DevArr<T>& band, int k, int64_t n) {
  c0ip::LineOp<T> op;
  op.v = band.p;
  op.lo = nullptr;
  op.width = 4 * k + 1;
  op.hw = 2 * k;
  op.n_in = n;
  return op;
}

template <typename T>
void launch_axis(c0ip_ctx ctx, const c0ip::AxisArgs<T>& a, cudaStream_t st) {
  int64_t total = a.dims[0] * a.dims[1] * a.dims[2];
  if (a.sax >= 0) {
    if (a.scnt <= 0) return;
    total = total / a.dims[a.sax] * a.scnt;
  }
  c0ip::axis_apply_kernel<T><<<grid_for(total), 256, 0, st>>>(a);
  ctx->launches++;
  CK(cudaGetLastError());
}

template <typename T>
c0ip::AxisArgs<T> axis_args(int64_t n0, int64_t n1, int64_t n2, int axis, T* out) {
  c0ip::AxisArgs<T> a{};
  a.dims[0] = n0; a.dims[1] = n1; a.dims[2] = n2;
  a.axis = axis;
  a.nterms = 0;
  a.z = nullptr;
  a.gamma = 0;
  a.beta = 0;
  a.out = out;
  a.sax = -1;
  a.s0 = 0;
  a.scnt = 0;
  return a;
}

template <typename T>
void add_term(c0ip::AxisArgs<T>& a, const T* in, c0ip::LineOp<T> op, T alpha) {
  a.in[a.nterms] = in;
  a.op[a.nterms] = op;
  a.alpha[a.nterms] = alpha;
  a.nterms++;
}

template <typename T>
void ensure_tmp(Level& L, int d) {
  Tables<T>& t = tab<T>(L);
  int need = (d == 2) ? 3 : 6;
  for (int i = 0; i < need; ++i) t.tmp[i].alloc(L.ndofs);
}

// y = A x, or r = b - A x if b != nullptr (sum factorisation; Eqs. c0iptensorvp(3D)).
// Rows: only the slow-axis interior rows [jlo, jhi) of y are written (default: all); x, b, y are indexed
// globally (a slab window passes pointers shifted by -row0 * row), the per-axis temporaries are full-size
// level arrays of which only the rows the last stage reads ([jlo - 2k, jhi + 2k)) are computed.
template <typename T>
c0ip::LineOp<T> band_op(const DevArr<T>& band, int hw, int64_t n) {
  c0ip::LineOp<T> op;
  op.v = band.p; op.lo = nullptr; op.width = 2 * hw + 1; op.hw = hw; op.n_in = n;
  return op;
}

// Poisson SIPG: A = M_y L_x + L_y M_x (2D), M_z M_y L_x + M_z L_y M_x + L_z M_y M_x (3D)
template <typename T>
void sipg_apply(c0ip_ctx ctx, Level& L, const T* x, const T* b, T* y, cudaStream_t st) {
  const int d = ctx->d, hw = 2 * ctx->k + 1;
  const int64_t n = L.n, n2 = (d == 3) ? n : 1;
  Tables<T>& t = tab<T>(L);
  ensure_tmp<T>(L, d);
  const auto Mo = band_op(t.M, hw, n), Lo = band_op(t.L, hw, n);
  auto a0 = axis_args<T>(n, n, n2, 0, t.tmp[0].p);            // L_x x
  add_term(a0, x, Lo, T(1));
  launch_axis(ctx, a0, st);
  auto a1 = axis_args<T>(n, n, n2, 0, t.tmp[1].p);            // M_x x
  add_term(a1, x, Mo, T(1));
  launch_axis(ctx, a1, st);
  const T sg = b ? T(-1) : T(1);
  if (d == 2) {
    auto a = axis_args<T>(n, n, 1, 1, y);
    add_term(a, (const T*)t.tmp[0].p, Mo, sg);
    add_term(a, (const T*)t.tmp[1].p, Lo, sg);
    if (b) { a.z = b; a.gamma = T(1); }
    launch_axis(ctx, a, st);
    return;
  }
  auto p = axis_args<T>(n, n, n, 1, t.tmp[2].p);             // P = M_y L_x x + L_y M_x x
  add_term(p, (const T*)t.tmp[0].p, Mo, T(1));
  add_term(p, (const T*)t.tmp[1].p, Lo, T(1));
  launch_axis(ctx, p, st);
  auto q = axis_args<T>(n, n, n, 1, t.tmp[3].p);             // Q = M_y M_x x
  add_term(q, (const T*)t.tmp[1].p, Mo, T(1));
  launch_axis(ctx, q, st);
  auto a = axis_args<T>(n, n, n, 2, y);                      // y = M_z P + L_z Q
  add_term(a, (const T*)t.tmp[2].p, Mo, sg);
  add_term(a, (const T*)t.tmp[3].p, Lo, sg);
  if (b) { a.z = b; a.gamma = T(1); }
  launch_axis(ctx, a, st);
}

template <typename T>
void generic_apply(c0ip_ctx ctx, Level& L, const T* x, const T* b, T* y, cudaStream_t st, int64_t jlo = 0,
                   int64_t jhi = -1) {
  const int d = ctx->d, k = ctx->k;
  const int64_t n = L.n;
  if (jhi < 0) jhi = n;
  if (jhi <= jlo) return;
  if (L.sipg) {
    if (jlo != 0 || jhi != n) throw std::runtime_error("SIPG levels have no windowed operator");
    sipg_apply<T>(ctx, L, x, b, y, st);
    return;
  }
  Tables<T>& t = tab<T>(L);
  ensure_tmp<T>(L, d);
  // per-axis operators (identical on uniform levels; graded levels have their own per axis)
  c0ip::LineOp<T> Mx[3], Lx[3], Bx[3];
  for (int a = 0; a < 3; ++a) {
    Mx[a] = square_op(L.graded ? t.Ma[a] : t.M, k, n);
    Lx[a] = square_op(L.graded ? t.La[a] : t.L, k, n);
    Bx[a] = square_op(L.graded ? t.Ba[a] : t.B, k, n);
  }
  const int64_t n2 = (d == 3) ? n : 1;
  const int sax = d - 1;                                         // slowest axis
  const int64_t tlo = std::max<int64_t>(0, jlo - 2 * k), thi = std::min<int64_t>(n, jhi + 2 * k);
  auto rows = [&](c0ip::AxisArgs<T>& a, int64_t lo, int64_t hi) { a.sax = sax; a.s0 = lo; a.scnt = hi - lo; };
  // x-stage: B_x x, L_x x, M_x x
  {
    const c0ip::LineOp<T>* ops[3] = {&Bx[0], &Lx[0], &Mx[0]};
    for (int i = 0; i < 3; ++i) {
      auto a = axis_args<T>(n, n, n2, 0, t.tmp[i].p);
      add_term(a, x, *ops[i], T(1));
      rows(a, tlo, thi);
      launch_axis(ctx, a, st);
    }
  }
  const T sg = b ? T(-1) : T(1);
  if (d == 2) {
    // y = M_y (B_x x) + 2 L_y (L_x x) + B_y (M_x x)
    auto a = axis_args<T>(n, n, 1, 1, y);
    add_term(a, (const T*)t.tmp[0].p, Mx[1], sg);
    add_term(a, (const T*)t.tmp[1].p, Lx[1], T(2) * sg);
    add_term(a, (const T*)t.tmp[2].p, Bx[1], sg);
    if (b) { a.z = b; a.gamma = T(1); }
    rows(a, jlo, jhi);
    launch_axis(ctx, a, st);
    return;
  }
  // y-stage: P = M_y B_x + B_y M_x + 2 L_y L_x ; Q = L_y M_x + M_y L_x ; R = M_y M_x
  {
    auto a = axis_args<T>(n, n, n, 1, t.tmp[3].p);
    add_term(a, (const T*)t.tmp[0].p, Mx[1], T(1));
    add_term(a, (const T*)t.tmp[2].p, Bx[1], T(1));
    add_term(a, (const T*)t.tmp[1].p, Lx[1], T(2));
    rows(a, tlo, thi);
    launch_axis(ctx, a, st);
    auto q = axis_args<T>(n, n, n, 1, t.tmp[4].p);
    add_term(q, (const T*)t.tmp[2].p, Lx[1], T(1));
    add_term(q, (const T*)t.tmp[1].p, Mx[1], T(1));
    rows(q, tlo, thi);
    launch_axis(ctx, q, st);
    auto r = axis_args<T>(n, n, n, 1, t.tmp[5].p);
    add_term(r, (const T*)t.tmp[2].p, Mx[1], T(1));
    rows(r, tlo, thi);
    launch_axis(ctx, r, st);
  }
  // z-stage: y = M_z P + 2 L_z Q + B_z R
  auto a = axis_args<T>(n, n, n, 2, y);
  add_term(a, (const T*)t.tmp[3].p, Mx[2], sg);
  add_term(a, (const T*)t.tmp[4].p, Lx[2], T(2) * sg);
  add_term(a, (const T*)t.tmp[5].p, Bx[2], sg);
  if (b) { a.z = b; a.gamma = T(1); }
  rows(a, jlo, jhi);
  launch_axis(ctx, a, st);
}

template <typename T>
void apply_op(c0ip_ctx ctx, Level& L, const T* x, const T* b, T* y, cudaStream_t st) {
  if (ctx->path == C0IP_PATH_AUTO && L.fused) {
    if (c0ip::fused_dim(*L.fused) == 2 && c0ip::fused_apply<T>(*L.fused, x, b, y, st, &ctx->launches)) return;
    if (c0ip::fused_dim(*L.fused) == 3 && c0ip::fused3_apply<T>(*L.fused, x, b, y, st, &ctx->launches)) return;
  }
  generic_apply<T>(ctx, L, x, b, y, st);
}

template <typename T>
void patch_solve(c0ip_ctx ctx, Level& L, const T* r, T* x, T omega, const int32_t* list,
                 int64_t count, int atomic, cudaStream_t st) {
  if (count == 0) return;
  Tables<T>& t = tab<T>(L);
  c0ip::PatchArgs<T> a{};
  a.d = ctx->d; a.k = ctx->k; a.np = L.sipg ? 2 * ctx->k + 2 : 2 * ctx->k - 1;
  a.pstride = L.sipg ? ctx->k + 1 : ctx->k;
  a.N = L.N; a.n = L.n;
  for (int v = 0; v < 4; ++v) { a.S[v] = t.S[v].p; a.lam[v] = t.lam[v].p; }
  for (int ax = 0; ax < 3; ++ax) {
    a.Sv[ax] = L.graded ? t.Sv[ax].p : nullptr;
    a.lamv[ax] = L.graded ? t.lamv[ax].p : nullptr;
  }
  a.r = r; a.x = x; a.omega = omega;
  a.list = list; a.count = count; a.atomic = atomic;
  const int nloc = ipow(a.np, a.d);
  const int block = 256;
  const int ppb = std::max(1, block / nloc);
  const size_t smem = 2 * size_t(ppb) * nloc * sizeof(T);
  if (smem > 48 * 1024)
    CK(cudaFuncSetAttribute(c0ip::patch_fdm_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t blocks = (count + ppb - 1) / ppb;
  c0ip::patch_fdm_kernel<T><<<(unsigned)blocks, block, smem, st>>>(a);
  ctx->launches++;
  CK(cudaGetLastError());
}

// 2D FP64: patch solves on the tensor cores (mma2d.cu)
template <typename T>
bool mma_patches(c0ip_ctx ctx, Level& L, const T* r, T* x, T omega, const int32_t* list, int64_t count, int atomic,
                 cudaStream_t st) {
  if constexpr (std::is_same<T, double>::value) {
    if (ctx->path == C0IP_PATH_AUTO && L.fused && c0ip::fused_dim(*L.fused) == 2 &&
        c0ip::mma_patch_fdm2d(*L.fused, omega, r, x, list, count, atomic, st)) {
      ctx->launches++;
      CK(cudaGetLastError());
      return true;
    }
  }
  return false;
}

// x += omega A~_v^{-1} R_v r over disjoint patches (tuned 3D kernel when available, else generic)
template <typename T>
void disjoint_patch_solve(c0ip_ctx ctx, Level& L, const T* r, T* x, T omega, const int32_t* list, int64_t count,
                          cudaStream_t st) {
  if (ctx->path == C0IP_PATH_AUTO && L.fused && c0ip::fused_dim(*L.fused) == 3 &&
      c0ip::fused3_patch_fdm<T>(*L.fused, omega, r, x, list, count, st, &ctx->launches))
    return;
  // 2D lists: patch_list2d, except FP64 k = 3, 4 where the DMMA patch solve is faster (at k = 2 the 3 -> 8
  // padding of the DMMA fragments makes it the slower one: MVS step 9.9 vs 7.8 GDoF/s measured)
  const bool fused2 = ctx->path == C0IP_PATH_AUTO && L.fused && c0ip::fused_dim(*L.fused) == 2;
  if (fused2 && ctx->k == 2 && c0ip::fused2_patch_list<T>(*L.fused, omega, r, x, list, count, st, &ctx->launches))
    return;
  if (mma_patches<T>(ctx, L, r, x, omega, list, count, 0, st)) return;
  if (fused2 && c0ip::fused2_patch_list<T>(*L.fused, omega, r, x, list, count, st, &ctx->launches))
    return;
  patch_solve<T>(ctx, L, r, x, omega, list, count, 0, st);
}

ExactDev& exact_tables(c0ip_ctx ctx, Level& L) {
  if (L.graded || L.sipg)
    throw std::runtime_error("the exact local solver needs a uniform C0IP level (variant-tuple tables)");
  if (!L.exact) {
    std::unique_ptr<ExactDev> e(new ExactDev());
    const int nc = 1 << (ctx->d + 1);
    std::vector<int32_t> col(L.npatch);
    for (int c = 0; c < nc; ++c)
      for (int64_t i = L.color_off[c]; i < L.color_off[c + 1]; ++i) col[L.colors_h[i]] = c;
    std::string err;
    if (!c0ip::build_exact_host(ctx->d, ctx->k, L.N, L.M, L.L, L.B, col, nc, e->host, err))
      throw std::runtime_error("coercivity: " + err);
    const size_t nt = e->host.tuples.size();
    e->inv64.resize(nt); e->inv32.resize(nt); e->all.resize(nt);
    for (size_t i = 0; i < nt; ++i) {
      e->inv64[i].upload(e->host.inv[i]);
      e->inv32[i].upload(cast_vec<float>(e->host.inv[i]));
      e->all[i].upload(e->host.all[i]);
    }
    e->by_color.resize(nc);
    for (int c = 0; c < nc; ++c) {
      e->by_color[c].resize(nt);
      for (size_t i = 0; i < nt; ++i) e->by_color[c][i].upload(e->host.by_color[c][i]);
    }
    e->off.upload(e->host.off);
    L.exact = std::move(e);
  }
  return *L.exact;
}

// x += omega sum_{v in lists} R_v^T A_v^{-1} R_v r with the exact local matrices (fused gather / DMMA GEMM /
// scatter-add per variant tuple, exact_local.cu)
template <typename T>
void exact_patch_solve(c0ip_ctx ctx, Level& L, const T* r, T* x, T omega, int color, cudaStream_t st) {
  ExactDev& e = exact_tables(ctx, L);
  for (size_t i = 0; i < e.host.tuples.size(); ++i) {
    const auto& lst = color < 0 ? e.all[i] : e.by_color[color][i];
    const int64_t cnt = color < 0 ? (int64_t)e.host.all[i].size() : (int64_t)e.host.by_color[color][i].size();
    if (cnt == 0) continue;
    c0ip::ExactArgs<T> a;
    if constexpr (std::is_same<T, double>::value) a.Ainv = e.inv64[i].p; else a.Ainv = e.inv32[i].p;
    a.nloc = e.host.nloc; a.off = e.off.p; a.list = lst.p; a.count = cnt;
    a.d = ctx->d; a.k = ctx->k; a.N = L.N; a.n = L.n; a.r = r; a.x = x; a.omega = omega;
    c0ip::launch_exact_patches<T>(a, st);
    ctx->launches++;
    CK(cudaGetLastError());
  }
}

template <typename T>
void smooth_impl(c0ip_ctx ctx, Level& L, c0ip_smoother sm, int steps, T omega, bool reverse,
                 const T* b, T* x, cudaStream_t st) {
  Tables<T>& t = tab<T>(L);
  t.sres.alloc(L.ndofs);
  const int d = ctx->d;
  if (ctx->local == C0IP_LOCAL_EXACT) {        // exact local solvers
    for (int s = 0; s < steps; ++s) {
      if (sm == C0IP_MVS) {
        const int nc = 1 << (d + 1);
        for (int ci = 0; ci < nc; ++ci) {
          const int c = reverse ? nc - 1 - ci : ci;
          if (L.color_off[c + 1] == L.color_off[c]) continue;
          apply_op<T>(ctx, L, x, b, t.sres.p, st);
          exact_patch_solve<T>(ctx, L, t.sres.p, x, omega, c, st);
        }
      } else {                                   // every AVS realisation: one residual, atomic scatter-add
        apply_op<T>(ctx, L, x, b, t.sres.p, st);
        exact_patch_solve<T>(ctx, L, t.sres.p, x, omega, -1, st);
      }
    }
    return;
  }
  for (int s = 0; s < steps; ++s) {
    if (sm == C0IP_MVS) {
      const int nc = 1 << (d + 1);
      for (int ci = 0; ci < nc; ++ci) {
        int c = reverse ? nc - 1 - ci : ci;
        int64_t cnt = L.color_off[c + 1] - L.color_off[c];
        if (cnt == 0) continue;
        if (ctx->path == C0IP_PATH_AUTO && L.fused &&
            c0ip::fused_mvs_color<T>(*L.fused, L.colors_d.p + L.color_off[c], cnt, omega, b, x, st,
                                     &ctx->launches))
          continue;
        if (ctx->path == C0IP_PATH_AUTO && L.fused && c0ip::fused_dim(*L.fused) == 3 &&
            c0ip::fused3_mvs_color<T>(*L.fused, L.colors_d.p + L.color_off[c], cnt, omega, b, x, st,
                                      &ctx->launches))
          continue;
        apply_op<T>(ctx, L, x, b, t.sres.p, st);                 // residual per colour
        disjoint_patch_solve<T>(ctx, L, t.sres.p, x, omega, L.colors_d.p + L.color_off[c], cnt, st);
      }
      continue;
    }
    if (sm == C0IP_AVS_DETERMINISTIC && ctx->path == C0IP_PATH_AUTO && L.fused &&
        c0ip::fused_avs<T>(*L.fused, omega, b, x, t.sres.p, st, &ctx->launches))
      continue;
    apply_op<T>(ctx, L, x, b, t.sres.p, st);                     // one residual per AVS step
    if (ctx->path == C0IP_PATH_AUTO && L.fused && c0ip::fused_dim(*L.fused) == 3 &&
        c0ip::fused3_fdm_window<T>(*L.fused, omega, t.sres.p, x, sm == C0IP_AVS_ATOMIC, st, &ctx->launches))
      continue;
    if (sm == C0IP_AVS_ATOMIC) {
      if (mma_patches<T>(ctx, L, t.sres.p, x, omega, nullptr, L.npatch, 1, st)) continue;
      patch_solve<T>(ctx, L, t.sres.p, x, omega, nullptr, L.npatch, 1, st);
    } else {   // coloured / deterministic generic: serialise writes over the 2^d parity classes
      for (int c = 0; c < (1 << d); ++c) {
        int64_t cnt = L.parity_off[c + 1] - L.parity_off[c];
        disjoint_patch_solve<T>(ctx, L, t.sres.p, x, omega, L.parity_d.p + L.parity_off[c], cnt, st);
      }
    }
  }
}

// transfer bands of the pass along `axis` (per axis on graded levels)
template <typename T>
c0ip::LineOp<T> e_op(Level& F, int axis) {
  Tables<T>& t = tab<T>(F);
  c0ip::LineOp<T> E;
  E.v = F.graded ? t.Ea[axis].p : t.E.p;
  E.lo = F.graded ? F.Ealo[axis].p : F.Elo.p;
  E.width = F.E.width; E.hw = 0; E.n_in = F.E.cols;
  return E;
}
template <typename T>
c0ip::LineOp<T> et_op(Level& F, int axis) {
  Tables<T>& t = tab<T>(F);
  c0ip::LineOp<T> Et;
  Et.v = F.graded ? t.Eta[axis].p : t.Et.p;
  Et.lo = F.graded ? F.Etalo[axis].p : F.Etlo.p;
  Et.width = F.Et.width; Et.hw = 0; Et.n_in = F.n;
  return Et;
}

// fine += P coarse  (P = E (x) E (x) E, natural embedding)
template <typename T>
void prolongate_add_impl(c0ip_ctx ctx, Level& F, const T* coarse, T* fine, cudaStream_t st) {
  if (ctx->path == C0IP_PATH_AUTO && ctx->d == 2 && !F.graded && !F.sipg &&
      c0ip::fused_transfer2d<T>(ctx->k, true, F.N / 2, coarse, fine, st, &ctx->launches))
    return;
  Tables<T>& t = tab<T>(F);
  ensure_tmp<T>(F, ctx->d);
  const int64_t nf = F.n, nc = F.E.cols;
  if (ctx->d == 2) {
    auto a = axis_args<T>(nf, nc, 1, 0, t.tmp[0].p);
    add_term(a, coarse, e_op<T>(F, 0), T(1));
    launch_axis(ctx, a, st);
    auto b = axis_args<T>(nf, nf, 1, 1, fine);
    add_term(b, (const T*)t.tmp[0].p, e_op<T>(F, 1), T(1));
    b.beta = T(1);
    launch_axis(ctx, b, st);
    return;
  }
  auto a = axis_args<T>(nf, nc, nc, 0, t.tmp[0].p);
  add_term(a, coarse, e_op<T>(F, 0), T(1));
  launch_axis(ctx, a, st);
  auto b = axis_args<T>(nf, nf, nc, 1, t.tmp[1].p);
  add_term(b, (const T*)t.tmp[0].p, e_op<T>(F, 1), T(1));
  launch_axis(ctx, b, st);
  auto c = axis_args<T>(nf, nf, nf, 2, fine);
  add_term(c, (const T*)t.tmp[1].p, e_op<T>(F, 2), T(1));
  c.beta = T(1);
  launch_axis(ctx, c, st);
}

// coarse = P^T fine (restriction = transpose of the embedding)
template <typename T>
void restrict_impl(c0ip_ctx ctx, Level& F, const T* fine, T* coarse, cudaStream_t st) {
  if (ctx->path == C0IP_PATH_AUTO && ctx->d == 2 && !F.graded && !F.sipg &&
      c0ip::fused_transfer2d<T>(ctx->k, false, F.N / 2, fine, coarse, st, &ctx->launches))
    return;
  Tables<T>& t = tab<T>(F);
  ensure_tmp<T>(F, ctx->d);
  const int64_t nf = F.n, nc = F.E.cols;
  if (ctx->d == 2) {
    auto a = axis_args<T>(nc, nf, 1, 0, t.tmp[0].p);
    add_term(a, fine, et_op<T>(F, 0), T(1));
    launch_axis(ctx, a, st);
    auto b = axis_args<T>(nc, nc, 1, 1, coarse);
    add_term(b, (const T*)t.tmp[0].p, et_op<T>(F, 1), T(1));
    launch_axis(ctx, b, st);
    return;
  }
  auto a = axis_args<T>(nc, nf, nf, 0, t.tmp[0].p);
  add_term(a, fine, et_op<T>(F, 0), T(1));
  launch_axis(ctx, a, st);
  auto b = axis_args<T>(nc, nc, nf, 1, t.tmp[1].p);
  add_term(b, (const T*)t.tmp[0].p, et_op<T>(F, 1), T(1));
  launch_axis(ctx, b, st);
  auto c = axis_args<T>(nc, nc, nc, 2, coarse);
  add_term(c, (const T*)t.tmp[1].p, et_op<T>(F, 2), T(1));
  launch_axis(ctx, c, st);
}

template <typename T>
void fill(c0ip_ctx ctx, T* p, int64_t n, T v, cudaStream_t st) {
  c0ip::fill_kernel<T><<<grid_for(n), 256, 0, st>>>(n, v, p);
  ctx->launches++;
  CK(cudaGetLastError());
}

template <typename T>
void axpby(c0ip_ctx ctx, int64_t n, T a, const T* x, T b, T* y, cudaStream_t st) {
  c0ip::axpby_kernel<T><<<grid_for(n), 256, 0, st>>>(n, a, x, b, y);
  ctx->launches++;
  CK(cudaGetLastError());
}

template <typename Tin, typename Tout>
void convert(c0ip_ctx ctx, int64_t n, const Tin* x, Tout* y, cudaStream_t st) {
  c0ip::convert_kernel<Tin, Tout><<<grid_for(n), 256, 0, st>>>(n, x, y);
  ctx->launches++;
  CK(cudaGetLastError());
}

// MG_l(x = 0, b): Algorithm 1; coarsest level: one smoothing step (reading Q12)
template <typename T>
void vcycle_rec(c0ip_ctx ctx, int l, const c0ip_mg_config& mg, T* x, const T* b, cudaStream_t st) {
  Level& L = ctx->levels[l];
  Tables<T>& t = tab<T>(L);
  fill<T>(ctx, x, L.ndofs, T(0), st);
  if (l == ctx->lmin) {
    smooth_impl<T>(ctx, L, mg.smoother, 1, (T)mg.omega, false, b, x, st);
    return;
  }
  smooth_impl<T>(ctx, L, mg.smoother, mg.steps, (T)mg.omega, false, b, x, st);
  t.vr.alloc(L.ndofs);
  apply_op<T>(ctx, L, x, b, t.vr.p, st);                    // r_l = b - A x
  Level& C = ctx->levels[l - 1];
  Tables<T>& tc = tab<T>(C);
  tc.vx.alloc(C.ndofs);
  tc.vb.alloc(C.ndofs);
  restrict_impl<T>(ctx, L, t.vr.p, tc.vb.p, st);
  vcycle_rec<T>(ctx, l - 1, mg, tc.vx.p, tc.vb.p, st);
  prolongate_add_impl<T>(ctx, L, tc.vx.p, x, st);
  smooth_impl<T>(ctx, L, mg.smoother, mg.steps, (T)mg.omega,
                 mg.symmetric && mg.smoother == C0IP_MVS, b, x, st);
}

void vcycle_top(c0ip_ctx ctx, const c0ip_mg_config& mg, const double* r, double* z, cudaStream_t st, int level = -1) {
  const int l = level < 0 ? ctx->lmax : level;
  Level& L = ctx->levels[l];
  if (mg.cycle_dtype == C0IP_F64) {
    vcycle_rec<double>(ctx, l, mg, z, r, st);
  } else {
    Tables<float>& t = L.t32;
    t.vx.alloc(L.ndofs);
    t.vb.alloc(L.ndofs);
    convert<double, float>(ctx, L.ndofs, r, t.vb.p, st);    // conversion at V-cycle entry
    vcycle_rec<float>(ctx, l, mg, t.vx.p, t.vb.p, st);
    convert<float, double>(ctx, L.ndofs, t.vx.p, z, st);
  }
}

// V-cycle on the PCG work vectors as a CUDA graph: the ~20 launches per level are captured once (on an
// internal stream, since the legacy stream cannot be captured) and replayed on the caller's stream.
bool same_mg(const c0ip_mg_config& a, const c0ip_mg_config& b) {
  return a.smoother == b.smoother && a.steps == b.steps && a.omega == b.omega && a.symmetric == b.symmetric &&
         a.cycle_dtype == b.cycle_dtype;
}

void vcycle_graph(c0ip_ctx ctx, const c0ip_mg_config& mg, const double* r, double* z, cudaStream_t st) {
  // the captured graph bakes in r and z: recapture if the config or the buffers change
  if (!ctx->vc_exec || !same_mg(ctx->vc_key, mg) || ctx->vc_r != r || ctx->vc_z != z) {
    ctx->vc_r = r;
    ctx->vc_z = z;
    if (ctx->vc_exec) { cudaGraphExecDestroy(ctx->vc_exec); ctx->vc_exec = nullptr; }
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    CK(cudaStreamSynchronize(st));
    if (ctx->local == C0IP_LOCAL_EXACT)           // tables uploaded before capture (no copies inside it)
      for (int l = ctx->lmin; l <= ctx->lmax; ++l) exact_tables(ctx, ctx->levels[l]);
    const int64_t l0 = ctx->launches;
    CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    try {
      vcycle_top(ctx, mg, r, z, ctx->cap_stream);
    } catch (...) {
      cudaGraph_t g;
      cudaStreamEndCapture(ctx->cap_stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraph_t g;
    CK(cudaStreamEndCapture(ctx->cap_stream, &g));
    cudaError_t e = cudaGraphInstantiate(&ctx->vc_exec, g, 0);
    cudaGraphDestroy(g);
    CK(e);
    ctx->vc_key = mg;
    ctx->vc_nodes = ctx->launches - l0;
    ctx->launches = l0;
  }
  CK(cudaGraphLaunch(ctx->vc_exec, st));
  ctx->launches += ctx->vc_nodes;
}

// dots[i] = <x_i, y_i>, i < nd, read back to host (synchronises the stream)
void dots(c0ip_ctx ctx, int64_t n, int nd, const double* x0, const double* y0, const double* x1,
          const double* y1, const double* x2, const double* y2, double* out, cudaStream_t st) {
  const int G = 296;
  ctx->dot_part.alloc(3 * G);
  ctx->dot_out.alloc(3);
  c0ip::dot_partial_kernel<<<G, 256, 0, st>>>(n, nd, x0, y0, x1 ? x1 : x0, y1 ? y1 : y0,
                                              x2 ? x2 : x0, y2 ? y2 : y0, ctx->dot_part.p);
  c0ip::dot_final_kernel<<<1, 256, 0, st>>>(G, ctx->dot_part.p, ctx->dot_out.p);
  ctx->launches += 2;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(ctx->dot_host, ctx->dot_out.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int i = 0; i < nd; ++i) out[i] = ctx->dot_host[i];
}

c0ip_status check_level(c0ip_ctx ctx, int32_t level) {
  if (!ctx) return fail(C0IP_ERR_ARG, "null context");
  if (level < ctx->lmin || level > ctx->lmax)
    return fail(C0IP_ERR_ARG, "level " + std::to_string(level) + " out of range [" +
                                  std::to_string(ctx->lmin) + "," + std::to_string(ctx->lmax) + "]");
  return C0IP_OK;
}

c0ip_status cuda_fail(const CudaError& e) {
  if (e.e == cudaErrorMemoryAllocation) return fail(C0IP_ERR_OOM, std::string("out of device memory in ") + e.where);
  return fail(C0IP_ERR_CUDA, std::string(cudaGetErrorString(e.e)) + " in " + e.where);
}

#define ABI_TRY try {
#define ABI_CATCH                                                                  \
  }                                                                                \
  catch (const CudaError& e) { return cuda_fail(e); }                              \
  catch (const std::bad_alloc&) { return fail(C0IP_ERR_OOM, "host allocation failed"); } \
  catch (const std::exception& e) { return fail(C0IP_ERR_STATE, e.what()); }

void build_level(c0ip_ctx ctx, int l, int64_t N) {
  Level& L = ctx->levels[l];
  const int k = ctx->k, d = ctx->d;
  L.l = l;
  L.N = N;
  L.sipg = ctx->sipg;
  L.n = ctx->sipg ? N * (k + 1) : k * N - 1;           // SIPG: N (k+1) discontinuous nodes per axis
  L.h = 1.0 / double(N);
  L.ndofs = 1;
  L.npatch = 1;
  for (int a = 0; a < d; ++a) { L.ndofs *= L.n; L.npatch *= (N - 1); }
  if (ctx->sipg) {
    // Poisson SIPG (reading Q30): DG mass and SIPG stiffness bands, exact FDM per variant
    c0ip::sipg_bands(ctx->ref, N, ctx->sigma, L.M, L.L);    // sigma_P = penalty_scale k (k+1) (reading Q30)
    L.B = L.L;
    if (!c0ip::band_is_spd(L.L))
      throw std::runtime_error("coercivity: 1D SIPG matrix is not positive definite (penalty too small)");
    std::string err;
    if (!c0ip::make_fdm_sipg(k, N, L.M, L.L, L.fdm, err)) throw std::runtime_error("coercivity: " + err);
  } else if (ctx->graded) {
    // graded / anisotropic Cartesian mesh: per-axis bands and per-vertex FDM factors, generic
    // per-axis kernels only (the fused tile kernels assume uniform coefficients)
    L.graded = true;
    const int64_t stride = (int64_t(1) << (ctx->lmax - l));
    std::string err;
    for (int a = 0; a < d; ++a) {
      L.nodes[a].clear();
      for (size_t i = 0; i < ctx->nodes[a].size(); i += size_t(stride)) L.nodes[a].push_back(ctx->nodes[a][i]);
      c0ip::global_bands_graded(ctx->ref, L.nodes[a], L.Ma[a], L.La[a], L.Ba[a]);
      if (!c0ip::band_is_spd(L.Ba[a]))
        throw std::runtime_error("coercivity: 1D C0IP matrix B is not positive definite (penalty too small)");
      std::vector<double> Sv, lv;
      if (!c0ip::make_fdm_vertices(k, N, L.Ma[a], L.La[a], L.Ba[a], Sv, lv, err))
        throw std::runtime_error("coercivity: " + err);
      for (auto* t : {&L.t64.Ma[a], &L.t64.La[a], &L.t64.Ba[a]}) (void)t;
      L.t64.Ma[a].upload(L.Ma[a].v); L.t64.La[a].upload(L.La[a].v); L.t64.Ba[a].upload(L.Ba[a].v);
      L.t32.Ma[a].upload(cast_vec<float>(L.Ma[a].v)); L.t32.La[a].upload(cast_vec<float>(L.La[a].v));
      L.t32.Ba[a].upload(cast_vec<float>(L.Ba[a].v));
      L.t64.Sv[a].upload(Sv); L.t64.lamv[a].upload(lv);
      L.t32.Sv[a].upload(cast_vec<float>(Sv)); L.t32.lamv[a].upload(cast_vec<float>(lv));
    }
    L.M = L.Ma[0]; L.L = L.La[0]; L.B = L.Ba[0];         // axis 0 (c0ip_get_matrices_1d)
  } else {
    c0ip::global_bands(ctx->ref, N, L.M, L.L, L.B);
    const double h = L.h;
    for (auto& v : L.M.v) v *= h;                       // M = h Mhat
    for (auto& v : L.L.v) v /= h;                       // L = Lhat / h
    for (auto& v : L.B.v) v /= h * h * h;               // B = Bhat / h^3
    if (!c0ip::band_is_spd(L.B))
      throw std::runtime_error("coercivity: 1D C0IP matrix B is not positive definite (penalty too small)");
    std::string err;
    if (!c0ip::make_fdm(ctx->ref, N, L.M, L.L, L.B, L.fdm, err)) throw std::runtime_error("coercivity: " + err);
  }
  L.t64.M.upload(L.M.v); L.t64.L.upload(L.L.v); L.t64.B.upload(L.B.v);
  L.t32.M.upload(cast_vec<float>(L.M.v)); L.t32.L.upload(cast_vec<float>(L.L.v)); L.t32.B.upload(cast_vec<float>(L.B.v));
  for (int v = 0; v < 4; ++v) {
    if (!L.fdm.present[v]) continue;
    L.t64.S[v].upload(L.fdm.S[v]); L.t64.lam[v].upload(L.fdm.lam[v]);
    L.t32.S[v].upload(cast_vec<float>(L.fdm.S[v])); L.t32.lam[v].upload(cast_vec<float>(L.fdm.lam[v]));
  }
  // colour and parity-class lists (reading C3)
  const int nc = 1 << (d + 1), npar = 1 << d;
  std::vector<std::vector<int32_t>> cl(nc), pl(npar);
  for (int64_t p = 0; p < L.npatch; ++p) {
    int64_t v[3] = {0, 0, 0}, q = p;
    for (int a = 0; a < d; ++a) { v[a] = 1 + q % (N - 1); q /= (N - 1); }
    int c = color_of(v, d);
    cl[c].push_back((int32_t)p);
    pl[c / 2].push_back((int32_t)p);
  }
  L.color_off.assign(nc + 1, 0);
  L.colors_h.clear();
  for (int c = 0; c < nc; ++c) {
    L.color_off[c + 1] = L.color_off[c] + (int64_t)cl[c].size();
    L.colors_h.insert(L.colors_h.end(), cl[c].begin(), cl[c].end());
  }
  L.parity_off.assign(npar + 1, 0);
  L.parity_h.clear();
  for (int c = 0; c < npar; ++c) {
    L.parity_off[c + 1] = L.parity_off[c] + (int64_t)pl[c].size();
    L.parity_h.insert(L.parity_h.end(), pl[c].begin(), pl[c].end());
  }
  L.colors_d.upload(L.colors_h);
  L.parity_d.upload(L.parity_h);
  if (!L.graded && !L.sipg) L.fused = c0ip::make_fused_level_impl(d, k, N, ctx->ref, L.fdm, L.h);
}

void build_transfer(c0ip_ctx ctx, int l) {
  Level& L = ctx->levels[l];
  if (L.graded) {                                      // per-axis embeddings of the nested graded meshes
    for (int a = 0; a < ctx->d; ++a) {
      L.Ea[a] = c0ip::embedding_graded(ctx->k, L.nodes[a]);
      L.Eta[a] = c0ip::transpose(L.Ea[a]);
      L.t64.Ea[a].upload(L.Ea[a].v); L.t32.Ea[a].upload(cast_vec<float>(L.Ea[a].v));
      L.t64.Eta[a].upload(L.Eta[a].v); L.t32.Eta[a].upload(cast_vec<float>(L.Eta[a].v));
      L.Ealo[a].upload(L.Ea[a].lo);
      L.Etalo[a].upload(L.Eta[a].lo);
    }
  }
  L.E = L.sipg ? c0ip::embedding_dg(ctx->k, ctx->levels[l - 1].N)
               : (L.graded ? L.Ea[0] : c0ip::embedding(ctx->k, ctx->levels[l - 1].N));
  L.Et = c0ip::transpose(L.E);
  L.t64.E.upload(L.E.v); L.t32.E.upload(cast_vec<float>(L.E.v));
  L.t64.Et.upload(L.Et.v); L.t32.Et.upload(cast_vec<float>(L.Et.v));
  L.Elo.upload(L.E.lo);
  L.Etlo.upload(L.Et.lo);
}

}  // namespace

// =============================================================================== ABI
extern "C" {

const char* c0ip_last_error(void) { return g_err.c_str(); }

static c0ip_status create_impl(const c0ip_config* cfg, const double* const* nodes, bool sipg, c0ip_ctx* out);

c0ip_status c0ip_create(const c0ip_config* cfg, c0ip_ctx* out) { return create_impl(cfg, nullptr, false, out); }

c0ip_status c0ip_create_sipg(const c0ip_config* cfg, c0ip_ctx* out) { return create_impl(cfg, nullptr, true, out); }

c0ip_status c0ip_create_graded(const c0ip_config* cfg, const double* const* nodes, c0ip_ctx* out) {
  if (!nodes) return fail(C0IP_ERR_ARG, "null nodes");
  return create_impl(cfg, nodes, false, out);
}

static c0ip_status create_impl(const c0ip_config* cfg, const double* const* nodes, bool sipg, c0ip_ctx* out) {
  if (!cfg || !out) return fail(C0IP_ERR_ARG, "null argument");
  if (cfg->dim != 2 && cfg->dim != 3) return fail(C0IP_ERR_ARG, "dim must be 2 or 3");
  if (cfg->degree < 2 || cfg->degree > 7) return fail(C0IP_ERR_ARG, "degree must be in [2,7]");
  if (cfg->finest_level < 1 || cfg->finest_level > 14) return fail(C0IP_ERR_ARG, "finest_level must be in [1,14]");
  if (cfg->cells_override < 0 || cfg->cells_override == 1) return fail(C0IP_ERR_ARG, "cells_override must be 0 or >= 2");
  if (cfg->penalty_scale < 0) return fail(C0IP_ERR_ARG, "penalty_scale must be >= 0");
  std::unique_ptr<c0ip_ctx_s> ctx(new (std::nothrow) c0ip_ctx_s());
  if (!ctx) return fail(C0IP_ERR_OOM, "host allocation failed");
  ABI_TRY
  CK(cudaSetDevice(cfg->device));
  ctx->cfg = *cfg;
  ctx->d = cfg->dim;
  ctx->k = cfg->degree;
  const double ps = cfg->penalty_scale > 0 ? cfg->penalty_scale : 1.0;
  ctx->sigma = ps * ctx->k * (ctx->k + 1);                    // reading Q4
  ctx->ref = c0ip::make_ref(ctx->k, ctx->sigma);
  ctx->lmax = cfg->finest_level;
  ctx->lmin = cfg->cells_override > 0 ? cfg->finest_level : 1;
  ctx->levels.resize(ctx->lmax + 1);
  ctx->sipg = sipg;
  if (nodes) {                                           // graded mesh: cell boundaries of the finest level
    const int64_t NL = cfg->cells_override > 0 ? cfg->cells_override : (int64_t(1) << cfg->finest_level);
    ctx->graded = true;
    for (int a = 0; a < ctx->d; ++a) {
      std::vector<double> X(NL + 1);
      for (int64_t i = 0; i <= NL; ++i) X[i] = nodes[a] ? nodes[a][i] : double(i) / double(NL);
      if (std::fabs(X[0]) > 1e-14 || std::fabs(X[NL] - 1.0) > 1e-14)
        return fail(C0IP_ERR_ARG, "graded nodes must start at 0 and end at 1");
      for (int64_t i = 0; i < NL; ++i)
        if (!(X[i + 1] > X[i])) return fail(C0IP_ERR_ARG, "graded nodes must be strictly increasing");
      ctx->nodes[a] = X;
    }
  }
  try {
    for (int l = ctx->lmin; l <= ctx->lmax; ++l)
      build_level(ctx.get(), l, cfg->cells_override > 0 ? cfg->cells_override : (int64_t(1) << l));
  } catch (const std::runtime_error& e) {
    std::string m = e.what();
    if (m.rfind("coercivity", 0) == 0) return fail(C0IP_ERR_COERCIVITY, m);
    throw;
  }
  for (int l = ctx->lmin + 1; l <= ctx->lmax; ++l) build_transfer(ctx.get(), l);
  CK(cudaMallocHost(&ctx->dot_host, 4 * sizeof(double)));
  *out = ctx.release();
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_destroy(c0ip_ctx ctx) {
  if (!ctx) return fail(C0IP_ERR_ARG, "null context");
  delete ctx;
  return C0IP_OK;
}

c0ip_status c0ip_set_path(c0ip_ctx ctx, c0ip_path path) {
  if (!ctx) return fail(C0IP_ERR_ARG, "null context");
  if (path != C0IP_PATH_AUTO && path != C0IP_PATH_GENERIC) return fail(C0IP_ERR_ARG, "bad path");
  if (path != ctx->path && ctx->vc_exec) {       // the cached V-cycle graph was captured on the old path
    cudaGraphExecDestroy(ctx->vc_exec);
    ctx->vc_exec = nullptr;
  }
  ctx->path = path;
  return C0IP_OK;
}

c0ip_status c0ip_set_local_solver(c0ip_ctx ctx, c0ip_local_solver solver) {
  if (!ctx) return fail(C0IP_ERR_ARG, "null context");
  if (solver != C0IP_LOCAL_FDM && solver != C0IP_LOCAL_EXACT) return fail(C0IP_ERR_ARG, "bad local solver");
  if (solver != ctx->local && ctx->vc_exec) {     // the cached V-cycle graph was captured with the old solver
    cudaGraphExecDestroy(ctx->vc_exec);
    ctx->vc_exec = nullptr;
  }
  ctx->local = solver;
  return C0IP_OK;
}

c0ip_status c0ip_level_info(c0ip_ctx ctx, int32_t level, int64_t* n_dofs, int64_t* n_1d,
                            int64_t* cells, int64_t* n_patches, int32_t* n_colors) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  Level& L = ctx->levels[level];
  if (n_dofs) *n_dofs = L.ndofs;
  if (n_1d) *n_1d = L.n;
  if (cells) *cells = L.N;
  if (n_patches) *n_patches = L.npatch;
  if (n_colors) *n_colors = 1 << (ctx->d + 1);
  return C0IP_OK;
}

c0ip_status c0ip_patch_dofs(c0ip_ctx ctx, int32_t level, int64_t patch, int64_t* out) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (!out) return fail(C0IP_ERR_ARG, "null output");
  Level& L = ctx->levels[level];
  if (patch < 0 || patch >= L.npatch) return fail(C0IP_ERR_ARG, "patch out of range");
  const int d = ctx->d, k = ctx->k, np = L.sipg ? 2 * k + 2 : 2 * k - 1, ps = L.sipg ? k + 1 : k;
  int64_t v[3] = {0, 0, 0}, q = patch;
  for (int a = 0; a < d; ++a) { v[a] = 1 + q % (L.N - 1); q /= (L.N - 1); }
  const int nloc = ipow(np, d);
  for (int l = 0; l < nloc; ++l) {
    int64_t g = 0, st = 1;
    int ll = l;
    for (int a = 0; a < d; ++a) {
      g += ((v[a] - 1) * ps + ll % np) * st;  // 1D range [(v-1)k, (v+1)k-2] (reading C2); SIPG [(v-1)(k+1), (v+1)(k+1))
      ll /= np;
      st *= L.n;
    }
    out[l] = g;
  }
  return C0IP_OK;
}

c0ip_status c0ip_color_patches(c0ip_ctx ctx, int32_t level, int32_t color, int64_t* out,
                               int64_t cap, int64_t* count) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (color < 0 || color >= (1 << (ctx->d + 1))) return fail(C0IP_ERR_ARG, "colour out of range");
  Level& L = ctx->levels[level];
  int64_t cnt = L.color_off[color + 1] - L.color_off[color];
  if (count) *count = cnt;
  if (out) {
    if (cap < cnt) return fail(C0IP_ERR_ARG, "capacity too small");
    for (int64_t i = 0; i < cnt; ++i) out[i] = L.colors_h[L.color_off[color] + i];
  }
  return C0IP_OK;
}

c0ip_status c0ip_get_fdm(c0ip_ctx ctx, int32_t level, int32_t variant, double* S, double* lambda) {
  if (ctx && ctx->graded) return fail(C0IP_ERR_STATE, "graded meshes have per-vertex FDM factors (no variants)");
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (variant < 0 || variant > 3) return fail(C0IP_ERR_ARG, "variant out of range");
  Level& L = ctx->levels[level];
  if (!L.fdm.present[variant]) return fail(C0IP_ERR_STATE, "variant not present on this level");
  if (S) std::memcpy(S, L.fdm.S[variant].data(), L.fdm.S[variant].size() * sizeof(double));
  if (lambda) std::memcpy(lambda, L.fdm.lam[variant].data(), L.fdm.lam[variant].size() * sizeof(double));
  return C0IP_OK;
}

c0ip_status c0ip_get_matrices_1d(c0ip_ctx ctx, int32_t level, double* M, double* Lm, double* B) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  Level& L = ctx->levels[level];
  if (L.n > 4096) return fail(C0IP_ERR_ARG, "n_1d too large for a dense export");
  const int64_t n = L.n;
  for (int which = 0; which < 3; ++which) {
    double* dst = which == 0 ? M : (which == 1 ? Lm : B);
    const c0ip::Band& src = which == 0 ? L.M : (which == 1 ? L.L : L.B);
    if (!dst) continue;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) dst[i * n + j] = src.at(i, j);
  }
  return C0IP_OK;
}

c0ip_status c0ip_rhs(c0ip_ctx ctx, int32_t level, double* b, void* stream) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (!b) return fail(C0IP_ERR_ARG, "null output");
  ABI_TRY
  Level& L = ctx->levels[level];
  cudaStream_t st = (cudaStream_t)stream;
  DevArr<double> tmp[3], tmpg[3];
  c0ip::LoadArgs la;
  for (int a = 0; a < 3; ++a) {
    const int aa = a < ctx->d ? a : 0;
    if (L.sipg) {                                   // -Delta u* = d pi^2 prod sin, u* = 0 on the boundary
      tmp[a].upload(c0ip::sine_load_1d_dg(ctx->k, L.N));
      tmpg[a].upload(std::vector<double>(L.n, 0.0));
    } else {
      tmp[a].upload(L.graded ? c0ip::sine_load_1d_graded(ctx->k, L.nodes[aa]) : c0ip::sine_load_1d(ctx->k, L.N));
      tmpg[a].upload(L.graded ? c0ip::boundary_normal_1d_graded(ctx->ref, L.nodes[aa])
                              : c0ip::boundary_normal_1d(ctx->ref, L.N));
    }
    la.f1[a] = tmp[a].p;
    la.g1[a] = tmpg[a].p;
  }
  const double c = L.sipg ? double(ctx->d) * M_PI * M_PI                // SIPG: f = d pi^2 prod sin
                          : double(ctx->d * ctx->d) * std::pow(M_PI, 4);   // f = d^2 pi^4 prod sin (Q1, Q8)
  const double cb = -M_PI;                                        // g = d_n u* = -pi prod_{b!=a} sin (Q8b)
  c0ip::outer_load_kernel<<<grid_for(L.ndofs), 256, 0, st>>>(ctx->d, L.n, la, c, cb, b);
  ctx->launches++;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  for (int a = 0; a < 3; ++a) { tmp[a].free(); tmpg[a].free(); }
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_apply(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, const void* x, void* y, void* stream) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (!x || !y) return fail(C0IP_ERR_ARG, "null vector");
  ABI_TRY
  Level& L = ctx->levels[level];
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == C0IP_F64) apply_op<double>(ctx, L, (const double*)x, nullptr, (double*)y, st);
  else if (dt == C0IP_F32) apply_op<float>(ctx, L, (const float*)x, nullptr, (float*)y, st);
  else return fail(C0IP_ERR_ARG, "bad dtype");
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_residual(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, const void* b, const void* x,
                          void* r, void* stream) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (!x || !b || !r) return fail(C0IP_ERR_ARG, "null vector");
  ABI_TRY
  Level& L = ctx->levels[level];
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == C0IP_F64) apply_op<double>(ctx, L, (const double*)x, (const double*)b, (double*)r, st);
  else if (dt == C0IP_F32) apply_op<float>(ctx, L, (const float*)x, (const float*)b, (float*)r, st);
  else return fail(C0IP_ERR_ARG, "bad dtype");
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_smooth(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, c0ip_smoother sm, int32_t steps,
                        double omega, int32_t reverse_colors, const void* b, void* x, void* stream) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (!x || !b) return fail(C0IP_ERR_ARG, "null vector");
  if (steps < 0) return fail(C0IP_ERR_ARG, "steps must be >= 0");
  if (sm < C0IP_AVS_ATOMIC || sm > C0IP_MVS) return fail(C0IP_ERR_ARG, "bad smoother");
  ABI_TRY
  Level& L = ctx->levels[level];
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == C0IP_F64)
    smooth_impl<double>(ctx, L, sm, steps, omega, reverse_colors != 0, (const double*)b, (double*)x, st);
  else if (dt == C0IP_F32)
    smooth_impl<float>(ctx, L, sm, steps, (float)omega, reverse_colors != 0, (const float*)b, (float*)x, st);
  else return fail(C0IP_ERR_ARG, "bad dtype");
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_restrict(c0ip_ctx ctx, int32_t fine_level, c0ip_dtype dt, const void* fine, void* coarse,
                          void* stream) {
  c0ip_status s = check_level(ctx, fine_level);
  if (s) return s;
  if (fine_level <= ctx->lmin) return fail(C0IP_ERR_ARG, "fine_level must be above the coarsest level");
  if (!fine || !coarse) return fail(C0IP_ERR_ARG, "null vector");
  ABI_TRY
  Level& L = ctx->levels[fine_level];
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == C0IP_F64) restrict_impl<double>(ctx, L, (const double*)fine, (double*)coarse, st);
  else if (dt == C0IP_F32) restrict_impl<float>(ctx, L, (const float*)fine, (float*)coarse, st);
  else return fail(C0IP_ERR_ARG, "bad dtype");
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_prolongate_add(c0ip_ctx ctx, int32_t fine_level, c0ip_dtype dt, const void* coarse,
                                void* fine, void* stream) {
  c0ip_status s = check_level(ctx, fine_level);
  if (s) return s;
  if (fine_level <= ctx->lmin) return fail(C0IP_ERR_ARG, "fine_level must be above the coarsest level");
  if (!fine || !coarse) return fail(C0IP_ERR_ARG, "null vector");
  ABI_TRY
  Level& L = ctx->levels[fine_level];
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == C0IP_F64) prolongate_add_impl<double>(ctx, L, (const double*)coarse, (double*)fine, st);
  else if (dt == C0IP_F32) prolongate_add_impl<float>(ctx, L, (const float*)coarse, (float*)fine, st);
  else return fail(C0IP_ERR_ARG, "bad dtype");
  return C0IP_OK;
  ABI_CATCH
}

static c0ip_status check_mg(c0ip_ctx ctx, const c0ip_mg_config* mg) {
  if (!ctx || !mg) return fail(C0IP_ERR_ARG, "null argument");
  if (ctx->lmin == ctx->lmax && ctx->cfg.cells_override > 0)
    return fail(C0IP_ERR_STATE, "multigrid needs the nested hierarchy (cells_override = 0)");
  if (mg->smoother < C0IP_AVS_ATOMIC || mg->smoother > C0IP_MVS) return fail(C0IP_ERR_ARG, "bad smoother");
  if (mg->steps < 1) return fail(C0IP_ERR_ARG, "steps must be >= 1");
  if (mg->cycle_dtype != C0IP_F64 && mg->cycle_dtype != C0IP_F32) return fail(C0IP_ERR_ARG, "bad cycle dtype");
  return C0IP_OK;
}

c0ip_status c0ip_vcycle(c0ip_ctx ctx, const c0ip_mg_config* mg, const double* r, double* z, void* stream) {
  c0ip_status s = check_mg(ctx, mg);
  if (s) return s;
  if (!r || !z) return fail(C0IP_ERR_ARG, "null vector");
  ABI_TRY
  vcycle_top(ctx, *mg, r, z, (cudaStream_t)stream);
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_pcg(c0ip_ctx ctx, const c0ip_mg_config* mg, const double* b, double* x, double rtol,
                     int32_t max_iter, c0ip_report* rep, double* res_history, void* stream) {
  c0ip_status s = check_mg(ctx, mg);
  if (s) return s;
  if (!b || !x) return fail(C0IP_ERR_ARG, "null vector");
  if (max_iter < 0 || !(rtol >= 0)) return fail(C0IP_ERR_ARG, "bad rtol / max_iter");
  ABI_TRY
  cudaStream_t st = (cudaStream_t)stream;
  auto t0 = std::chrono::steady_clock::now();
  Level& L = ctx->levels[ctx->lmax];
  const int64_t n = L.ndofs;
  ctx->pcg_r.alloc(n); ctx->pcg_z.alloc(n); ctx->pcg_p.alloc(n); ctx->pcg_Ap.alloc(n);
  double *r = ctx->pcg_r.p, *z = ctx->pcg_z.p, *p = ctx->pcg_p.p, *Ap = ctx->pcg_Ap.p;
  // Saad Alg. 9.1 (textbook PCG), x0 given (reading Q19: callers pass 0)
  apply_op<double>(ctx, L, x, b, r, st);                          // r = b - A x
  vcycle_top(ctx, *mg, r, z, st);                                 // z = MG(r)
  CK(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  double dd[3];
  dots(ctx, n, 2, r, z, r, r, nullptr, nullptr, dd, st);
  double rz = dd[0], r0 = std::sqrt(dd[1]), rn = r0;
  if (res_history) res_history[0] = r0;
  int it = 0;
  while (it < max_iter && rn > rtol * r0) {
    apply_op<double>(ctx, L, p, nullptr, Ap, st);
    dots(ctx, n, 1, p, Ap, nullptr, nullptr, nullptr, nullptr, dd, st);
    const double alpha = rz / dd[0];
    axpby<double>(ctx, n, alpha, p, 1.0, x, st);
    axpby<double>(ctx, n, -alpha, Ap, 1.0, r, st);
    ++it;
    dots(ctx, n, 1, r, r, nullptr, nullptr, nullptr, nullptr, dd, st);
    rn = std::sqrt(dd[0]);
    if (res_history) res_history[it] = rn;
    if (rn <= rtol * r0) break;
    vcycle_graph(ctx, *mg, r, z, st);
    dots(ctx, n, 1, r, z, nullptr, nullptr, nullptr, nullptr, dd, st);
    const double beta = dd[0] / rz;
    rz = dd[0];
    axpby<double>(ctx, n, 1.0, z, beta, p, st);                   // p = z + beta p
  }
  CK(cudaStreamSynchronize(st));
  auto t1 = std::chrono::steady_clock::now();
  if (rep) {
    rep->iterations = it;
    rep->converged = (rn <= rtol * r0) ? 1 : 0;
    rep->r0 = r0;
    rep->rn = rn;
    double ratio = (r0 > 0) ? rn / r0 : 0.0;
    rep->nu = (it == 0 || ratio <= 0) ? 0.0 : -8.0 / std::log10(std::pow(ratio, 1.0 / it));
    rep->seconds = std::chrono::duration<double>(t1 - t0).count();
  }
  return C0IP_OK;
  ABI_CATCH
}

// w -= V (V^T w) over the nv basis vectors V_0..V_{nv-1} (classical Gram-Schmidt pass): batched dots (8 vectors
// per pass over w), one host round trip, batched update (64 vectors per pass); hs = V^T w
static void project(c0ip_ctx ctx, int64_t n, int nv, double* w, const double* V, std::vector<double>& hs,
                    cudaStream_t st) {
  const int G = 296;
  ctx->dot_part.alloc(8 * G);
  ctx->gm_h.alloc(nv);
  for (int c0 = 0; c0 < nv; c0 += 8) {
    const int cnt = std::min(8, nv - c0);
    c0ip::mdot_partial_kernel<8><<<G, 256, 0, st>>>(n, cnt, w, V + size_t(c0) * n, ctx->dot_part.p);
    c0ip::mdot_final_kernel<<<cnt, 256, 0, st>>>(G, ctx->dot_part.p, ctx->gm_h.p + c0);
    ctx->launches += 2;
  }
  CK(cudaGetLastError());
  hs.assign(nv, 0.0);
  CK(cudaMemcpyAsync(hs.data(), ctx->gm_h.p, nv * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int c0 = 0; c0 < nv; c0 += 64) {
    const int cnt = std::min(64, nv - c0);
    c0ip::Coefs64 cf{};
    for (int c = 0; c < cnt; ++c) cf.c[c] = hs[c0 + c];
    c0ip::maxpy_kernel<<<grid_for(n), 256, 0, st>>>(n, cnt, cf, V + size_t(c0) * n, w);
    ctx->launches++;
  }
  CK(cudaGetLastError());
}

c0ip_status c0ip_gmres(c0ip_ctx ctx, const c0ip_mg_config* mg, const double* b, double* x, double rtol,
                       int32_t max_iter, int32_t restart, c0ip_report* rep, double* res_history, void* stream) {
  c0ip_status s = check_mg(ctx, mg);
  if (s) return s;
  if (!b || !x) return fail(C0IP_ERR_ARG, "null vector");
  if (max_iter < 0 || restart < 1 || !(rtol >= 0)) return fail(C0IP_ERR_ARG, "bad rtol / max_iter / restart");
  ABI_TRY
  cudaStream_t st = (cudaStream_t)stream;
  auto t0 = std::chrono::steady_clock::now();
  Level& L = ctx->levels[ctx->lmax];
  const int64_t n = L.ndofs;
  const int m = restart;          // workspace sized by restart (reused across calls: no allocation
                                  // inside a timed solve after the first call with this restart)
  // Flexible right-preconditioned GMRES(m) (Saad Alg. 9.6), classical Gram-Schmidt with one re-orthogonalisation
  // (CGS2: two batched projections and one norm per Arnoldi step = 3 host round trips), Givens rotations
  // (GMRES outer solver for the multiplicative smoother)
  ctx->gm_V.alloc(n * (m + 1));
  ctx->gm_Z.alloc(n * m);
  ctx->gm_w.alloc(n);
  ctx->pcg_r.alloc(n);
  ctx->pcg_z.alloc(n);
  double* V = ctx->gm_V.p;
  double* Z = ctx->gm_Z.p;
  double* w = ctx->gm_w.p;
  std::vector<double> H((m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
  auto h = [&](int i, int j) -> double& { return H[size_t(i) * m + j]; };
  double dd[3];
  auto residual_norm = [&]() {                       // V_0 = b - A x, returns ||V_0||
    apply_op<double>(ctx, L, x, b, V, st);
    dots(ctx, n, 1, V, V, nullptr, nullptr, nullptr, nullptr, dd, st);
    return std::sqrt(dd[0]);
  };
  double beta = residual_norm();
  const double r0 = beta;
  double rn = beta;
  if (res_history) res_history[0] = r0;
  int it = 0;
  // stopping test on the least-squares residual |g_{j+1}| (the recursively updated residual, as in
  // PCG): the true residual of a smooth solution is only known to ~eps || |A| |x| ||
  while (it < max_iter && rn > rtol * r0 && beta > 0) {
    const int mm = std::min(m, max_iter - it);
    axpby<double>(ctx, n, 0.0, b, 1.0 / beta, V, st);            // V_0 = r / beta
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int jd = 0;
    for (int j = 0; j < mm; ++j) {
      double* vj = V + size_t(j) * n;
      double* zj = Z + size_t(j) * n;
      // z_j = MG(v_j): the first application runs uncaptured (allocates the level workspaces), the
      // rest replay the captured V-cycle graph on the fixed staging buffers pcg_r -> pcg_z
      if (it == 0) {
        vcycle_top(ctx, *mg, vj, zj, st);
      } else {
        CK(cudaMemcpyAsync(ctx->pcg_r.p, vj, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        vcycle_graph(ctx, *mg, ctx->pcg_r.p, ctx->pcg_z.p, st);
        CK(cudaMemcpyAsync(zj, ctx->pcg_z.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      }
      apply_op<double>(ctx, L, zj, nullptr, w, st);              // w = A z_j
      for (int i = 0; i <= j; ++i) h(i, j) = 0.0;
      for (int pass = 0; pass < 2; ++pass) {                     // CGS2: two batched projection passes
        std::vector<double> hs;
        project(ctx, n, j + 1, w, V, hs, st);
        for (int i = 0; i <= j; ++i) h(i, j) += hs[i];
      }
      dots(ctx, n, 1, w, w, nullptr, nullptr, nullptr, nullptr, dd, st);
      h(j + 1, j) = std::sqrt(dd[0]);
      double* vn = V + size_t(j + 1) * n;
      CK(cudaMemcpyAsync(vn, w, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      if (h(j + 1, j) > 0) axpby<double>(ctx, n, 0.0, w, 1.0 / h(j + 1, j), vn, st);
      for (int i = 0; i < j; ++i) {                              // previous rotations
        const double t = cs[i] * h(i, j) + sn[i] * h(i + 1, j);
        h(i + 1, j) = -sn[i] * h(i, j) + cs[i] * h(i + 1, j);
        h(i, j) = t;
      }
      const double den = std::hypot(h(j, j), h(j + 1, j));
      cs[j] = h(j, j) / den;
      sn[j] = h(j + 1, j) / den;
      h(j, j) = den;
      h(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++it;
      jd = j + 1;
      rn = std::fabs(g[j + 1]);
      if (res_history) res_history[it] = rn;
      if (rn <= rtol * r0) break;
    }
    for (int i = jd - 1; i >= 0; --i) {                          // back substitution H y = g
      double t = g[i];
      for (int l = i + 1; l < jd; ++l) t -= h(i, l) * y[l];
      y[i] = t / h(i, i);
    }
    for (int i = 0; i < jd; ++i) axpby<double>(ctx, n, y[i], Z + size_t(i) * n, 1.0, x, st);
    beta = residual_norm();                                       // true residual of the restart / exit
  }
  CK(cudaStreamSynchronize(st));
  auto t1 = std::chrono::steady_clock::now();
  if (rep) {
    rep->iterations = it;
    rep->converged = (rn <= rtol * r0) ? 1 : 0;
    rep->r0 = r0;
    rep->rn = beta;                                               // true residual norm at exit
    const double ratio = (r0 > 0) ? rn / r0 : 0.0;
    rep->nu = (it == 0 || ratio <= 0) ? 0.0 : -8.0 / std::log10(std::pow(ratio, 1.0 / it));
    rep->seconds = std::chrono::duration<double>(t1 - t0).count();
  }
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_slab_ghosts(c0ip_ctx ctx, int32_t* ghost_avs, int32_t* ghost_apply) {
  if (!ctx) return fail(C0IP_ERR_ARG, "null context");
  if (ghost_avs) *ghost_avs = 4 * ctx->k - 2;
  if (ghost_apply) *ghost_apply = 2 * ctx->k;
  return C0IP_OK;
}

}  // extern "C"

template <typename T>
static void slab_apply_impl(c0ip_ctx ctx, Level& L, const T* x, const T* b, T* y, const c0ip::SlabWindow& w,
                            cudaStream_t st) {
  if (c0ip::fused_dim(*L.fused) == 3)
    c0ip::fused3_apply<T>(*L.fused, x, b, y, st, &ctx->launches, &w);
  else
    c0ip::fused_apply<T>(*L.fused, x, b, y, st, &ctx->launches, &w);
}

// r = b - A x on the rows the owned patches read (wr), then the owned rows of x += omega sum_v R_v^T u_v
// (2D: gather-form FDM, 3D: parity-class patch FDM restricted to the owned planes; both deterministic)
template <typename T>
static void slab_avs(c0ip_ctx ctx, Level& L, T omega, const c0ip::SlabWindow& wr, const c0ip::SlabWindow& wo,
                     const T* b, T* x, T* r, cudaStream_t st) {
  slab_apply_impl<T>(ctx, L, x, b, r, wr, st);
  if (c0ip::fused_dim(*L.fused) == 3)
    c0ip::fused3_fdm_window<T>(*L.fused, omega, r, x, false, st, &ctx->launches, &wo);
  else
    c0ip::fused_fdm<T>(*L.fused, omega, r, x, st, &ctx->launches, &wo);
}

extern "C" {

static c0ip_status check_window(c0ip_ctx ctx, Level& L, int64_t row0, int64_t lrows, int64_t out_lo,
                                int64_t out_hi, int64_t ghost) {
  const int64_t KN = int64_t(ctx->k) * L.N;
  if (row0 < 0 || lrows < 1 || row0 + lrows > L.n) return fail(C0IP_ERR_ARG, "slab window outside the level");
  if (out_lo < 1 || out_hi > KN || out_lo > out_hi) return fail(C0IP_ERR_ARG, "owned rows outside the level");
  const int64_t need_lo = std::max<int64_t>(1, out_lo - ghost), need_hi = std::min<int64_t>(KN - 1, out_hi - 1 + ghost);
  if (row0 + 1 > need_lo || row0 + lrows < need_hi)
    return fail(C0IP_ERR_ARG, "slab window lacks ghost rows (need node rows [" + std::to_string(need_lo) + ", " +
                                  std::to_string(need_hi) + "])");
  if (!L.fused || !c0ip::fused_supports_slab(*L.fused))
    return fail(C0IP_ERR_STATE, "slab calls need a fused level (2D: N >= 8, k <= 7; 3D: N >= 8, k <= 5)");
  return C0IP_OK;
}

c0ip_status c0ip_slab_avs_step(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, double omega, int64_t row0,
                               int64_t lrows, int64_t out_lo, int64_t out_hi, const void* b_ext, void* x_ext,
                               void* r_ext, void* stream) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (!b_ext || !x_ext || !r_ext) return fail(C0IP_ERR_ARG, "null vector");
  Level& L = ctx->levels[level];
  if ((s = check_window(ctx, L, row0, lrows, out_lo, out_hi, 4 * ctx->k - 2))) return s;
  ABI_TRY
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t KN = int64_t(ctx->k) * L.N, gr = 2 * ctx->k - 2;
  c0ip::SlabWindow wr{row0, lrows, std::max<int64_t>(1, out_lo - gr), std::min<int64_t>(KN, out_hi + gr)};
  c0ip::SlabWindow wo{row0, lrows, out_lo, out_hi};
  if (dt != C0IP_F64 && dt != C0IP_F32) return fail(C0IP_ERR_ARG, "bad dtype");
  if (dt == C0IP_F64)
    slab_avs<double>(ctx, L, omega, wr, wo, (const double*)b_ext, (double*)x_ext, (double*)r_ext, st);
  else
    slab_avs<float>(ctx, L, (float)omega, wr, wo, (const float*)b_ext, (float*)x_ext, (float*)r_ext, st);
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_slab_fdm(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, double omega, int64_t row0, int64_t lrows,
                          int64_t out_lo, int64_t out_hi, const void* r_ext, void* x_ext, void* stream) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (!r_ext || !x_ext) return fail(C0IP_ERR_ARG, "null vector");
  Level& L = ctx->levels[level];
  if ((s = check_window(ctx, L, row0, lrows, out_lo, out_hi, 2 * ctx->k - 2))) return s;
  ABI_TRY
  cudaStream_t st = (cudaStream_t)stream;
  c0ip::SlabWindow wo{row0, lrows, out_lo, out_hi};
  const bool three = c0ip::fused_dim(*L.fused) == 3;
  if (dt == C0IP_F64) {
    if (three) c0ip::fused3_fdm_window<double>(*L.fused, omega, (const double*)r_ext, (double*)x_ext, false, st,
                                               &ctx->launches, &wo);
    else c0ip::fused_fdm<double>(*L.fused, omega, (const double*)r_ext, (double*)x_ext, st, &ctx->launches, &wo);
  } else if (dt == C0IP_F32) {
    if (three) c0ip::fused3_fdm_window<float>(*L.fused, (float)omega, (const float*)r_ext, (float*)x_ext, false, st,
                                              &ctx->launches, &wo);
    else c0ip::fused_fdm<float>(*L.fused, (float)omega, (const float*)r_ext, (float*)x_ext, st, &ctx->launches, &wo);
  } else {
    return fail(C0IP_ERR_ARG, "bad dtype");
  }
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_slab_apply(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, int64_t row0, int64_t lrows, int64_t out_lo,
                            int64_t out_hi, const void* b_ext, const void* x_ext, void* y_ext, void* stream) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (!x_ext || !y_ext) return fail(C0IP_ERR_ARG, "null vector");
  Level& L = ctx->levels[level];
  if ((s = check_window(ctx, L, row0, lrows, out_lo, out_hi, 2 * ctx->k))) return s;
  ABI_TRY
  cudaStream_t st = (cudaStream_t)stream;
  c0ip::SlabWindow w{row0, lrows, out_lo, out_hi};
  if (dt == C0IP_F64)
    slab_apply_impl<double>(ctx, L, (const double*)x_ext, (const double*)b_ext, (double*)y_ext, w, st);
  else if (dt == C0IP_F32)
    slab_apply_impl<float>(ctx, L, (const float*)x_ext, (const float*)b_ext, (float*)y_ext, w, st);
  else
    return fail(C0IP_ERR_ARG, "bad dtype");
  return C0IP_OK;
  ABI_CATCH
}

}  // extern "C"

// ------------------------------------------------------------------------------------- slab extension
// Colour-lockstep MVS, windowed transfers and the V-cycle from an inner level: the pieces of the
// distributed V-cycle / Krylov solvers (paper_2412_05082_b200/dist.py drives them).
// Window convention as above: x_ext[(j - 1 - row0) * row + ...] holds node row j of the slow axis.  Kernels
// that index the level globally get "virtual" pointers x_ext - row0 * row; they only touch rows inside the
// window (checked by the callers' ghost widths).
namespace {

int64_t slow_row_len(const c0ip_ctx ctx, const Level& L) { return ctx->d == 2 ? L.n : L.n * L.n; }

std::map<std::tuple<int, int64_t, int64_t>, std::unique_ptr<WinLists>>& win_cache(c0ip_ctx ctx) {
  return ctx->wins;
}

WinLists& win_lists(c0ip_ctx ctx, Level& L, int64_t out_lo, int64_t out_hi) {
  auto key = std::make_tuple(L.l, out_lo, out_hi);
  auto& cache = win_cache(ctx);
  auto it = cache.find(key);
  if (it != cache.end()) return *it->second;
  std::unique_ptr<WinLists> w(new WinLists());
  const int nc = 1 << (ctx->d + 1), k = ctx->k;
  w->h.assign(nc, {});
  int64_t stride = 1;
  for (int a = 0; a < ctx->d - 1; ++a) stride *= (L.N - 1);
  for (int c = 0; c < nc; ++c)
    for (int64_t i = L.color_off[c]; i < L.color_off[c + 1]; ++i) {
      const int32_t p = L.colors_h[i];
      const int64_t vs = 1 + p / stride;                       // slow-axis vertex of the patch
      if ((vs + 1) * k - 1 >= out_lo && (vs - 1) * k + 1 <= out_hi - 1) w->h[c].push_back(p);
    }
  w->dev.resize(nc);
  for (int c = 0; c < nc; ++c) w->dev[c].upload(w->h[c]);
  WinLists& ref = *w;
  cache[key] = std::move(w);
  return ref;
}

// one MVS colour on a slab: residual on the colour's patches (footprint), FDM solve, update of their DoFs
// (owned rows +- (k-1); rows outside the owned range are ghost copies refreshed by the next exchange)
template <typename T>
void slab_mvs_color_impl(c0ip_ctx ctx, Level& L, int color, T omega, int64_t row0, int64_t lrows, int64_t out_lo,
                         int64_t out_hi, const T* b_ext, T* x_ext, T* r_ext, cudaStream_t st) {
  WinLists& wl = win_lists(ctx, L, out_lo, out_hi);
  const int64_t cnt = (int64_t)wl.h[color].size();
  if (cnt == 0) return;
  const int32_t* list = wl.dev[color].p;
  const int64_t row = slow_row_len(ctx, L);
  const T* bv = b_ext - row0 * row;
  T* xv = x_ext - row0 * row;
  T* rv = r_ext - row0 * row;
  const int k = ctx->k;
  if (ctx->path == C0IP_PATH_AUTO && L.fused && c0ip::fused_dim(*L.fused) == 2 &&
      c0ip::fused_mvs_color<T>(*L.fused, list, cnt, omega, bv, xv, st, &ctx->launches))
    return;
  if (ctx->path == C0IP_PATH_AUTO && L.fused && c0ip::fused_dim(*L.fused) == 3 &&
      c0ip::fused3_mvs_color<T>(*L.fused, list, cnt, omega, bv, xv, st, &ctx->launches))
    return;
  // residual on the patch DoF rows: node rows [out_lo - (k-1), out_hi + k - 1] (the slab cuts are vertex rows);
  // the same kernel as the single-domain step (fused apply3d on the window, else the generic per-axis kernels)
  const int64_t KN = int64_t(k) * L.N;
  const c0ip::SlabWindow wr{row0, lrows, std::max<int64_t>(1, out_lo - (k - 1)), std::min<int64_t>(KN, out_hi + k)};
  const bool fused = ctx->path == C0IP_PATH_AUTO && L.fused;
  if (!(fused && c0ip::fused_dim(*L.fused) == 3 &&
        c0ip::fused3_apply<T>(*L.fused, x_ext, b_ext, r_ext, st, &ctx->launches, &wr)) &&
      !(fused && c0ip::fused_dim(*L.fused) == 2 &&
        c0ip::fused_apply<T>(*L.fused, x_ext, b_ext, r_ext, st, &ctx->launches, &wr)))
    generic_apply<T>(ctx, L, xv, bv, rv, st, wr.out_lo - 1, wr.out_hi - 1);
  if (ctx->local == C0IP_LOCAL_EXACT) throw std::runtime_error("slab MVS with exact local solvers is not supported");
  // the patch-solve kernel of the single-domain colour step, so the owned rows stay bitwise equal
  disjoint_patch_solve<T>(ctx, L, rv, xv, omega, list, cnt, st);
}

// coarse node rows [c_out_lo, c_out_hi) of P^T fine (restriction) from a fine window
template <typename T>
void slab_restrict_impl(c0ip_ctx ctx, Level& F, const T* fv, T* cv, int64_t ic_lo, int64_t ic_hi, cudaStream_t st) {
  Tables<T>& t = tab<T>(F);
  ensure_tmp<T>(F, ctx->d);
  const int64_t nf = F.n, nc = F.E.cols;
  const int width = F.Et.width;
  const int64_t fr_lo = F.Et.lo[ic_lo], fr_hi = F.Et.lo[ic_hi - 1] + width;
  if (ctx->d == 2) {
    auto a = axis_args<T>(nc, nf, 1, 0, t.tmp[0].p);
    add_term(a, fv, et_op<T>(F, 0), T(1));
    a.sax = 1; a.s0 = fr_lo; a.scnt = fr_hi - fr_lo;
    launch_axis(ctx, a, st);
    auto b = axis_args<T>(nc, nc, 1, 1, cv);
    add_term(b, (const T*)t.tmp[0].p, et_op<T>(F, 1), T(1));
    b.sax = 1; b.s0 = ic_lo; b.scnt = ic_hi - ic_lo;
    launch_axis(ctx, b, st);
    return;
  }
  auto a = axis_args<T>(nc, nf, nf, 0, t.tmp[0].p);
  add_term(a, fv, et_op<T>(F, 0), T(1));
  a.sax = 2; a.s0 = fr_lo; a.scnt = fr_hi - fr_lo;
  launch_axis(ctx, a, st);
  auto b = axis_args<T>(nc, nc, nf, 1, t.tmp[1].p);
  add_term(b, (const T*)t.tmp[0].p, et_op<T>(F, 1), T(1));
  b.sax = 2; b.s0 = fr_lo; b.scnt = fr_hi - fr_lo;
  launch_axis(ctx, b, st);
  auto c = axis_args<T>(nc, nc, nc, 2, cv);
  add_term(c, (const T*)t.tmp[1].p, et_op<T>(F, 2), T(1));
  c.sax = 2; c.s0 = ic_lo; c.scnt = ic_hi - ic_lo;
  launch_axis(ctx, c, st);
}

// fine interior rows [if_lo, if_hi) += (P coarse) (prolongation = embedding)
template <typename T>
void slab_prolongate_impl(c0ip_ctx ctx, Level& F, const T* cv, T* fv, int64_t if_lo, int64_t if_hi, cudaStream_t st) {
  Tables<T>& t = tab<T>(F);
  ensure_tmp<T>(F, ctx->d);
  const int64_t nf = F.n, nc = F.E.cols;
  const int width = F.E.width;
  const int64_t cr_lo = F.E.lo[if_lo], cr_hi = F.E.lo[if_hi - 1] + width;
  if (ctx->d == 2) {
    auto a = axis_args<T>(nf, nc, 1, 0, t.tmp[0].p);
    add_term(a, cv, e_op<T>(F, 0), T(1));
    a.sax = 1; a.s0 = cr_lo; a.scnt = cr_hi - cr_lo;
    launch_axis(ctx, a, st);
    auto b = axis_args<T>(nf, nf, 1, 1, fv);
    add_term(b, (const T*)t.tmp[0].p, e_op<T>(F, 1), T(1));
    b.beta = T(1);
    b.sax = 1; b.s0 = if_lo; b.scnt = if_hi - if_lo;
    launch_axis(ctx, b, st);
    return;
  }
  auto a = axis_args<T>(nf, nc, nc, 0, t.tmp[0].p);
  add_term(a, cv, e_op<T>(F, 0), T(1));
  a.sax = 2; a.s0 = cr_lo; a.scnt = cr_hi - cr_lo;
  launch_axis(ctx, a, st);
  auto b = axis_args<T>(nf, nf, nc, 1, t.tmp[1].p);
  add_term(b, (const T*)t.tmp[0].p, e_op<T>(F, 1), T(1));
  b.sax = 2; b.s0 = cr_lo; b.scnt = cr_hi - cr_lo;
  launch_axis(ctx, b, st);
  auto c = axis_args<T>(nf, nf, nf, 2, fv);
  add_term(c, (const T*)t.tmp[1].p, e_op<T>(F, 2), T(1));
  c.beta = T(1);
  c.sax = 2; c.s0 = if_lo; c.scnt = if_hi - if_lo;
  launch_axis(ctx, c, st);
}

}  // namespace

extern "C" {

c0ip_status c0ip_slab_mvs_color(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, double omega, int32_t color,
                                int64_t row0, int64_t lrows, int64_t out_lo, int64_t out_hi, const void* b_ext,
                                void* x_ext, void* r_ext, void* stream) {
  c0ip_status s = check_level(ctx, level);
  if (s) return s;
  if (!b_ext || !x_ext || !r_ext) return fail(C0IP_ERR_ARG, "null vector");
  if (color < 0 || color >= (1 << (ctx->d + 1))) return fail(C0IP_ERR_ARG, "bad colour");
  Level& L = ctx->levels[level];
  if ((s = check_window(ctx, L, row0, lrows, out_lo, out_hi, 4 * ctx->k - 2))) return s;
  ABI_TRY
  cudaStream_t st = (cudaStream_t)stream;
  if (dt == C0IP_F64)
    slab_mvs_color_impl<double>(ctx, L, color, omega, row0, lrows, out_lo, out_hi, (const double*)b_ext,
                                (double*)x_ext, (double*)r_ext, st);
  else if (dt == C0IP_F32)
    slab_mvs_color_impl<float>(ctx, L, color, (float)omega, row0, lrows, out_lo, out_hi, (const float*)b_ext,
                               (float*)x_ext, (float*)r_ext, st);
  else
    return fail(C0IP_ERR_ARG, "bad dtype");
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_slab_restrict(c0ip_ctx ctx, int32_t fine_level, c0ip_dtype dt, int64_t f_row0, int64_t f_lrows,
                               const void* fine_ext, int64_t c_row0, int64_t c_lrows, int64_t c_out_lo,
                               int64_t c_out_hi, void* coarse_ext, void* stream) {
  c0ip_status s = check_level(ctx, fine_level);
  if (s) return s;
  if (fine_level - 1 < ctx->lmin || ctx->cfg.cells_override > 0) return fail(C0IP_ERR_STATE, "no coarser level");
  if (!fine_ext || !coarse_ext) return fail(C0IP_ERR_ARG, "null vector");
  Level& F = ctx->levels[fine_level];
  Level& Cl = ctx->levels[fine_level - 1];
  const int64_t ic_lo = c_out_lo - 1, ic_hi = c_out_hi - 1;      // interior coarse rows
  if (ic_lo < 0 || ic_hi > Cl.n || ic_lo >= ic_hi) return fail(C0IP_ERR_ARG, "coarse rows outside the level");
  if (c_row0 < 0 || c_row0 > ic_lo || c_row0 + c_lrows < ic_hi) return fail(C0IP_ERR_ARG, "coarse window");
  const int64_t fr_lo = F.Et.lo[ic_lo], fr_hi = F.Et.lo[ic_hi - 1] + F.Et.width;
  if (f_row0 > fr_lo || f_row0 + f_lrows < std::min<int64_t>(fr_hi, F.n))
    return fail(C0IP_ERR_ARG, "fine window lacks the rows the restriction reads (need interior rows [" +
                                  std::to_string(fr_lo) + ", " + std::to_string(fr_hi) + "))");
  ABI_TRY
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rf = slow_row_len(ctx, F), rc = slow_row_len(ctx, Cl);
  if (dt == C0IP_F64)
    slab_restrict_impl<double>(ctx, F, (const double*)fine_ext - f_row0 * rf, (double*)coarse_ext - c_row0 * rc,
                               ic_lo, ic_hi, st);
  else if (dt == C0IP_F32)
    slab_restrict_impl<float>(ctx, F, (const float*)fine_ext - f_row0 * rf, (float*)coarse_ext - c_row0 * rc,
                              ic_lo, ic_hi, st);
  else
    return fail(C0IP_ERR_ARG, "bad dtype");
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_slab_prolongate_add(c0ip_ctx ctx, int32_t fine_level, c0ip_dtype dt, int64_t c_row0,
                                     int64_t c_lrows, const void* coarse_ext, int64_t f_row0, int64_t f_lrows,
                                     int64_t f_out_lo, int64_t f_out_hi, void* fine_ext, void* stream) {
  c0ip_status s = check_level(ctx, fine_level);
  if (s) return s;
  if (fine_level - 1 < ctx->lmin || ctx->cfg.cells_override > 0) return fail(C0IP_ERR_STATE, "no coarser level");
  if (!fine_ext || !coarse_ext) return fail(C0IP_ERR_ARG, "null vector");
  Level& F = ctx->levels[fine_level];
  Level& Cl = ctx->levels[fine_level - 1];
  const int64_t if_lo = f_out_lo - 1, if_hi = f_out_hi - 1;
  if (if_lo < 0 || if_hi > F.n || if_lo >= if_hi) return fail(C0IP_ERR_ARG, "fine rows outside the level");
  if (f_row0 < 0 || f_row0 > if_lo || f_row0 + f_lrows < if_hi) return fail(C0IP_ERR_ARG, "fine window");
  const int64_t cr_lo = F.E.lo[if_lo], cr_hi = F.E.lo[if_hi - 1] + F.E.width;
  if (c_row0 > cr_lo || c_row0 + c_lrows < std::min<int64_t>(cr_hi, Cl.n))
    return fail(C0IP_ERR_ARG, "coarse window lacks the rows the prolongation reads (need interior rows [" +
                                  std::to_string(cr_lo) + ", " + std::to_string(cr_hi) + "))");
  ABI_TRY
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rf = slow_row_len(ctx, F), rc = slow_row_len(ctx, Cl);
  if (dt == C0IP_F64)
    slab_prolongate_impl<double>(ctx, F, (const double*)coarse_ext - c_row0 * rc, (double*)fine_ext - f_row0 * rf,
                                 if_lo, if_hi, st);
  else if (dt == C0IP_F32)
    slab_prolongate_impl<float>(ctx, F, (const float*)coarse_ext - c_row0 * rc, (float*)fine_ext - f_row0 * rf,
                                if_lo, if_hi, st);
  else
    return fail(C0IP_ERR_ARG, "bad dtype");
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_vcycle_level(c0ip_ctx ctx, const c0ip_mg_config* mg, int32_t level, const double* r, double* z,
                              void* stream) {
  c0ip_status s = check_mg(ctx, mg);
  if (s) return s;
  if ((s = check_level(ctx, level))) return s;
  if (!r || !z) return fail(C0IP_ERR_ARG, "null vector");
  ABI_TRY
  vcycle_top(ctx, *mg, r, z, (cudaStream_t)stream, level);
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_slab_transfer_rows(c0ip_ctx ctx, int32_t fine_level, int64_t c_out_lo, int64_t c_out_hi,
                                    int64_t f_out_lo, int64_t f_out_hi, int64_t* fine_need, int64_t* coarse_need) {
  c0ip_status s = check_level(ctx, fine_level);
  if (s) return s;
  if (fine_level - 1 < ctx->lmin || ctx->cfg.cells_override > 0) return fail(C0IP_ERR_STATE, "no coarser level");
  Level& F = ctx->levels[fine_level];
  Level& Cl = ctx->levels[fine_level - 1];
  const int64_t ic_lo = c_out_lo - 1, ic_hi = c_out_hi - 1, if_lo = f_out_lo - 1, if_hi = f_out_hi - 1;
  if (ic_lo < 0 || ic_hi > Cl.n || ic_lo >= ic_hi || if_lo < 0 || if_hi > F.n || if_lo >= if_hi)
    return fail(C0IP_ERR_ARG, "rows outside the level");
  if (fine_need) {            // node rows of the fine vector the restriction of [c_out_lo, c_out_hi) reads
    fine_need[0] = F.Et.lo[ic_lo] + 1;
    fine_need[1] = std::min<int64_t>(F.Et.lo[ic_hi - 1] + F.Et.width, F.n) + 1;
  }
  if (coarse_need) {          // node rows of the coarse vector the prolongation onto [f_out_lo, f_out_hi) reads
    coarse_need[0] = F.E.lo[if_lo] + 1;
    coarse_need[1] = std::min<int64_t>(F.E.lo[if_hi - 1] + F.E.width, Cl.n) + 1;
  }
  return C0IP_OK;
}

c0ip_status c0ip_vec_axpby(c0ip_ctx ctx, c0ip_dtype dt, int64_t n, double alpha, const void* x, double beta,
                          void* y, void* stream) {
  if (!ctx || !x || !y || n < 0) return fail(C0IP_ERR_ARG, "null argument / negative length");
  ABI_TRY
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) return C0IP_OK;
  if (dt == C0IP_F64) axpby<double>(ctx, n, alpha, (const double*)x, beta, (double*)y, st);
  else if (dt == C0IP_F32) axpby<float>(ctx, n, (float)alpha, (const float*)x, (float)beta, (float*)y, st);
  else return fail(C0IP_ERR_ARG, "bad dtype");
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_vec_dots(c0ip_ctx ctx, int64_t n, int32_t ndots, const double* x0, const double* y0,
                          const double* x1, const double* y1, double* out, void* stream) {
  if (!ctx || !out || !x0 || !y0 || n < 0 || ndots < 1 || ndots > 2 || (ndots == 2 && (!x1 || !y1)))
    return fail(C0IP_ERR_ARG, "bad dot arguments");
  ABI_TRY
  if (n == 0) { for (int i = 0; i < ndots; ++i) out[i] = 0.0; return C0IP_OK; }
  dots(ctx, n, ndots, x0, y0, x1, y1, nullptr, nullptr, out, (cudaStream_t)stream);
  return C0IP_OK;
  ABI_CATCH
}

c0ip_status c0ip_launch_count(c0ip_ctx ctx, int64_t* count) {
  if (!ctx || !count) return fail(C0IP_ERR_ARG, "null argument");
  *count = ctx->launches;
  return C0IP_OK;
}

}  // extern "C"
