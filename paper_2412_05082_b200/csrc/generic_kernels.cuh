// Generic (any N, any k) CUDA kernels for sm_100a: per-axis banded line operators, the patch
// FDM local solve, transfers and vector ops.  They serve the coarse multigrid levels and act
// as the fallback-free baseline path (C0IP_PATH_GENERIC).  The fused tile kernels for large
// levels live in fused_kernels.cuh.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace c0ip {

// A 1D line operator along one axis: square band (lo == nullptr: row i couples columns
// i - hw .. i + hw, zero-padded) or rectangular band (row i couples lo[i] .. lo[i]+width-1).
template <typename T>
struct LineOp {
  const T* v = nullptr;
  const int64_t* lo = nullptr;
  int width = 0;
  int hw = 0;
  int64_t n_in = 0;
};

template <typename T>
struct AxisArgs {
  int64_t dims[3];        // output dims, dims[0] = x (fastest)
  int axis;
  int nterms;
  const T* in[3];
  LineOp<T> op[3];
  T alpha[3];
  const T* z;             // optional: out = gamma * z + sum_t ...
  T gamma;
  T beta;                 // out = beta * out + ... (beta != 0 reads out)
  T* out;
  int sax;                // slab range: iterate only c[sax] in [s0, s0 + scnt) (sax < 0: every index)
  int64_t s0, scnt;
};

// out[idx] = beta*out + gamma*z + sum_t alpha_t * sum_q op_t(i_a, q) * in_t[idx with i_a -> col]
// Sum factorisation of PAPER.md:344 (one 1D contraction per launch and term).
template <typename T>
__global__ void __launch_bounds__(256) axis_apply_kernel(AxisArgs<T> a) {
  int64_t it[3] = {a.dims[0], a.dims[1], a.dims[2]};
  if (a.sax >= 0) it[a.sax] = a.scnt;
  const int64_t total = it[0] * it[1] * it[2];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[3];
    c[0] = q % it[0];
    c[1] = (q / it[0]) % it[1];
    c[2] = q / (it[0] * it[1]);
    if (a.sax >= 0) c[a.sax] += a.s0;
    const int64_t idx = c[0] + a.dims[0] * (c[1] + a.dims[1] * c[2]);
    T acc = 0;
    for (int t = 0; t < a.nterms; ++t) {
      const LineOp<T>& op = a.op[t];
      int64_t din[3] = {a.dims[0], a.dims[1], a.dims[2]};
      din[a.axis] = op.n_in;
      int64_t stride = (a.axis == 0) ? 1 : (a.axis == 1 ? din[0] : din[0] * din[1]);
      int64_t ci[3] = {c[0], c[1], c[2]};
      ci[a.axis] = 0;
      const T* base = a.in[t] + ci[0] + din[0] * (ci[1] + din[1] * ci[2]);
      const int64_t i = c[a.axis];
      const T* row = op.v + i * op.width;
      T s = 0;
      if (op.lo) {
        const int64_t lo = op.lo[i];
        for (int q = 0; q < op.width; ++q) s += row[q] * base[(lo + q) * stride];
      } else {
        for (int q = 0; q < op.width; ++q) {
          int64_t j = i - op.hw + q;
          if (j >= 0 && j < op.n_in) s += row[q] * base[j * stride];
        }
      }
      acc += a.alpha[t] * s;
    }
    if (a.z) acc += a.gamma * a.z[idx];
    if (a.beta != T(0)) acc += a.beta * a.out[idx];
    a.out[idx] = acc;
  }
}

// ----------------------------------------------------------------------------- patch FDM
template <typename T>
struct PatchArgs {
  int d, k, np;
  int pstride;            // patch origin stride per vertex: k (C0IP nodes) or k+1 (SIPG DG nodes)
  int64_t N, n;           // cells, 1D interior dofs
  const T* S[4];          // per axis variant: S[l*np + i]  (np x np)
  const T* lam[4];
  const T* Sv[3];         // graded meshes: per axis, per vertex v: Sv[a][(v-1) np^2 + l np + i]
  const T* lamv[3];       //   and lamv[a][(v-1) np + i]; nullptr: the variant tables above
  const T* r;             // residual (global)
  T* x;                   // updated: x[g] += omega * u
  T omega;
  const int32_t* list;    // patch ids, or nullptr for 0..count-1
  int64_t count;
  int atomic;             // 1: atomicAdd (overlapping patches), 0: plain (disjoint)
};

__device__ __forceinline__ int axis_variant(int64_t v, int64_t N) {
  return (N == 2) ? 3 : (v == 1 ? 0 : (v == N - 1 ? 2 : 1));
}

// One or more patches per CTA: gather R_v r, FDM  u = (x)S (sum Lambda)^{-1} (x)S^T r_v
// (Eq. inverse, applied to A~_v of Eq. localsolverbila), scatter R_v^T u.
template <typename T>
__global__ void __launch_bounds__(256) patch_fdm_kernel(PatchArgs<T> a) {
  extern __shared__ unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int np = a.np;
  int nloc = np;
  for (int i = 1; i < a.d; ++i) nloc *= np;
  const int ppb = max(1, (int)blockDim.x / nloc);        // patches per block
  T* buf0 = sm;
  T* buf1 = sm + ppb * nloc;
  const int64_t first = (int64_t)blockIdx.x * ppb;
  const int64_t Nm1 = a.N - 1;
  const int items = ppb * nloc;

  auto patch_id = [&](int pp) -> int64_t {
    int64_t q = first + pp;
    if (q >= a.count) return -1;
    return a.list ? (int64_t)a.list[q] : q;
  };
  auto vert = [&](int64_t pid, int ax) -> int64_t {
    int64_t s = 1;
    for (int i = 0; i < ax; ++i) s *= Nm1;
    return 1 + (pid / s) % Nm1;
  };
  auto gid = [&](int64_t pid, int l) -> int64_t {
    int64_t g = 0, st = 1;
    for (int ax = 0; ax < a.d; ++ax) {
      int la = l % np; l /= np;
      g += ((vert(pid, ax) - 1) * a.pstride + la) * st;
      st *= a.n;
    }
    return g;
  };
  // gather
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    int pp = it / nloc, l = it % nloc;
    int64_t pid = patch_id(pp);
    buf0[it] = (pid >= 0) ? a.r[gid(pid, l)] : T(0);
  }
  __syncthreads();
  // S^T along each axis
  for (int ax = 0; ax < a.d; ++ax) {
    int st = 1;
    for (int i = 0; i < ax; ++i) st *= np;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      int pp = it / nloc, l = it % nloc;
      int64_t pid = patch_id(pp);
      T s = 0;
      if (pid >= 0) {
        const int64_t vv = vert(pid, ax);
        const T* S = a.Sv[ax] ? a.Sv[ax] + (vv - 1) * np * np : a.S[axis_variant(vv, a.N)];
        int li = (l / st) % np;
        int base = pp * nloc + l - li * st;
        for (int m = 0; m < np; ++m) s += S[m * np + li] * buf0[base + m * st];
      }
      buf1[it] = s;
    }
    __syncthreads();
    T* t = buf0; buf0 = buf1; buf1 = t;
  }
  // divide by lambda_{i1} + ... + lambda_{id}
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    int pp = it / nloc, l = it % nloc;
    int64_t pid = patch_id(pp);
    if (pid < 0) continue;
    T den = 0;
    int ll = l;
    for (int ax = 0; ax < a.d; ++ax) {
      const int64_t vv = vert(pid, ax);
      den += a.lamv[ax] ? a.lamv[ax][(vv - 1) * np + ll % np] : a.lam[axis_variant(vv, a.N)][ll % np];
      ll /= np;
    }
    buf0[it] = buf0[it] / den;
  }
  __syncthreads();
  // S along each axis
  for (int ax = 0; ax < a.d; ++ax) {
    int st = 1;
    for (int i = 0; i < ax; ++i) st *= np;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      int pp = it / nloc, l = it % nloc;
      int64_t pid = patch_id(pp);
      T s = 0;
      if (pid >= 0) {
        const int64_t vv = vert(pid, ax);
        const T* S = a.Sv[ax] ? a.Sv[ax] + (vv - 1) * np * np : a.S[axis_variant(vv, a.N)];
        int li = (l / st) % np;
        int base = pp * nloc + l - li * st;
        for (int m = 0; m < np; ++m) s += S[li * np + m] * buf0[base + m * st];
      }
      buf1[it] = s;
    }
    __syncthreads();
    T* t = buf0; buf0 = buf1; buf1 = t;
  }
  // scatter-add R_v^T (PAPER.md:206-213 / 228-239, sign "+" per reading Q2)
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    int pp = it / nloc, l = it % nloc;
    int64_t pid = patch_id(pp);
    if (pid < 0) continue;
    T val = a.omega * buf0[it];
    int64_t g = gid(pid, l);
    if (a.atomic) atomicAdd(a.x + g, val);
    else a.x[g] += val;
  }
}

// ----------------------------------------------------------------------------- vector ops
template <typename T>
__global__ void axpby_kernel(int64_t n, T a, const T* __restrict__ x, T b, T* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i] + (b == T(0) ? T(0) : b * y[i]);
}

template <typename Tin, typename Tout>
__global__ void convert_kernel(int64_t n, const Tin* __restrict__ x, Tout* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (Tout)x[i];
}

template <typename T>
__global__ void fill_kernel(int64_t n, T v, T* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = v;
}

// Deterministic two-pass dot products: pass 1 writes one partial per block (fixed order),
// pass 2 sums the partials in one block.  Up to 3 dots at once: <x0,y0>, <x1,y1>, <x2,y2>.
__global__ void __launch_bounds__(256) dot_partial_kernel(int64_t n, int nd, const double* x0,
                                                          const double* y0, const double* x1,
                                                          const double* y1, const double* x2,
                                                          const double* y2, double* partial) {
  __shared__ double sh[3][256];
  double s[3] = {0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    s[0] += x0[i] * y0[i];
    if (nd > 1) s[1] += x1[i] * y1[i];
    if (nd > 2) s[2] += x2[i] * y2[i];
  }
  for (int j = 0; j < 3; ++j) sh[j][threadIdx.x] = s[j];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int j = 0; j < 3; ++j) sh[j][threadIdx.x] += sh[j][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int j = 0; j < 3; ++j) partial[j * gridDim.x + blockIdx.x] = sh[j][0];
}

__global__ void __launch_bounds__(256) dot_final_kernel(int nparts, const double* partial, double* out) {
  __shared__ double sh[3][256];
  for (int j = 0; j < 3; ++j) {
    double s = 0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[j * nparts + i];
    sh[j][threadIdx.x] = s;
  }
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int j = 0; j < 3; ++j) sh[j][threadIdx.x] += sh[j][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int j = 0; j < 3; ++j) out[j] = sh[j][0];
}

// Batched projections of the GMRES Arnoldi step (classical Gram-Schmidt, CGS2): partial sums of <w, V_c> for
// c < nv (<= CH) in one pass over w (block partials in fixed order: deterministic), then one final reduction
// per vector, and w -= sum_c coef_c V_c in one pass.
template <int CH>
__global__ void __launch_bounds__(256) mdot_partial_kernel(int64_t n, int nv, const double* __restrict__ w,
                                                           const double* __restrict__ V, double* partial) {
  __shared__ double sh[CH][256];
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double wi = w[i];
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (c < nv) acc[c] += wi * V[c * n + i];
  }
#pragma unroll
  for (int c = 0; c < CH; ++c) sh[c][threadIdx.x] = acc[c];
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s)
#pragma unroll
      for (int c = 0; c < CH; ++c) sh[c][threadIdx.x] += sh[c][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < nv && threadIdx.x < CH) partial[threadIdx.x * gridDim.x + blockIdx.x] = sh[threadIdx.x][0];
}

__global__ void __launch_bounds__(256) mdot_final_kernel(int G, const double* partial, double* out) {
  __shared__ double sh[256];
  double s = 0;
  for (int i = threadIdx.x; i < G; i += blockDim.x) s += partial[blockIdx.x * G + i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

struct Coefs64 {
  double c[64];
};

__global__ void maxpy_kernel(int64_t n, int nv, const __grid_constant__ Coefs64 cf, const double* __restrict__ V,
                             double* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = w[i];
    for (int c = 0; c < nv; ++c) s -= cf.c[c] * V[c * n + i];
    w[i] = s;
  }
}

// b[g] = c * prod_a f1[i_a] + cb * sum_a g1[i_a] prod_{b != a} f1[i_b]
// (separable paper load plus the separable Nitsche boundary data, reading Q8b)
// (per-axis 1D factors f1[a], g1[a]: graded meshes have different ones per axis)
struct LoadArgs {
  const double* f1[3];
  const double* g1[3];
};
__global__ void outer_load_kernel(int d, int64_t n, LoadArgs la, double c, double cb, double* b) {
  int64_t total = n * n * (d == 3 ? n : 1);
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    int64_t i0 = g % n, i1 = (g / n) % n, i2 = g / (n * n);
    const double f0 = la.f1[0][i0], fy = la.f1[1][i1], fz = d == 3 ? la.f1[2][i2] : 1.0;
    double v = c * f0 * fy * fz;
    double w = la.g1[0][i0] * fy * fz + f0 * la.g1[1][i1] * fz;
    if (d == 3) w += f0 * fy * la.g1[2][i2];
    b[g] = v + cb * w;
  }
}

}  // namespace c0ip
