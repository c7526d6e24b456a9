// Dispatch interface of the fused tile kernels (fused_kernels.cu).  A FusedLevel holds the
// per-level constants of the fused path; the fused_* entry points return false when the
// level / degree / dimension is not covered, in which case the caller uses the generic path.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>

#include "host_setup.hpp"

namespace c0ip {

struct FusedLevel;    // opaque; defined in fused_kernels.cu

struct FusedLevelDeleter {
  void operator()(FusedLevel* p) const;
};

std::unique_ptr<FusedLevel, FusedLevelDeleter> make_fused_level_impl(int d, int k, int64_t N,
                                                                     const RefData& ref,
                                                                     const Fdm& fdm, double h);

// Slab window (multi-GPU z-slabs): arrays hold global interior rows [row0, row0 + lrows) of the slowest
// axis; outputs are written for node rows j in [out_lo, out_hi).  nullptr = the whole domain.
struct SlabWindow {
  int64_t row0, lrows, out_lo, out_hi;
};
bool fused_supports_slab(const FusedLevel& F);

template <typename T>
bool fused_apply(FusedLevel& F, const T* x, const T* b, T* y, cudaStream_t st, int64_t* launches,
                 const SlabWindow* win = nullptr);
template <typename T>
bool fused_fdm(FusedLevel& F, T omega, const T* r, T* x, cudaStream_t st, int64_t* launches,
               const SlabWindow* win = nullptr);
template <typename T>
bool fused_avs(FusedLevel& F, T omega, const T* b, T* x, T* scratch, cudaStream_t st,
               int64_t* launches);
// one colour of the coloured MVS (patch list of the colour on the device)
template <typename T>
bool fused_mvs_color(FusedLevel& F, const int32_t* list, int64_t count, T omega, const T* b, T* x,
                     cudaStream_t st, int64_t* launches);

// 2D: x += omega A~_v^{-1} R_v r over a list of mutually disjoint patches (one MVS colour, k >= 5)
template <typename T>
bool fused2_patch_list(FusedLevel& F, T omega, const T* r, T* x, const int32_t* list, int64_t count,
                       cudaStream_t st, int64_t* launches);

// 3D (fused3d.cu): matvec / residual, and the per-patch FDM update x += omega A~_v^{-1} R_v r over a
// list of mutually disjoint patches (a parity class or a colour)
template <typename T>
bool fused3_apply(FusedLevel& F, const T* x, const T* b, T* y, cudaStream_t st, int64_t* launches,
                  const SlabWindow* win = nullptr);
template <typename T>
bool fused3_patch_fdm(FusedLevel& F, T omega, const T* r, T* x, const int32_t* list, int64_t count,
                      cudaStream_t st, int64_t* launches, int atomic = 0);
// additive FDM update of every patch touching the owned planes of the window (nullptr: all patches),
// writes restricted to the owned planes; atomic scatter, or 8 parity-class launches with plain stores
template <typename T>
bool fused3_fdm_window(FusedLevel& F, T omega, const T* r, T* x, bool atomic, cudaStream_t st, int64_t* launches,
                       const SlabWindow* win = nullptr);
int fused_dim(const FusedLevel& F);
// one colour of the 3D coloured MVS fused per patch (residual on the footprint + FDM + update), k <= 3
template <typename T>
bool fused3_mvs_color(FusedLevel& F, const int32_t* list, int64_t count, T omega, const T* b, T* x,
                      cudaStream_t st, int64_t* launches);

// FP64 tensor-core (DMMA) kernels (mma2d.cu); false if the level / degree is not covered
// (2D, k = 3, 4) or C0IP_NO_MMA is set
bool mma_enabled();
bool mma_fdm2d(const FusedLevel& F, double omega, const double* r, double* x, const SlabWindow& w,
               cudaStream_t st);
// x += omega A~_v^{-1} R_v r over a patch list (nullptr: all patches); atomic: red.global.add (patches
// may overlap), else plain read-modify-write (the list must be mutually disjoint)
bool mma_patch_fdm2d(const FusedLevel& F, double omega, const double* r, double* x, const int32_t* list,
                     int64_t count, int atomic, cudaStream_t st);
bool mma_mvs2d(const FusedLevel& F, const int32_t* list, int64_t count, double omega, const double* b, double* x,
               cudaStream_t st);

// 2D transfers (transfer2d.cu): prolong = true: fine += P coarse; false: coarse = P^T fine.
// Nc = coarse cells per axis (>= 4), returns false if not covered.
template <typename T>
bool fused_transfer2d(int k, bool prolong, int64_t Nc, const T* src, T* dst, cudaStream_t st, int64_t* launches);

}  // namespace c0ip
