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

template <typename T>
bool fused_apply(FusedLevel& F, const T* x, const T* b, T* y, cudaStream_t st, int64_t* launches);
template <typename T>
bool fused_avs(FusedLevel& F, T omega, const T* b, T* x, T* scratch, cudaStream_t st,
               int64_t* launches);
template <typename T>
bool fused_mvs_color(FusedLevel& F, int color, T omega, const T* b, T* x, cudaStream_t st,
                     int64_t* launches);

}  // namespace c0ip
