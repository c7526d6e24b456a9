// Exact local solvers: dense A_v^{-1} per patch variant tuple
// and the fused gather / DMMA-GEMM / scatter-add kernel (exact_local.cu).  This file shares no code with
// oracle/.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "host_setup.hpp"

namespace c0ip {

template <typename T>
struct ExactArgs {
  const T* Ainv = nullptr;        // nloc x nloc, row-major (A_v^{-1} of one variant tuple, level scaling)
  int nloc = 0;                   // (2k-1)^d
  const int64_t* off = nullptr;   // nloc offsets of the patch-local DoFs (x fastest) from the patch origin
  const int32_t* list = nullptr;  // patch ids (all of this variant tuple)
  int64_t count = 0;
  int d = 2, k = 2;
  int64_t N = 0, n = 0;           // cells per axis, interior nodes per axis
  const T* r = nullptr;           // residual (full level vector)
  T* x = nullptr;                 // updated in place: x += omega R_v^T A_v^{-1} R_v r
  T omega = 0;
};

template <typename T>
void launch_exact_patches(const ExactArgs<T>& a, cudaStream_t st);

// Host tables of one level: A_v^{-1} per variant tuple (index sum_a var_a 4^a, var in {0 left, 1 interior,
// 2 right, 3 both}), the local offsets, and the patch lists grouped by tuple (all patches; per colour).
struct ExactHost {
  int nloc = 0;
  std::vector<int> tuples;                       // tuple indices present on this level
  std::vector<std::vector<double>> inv;          // per present tuple, nloc^2
  std::vector<int64_t> off;                      // nloc
  std::vector<std::vector<int32_t>> all;         // per present tuple: patch ids (AVS)
  std::vector<std::vector<std::vector<int32_t>>> by_color;   // [colour][tuple] patch ids (MVS)
};

// Builds the tables from the level's (h-scaled) banded 1D M, L, B.  colour_of_patch(p) gives the MVS
// colour.  Returns false with a message if an A_v is not SPD.
bool build_exact_host(int d, int k, int64_t N, const Band& M, const Band& L, const Band& B,
                      const std::vector<int32_t>& colour_of_patch, int ncolours, ExactHost& out,
                      std::string& err);

}  // namespace c0ip
