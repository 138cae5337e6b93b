// Fused 3-D level pass (fused3d.cu): the plane pass + column passes that
// replace the general per-step kernels on large 3-D levels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mgrx_b200 {

// Geometry and work decomposition of one fused level pass.
struct F3Geom {
  int64_t n0 = 0, n1 = 0, n2 = 0;  // fine extents (level l)
  int64_t m0 = 0, m1 = 0, m2 = 0;  // coarse extents (level l-1)
  int64_t chunk = 0;               // coarse planes (axis 0) per work unit
  int tile_rows = 0;               // coarse rows (axis 1) per work unit
  int ntile1 = 0;                  // tiles along axis 1
  int units = 0;                   // work units = chunks * ntile1
  int threads = 0;                 // plane-pass CTA size (strips of 30 coarse columns)
  int ctas_per_sm = 1;             // plane-pass CTAs resident per SM
  int grid = 0;                    // persistent plane-pass CTAs
};

struct Fused3DPlan {
  bool enabled = false;
  size_t scratch_bytes = 0;  // fp64 load-vector volume G + work counter
  size_t scratch_off = 0;    // filled by the caller's scratch layout
  F3Geom g;
};

Fused3DPlan fused3d_plan(const LevelGeom& g, int esize);

template <typename T>
cudaError_t fused3d_decompose_level(const T* blk, T* shell, T* coarse, void* scratch, const LevelGeom& g,
                                    const Fused3DPlan& fp, const ThomasLevel& th, const Exec& ex);
template <typename T>
cudaError_t fused3d_recompose_level(const T* shell, T* coarse, T* fine, void* scratch, const LevelGeom& g,
                                    const Fused3DPlan& fp, const ThomasLevel& th, const Exec& ex);
// recompose_level split in its shell-only correction and the sequential finish
template <typename T>
cudaError_t fused3d_recompose_correction(const T* shell, void* scratch, const Fused3DPlan& fp, const ThomasLevel& th,
                                         const Exec& ex);
template <typename T>
cudaError_t fused3d_recompose_finish(const T* shell, T* coarse, T* fine, void* scratch, const Fused3DPlan& fp,
                                     const ThomasLevel& th, const Exec& ex);

}  // namespace mgrx_b200
