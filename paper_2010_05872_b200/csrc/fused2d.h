// Fused 2-D level pass on nonuniform coordinates (fused2d.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mgrx_b200 {

struct F2Geom {
  int n0 = 0, n1 = 0;  // fine extents
  int m0 = 0, m1 = 0;  // coarse extents
  int strips = 0;      // CTAs across axis 1 (240 coarse columns each)
  int chunk = 0;       // coarse rows per CTA (its two halo fine rows are recomputed)
  int chunks = 0;      // CTAs along axis 0
};

// Per-level coordinate tables (NuLevel of api.cu's nonuniform upload).
struct F2Tabs {
  const double *wl0 = nullptr, *wr0 = nullptr, *wl1 = nullptr, *wr1 = nullptr;  // interpolation weights at odd j
  const double *s0 = nullptr, *s1 = nullptr;                                    // load stencils (5 per coarse node)
};

struct Fused2DPlan {
  bool enabled = false;
  size_t scratch_bytes = 0;  // the fp64 volume G (m0 x m1)
  size_t scratch_off = 0;
  F2Geom g;
};

Fused2DPlan fused2d_plan(const LevelGeom& g);

template <typename T>
cudaError_t fused2d_decompose_level(const T* blk, T* shell, T* coarse, void* scratch, const Fused2DPlan& fp,
                                    const NuLevel& nu, const Exec& ex);
template <typename T>
cudaError_t fused2d_recompose_level(const T* shell, T* coarse, T* fine, void* scratch, const Fused2DPlan& fp,
                                    const NuLevel& nu, const Exec& ex);

}  // namespace mgrx_b200
