// Fused 3-D level pass (fused3d.cu): the plane pass + column passes that
// replace the general per-step kernels on large 3-D levels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mgrx_b200 {

struct Fused3DPlan {
  bool enabled = false;
  size_t scratch_bytes = 0;  // fp64 load-vector volume + nodal staging
  size_t scratch_off = 0;    // filled by the caller's scratch layout
  int tile_rows = 0;         // coarse rows per plane-pass CTA (axis 1)
  int chunk_planes = 0;      // coarse planes per plane-pass CTA (axis 0)
  int grid_plane = 0;        // plane-pass CTAs
};

Fused3DPlan fused3d_plan(const LevelGeom& g, int esize);

template <typename T>
cudaError_t fused3d_decompose_level(const T* blk, T* shell, T* coarse, void* scratch, const LevelGeom& g,
                                    const Fused3DPlan& fp, const ThomasLevel& th, const Exec& ex);
template <typename T>
cudaError_t fused3d_recompose_level(const T* shell, T* coarse, T* fine, void* scratch, const LevelGeom& g,
                                    const Fused3DPlan& fp, const ThomasLevel& th, const Exec& ex);

}  // namespace mgrx_b200
