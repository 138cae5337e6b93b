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
  int dec3 = 0;                    // decompose plane pass: the 3-CTA / 3-slot variant
  int64_t dec_chunk = 0;           // its axis-0 chunk (units sized for 3 CTAs per SM)
  int grid = 0;                    // persistent plane-pass CTAs
  // slab mode: the plane passes cover coarse planes
  // [a_base, a_end), the interpolation fine planes [p_base, p_end)
  int64_t a_base = 0, a_end = -1, p_base = 0, p_end = -1;
  unsigned* nonfinite = nullptr;  // decompose plane pass with the finiteness check: set to 1 on inf / NaN
  // slab mode with slab-sized buffers: the shell entries of odd fine planes
  // live at (global shell position + odd_shift) relative to the shell base
  // (the even planes' region and the odd planes' region of a rank are two
  // separate runs of the level-centric buffer); 0 = one global buffer
  int64_t odd_shift = 0;
};

struct Fused3DPlan {
  bool enabled = false;
  size_t scratch_bytes = 0;  // fp64 load-vector volume G
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

// Slab mode: the passes of one fused level restricted to a slab of coarse
// planes [k0, k1) (fine planes [p0, p1) for the interpolation), on the
// caller's G (m0 x m1 x m2 fp64, global plane indexing).
template <typename T>
cudaError_t fused3d_slab_dec_plane(const T* blk, T* shell, T* coarse, double* G, const Fused3DPlan& fp, int64_t k0,
                                   int64_t k1, const Exec& ex);
template <typename T>
cudaError_t fused3d_slab_rec_plane(const T* shell, double* G, const Fused3DPlan& fp, int64_t k0, int64_t k1,
                                   const Exec& ex);
cudaError_t fused3d_slab_inplane(double* G, const Fused3DPlan& fp, const ThomasLevel& th, int64_t k0, int64_t k1,
                                 const Exec& ex);
// axis-0 solve of a [m0][width] column block of G (transposed), in place
cudaError_t fused3d_slab_axis0(double* Gt, int64_t width, const Fused3DPlan& fp, const ThomasLevel& th,
                               const Exec& ex);
template <typename T>
cudaError_t fused3d_slab_interp(const T* shell, const T* coarse, T* fine, const Fused3DPlan& fp, int64_t p0, int64_t p1,
                                const Exec& ex);

// Thomas along the middle axis of [outer][m][inner] (rows when inner == 1).
// w / id: the uniform ThomasAux tables of a plan (api.cu get_plan): id[m ..
// m + 64) holds the end-correction tables of the Toeplitz form, used for m >= 40.
cudaError_t f3_axis_solve(double* y, int64_t outer, int64_t m, int64_t inner, const double* w, const double* id,
                          const Exec& ex);
// Axis-0 Thomas of the columns of a [m0][inner] fp64 array (the segmented
// column pass); cudaErrorNotSupported when m0 is outside its range.
cudaError_t f3_axis0_solve(double* y, int64_t m0, int64_t inner, const double* w, const double* id,
                           const Exec& ex);

// K-pack of slab mode's all-to-all: the column blocks [cb[q], cb[q+1]) of a
// rows x pitch fp64 array packed back to back (unpack: the inverse).
cudaError_t slab_pack(const double* src, int64_t rows, int64_t pitch, const uint64_t* cb, int nparts, double* dst,
                      bool unpack, const Exec& ex);

}  // namespace mgrx_b200
