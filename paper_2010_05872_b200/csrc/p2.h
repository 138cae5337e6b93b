// Second-generation fused 3-D level pass ("p2", fused_p2.cu) for fp32 levels
// with odd extents: two passes over the level instead of four.
//
//   plane pass  coefficients + shell/coarse stores (decompose) or the
//               component read from the shell (recompose), the load vector
//               L0 L1 L2 c, the axis-2 Thomas solve, and the axis-0 forward
//               elimination inside the CTA's chunk of coarse planes.
//   carries     per (row, column) the axis-0 recurrences across chunks.
//   strip pass  per (chunk, 32 columns): axis-0 back substitution, the
//               axis-1 solve, coarse += sign * z.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace mgrx_b200 {

struct P2Geom {
  int n0 = 0, n1 = 0, n2 = 0;  // fine extents
  int m0 = 0, m1 = 0, m2 = 0;  // coarse extents
  int T = 0;                   // coarse rows per tile (the last tile has T + 1)
  int ntile = 0;               // (m1 - 1) / T
  int C = 0;                   // coarse planes per chunk (the last chunk has the remainder)
  int nchunk = 0;
  int nw = 0;                  // warps per plane-pass CTA (30 coarse columns each)
  int64_t in_sp = 0, in_sr = 0;  // fine block plane / row pitch (elements)
  int64_t co_sp = 0, co_sr = 0;  // coarse block plane / row pitch (elements)
  int PG = 0;                    // row pitch of the fp64 planes (doubles)
  int64_t GP = 0;                // plane pitch of the fp64 planes (= m1 * PG)
};

struct P2Bufs {
  double* G = nullptr;   // [m0][m1][PG]  T1 T2 of the chunk-local axis-0 forward elimination
  double* S = nullptr;   // [nchunk]      per chunk: sum_i Gamma_i g_i (back-substitution seed)
  double* EU = nullptr;  // [nchunk]      chunk c's share of coarse plane a0(c) - 1
  double* ED = nullptr;  // [nchunk]      chunk c's share of coarse plane a1(c)
  double* X = nullptr;   // [nchunk]      forward carry entering chunk c
  double* XB = nullptr;  // [nchunk]      back-substitution value just above chunk c
};

struct P2Tabs {
  const double *w0 = nullptr, *id0 = nullptr, *gam0 = nullptr, *A0 = nullptr;  // axis 0 (m0)
  const double *w1 = nullptr, *id1 = nullptr;                                   // axis 1 (m1)
  const double *w2 = nullptr, *id2 = nullptr;                                   // axis 2 (m2)
  const double* ch = nullptr;  // per chunk: Aend, SG, Gend, Dl, wa1 (5 x nchunk)
  const double *af1 = nullptr, *bb1 = nullptr;  // axis-1 segment carry weights per row (m1)
  const double *sf = nullptr, *sb = nullptr;    // axis-1 segment scan factors (5 x 32)
};

struct P2Plan {
  bool enabled = false;
  P2Geom g;
  size_t scratch_bytes = 0;  // buffers of P2Bufs
  size_t scratch_off = 0;    // set by the caller
  std::vector<double> tabs;  // host tables (uploaded by the caller)
  size_t tab_off = 0;        // offset (doubles) of this level's tables in the caller's upload
  size_t o_w0 = 0, o_id0 = 0, o_gam0 = 0, o_A0 = 0, o_w1 = 0, o_id1 = 0, o_w2 = 0, o_id2 = 0, o_ch = 0;
  size_t o_af1 = 0, o_bb1 = 0, o_sf = 0, o_sb = 0;
};

// Plan of one level (geometry as LevelGeom): enabled for fp32 3-D levels
// with odd extents and m1, m2 in {33, 65, 129, 257}.
P2Plan p2_plan(const LevelGeom& lg, int esize);
void p2_bind(const P2Plan& p, void* scratch, const double* d_tabs, P2Bufs* b, P2Tabs* t);
// zero the completion counters once after (re)allocating the scratch
cudaError_t p2_init(const P2Plan& p, void* scratch, cudaStream_t s);

cudaError_t p2_decompose_level(const float* blk, float* shell, float* coarse, const P2Plan& p, const P2Bufs& b,
                               const P2Tabs& t, const Exec& ex);
// recompose: the shell-only correction (plane pass + carries) and the
// sequential finish (column pass, coarse -= z); interpolation is the caller's
cudaError_t p2_recompose_correction(const float* shell, const P2Plan& p, const P2Bufs& b, const P2Tabs& t,
                                    const Exec& ex);
cudaError_t p2_recompose_apply(float* coarse, const P2Plan& p, const P2Bufs& b, const P2Tabs& t, const Exec& ex);

}  // namespace mgrx_b200
