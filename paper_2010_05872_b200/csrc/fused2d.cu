// Fused 2-D level pass on nonuniform coordinates (BASELINE config 3) for
// sm_100a.
//
// Replaces, on large 2-D levels of a nonuniform-coordinate call, the general
// per-step sequence (coefficients with the coordinate-derived interpolation
// weights, the materialised fp64 component, one load + Thomas sweep per axis,
// apply; the restatement of transform.hpp:216-304 / :331-477 documented in
// oracle/mgrx_oracle.c mo_*_nu) with
//
//   decompose  f2_dec    streams the level's fine rows: coefficients (the
//                        general path's corner order and weights), shell and
//                        coarse stores, the load vector L0 L1 c of the
//                        component in registers (axis 1 through warp
//                        shuffles, axis 0 accumulated over the rows); a
//                        finished coarse row goes to the fp64 volume G
//              f2_rows   Thomas along axis 1 on G (a warp per row)
//              f2_cols   Thomas along axis 0 on G + coarse += z
//   recompose  f2_rec    the same load vector from the shell
//              f2_rows, f2_cols (coarse -= z)
//              f2_interp fine = coarse nodes + shell + the weighted prediction
//
// The correction z = T0 T1 L0 L1 c is the restatement's S1 S0 c with the
// axis operators applied in a different order (they act on different axes
// and commute exactly): results differ from the restatement by rounding only
// (tests/test_gpu_configs.py: 1e-12 of the range for fp64).  The G volume of
// the finest 4097^2 level (33.6 MB) stays in L2 between the passes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "fused2d.h"

namespace mgrx_b200 {

namespace {

constexpr int kF2Warps = 8;             // row passes: 8 warps x 30 owned coarse columns per CTA
constexpr int kF2Strip = 30 * kF2Warps;  // coarse columns per CTA
constexpr int kColLS = 17;              // axis-0 solve: values per segment
constexpr int kColW = 8;                // columns per block
constexpr unsigned kFull = 0xffffffffu;

template <typename T> __device__ __forceinline__ T to_tt(double v);
template <> __device__ __forceinline__ float to_tt<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ double to_tt<double>(double v) { return v; }

// Shell offset of fine row p of a 2-D level (pack_level_centric,
// reorder.hpp:180-215): reordered row r0 = p even ? p/2 : m0 + p/2; a row
// with r0 < m0 holds only its odd columns.
__device__ __forceinline__ int64_t f2_row_start(const F2Geom& g, int p) {
  const int64_t r0 = (p & 1) ? g.m0 + (p >> 1) : (p >> 1);
  return r0 < g.m0 ? r0 * (g.n1 - g.m1) : int64_t(g.m0) * (g.n1 - g.m1) + (r0 - g.m0) * g.n1;
}

// Row pass (decompose: coefficients + load vector; recompose: load vector
// from the shell).  CTA = (strip of 240 coarse columns, chunk of 32 coarse
// rows); warp w owns coarse columns base + 30 w + [0, 30) on lanes 1..30,
// lanes 0 and 31 recompute the neighbours (their values reach the owners
// through shuffles).  Fine rows are loaded two ahead in registers.
template <typename T, bool DEC>
__global__ void __launch_bounds__(32 * kF2Warps) k_f2_pass(const T* __restrict__ src, T* __restrict__ shell,
                                                           T* __restrict__ coarse, double* __restrict__ G,
                                                           const F2Geom g, const F2Tabs t) {
  const int strip = int(blockIdx.x) % g.strips, chunk = int(blockIdx.x) / g.strips;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = strip * kF2Strip + 30 * warp - 1 + lane;
  const bool valid = c >= 0 && c < g.m1;
  const bool owned = valid && lane >= 1 && lane <= 30;
  const bool has_odd = valid && 2 * c + 1 < g.n1;
  const int cc = valid ? c : 0;
  const int k0 = chunk * g.chunk, k1 = min(g.m0, k0 + g.chunk);
  const int plo = max(0, 2 * k0 - 2), phi = min(g.n0 - 1, 2 * k1);
  const int own_lo = 2 * k0, own_hi = (k1 == g.m0) ? g.n0 : 2 * k1;  // fine rows whose shell this CTA writes
  // per-lane weights: axis-1 interpolation at 2c+1, the axis-1 load stencil of c
  const double wl1 = has_odd ? t.wl1[2 * cc + 1] : 0.0, wr1 = has_odd ? t.wr1[2 * cc + 1] : 0.0;
  double s1[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) s1[k] = valid ? t.s1[5 * cc + k] : 0.0;
  const bool rdeg = 2 * cc + 2 >= g.n1;  // the right corner column does not exist (even n1)
  // loads of fine row p: the column pair's two values (decompose: the level
  // block; recompose: the component from the shell, 0 on nodes)
  auto load = [&](int p, double& e, double& o) {
    e = 0.0;
    o = 0.0;
    if (p > phi || !valid) return;
    if (DEC) {
      const T* r = src + int64_t(p) * g.n1 + 2 * cc;
      e = double(r[0]);
      if (has_odd) o = double(r[1]);
    } else {
      const T* r = src + f2_row_start(g, p);
      if (p & 1) {
        e = double(r[cc]);
        if (has_odd) o = double(r[g.m1 + cc]);
      } else if (has_odd) {
        o = double(r[cc]);
      }
    }
  };
  pdl_wait();
  double e0, o0, e1, o1, e2, o2, e3, o3;
  load(plo, e0, o0);
  load(plo + 1, e1, o1);
  load(plo + 2, e2, o2);
  load(plo + 3, e3, o3);
  double prev_e = 0.0;                      // decompose: nodal value of the last even row (own column)
  double Ap = 0.0, Ac = 0.0, An = 0.0;      // axis-0 accumulators: coarse rows k-1, k, k+1
  for (int p = plo; p <= phi; ++p) {
    const int k = p >> 1;
    const bool odd = p & 1;
    double ce, co;  // the component at (p, 2c), (p, 2c+1)
    if (DEC) {
      const bool own_row = owned && p >= own_lo && p < own_hi;
      if (!odd) {
        // (p, 2c) nodal; (p, 2c+1): interpolation along axis 1
        const double vR = __shfl_down_sync(kFull, e0, 1);
        const double vr = rdeg ? e0 : vR;
        const double pred = __dadd_rn(__dmul_rn(wl1, e0), __dmul_rn(wr1, vr));
        const T tO = to_tt<T>(__dsub_rn(o0, pred));
        ce = 0.0;
        co = has_odd ? double(tO) : 0.0;
        if (own_row) {
          if (k >= k0 && k < k1) coarse[int64_t(k) * g.m1 + c] = to_tt<T>(e0);
          if (has_odd) shell[f2_row_start(g, p) + c] = tO;
        }
        prev_e = e0;
      } else {
        // rows 2k and 2k+2 (2k when 2k+2 is past the end: degenerate corner)
        const double vL = prev_e, vRw = (p + 1 <= g.n0 - 1) ? e1 : prev_e;
        const double wl0 = t.wl0[p], wr0 = t.wr0[p];
        const double pe = __dadd_rn(__dmul_rn(wl0, vL), __dmul_rn(wr0, vRw));
        const T tE = to_tt<T>(__dsub_rn(e0, pe));
        const double vLr0 = __shfl_down_sync(kFull, vL, 1), vRr0 = __shfl_down_sync(kFull, vRw, 1);
        const double vLr = rdeg ? vL : vLr0, vRr = rdeg ? vRw : vRr0;
        // corners in cmask order (axis 0 = bit 0): (L,L) (R,L) (L,R) (R,R)
        double po = __dmul_rn(__dmul_rn(wl0, wl1), vL);
        po = __dadd_rn(po, __dmul_rn(__dmul_rn(wr0, wl1), vRw));
        po = __dadd_rn(po, __dmul_rn(__dmul_rn(wl0, wr1), vLr));
        po = __dadd_rn(po, __dmul_rn(__dmul_rn(wr0, wr1), vRr));
        const T tO = to_tt<T>(__dsub_rn(o0, po));
        ce = valid ? double(tE) : 0.0;
        co = has_odd ? double(tO) : 0.0;
        if (own_row) {
          T* sr = shell + f2_row_start(g, p);
          sr[c] = tE;
          if (has_odd) sr[g.m1 + c] = tO;
        }
      }
    } else {
      ce = e0;
      co = o0;
    }
    // axis-1 load stencil at c: component at fine columns 2c-2 .. 2c+2
    const double ceL = __shfl_up_sync(kFull, ce, 1), coL = __shfl_up_sync(kFull, co, 1);
    const double ceR = __shfl_down_sync(kFull, ce, 1);
    double h = s1[0] * ceL;
    h = fma(s1[1], coL, h);
    h = fma(s1[2], ce, h);
    h = fma(s1[3], co, h);
    h = fma(s1[4], ceR, h);
    // axis-0 load stencil: fine row p feeds coarse rows k-1, k, k+1 (even p)
    // or k, k+1 (odd p)
    if (!odd) {
      if (k >= 1) Ap = fma(t.s0[5 * (k - 1) + 4], h, Ap);
      Ac = fma(t.s0[5 * k + 2], h, Ac);
      if (k + 1 < g.m0) An = fma(t.s0[5 * (k + 1) + 0], h, An);
      if (owned && k - 1 >= k0 && k - 1 < k1) G[int64_t(k - 1) * g.m1 + c] = Ap;
      if (p == g.n0 - 1 && owned && k >= k0 && k < k1) G[int64_t(k) * g.m1 + c] = Ac;
    } else {
      Ac = fma(t.s0[5 * k + 3], h, Ac);
      if (k + 1 < g.m0) An = fma(t.s0[5 * (k + 1) + 1], h, An);
      if (p == g.n0 - 1 && owned && k >= k0 && k < k1) G[int64_t(k) * g.m1 + c] = Ac;
      Ap = Ac;
      Ac = An;
      An = 0.0;
    }
    e0 = e1;
    o0 = o1;
    e1 = e2;
    o1 = o2;
    e2 = e3;
    o2 = o3;
    load(p + 4, e3, o3);
  }
  pdl_trigger();
}

// fine = coarse nodes + shell + the weighted prediction from the corrected
// coarse block (general recompose interpolation, same corner order).
template <typename T>
__global__ void __launch_bounds__(256) k_f2_interp(const T* __restrict__ shell, const T* __restrict__ coarse,
                                                   T* __restrict__ fine, const F2Geom g, const F2Tabs t) {
  pdl_wait();
  const int p = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;  // fine row, coarse column
  if (c >= g.m1) return;
  const int k = p >> 1;
  const bool has_odd = 2 * c + 1 < g.n1;
  const int cr = (2 * c + 2 < g.n1) ? c + 1 : c;
  const T* sr = shell + f2_row_start(g, p);
  T* fr = fine + int64_t(p) * g.n1 + 2 * c;
  const T* ck = coarse + int64_t(k) * g.m1;
  if (!(p & 1)) {
    const double a = double(ck[c]);
    fr[0] = ck[c];
    if (has_odd) {
      const double b = double(ck[cr]);
      const double pred = __dadd_rn(__dmul_rn(t.wl1[2 * c + 1], a), __dmul_rn(t.wr1[2 * c + 1], b));
      fr[1] = to_tt<T>(__dadd_rn(double(sr[c]), pred));
    }
  } else {
    const T* ck1 = (p + 1 <= g.n0 - 1) ? ck + g.m1 : ck;
    const double wl0 = t.wl0[p], wr0 = t.wr0[p];
    const double vL = double(ck[c]), vR = double(ck1[c]);
    const double pe = __dadd_rn(__dmul_rn(wl0, vL), __dmul_rn(wr0, vR));
    fr[0] = to_tt<T>(__dadd_rn(double(sr[c]), pe));
    if (has_odd) {
      const double wl1 = t.wl1[2 * c + 1], wr1 = t.wr1[2 * c + 1];
      const double vLr = double(ck[cr]), vRr = double(ck1[cr]);
      double po = __dmul_rn(__dmul_rn(wl0, wl1), vL);
      po = __dadd_rn(po, __dmul_rn(__dmul_rn(wr0, wl1), vR));
      po = __dadd_rn(po, __dmul_rn(__dmul_rn(wl0, wr1), vLr));
      po = __dadd_rn(po, __dmul_rn(__dmul_rn(wr0, wr1), vRr));
      fr[1] = to_tt<T>(__dadd_rn(double(sr[g.m1 + c]), po));
    }
  }
  pdl_trigger();
}

// Affine map y -> a + b y of a recurrence segment.
struct Aff2 {
  double a, b;
};

// Axis-1 Thomas (nonuniform ThomasAux: forward y_i = f_i - w_i y_{i-1},
// back z_i = (y_i - off_i z_{i+1}) / d_i) of every G row: a warp per row,
// staged in shared memory; lane segments run from a zero carry, a shuffle
// scan of their affine maps gives each its true carry, then the exact rerun.
__global__ void __launch_bounds__(256) k_f2_rows(double* __restrict__ G, int rows, int m, const double* __restrict__ gw,
                                                 const double* __restrict__ gid, const double* __restrict__ goff) {
  extern __shared__ double rs[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // the Thomas tables in shared memory: a lane walks its own segment, so
  // global loads of them would be 32 separate lines per instruction
  double* w = rs;
  double* id = w + m;
  double* off = id + m;
  double* x = off + m + warp * m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    w[i] = gw[i];
    id[i] = gid[i];
    off[i] = goff[i];
  }
  __syncthreads();
  const int seg = ((m + 31) >> 5) | 1;  // odd: lanes' segments start in distinct shared-memory banks
  const int s0 = min(m, lane * seg), s1 = min(m, s0 + seg);
  pdl_wait();
  for (int r = blockIdx.x * nw + warp; r < rows; r += gridDim.x * nw) {
    double* gr = G + int64_t(r) * m;
    for (int i0 = lane; i0 < m; i0 += 32 * 8) {  // 8 loads in flight per lane
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = (i0 + 32 * u < m) ? gr[i0 + 32 * u] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + 32 * u < m) x[i0 + 32 * u] = t[u];
    }
    __syncwarp();
    Aff2 f{0.0, 1.0};
    for (int i = s0; i < s1; ++i) {
      const double wi = w[i];
      f.a = x[i] - wi * f.a;
      f.b = -wi * f.b;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double pa = __shfl_up_sync(kFull, f.a, o), pb = __shfl_up_sync(kFull, f.b, o);
      if (lane >= o) {
        f.a = f.a + f.b * pa;
        f.b = f.b * pb;
      }
    }
    double y = __shfl_up_sync(kFull, f.a, 1);
    if (lane == 0) y = 0.0;
    for (int i = s0; i < s1; ++i) {
      y = x[i] - w[i] * y;
      x[i] = y;
    }
    Aff2 b{0.0, 1.0};
    for (int i = s1 - 1; i >= s0; --i) {
      const double di = id[i], oi = off[i];
      b.a = (x[i] - oi * b.a) * di;
      b.b = -oi * di * b.b;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double na = __shfl_down_sync(kFull, b.a, o), nb = __shfl_down_sync(kFull, b.b, o);
      if (lane + o < 32) {
        b.a = b.a + b.b * na;
        b.b = b.b * nb;
      }
    }
    double z = __shfl_down_sync(kFull, b.a, 1);
    if (lane == 31) z = 0.0;
    for (int i = s1 - 1; i >= s0; --i) {
      z = (x[i] - off[i] * z) * id[i];
      x[i] = z;
    }
    __syncwarp();
    for (int i = lane; i < m; i += 32) gr[i] = x[i];
    __syncwarp();
  }
  pdl_trigger();
}

// Hillis-Steele scans of segment maps (a, b) per column in shared memory
// (A/B: [S][kColW]); returns the carry entering segment s: forward, the
// composition of segments 0..s-1 applied to 0; backward, of segments
// S-1..s+1.  Called by the whole block.
__device__ __forceinline__ double scan_fwd(double* A, double* B, double a, double b, int s, int S, int col) {
  for (int o = 1; o < S; o <<= 1) {
    A[s * kColW + col] = a;
    B[s * kColW + col] = b;
    __syncthreads();
    if (s >= o) {  // (earlier o-block) then (this): a' = a + b * a_prev, b' = b * b_prev
      const double pa = A[(s - o) * kColW + col], pb = B[(s - o) * kColW + col];
      a = a + b * pa;
      b = b * pb;
    }
    __syncthreads();
  }
  A[s * kColW + col] = a;
  __syncthreads();
  const double carry = s > 0 ? A[(s - 1) * kColW + col] : 0.0;
  __syncthreads();
  return carry;
}
__device__ __forceinline__ double scan_bwd(double* A, double* B, double a, double b, int s, int S, int col) {
  for (int o = 1; o < S; o <<= 1) {
    A[s * kColW + col] = a;
    B[s * kColW + col] = b;
    __syncthreads();
    if (s + o < S) {
      const double na = A[(s + o) * kColW + col], nb = B[(s + o) * kColW + col];
      a = a + b * na;
      b = b * nb;
    }
    __syncthreads();
  }
  A[s * kColW + col] = a;
  __syncthreads();
  const double carry = s + 1 < S ? A[(s + 1) * kColW + col] : 0.0;
  __syncthreads();
  return carry;
}

// Axis-0 Thomas of every G column (length m0, stride m1) + coarse += sign z
// (apply_correction, transform.hpp:435-477).  Block = 8 columns x S
// segments of <= kColLS values in registers; segment maps folded through
// shared memory.
template <typename T>
__global__ void __launch_bounds__(1024) k_f2_cols(const double* __restrict__ G, T* __restrict__ coarse, double sign,
                                                  int m0, int m1, const double* __restrict__ w,
                                                  const double* __restrict__ id, const double* __restrict__ off) {
  extern __shared__ double cs[];
  const int S = blockDim.x / kColW;
  double* A = cs;
  double* B = A + S * kColW;
  const int col = threadIdx.x % kColW, s = threadIdx.x / kColW;
  const int c = blockIdx.x * kColW + col;
  const bool valid = c < m1;
  const int s0 = min(m0, s * kColLS), len = min(m0, s0 + kColLS) - s0;
  double v[kColLS];
  pdl_wait();
  const double* gp = G + int64_t(s0) * m1 + (valid ? c : 0);
#pragma unroll
  for (int k = 0; k < kColLS; ++k) v[k] = (valid && k < len) ? gp[int64_t(k) * m1] : 0.0;
  double ya = 0.0, yb = 1.0;
#pragma unroll
  for (int k = 0; k < kColLS; ++k)
    if (k < len) {
      const double wi = w[s0 + k];
      ya = v[k] - wi * ya;
      yb = -wi * yb;
    }
  // inclusive scan over the segments (composition in segment order), then
  // each segment's carry is the previous segment's prefix applied to 0
  double y = scan_fwd(A, B, ya, yb, s, S, col);
#pragma unroll
  for (int k = 0; k < kColLS; ++k)
    if (k < len) {
      y = v[k] - w[s0 + k] * y;
      v[k] = y;
    }
  double za = 0.0, zb = 1.0;
#pragma unroll
  for (int k = kColLS - 1; k >= 0; --k)
    if (k < len) {
      const double di = id[s0 + k], oi = off[s0 + k];
      za = (v[k] - oi * za) * di;
      zb = -oi * di * zb;
    }
  double z = scan_bwd(A, B, za, zb, s, S, col);
  pdl_trigger();
  if (!valid) return;
  T* cp = coarse + int64_t(s0) * m1 + c;
#pragma unroll
  for (int k = kColLS - 1; k >= 0; --k)
    if (k < len) {
      z = (v[k] - off[s0 + k] * z) * id[s0 + k];
      cp[int64_t(k) * m1] = to_tt<T>(double(cp[int64_t(k) * m1]) + sign * z);
    }
}

template <typename T>
cudaError_t launch_pass(const T* src, T* shell, T* coarse, double* G, const F2Geom& g, const F2Tabs& t, bool dec,
                        const Exec& ex) {
  const unsigned grid = unsigned(g.strips * g.chunks);
  if (dec)
    MGRX_LAUNCH(ex, "f2_dec", pdl_launch(k_f2_pass<T, true>, dim3(grid), dim3(32 * kF2Warps), 0, ex.s, !ex.prof,
                                         src, shell, coarse, G, g, t));
  else
    MGRX_LAUNCH(ex, "f2_rec", pdl_launch(k_f2_pass<T, false>, dim3(grid), dim3(32 * kF2Warps), 0, ex.s, !ex.prof,
                                         src, shell, coarse, G, g, t));
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_solves(double* G, T* coarse, double sign, const F2Geom& g, const NuLevel& nu, const Exec& ex) {
  // axis 1: a warp per row
  const size_t rsm = size_t(8 + 3) * g.m1 * 8;
  cudaError_t e = cudaFuncSetAttribute(k_f2_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, int(rsm));
  if (e != cudaSuccess) return e;
  const int rblocks = std::min((g.m0 + 7) / 8, kNumSMs * 8);
  MGRX_LAUNCH(ex, "f2_rows", pdl_launch(k_f2_rows, dim3(unsigned(rblocks)), dim3(256), rsm, ex.s, !ex.prof, G, g.m0,
                                        g.m1, nu.ax[1].tw, nu.ax[1].tid, nu.ax[1].off));
  // axis 0 + apply: 8 columns x ceil(m0 / kColLS) segments per block
  const int S = (g.m0 + kColLS - 1) / kColLS;
  const unsigned cblocks = unsigned((g.m1 + kColW - 1) / kColW);
  MGRX_LAUNCH(ex, "f2_cols", pdl_launch(k_f2_cols<T>, dim3(cblocks), dim3(unsigned(S * kColW)),
                                        size_t(2) * S * kColW * 8, ex.s, !ex.prof, static_cast<const double*>(G),
                                        coarse, sign, g.m0, g.m1, nu.ax[0].tw, nu.ax[0].tid, nu.ax[0].off));
  return cudaGetLastError();
}

F2Tabs tabs_of(const NuLevel& nu) {
  F2Tabs t;
  t.wl0 = nu.ax[0].wl;
  t.wr0 = nu.ax[0].wr;
  t.wl1 = nu.ax[1].wl;
  t.wr1 = nu.ax[1].wr;
  t.s0 = nu.ax[0].s;
  t.s1 = nu.ax[1].s;
  return t;
}

}  // namespace

Fused2DPlan fused2d_plan(const LevelGeom& lg) {
  Fused2DPlan fp;
  if (lg.d != 2 || std::getenv("MGRX_NO_F2")) return fp;
  F2Geom& g = fp.g;
  g.n0 = int(lg.n[0]);
  g.n1 = int(lg.n[1]);
  g.m0 = int(lg.m[0]);
  g.m1 = int(lg.m[1]);
  // long enough rows for the strips, columns that fit one axis-0 block, and
  // enough work to beat the per-step kernels
  if (g.n0 < 5 || g.n1 < 5 || g.m0 > 128 * kColLS || int64_t(g.n0) * g.n1 < (int64_t(1) << 13)) return fp;
  g.strips = (g.m1 + kF2Strip - 1) / kF2Strip;
  // coarse rows per CTA: about two waves of 8 resident CTAs per SM (a CTA
  // streams its rows one after the other, latency bound), 2..32
  g.chunk = int(std::max<int64_t>(2, std::min<int64_t>(32, int64_t(g.m0) * g.strips / (kNumSMs * 16))));
  if (const char* e = std::getenv("MGRX_F2_CHUNK")) g.chunk = std::max(1, std::atoi(e));
  g.chunks = (g.m0 + g.chunk - 1) / g.chunk;
  fp.enabled = true;
  fp.scratch_bytes = size_t(g.m0) * g.m1 * 8;
  return fp;
}

template <typename T>
cudaError_t fused2d_decompose_level(const T* blk, T* shell, T* coarse, void* scratch, const Fused2DPlan& fp,
                                    const NuLevel& nu, const Exec& ex) {
  double* G = static_cast<double*>(scratch);
  cudaError_t e = launch_pass<T>(blk, shell, coarse, G, fp.g, tabs_of(nu), true, ex);
  if (e != cudaSuccess) return e;
  return launch_solves<T>(G, coarse, 1.0, fp.g, nu, ex);
}

template <typename T>
cudaError_t fused2d_recompose_level(const T* shell, T* coarse, T* fine, void* scratch, const Fused2DPlan& fp,
                                    const NuLevel& nu, const Exec& ex) {
  double* G = static_cast<double*>(scratch);
  cudaError_t e = launch_pass<T>(shell, nullptr, nullptr, G, fp.g, tabs_of(nu), false, ex);
  if (e != cudaSuccess) return e;
  e = launch_solves<T>(G, coarse, -1.0, fp.g, nu, ex);
  if (e != cudaSuccess) return e;
  const dim3 grid(unsigned((fp.g.m1 + 255) / 256), unsigned(fp.g.n0));
  MGRX_LAUNCH(ex, "f2_interp", pdl_launch(k_f2_interp<T>, grid, dim3(256), 0, ex.s, !ex.prof, shell,
                                          static_cast<const T*>(coarse), fine, fp.g, tabs_of(nu)));
  return cudaGetLastError();
}

template cudaError_t fused2d_decompose_level<float>(const float*, float*, float*, void*, const Fused2DPlan&,
                                                    const NuLevel&, const Exec&);
template cudaError_t fused2d_decompose_level<double>(const double*, double*, double*, void*, const Fused2DPlan&,
                                                     const NuLevel&, const Exec&);
template cudaError_t fused2d_recompose_level<float>(const float*, float*, float*, void*, const Fused2DPlan&,
                                                    const NuLevel&, const Exec&);
template cudaError_t fused2d_recompose_level<double>(const double*, double*, double*, void*, const Fused2DPlan&,
                                                     const NuLevel&, const Exec&);

}  // namespace mgrx_b200
