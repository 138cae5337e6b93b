// General per-step kernels: any rank 1..8, any extents >= 2, fp32/fp64,
// uniform and nonuniform coordinates.
//
// These follow the reference's per-element arithmetic exactly (same
// constants, same summation order, no FMA contraction, same axis order for
// the correction sweeps), so on the uniform path their output is
// bit-identical to the reference's decompose/recompose.  They are the
// correctness backbone and the path for shapes the fused 3-D kernels
// (fused3d.cu) do not take.
//
// Layout: every level block lives compact and in natural order (the
// reference keeps it as the reordered corner of the full array,
// reorder.hpp:131); the multilevel component is a separate fp64 array in
// natural order (the reference materialises it in reordered order,
// transform.hpp:343-381).  The level-centric output layout is produced
// directly by computing each coefficient's shell position.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace mgrx_b200 {

// --------------------------------------------------------------- indexing

// D > 0: rank known at compile time (loops unroll, indices stay in
// registers); D == 0: runtime rank g.d.
#define MGRX_ND(g) (D > 0 ? D : (g).d)

template <bool kIdx32, int D = 0>
__device__ __forceinline__ void unravel(int64_t p, const LevelGeom& g, int64_t* j) {
  if (kIdx32) {
    uint32_t q = uint32_t(p);
#pragma unroll
    for (int i = MGRX_ND(g) - 1; i > 0; --i) {
      const uint32_t qq = g.fn[i].div(q);
      j[i] = int64_t(q - qq * uint32_t(g.n[i]));
      q = qq;
    }
    j[0] = q;
  } else {
    for (int i = MGRX_ND(g) - 1; i > 0; --i) {
      j[i] = p % g.n[i];
      p /= g.n[i];
    }
    j[0] = p;
  }
}

// Shell position of a coefficient node (pack_level_centric,
// reorder.hpp:180-215): rows of the reordered level block in row-major
// order; a row whose leading reordered indices are all nodal contributes
// only its coefficient tail [m_{d-1}, n_{d-1}).
template <int D = 0>
__device__ __forceinline__ int64_t shell_pos(const LevelGeom& g, const int64_t* j) {
  const int d = MGRX_ND(g);
  int64_t row = 0, before = 0;
  bool inside = true;
#pragma unroll
  for (int i = 0; i + 1 < d; ++i) {
    const int64_t r = (j[i] & 1) ? g.m[i] + (j[i] >> 1) : (j[i] >> 1);
    row = row * g.n[i] + r;
    if (inside) {
      if (r < g.m[i]) {
        before += r * g.pm[i];
      } else {
        before += g.m[i] * g.pm[i];
        inside = false;
      }
    }
  }
  const int64_t jl = j[d - 1];
  const int64_t rl = (jl & 1) ? g.m[d - 1] + (jl >> 1) : (jl >> 1);
  return row * g.n[d - 1] - before * g.m[d - 1] + (inside ? rl - g.m[d - 1] : rl);
}

// Multilinear prediction at node j from nodal values.  Uniform path:
// corner_average (transform.hpp:206-212) with update_coefficients' corner
// enumeration (:223-301) — set axes ascending, cmask ascending, a degenerate
// even-axis end counting its single neighbour twice, sum * 2^-k.
// src is either the natural fine block (coarse == false) or the compact
// coarse block (coarse == true).
template <typename T, bool kNu, int D = 0>
__device__ __forceinline__ double predict(const T* __restrict__ src, bool coarse, const LevelGeom& g,
                                          const NuLevel& nu, const int64_t* j) {
  // per axis (compile-time indices, registers): is it odd, the offset of the
  // right corner (0 on a degenerate even-axis end), its bit in the cmask
  // (odd axes ascending)
  int k = 0;
  int64_t base = 0;
  int64_t dl[kMaxD];
  int bit[kMaxD];
#pragma unroll
  for (int i = 0; i < MGRX_ND(g); ++i) {
    const int64_t stride = coarse ? g.cst[i] : g.st[i];
    const bool odd = j[i] & 1;
    dl[i] = (odd && j[i] + 1 < g.n[i]) ? (coarse ? g.cst[i] : 2 * g.st[i]) : 0;
    bit[i] = odd ? k : -1;
    k += odd ? 1 : 0;
    base += (coarse ? (odd ? (j[i] - 1) >> 1 : j[i] >> 1) : (odd ? j[i] - 1 : j[i])) * stride;
  }
  // corners in cmask order, summed in that order
  double sum = 0.0;
  for (unsigned cm = 0; cm < (1u << k); ++cm) {
    int64_t off = base;
    double wprod = 1.0;
#pragma unroll
    for (int i = 0; i < MGRX_ND(g); ++i) {
      if (bit[i] < 0) continue;
      const bool right = (cm >> bit[i]) & 1u;
      if (right) off += dl[i];
      if (kNu) wprod = mul_(wprod, right ? nu.ax[i].wr[j[i]] : nu.ax[i].wl[j[i]]);
    }
    const double v = double(src[off]);
    sum = kNu ? add_(sum, mul_(wprod, v)) : add_(sum, v);
  }
  return kNu ? sum : mul_(sum, 1.0 / double(1u << k));
}

// ------------------------------------------------------------ decompose
// reorder_level + compute_coefficients (transform.hpp:310) + the component
// materialisation of compute_correction (:343-381) + the shell part of
// pack_level_centric, one thread per fine node.
template <typename T, bool kIdx32, bool kNu, int D>
__global__ void __launch_bounds__(256) k_dec_coef(const T* __restrict__ blk, T* __restrict__ shell,
                                                  T* __restrict__ coarse, double* __restrict__ comp,
                                                  const LevelGeom g, const NuLevel nu) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < g.N; p += stride) {
    int64_t j[kMaxD];
    unravel<kIdx32, D>(p, g, j);
    bool nodal = true;
    for (int i = 0; i < MGRX_ND(g); ++i) nodal &= !(j[i] & 1);
    if (nodal) {
      int64_t c = 0;
      for (int i = 0; i < MGRX_ND(g); ++i) c += (j[i] >> 1) * g.cst[i];
      coarse[c] = blk[p];
      comp[p] = 0.0;
    } else {
      const double pred = predict<T, kNu, D>(blk, false, g, nu, j);
      const T v = to_t<T>(sub_(double(blk[p]), pred));
      comp[p] = double(v);
      shell[shell_pos<D>(g, j)] = v;
    }
  }
}

// One tensor-product sweep of compute_correction (transform.hpp:392-428)
// along an axis: load vector (load_entry :84-96) + Thomas solve
// (batched_solve :116-130), one thread per line; consecutive threads take
// consecutive positions of the trailing axes so accesses coalesce whenever
// the swept axis is not the last one.
template <bool kNu>
__global__ void __launch_bounds__(128) k_sweep(const double* __restrict__ x, double* __restrict__ y,
                                               int64_t outer, int64_t inner, int64_t n, int64_t m,
                                               const double* __restrict__ w, const double* __restrict__ inv_d,
                                               const NuAxis nu) {
  const int64_t lines = outer * inner;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t0 < lines; t0 += stride) {
    const int64_t o = t0 / inner, t = t0 - o * inner;
    const double* c = x + o * n * inner + t;
    double* f = y + o * m * inner + t;
    double prev = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      if (kNu) {
        const double* s = nu.s + 5 * i;
        for (int k = 0; k < 5; ++k) {
          const int64_t jj = 2 * i + k - 2;
          if (jj >= 0 && jj < n) acc = add_(acc, mul_(s[k], c[jj * inner]));
        }
        if (i > 0) acc = sub_(acc, mul_(nu.tw[i], prev));
      } else {
        if (i >= 1) {
          acc = add_(acc, mul_(kW12, c[(2 * i - 2) * inner]));
          acc = add_(acc, mul_(0.5, c[(2 * i - 1) * inner]));
        }
        acc = add_(acc, mul_((i == 0 || i + 1 == m) ? kW5_12 : kW5_6, c[(2 * i) * inner]));
        if (2 * i + 1 < n) acc = add_(acc, mul_(0.5, c[(2 * i + 1) * inner]));
        if (2 * i + 2 < n) acc = add_(acc, mul_(kW12, c[(2 * i + 2) * inner]));
        if (i > 0) acc = sub_(acc, mul_(w[i], prev));
      }
      f[i * inner] = acc;
      prev = acc;
    }
    double nxt = mul_(prev, kNu ? nu.tid[m - 1] : inv_d[m - 1]);
    f[(m - 1) * inner] = nxt;
    for (int64_t i = m - 2; i >= 0; --i) {
      const double v = kNu ? mul_(sub_(f[i * inner], mul_(nu.off[i], nxt)), nu.tid[i])
                           : mul_(sub_(f[i * inner], mul_(kOff, nxt)), inv_d[i]);
      f[i * inner] = v;
      nxt = v;
    }
  }
}

// Parallel form of a sweep (path "auto"): the load vector as one fully
// parallel stencil pass (same arithmetic and order as k_sweep, so the load
// is bit-identical), then the Thomas solve split into segments per line
// (affine carries folded through shared memory, each segment rerun from its
// true carry) — rounding-level differences from the serial sweep only.
template <bool kNu>
__global__ void __launch_bounds__(256) k_axis_load(const double* __restrict__ x, double* __restrict__ y,
                                                   int64_t outer, int64_t inner, int64_t n, int64_t m,
                                                   const double* __restrict__ s5) {
  const int64_t total = outer * m * inner;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += stride) {
    const int64_t t = q % inner, oi = q / inner;
    const int64_t i = oi % m, o = oi / m;
    const double* c = x + o * n * inner + t;
    double acc = 0.0;
    if (kNu) {
      const double* sk = s5 + 5 * i;
      for (int k = 0; k < 5; ++k) {
        const int64_t jj = 2 * i + k - 2;
        if (jj >= 0 && jj < n) acc = add_(acc, mul_(sk[k], c[jj * inner]));
      }
    } else {
      if (i >= 1) {
        acc = add_(acc, mul_(kW12, c[(2 * i - 2) * inner]));
        acc = add_(acc, mul_(0.5, c[(2 * i - 1) * inner]));
      }
      acc = add_(acc, mul_((i == 0 || i + 1 == m) ? kW5_12 : kW5_6, c[(2 * i) * inner]));
      if (2 * i + 1 < n) acc = add_(acc, mul_(0.5, c[(2 * i + 1) * inner]));
      if (2 * i + 2 < n) acc = add_(acc, mul_(kW12, c[(2 * i + 2) * inner]));
    }
    y[q] = acc;
  }
}

// Thomas (batched_solve, transform.hpp:116-130; nonuniform: super-diagonal
// table `off`) along lines of m values at stride `inner`, in place.  16
// lines per block, S = 2 blockDim.y segments per line; values stream from
// global memory (L1/L2) in each of the four segment passes.
__global__ void __launch_bounds__(1024) k_axis_solve(double* __restrict__ y, int64_t nlines, int64_t m, int64_t inner,
                                                     const double* __restrict__ w, const double* __restrict__ inv_d,
                                                     const double* __restrict__ off) {
  __shared__ double A[64][16], B[64][16];
  const int lane = threadIdx.x, c16 = lane & 15, s = 2 * threadIdx.y + (lane >> 4), S = 2 * blockDim.y;
  const int64_t line = int64_t(blockIdx.x) * 16 + c16;
  const bool valid = line < nlines;
  const int64_t base = valid ? (line / inner) * m * inner + line % inner : 0;
  const int64_t seg = (m + S - 1) / S;
  const int64_t s0 = min(m, int64_t(s) * seg), s1 = min(m, s0 + seg);
  double* p = y + base;
  // forward y_i = f_i - w_i y_{i-1}: segment map from a zero carry
  double ya = 0.0, yb = 1.0;
  for (int64_t i = s0; i < s1; ++i) {
    const double f = valid ? p[i * inner] : 0.0;
    const double wi = w[i];
    ya = f - wi * ya;
    yb = -wi * yb;
  }
  A[s][c16] = ya;
  B[s][c16] = yb;
  __syncthreads();
  double c = 0.0;
  for (int q = 0; q < s; ++q) c = A[q][c16] + B[q][c16] * c;
  __syncthreads();
  for (int64_t i = s0; i < s1; ++i) {
    const double f = valid ? p[i * inner] : 0.0;
    c = f - w[i] * c;
    if (valid) p[i * inner] = c;
  }
  // back substitution z_i = (y_i - off_i z_{i+1}) / d_i, z_m = 0
  double za = 0.0, zb = 1.0;
  for (int64_t i = s1 - 1; i >= s0; --i) {
    const double yv = valid ? p[i * inner] : 0.0;
    const double id = inv_d[i], oi = off ? off[i] : kOff;
    za = (yv - oi * za) * id;
    zb = -oi * id * zb;
  }
  A[s][c16] = za;
  B[s][c16] = zb;
  __syncthreads();
  double z = 0.0;
  for (int q = S - 1; q > s; --q) z = A[q][c16] + B[q][c16] * z;
  for (int64_t i = s1 - 1; i >= s0; --i) {
    const double yv = valid ? p[i * inner] : 0.0;
    z = (yv - (off ? off[i] : kOff) * z) * inv_d[i];
    if (valid) p[i * inner] = z;
  }
}

// Last-axis variant (contiguous lines): one warp per line, the line staged
// in shared memory, lanes own contiguous segments (affine carries combined
// with a warp shuffle scan, then exact reruns).
__global__ void __launch_bounds__(128) k_axis_solve_rows(double* __restrict__ y, int64_t nlines, int m,
                                                         const double* __restrict__ w,
                                                         const double* __restrict__ inv_d,
                                                         const double* __restrict__ off) {
  extern __shared__ double rowbuf[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* x = rowbuf + int64_t(warp) * m;
  const int seg = (m + 31) >> 5;
  const int s0 = min(m, lane * seg), s1 = min(m, s0 + seg);
  for (int64_t line = int64_t(blockIdx.x) * nw + warp; line < nlines; line += int64_t(gridDim.x) * nw) {
    double* gl = y + line * m;
    for (int i = lane; i < m; i += 32) x[i] = gl[i];
    __syncwarp();
    // forward
    double fa = 0.0, fb = 1.0;
    for (int i = s0; i < s1; ++i) {
      const double wi = w[i];
      fa = x[i] - wi * fa;
      fb = -wi * fb;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double pa = __shfl_up_sync(0xffffffffu, fa, o), pb = __shfl_up_sync(0xffffffffu, fb, o);
      if (lane >= o) {
        fa = fa + fb * pa;
        fb = fb * pb;
      }
    }
    double c = __shfl_up_sync(0xffffffffu, fa, 1);
    if (lane == 0) c = 0.0;
    for (int i = s0; i < s1; ++i) {
      c = x[i] - w[i] * c;
      x[i] = c;
    }
    // backward z_i = (y_i - off_i z_{i+1}) / d_i
    double ga = 0.0, gb = 1.0;
    for (int i = s1 - 1; i >= s0; --i) {
      const double id = inv_d[i], oi = off ? off[i] : kOff;
      ga = (x[i] - oi * ga) * id;
      gb = -oi * id * gb;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double na = __shfl_down_sync(0xffffffffu, ga, o), nb = __shfl_down_sync(0xffffffffu, gb, o);
      if (lane + o < 32) {
        ga = ga + gb * na;
        gb = gb * nb;
      }
    }
    double z = __shfl_down_sync(0xffffffffu, ga, 1);
    if (lane == 31) z = 0.0;
    for (int i = s1 - 1; i >= s0; --i) {
      z = (x[i] - (off ? off[i] : kOff) * z) * inv_d[i];
      x[i] = z;
    }
    __syncwarp();
    for (int i = lane; i < m; i += 32) gl[i] = x[i];
    __syncwarp();
  }
}

// apply_correction (transform.hpp:435-477): corner <- T(double(corner) + s*z).
template <typename T>
__global__ void __launch_bounds__(256) k_apply(T* __restrict__ coarse, const double* __restrict__ z, int64_t nc,
                                               double sign) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < nc; p += stride)
    coarse[p] = to_t<T>(add_(double(coarse[p]), mul_(sign, z[p])));
}

// ------------------------------------------------------------ recompose
// Component of a level from its shell (unpack_level_centric reorder.hpp:221
// + the materialisation of compute_correction).
template <typename T, bool kIdx32, int D>
__global__ void __launch_bounds__(256) k_rec_comp(const T* __restrict__ shell, double* __restrict__ comp,
                                                  const LevelGeom g) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < g.N; p += stride) {
    int64_t j[kMaxD];
    unravel<kIdx32, D>(p, g, j);
    bool nodal = true;
    for (int i = 0; i < MGRX_ND(g); ++i) nodal &= !(j[i] & 1);
    comp[p] = nodal ? 0.0 : double(shell[shell_pos<D>(g, j)]);
  }
}

// add_interpolant (transform.hpp:317) + inverse_reorder_level
// (reorder.hpp:138): fine natural block from corrected coarse nodes and the
// shell coefficients.
template <typename T, bool kIdx32, bool kNu, int D>
__global__ void __launch_bounds__(256) k_rec_interp(const T* __restrict__ shell, const T* __restrict__ coarse,
                                                    T* __restrict__ fine, const LevelGeom g, const NuLevel nu) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < g.N; p += stride) {
    int64_t j[kMaxD];
    unravel<kIdx32, D>(p, g, j);
    bool nodal = true;
    for (int i = 0; i < MGRX_ND(g); ++i) nodal &= !(j[i] & 1);
    if (nodal) {
      int64_t c = 0;
      for (int i = 0; i < MGRX_ND(g); ++i) c += (j[i] >> 1) * g.cst[i];
      fine[p] = coarse[c];
    } else {
      const double pred = predict<T, kNu, D>(coarse, true, g, nu, j);
      fine[p] = to_t<T>(add_(double(shell[shell_pos<D>(g, j)]), pred));
    }
  }
}

// ------------------------------------------------------------------ tail
// All small levels of a hierarchy in one CTA: the level blocks, the fp64
// component and the sweep buffer live in shared memory, and each step of the
// per-level sequence above (coefficients, the d sweeps, apply) is a
// block-wide loop separated by __syncthreads.  Same arithmetic as the
// per-step kernels, so results stay bit-identical to the reference.
struct TailLevel {
  LevelGeom g;
  ThomasLevel th;
  int64_t shell_off;  // node_count(l-1): shell position in the level-centric buffer
};

template <int D, bool kNu>
__device__ __forceinline__ void tail_sweeps(double* comp, double* tmp, const LevelGeom& g, const ThomasLevel& th,
                                            const NuLevel& nu, double** result) {
  int cur[kMaxD];
#pragma unroll
  for (int i = 0; i < MGRX_ND(g); ++i) cur[i] = int(g.n[i]);
  double* x = comp;
  double* y = tmp;
#pragma unroll
  for (int a = 0; a < MGRX_ND(g); ++a) {
    int outer = 1, inner = 1;
#pragma unroll
    for (int i = 0; i < MGRX_ND(g); ++i) {
      if (i < a) outer *= cur[i];
      if (i > a) inner *= cur[i];
    }
    const int n = int(g.n[a]), m = int(g.m[a]);
    const double* w = th.w[a];
    const double* inv_d = th.inv_d[a];
    for (int t0 = threadIdx.x; t0 < outer * inner; t0 += blockDim.x) {
      const int o = t0 / inner, t = t0 - o * inner;
      const double* c = x + o * n * inner + t;
      double* f = y + o * m * inner + t;
      double prev = 0.0;
      for (int i = 0; i < m; ++i) {
        double acc = 0.0;
        if (kNu) {  // same arithmetic as k_sweep<true>
          const double* sk = nu.ax[a].s + 5 * i;
          for (int k = 0; k < 5; ++k) {
            const int jj = 2 * i + k - 2;
            if (jj >= 0 && jj < n) acc = add_(acc, mul_(sk[k], c[jj * inner]));
          }
          if (i > 0) acc = sub_(acc, mul_(nu.ax[a].tw[i], prev));
        } else {
          if (i >= 1) {
            acc = add_(acc, mul_(kW12, c[(2 * i - 2) * inner]));
            acc = add_(acc, mul_(0.5, c[(2 * i - 1) * inner]));
          }
          acc = add_(acc, mul_((i == 0 || i + 1 == m) ? kW5_12 : kW5_6, c[(2 * i) * inner]));
          if (2 * i + 1 < n) acc = add_(acc, mul_(0.5, c[(2 * i + 1) * inner]));
          if (2 * i + 2 < n) acc = add_(acc, mul_(kW12, c[(2 * i + 2) * inner]));
          if (i > 0) acc = sub_(acc, mul_(w[i], prev));
        }
        f[i * inner] = acc;
        prev = acc;
      }
      double nxt = mul_(prev, kNu ? nu.ax[a].tid[m - 1] : inv_d[m - 1]);
      f[(m - 1) * inner] = nxt;
      for (int i = m - 2; i >= 0; --i) {
        const double v = kNu ? mul_(sub_(f[i * inner], mul_(nu.ax[a].off[i], nxt)), nu.ax[a].tid[i])
                             : mul_(sub_(f[i * inner], mul_(kOff, nxt)), inv_d[i]);
        f[i * inner] = v;
        nxt = v;
      }
    }
    __syncthreads();
    cur[a] = g.m[a];
    double* tswap = x;
    x = y;
    y = tswap;
  }
  *result = x;
}

// Decompose levels levels[0] (finest, block read from `blk`) down to the
// last entry; shells go to out + shell_off, the final coarse block to `coarse_out`.
template <typename T, int D, bool kNu>
__global__ void __launch_bounds__(1024) k_tail_decompose(const T* __restrict__ blk, T* __restrict__ out,
                                                         T* __restrict__ coarse_out, const TailLevel* __restrict__ lv,
                                                         const NuLevel* __restrict__ nul, int nlev, int64_t nmax) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* comp = reinterpret_cast<double*>(smem);
  double* tmp = comp + nmax;
  T* A = reinterpret_cast<T*>(tmp + nmax);
  T* B = A + nmax;
  pdl_wait();
  for (int64_t p = threadIdx.x; p < lv[0].g.N; p += blockDim.x) A[p] = blk[p];
  __syncthreads();
  T* cur = A;
  T* nxt = B;
  for (int k = 0; k < nlev; ++k) {
    const LevelGeom& g = lv[k].g;
    const NuLevel nu = kNu ? nul[k] : NuLevel{};
    T* shell = out + lv[k].shell_off;
    for (int64_t p = threadIdx.x; p < g.N; p += blockDim.x) {
      int64_t j[kMaxD];
      unravel<true, D>(p, g, j);
      bool nodal = true;
      for (int i = 0; i < MGRX_ND(g); ++i) nodal &= !(j[i] & 1);
      if (nodal) {
        int64_t cc = 0;
        for (int i = 0; i < MGRX_ND(g); ++i) cc += (j[i] >> 1) * g.cst[i];
        nxt[cc] = cur[p];
        comp[p] = 0.0;
      } else {
        const double pred = predict<T, kNu, D>(cur, false, g, nu, j);
        const T v = to_t<T>(sub_(double(cur[p]), pred));
        comp[p] = double(v);
        shell[shell_pos<D>(g, j)] = v;
      }
    }
    __syncthreads();
    double* z = nullptr;
    tail_sweeps<D, kNu>(comp, tmp, g, lv[k].th, nu, &z);
    for (int64_t p = threadIdx.x; p < g.Nc; p += blockDim.x) nxt[p] = to_t<T>(add_(double(nxt[p]), mul_(1.0, z[p])));
    __syncthreads();
    T* t = cur;
    cur = nxt;
    nxt = t;
  }
  for (int64_t p = threadIdx.x; p < lv[nlev - 1].g.Nc; p += blockDim.x) coarse_out[p] = cur[p];
}

// Recompose from the coarse block (`coarse_in`, level of the first entry's
// coarse side) up through the entries (coarsest first); the last fine block
// goes to `fine_out`.
template <typename T, int D, bool kNu>
__global__ void __launch_bounds__(1024) k_tail_recompose(const T* __restrict__ coeffs, const T* __restrict__ coarse_in,
                                                         T* __restrict__ fine_out, const TailLevel* __restrict__ lv,
                                                         const NuLevel* __restrict__ nul, int nlev, int64_t nmax) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* comp = reinterpret_cast<double*>(smem);
  double* tmp = comp + nmax;
  T* A = reinterpret_cast<T*>(tmp + nmax);
  T* B = A + nmax;
  pdl_wait();
  for (int64_t p = threadIdx.x; p < lv[0].g.Nc; p += blockDim.x) A[p] = coarse_in[p];
  __syncthreads();
  T* cur = A;  // coarse block of the current level
  T* fin = B;
  for (int k = 0; k < nlev; ++k) {
    const LevelGeom& g = lv[k].g;
    const NuLevel nu = kNu ? nul[k] : NuLevel{};
    const T* shell = coeffs + lv[k].shell_off;
    for (int64_t p = threadIdx.x; p < g.N; p += blockDim.x) {
      int64_t j[kMaxD];
      unravel<true, D>(p, g, j);
      bool nodal = true;
      for (int i = 0; i < MGRX_ND(g); ++i) nodal &= !(j[i] & 1);
      comp[p] = nodal ? 0.0 : double(shell[shell_pos<D>(g, j)]);
    }
    __syncthreads();
    double* z = nullptr;
    tail_sweeps<D, kNu>(comp, tmp, g, lv[k].th, nu, &z);
    for (int64_t p = threadIdx.x; p < g.Nc; p += blockDim.x) cur[p] = to_t<T>(add_(double(cur[p]), mul_(-1.0, z[p])));
    __syncthreads();
    T* dst = (k == nlev - 1) ? fine_out : fin;
    for (int64_t p = threadIdx.x; p < g.N; p += blockDim.x) {
      int64_t j[kMaxD];
      unravel<true, D>(p, g, j);
      bool nodal = true;
      for (int i = 0; i < MGRX_ND(g); ++i) nodal &= !(j[i] & 1);
      if (nodal) {
        int64_t cc = 0;
        for (int i = 0; i < MGRX_ND(g); ++i) cc += (j[i] >> 1) * g.cst[i];
        dst[p] = cur[cc];
      } else {
        const double pred = predict<T, kNu, D>(cur, true, g, nu, j);
        dst[p] = to_t<T>(add_(double(shell[shell_pos<D>(g, j)]), pred));
      }
    }
    __syncthreads();
    T* t = cur;
    cur = fin;
    fin = t;
  }
}

size_t tail_smem_bytes(int64_t nmax, int esize) { return size_t(nmax) * (16 + 2 * size_t(esize)); }

template <typename T, int D>
static cudaError_t tail_dec_t(const T* blk, T* out, T* coarse_out, const void* d_levels, const void* d_nu, int nlev,
                              int64_t nmax, const Exec& ex) {
  const size_t sm = tail_smem_bytes(nmax, sizeof(T));
  const TailLevel* lv = static_cast<const TailLevel*>(d_levels);
  const NuLevel* nul = static_cast<const NuLevel*>(d_nu);
  if (nul) {
    cudaError_t e = cudaFuncSetAttribute(k_tail_decompose<T, D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(sm));
    if (e != cudaSuccess) return e;
    MGRX_LAUNCH(ex, "tail_dec", pdl_launch(k_tail_decompose<T, D, true>, dim3(1), dim3(1024), sm, ex.s, !ex.prof, blk,
                                           out, coarse_out, lv, nul, nlev, nmax));
  } else {
    cudaError_t e = cudaFuncSetAttribute(k_tail_decompose<T, D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(sm));
    if (e != cudaSuccess) return e;
    MGRX_LAUNCH(ex, "tail_dec", pdl_launch(k_tail_decompose<T, D, false>, dim3(1), dim3(1024), sm, ex.s, !ex.prof, blk,
                                           out, coarse_out, lv, nul, nlev, nmax));
  }
  return cudaGetLastError();
}

template <typename T, int D>
static cudaError_t tail_rec_t(const T* coeffs, const T* coarse_in, T* fine_out, const void* d_levels, const void* d_nu,
                              int nlev, int64_t nmax, const Exec& ex) {
  const size_t sm = tail_smem_bytes(nmax, sizeof(T));
  const TailLevel* lv = static_cast<const TailLevel*>(d_levels);
  const NuLevel* nul = static_cast<const NuLevel*>(d_nu);
  if (nul) {
    cudaError_t e = cudaFuncSetAttribute(k_tail_recompose<T, D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(sm));
    if (e != cudaSuccess) return e;
    MGRX_LAUNCH(ex, "tail_rec", pdl_launch(k_tail_recompose<T, D, true>, dim3(1), dim3(1024), sm, ex.s, !ex.prof,
                                           coeffs, coarse_in, fine_out, lv, nul, nlev, nmax));
  } else {
    cudaError_t e = cudaFuncSetAttribute(k_tail_recompose<T, D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(sm));
    if (e != cudaSuccess) return e;
    MGRX_LAUNCH(ex, "tail_rec", pdl_launch(k_tail_recompose<T, D, false>, dim3(1), dim3(1024), sm, ex.s, !ex.prof,
                                           coeffs, coarse_in, fine_out, lv, nul, nlev, nmax));
  }
  return cudaGetLastError();
}

// Rank-specialised tails for 1-3 dimensions (the common cases), runtime
// rank otherwise; d_nu: per-level nonuniform tables (same order as the
// levels) or null for uniform coordinates.
template <typename T>
cudaError_t tail_decompose(const T* blk, T* out, T* coarse_out, const void* d_levels, const void* d_nu, int nlev,
                           int64_t nmax, int d, const Exec& ex) {
  switch (d) {
    case 1: return tail_dec_t<T, 1>(blk, out, coarse_out, d_levels, d_nu, nlev, nmax, ex);
    case 2: return tail_dec_t<T, 2>(blk, out, coarse_out, d_levels, d_nu, nlev, nmax, ex);
    case 3: return tail_dec_t<T, 3>(blk, out, coarse_out, d_levels, d_nu, nlev, nmax, ex);
    default: return tail_dec_t<T, 0>(blk, out, coarse_out, d_levels, d_nu, nlev, nmax, ex);
  }
}

template <typename T>
cudaError_t tail_recompose(const T* coeffs, const T* coarse_in, T* fine_out, const void* d_levels, const void* d_nu,
                           int nlev, int64_t nmax, int d, const Exec& ex) {
  switch (d) {
    case 1: return tail_rec_t<T, 1>(coeffs, coarse_in, fine_out, d_levels, d_nu, nlev, nmax, ex);
    case 2: return tail_rec_t<T, 2>(coeffs, coarse_in, fine_out, d_levels, d_nu, nlev, nmax, ex);
    case 3: return tail_rec_t<T, 3>(coeffs, coarse_in, fine_out, d_levels, d_nu, nlev, nmax, ex);
    default: return tail_rec_t<T, 0>(coeffs, coarse_in, fine_out, d_levels, d_nu, nlev, nmax, ex);
  }
}

size_t tail_level_bytes() { return sizeof(TailLevel); }

void tail_fill_level(void* dst, const LevelGeom& g, const ThomasLevel& th, int64_t shell_off) {
  TailLevel t;
  t.g = g;
  t.th = th;
  t.shell_off = shell_off;
  *static_cast<TailLevel*>(dst) = t;
}

// ------------------------------------------------------------- launchers

// Rank-specialised variants (32-bit indexing, d = 2, 3, 4: the index
// arithmetic unrolls and stays in registers); the runtime-rank kernels
// cover the rest and 64-bit node counts.
#define MGRX_BY_RANK(LAUNCH)                          \
  if (g.N < (int64_t(1) << 32) && g.d == 2) {          \
    LAUNCH(true, 2);                                   \
  } else if (g.N < (int64_t(1) << 32) && g.d == 3) {   \
    LAUNCH(true, 3);                                   \
  } else if (g.N < (int64_t(1) << 32) && g.d == 4) {   \
    LAUNCH(true, 4);                                   \
  } else if (g.N < (int64_t(1) << 32)) {               \
    LAUNCH(true, 0);                                   \
  } else {                                             \
    LAUNCH(false, 0);                                  \
  }

template <typename T>
static void launch_dec_coef(const T* blk, T* shell, T* coarse, double* comp, const LevelGeom& g, const NuLevel* nu,
                            const Exec& ex) {
  const int grid = grid_for(g.N, 256);
  const NuLevel z = nu ? *nu : NuLevel{};
#define L_(I32, D)                                                                                              \
  if (nu)                                                                                                       \
    MGRX_LAUNCH(ex, "gen_dec_coef", k_dec_coef<T, I32, true, D><<<grid, 256, 0, ex.s>>>(blk, shell, coarse, comp, g, z)); \
  else                                                                                                          \
    MGRX_LAUNCH(ex, "gen_dec_coef", k_dec_coef<T, I32, false, D><<<grid, 256, 0, ex.s>>>(blk, shell, coarse, comp, g, z))
  MGRX_BY_RANK(L_)
#undef L_
}

template <typename T>
static void launch_rec_comp(const T* shell, double* comp, const LevelGeom& g, const Exec& ex) {
  const int grid = grid_for(g.N, 256);
#define L_(I32, D) MGRX_LAUNCH(ex, "gen_rec_comp", k_rec_comp<T, I32, D><<<grid, 256, 0, ex.s>>>(shell, comp, g))
  MGRX_BY_RANK(L_)
#undef L_
}

template <typename T>
static void launch_rec_interp(const T* shell, const T* coarse, T* fine, const LevelGeom& g, const NuLevel* nu,
                              const Exec& ex) {
  const int grid = grid_for(g.N, 256);
  const NuLevel z = nu ? *nu : NuLevel{};
#define L_(I32, D)                                                                                              \
  if (nu)                                                                                                       \
    MGRX_LAUNCH(ex, "gen_rec_interp", k_rec_interp<T, I32, true, D><<<grid, 256, 0, ex.s>>>(shell, coarse, fine, g, z)); \
  else                                                                                                          \
    MGRX_LAUNCH(ex, "gen_rec_interp", k_rec_interp<T, I32, false, D><<<grid, 256, 0, ex.s>>>(shell, coarse, fine, g, z))
  MGRX_BY_RANK(L_)
#undef L_
}

// compute_correction sweeps on `comp` (natural fine extents); the result
// (coarse extents, row-major) ends in *result, which points into comp or tmp.
static void run_sweeps(double* comp, double* tmp, const LevelGeom& g, const ThomasLevel* th, const NuLevel* nu,
                       double** result, const Exec& ex, bool fast) {
  int64_t cur[kMaxD];
  for (int i = 0; i < g.d; ++i) cur[i] = g.n[i];
  double* x = comp;
  double* y = tmp;
  for (int a = 0; a < g.d; ++a) {
    int64_t outer = 1, inner = 1;
    for (int i = 0; i < a; ++i) outer *= cur[i];
    for (int i = a + 1; i < g.d; ++i) inner *= cur[i];
    const int64_t lines = outer * inner;
    const int grid = grid_for(lines, 128, 32);
    // the serial per-line sweep saturates the GPU when there are many lines;
    // few long lines (2-D levels) need the segmented solve
    if (fast && lines < (int64_t(1) << 17)) {
      const int64_t outs = outer * g.m[a] * inner;
      if (nu)
        MGRX_LAUNCH(ex, "gen_load", k_axis_load<true><<<grid_for(outs, 256), 256, 0, ex.s>>>(x, y, outer, inner, g.n[a], g.m[a], nu->ax[a].s));
      else
        MGRX_LAUNCH(ex, "gen_load", k_axis_load<false><<<grid_for(outs, 256), 256, 0, ex.s>>>(x, y, outer, inner, g.n[a], g.m[a], nullptr));
      const int SY = int(std::max<int64_t>(1, std::min<int64_t>(32, (g.m[a] + 31) / 32)));
      const double* w = nu ? nu->ax[a].tw : th->w[a];
      const double* id = nu ? nu->ax[a].tid : th->inv_d[a];
      const double* of = nu ? nu->ax[a].off : nullptr;
      const size_t row_smem = size_t(4) * size_t(g.m[a]) * 8;
      if (inner == 1 && row_smem <= size_t(200) * 1024) {
        cudaFuncSetAttribute(k_axis_solve_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, int(row_smem));
        const int64_t blocks = std::min<int64_t>((lines + 3) / 4, int64_t(kNumSMs) * 8);
        MGRX_LAUNCH(ex, "gen_solve", k_axis_solve_rows<<<unsigned(blocks), 128, row_smem, ex.s>>>(y, lines, int(g.m[a]), w, id, of));
      } else {
        MGRX_LAUNCH(ex, "gen_solve", k_axis_solve<<<unsigned((lines + 15) / 16), dim3(32, SY), 0, ex.s>>>(y, lines, g.m[a], inner, w, id, of));
      }
    } else if (nu)
      MGRX_LAUNCH(ex, "gen_sweep", k_sweep<true><<<grid, 128, 0, ex.s>>>(x, y, outer, inner, g.n[a], g.m[a], nullptr, nullptr, nu->ax[a]));
    else
      MGRX_LAUNCH(ex, "gen_sweep", k_sweep<false><<<grid, 128, 0, ex.s>>>(x, y, outer, inner, g.n[a], g.m[a], th->w[a], th->inv_d[a], NuAxis{}));
    cur[a] = g.m[a];
    double* t = x;
    x = y;
    y = t;
  }
  *result = x;
}

template <typename T>
cudaError_t general_decompose_level(const T* blk, T* shell, T* coarse, double* comp, double* tmp, const LevelGeom& g,
                                    const ThomasLevel* th, const NuLevel* nu, const Exec& ex, bool fast) {
  launch_dec_coef<T>(blk, shell, coarse, comp, g, nu, ex);
  double* z = nullptr;
  run_sweeps(comp, tmp, g, th, nu, &z, ex, fast);
  MGRX_LAUNCH(ex, "gen_apply", k_apply<T><<<grid_for(g.Nc, 256), 256, 0, ex.s>>>(coarse, z, g.Nc, 1.0));
  return cudaGetLastError();
}

template <typename T>
cudaError_t general_recompose_level(const T* shell, T* coarse, T* fine, double* comp, double* tmp, const LevelGeom& g,
                                    const ThomasLevel* th, const NuLevel* nu, const Exec& ex, bool fast) {
  launch_rec_comp<T>(shell, comp, g, ex);
  double* z = nullptr;
  run_sweeps(comp, tmp, g, th, nu, &z, ex, fast);
  MGRX_LAUNCH(ex, "gen_apply", k_apply<T><<<grid_for(g.Nc, 256), 256, 0, ex.s>>>(coarse, z, g.Nc, -1.0));
  launch_rec_interp<T>(shell, coarse, fine, g, nu, ex);
  return cudaGetLastError();
}

#define MGRX_INST(T)                                                                                           \
  template cudaError_t general_decompose_level<T>(const T*, T*, T*, double*, double*, const LevelGeom&,         \
                                                  const ThomasLevel*, const NuLevel*, const Exec&, bool);       \
  template cudaError_t general_recompose_level<T>(const T*, T*, T*, double*, double*, const LevelGeom&,         \
                                                  const ThomasLevel*, const NuLevel*, const Exec&, bool);
MGRX_INST(float)
MGRX_INST(double)
#undef MGRX_INST

template cudaError_t tail_decompose<float>(const float*, float*, float*, const void*, const void*, int, int64_t, int,
                                           const Exec&);
template cudaError_t tail_decompose<double>(const double*, double*, double*, const void*, const void*, int, int64_t,
                                            int, const Exec&);
template cudaError_t tail_recompose<float>(const float*, const float*, float*, const void*, const void*, int, int64_t,
                                           int, const Exec&);
template cudaError_t tail_recompose<double>(const double*, const double*, double*, const void*, const void*, int,
                                            int64_t, int, const Exec&);

}  // namespace mgrx_b200
