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
#include "fused3d.h"
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

// k_sweep for contiguous lines (inner == 1): LINES consecutive lines are
// staged in shared memory with coalesced copies (a thread walking its own
// line directly would touch a different cache line per lane per step), each
// thread runs k_sweep's exact per-line arithmetic on its line, and the
// result lines go back coalesced.  Row strides are padded to odd lengths so
// the per-thread walks hit distinct banks.
template <bool kNu>
__global__ void __launch_bounds__(128) k_sweep_rows(const double* __restrict__ x, double* __restrict__ y, int64_t lines,
                                                    int n, int m, const double* __restrict__ w,
                                                    const double* __restrict__ inv_d, const NuAxis nu) {
  extern __shared__ double sw[];
  const int L = blockDim.x;
  const int ns = n | 1, ms = m | 1;
  double* in = sw;
  double* out = sw + int64_t(L) * ns;
  const int64_t l0 = int64_t(blockIdx.x) * L;
  const int nl = int(min(int64_t(L), lines - l0));
  const double* xs = x + l0 * n;
  for (int e = threadIdx.x; e < nl * n; e += L) {
    const int r = e / n;
    in[r * ns + (e - r * n)] = xs[e];
  }
  __syncthreads();
  if (threadIdx.x < nl) {
    const double* c = in + threadIdx.x * ns;
    double* f = out + threadIdx.x * ms;
    double prev = 0.0;
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      if (kNu) {
        const double* sk = nu.s + 5 * i;
        for (int k = 0; k < 5; ++k) {
          const int jj = 2 * i + k - 2;
          if (jj >= 0 && jj < n) acc = add_(acc, mul_(sk[k], c[jj]));
        }
        if (i > 0) acc = sub_(acc, mul_(nu.tw[i], prev));
      } else {
        if (i >= 1) {
          acc = add_(acc, mul_(kW12, c[2 * i - 2]));
          acc = add_(acc, mul_(0.5, c[2 * i - 1]));
        }
        acc = add_(acc, mul_((i == 0 || i + 1 == m) ? kW5_12 : kW5_6, c[2 * i]));
        if (2 * i + 1 < n) acc = add_(acc, mul_(0.5, c[2 * i + 1]));
        if (2 * i + 2 < n) acc = add_(acc, mul_(kW12, c[2 * i + 2]));
        if (i > 0) acc = sub_(acc, mul_(w[i], prev));
      }
      f[i] = acc;
      prev = acc;
    }
    double nxt = mul_(prev, kNu ? nu.tid[m - 1] : inv_d[m - 1]);
    f[m - 1] = nxt;
    for (int i = m - 2; i >= 0; --i) {
      const double v = kNu ? mul_(sub_(f[i], mul_(nu.off[i], nxt)), nu.tid[i]) : mul_(sub_(f[i], mul_(kOff, nxt)), inv_d[i]);
      f[i] = v;
      nxt = v;
    }
  }
  __syncthreads();
  double* ys = y + l0 * m;
  for (int e = threadIdx.x; e < nl * m; e += L) {
    const int r = e / m;
    ys[e] = out[r * ms + (e - r * m)];
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

// Coefficients (or, on recompose, the component read back from the shell)
// fused with the axis-0 load vector (path "auto", rank >= 2): each thread
// owns one position t of the trailing axes and a chunk of coarse rows
// [i0, i1) along axis 0, streams the fine rows 2 i0 - 2 .. 2 i1 through
// three rolling accumulators and writes the finished load entries f0[i][t]
// — the fp64 component is never materialised.  Per entry the products are
// added in load_entry's order (k = -2 .. 2, transform.hpp:84-96) starting
// from 0.0, exactly as k_axis_load does, so f0 is bit-identical to
// k_axis_load over k_dec_coef's component; coefficients are bit-identical
// to k_dec_coef.  Halo rows are recomputed by the neighbouring chunk, only
// the owned rows [2 i0, 2 i1) are written to the shell / coarse block.
template <typename T, bool kRec, bool kNu, int D>
__global__ void __launch_bounds__(256) k_coef_load0(const T* __restrict__ blk, T* __restrict__ shell,
                                                    T* __restrict__ coarse, double* __restrict__ f0,
                                                    const LevelGeom g, const NuLevel nu, int64_t inner, int chunk) {
  const int64_t n0 = g.n[0], m0 = g.m[0];
  const int64_t nch = (m0 + chunk - 1) / chunk;
  const int64_t total = nch * inner;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const double* s5 = kNu ? nu.ax[0].s : nullptr;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += stride) {
    const int64_t ch = q / inner, t = q - ch * inner;
    const int64_t i0 = ch * chunk, i1 = min(m0, i0 + chunk);
    int64_t j[kMaxD];
    bool even_tail = true;
    int64_t ct = 0;
    {
      int64_t r = t;
#pragma unroll
      for (int i = MGRX_ND(g) - 1; i >= 1; --i) {
        j[i] = r % g.n[i];
        r /= g.n[i];
        even_tail &= !(j[i] & 1);
        ct += (j[i] >> 1) * g.cst[i];
      }
    }
    const int64_t p_lo = i0 > 0 ? 2 * i0 - 2 : 0;
    const int64_t p_hi = min(n0 - 1, 2 * i1);
    double a_prev = 0.0, a_cur = 0.0, a_next = 0.0;  // rows k-1, k, k+1 for k = p >> 1
    for (int64_t p = p_lo; p <= p_hi; ++p) {
      const bool owned = p >= 2 * i0 && p < 2 * i1;
      j[0] = p;
      double c;
      if (!(p & 1) && even_tail) {  // nodal: component 0
        if (!kRec && owned) coarse[(p >> 1) * g.cst[0] + ct] = blk[p * inner + t];
        c = 0.0;
      } else if (kRec) {
        c = double(blk[shell_pos<D>(g, j)]);
      } else {
        const double pred = predict<T, kNu, D>(blk, false, g, nu, j);
        const T v = to_t<T>(sub_(double(blk[p * inner + t]), pred));
        if (owned) shell[shell_pos<D>(g, j)] = v;
        c = double(v);
      }
      const int64_t k = p >> 1;
      if (!(p & 1)) {
        if (k >= 1) {  // last term (offset +2) of row k-1
          a_prev = add_(a_prev, mul_(kNu ? s5[5 * (k - 1) + 4] : kW12, c));
          if (k - 1 >= i0 && k - 1 < i1) f0[(k - 1) * inner + t] = a_prev;
        }
        a_cur = add_(a_cur, mul_(kNu ? s5[5 * k + 2] : ((k == 0 || k + 1 == m0) ? kW5_12 : kW5_6), c));
        a_next = (k + 1 < m0) ? add_(0.0, mul_(kNu ? s5[5 * (k + 1)] : kW12, c)) : 0.0;
      } else {
        a_cur = add_(a_cur, mul_(kNu ? s5[5 * k + 3] : 0.5, c));
        if (k + 1 < m0) a_next = add_(a_next, mul_(kNu ? s5[5 * (k + 1) + 1] : 0.5, c));
        // advance: the next even row 2k+2 makes k+1 the current row
        if (p < p_hi) {
          a_prev = a_cur;
          a_cur = a_next;
          a_next = 0.0;
        }
      }
      if (p == n0 - 1 && k >= i0 && k < i1) f0[k * inner + t] = a_cur;  // the last row: row k is complete
    }
  }
}

// ---- 2-D specialisations (path "auto"): the same arithmetic as predict<T,
// kNu, 2> / shell_pos<2> written out per parity case (the generic corner
// loop costs ~250 instructions per node), bit-identical.  Corner order =
// cmask order (axis 0 is bit 0 when odd); shell positions: an even row
// holds only its odd-column tail, (r, k) -> r (n1 - m1) + k; odd row r of
// the reordered block starts at (m0 + r) n1 - m0 m1.

// k_axis_load (uniform weights) with 32-bit index math (total < 2^32):
// y[o][i][t] = load_entry of x[o][.][t] at coarse i (transform.hpp:84-96,
// the same operation order).
__global__ void __launch_bounds__(256) k_axis_load32(const double* __restrict__ x, double* __restrict__ y,
                                                     uint32_t total, uint32_t inner, uint32_t n, uint32_t m,
                                                     const FastDiv div_inner, const FastDiv div_m) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += stride) {
    const uint32_t oi = div_inner.div(q), t = q - oi * inner;
    const uint32_t o = div_m.div(oi), i = oi - o * m;
    const double* c = x + (uint64_t(o) * n) * inner + t;
    double acc = 0.0;
    if (i >= 1) {
      acc = add_(acc, mul_(kW12, c[uint64_t(2 * i - 2) * inner]));
      acc = add_(acc, mul_(0.5, c[uint64_t(2 * i - 1) * inner]));
    }
    acc = add_(acc, mul_((i == 0 || i + 1 == m) ? kW5_12 : kW5_6, c[uint64_t(2 * i) * inner]));
    if (2 * i + 1 < n) acc = add_(acc, mul_(0.5, c[uint64_t(2 * i + 1) * inner]));
    if (2 * i + 2 < n) acc = add_(acc, mul_(kW12, c[uint64_t(2 * i + 2) * inner]));
    y[q] = acc;
  }
}

// Rolling axis-0 load accumulators of one column (see k_coef_load0): rows
// k-1, k, k+1 around fine row p, k = p >> 1; finished rows go to f0.
struct Roll0 {
  double prev = 0.0, cur = 0.0, next = 0.0;
};

template <bool kNu>
__device__ __forceinline__ void roll0(Roll0& A, double c, int64_t p, int64_t p_hi, int64_t n0, int64_t m0, int64_t i0,
                                      int64_t i1, const double* __restrict__ s5, double* __restrict__ f0col,
                                      int64_t ld) {
  const int64_t k = p >> 1;
  if (!(p & 1)) {
    if (k >= 1) {
      A.prev = add_(A.prev, mul_(kNu ? s5[5 * (k - 1) + 4] : kW12, c));
      if (k - 1 >= i0 && k - 1 < i1) f0col[(k - 1) * ld] = A.prev;
    }
    A.cur = add_(A.cur, mul_(kNu ? s5[5 * k + 2] : ((k == 0 || k + 1 == m0) ? kW5_12 : kW5_6), c));
    A.next = (k + 1 < m0) ? add_(0.0, mul_(kNu ? s5[5 * (k + 1)] : kW12, c)) : 0.0;
  } else {
    A.cur = add_(A.cur, mul_(kNu ? s5[5 * k + 3] : 0.5, c));
    if (k + 1 < m0) A.next = add_(A.next, mul_(kNu ? s5[5 * (k + 1) + 1] : 0.5, c));
    if (p < p_hi) {
      A.prev = A.cur;
      A.cur = A.next;
      A.next = 0.0;
    }
  }
  if (p == n0 - 1 && k >= i0 && k < i1) f0col[k * ld] = A.cur;
}

// k_coef_load0 for rank 2.  Each thread owns a column pair (2k, 2k+1) so
// every branch is uniform across a warp (a per-column mapping alternates
// the parity case lane by lane) and the corner loads are shared between the
// pair.  Arithmetic is predict<T, kNu, 2>'s written out per case.
template <typename T, bool kRec, bool kNu>
__global__ void __launch_bounds__(256) k2_coef_load0(const T* __restrict__ blk, T* __restrict__ shell,
                                                     T* __restrict__ coarse, double* __restrict__ f0,
                                                     const LevelGeom g, const NuLevel nu, int chunk) {
  const int64_t n0 = g.n[0], m0 = g.m[0], n1 = g.n[1], m1 = g.m[1];
  const int64_t total = ((m0 + chunk - 1) / chunk) * m1;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const double* s5 = kNu ? nu.ax[0].s : nullptr;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += stride) {
    const int64_t ch = q / m1, k = q - ch * m1;
    const int64_t i0 = ch * chunk, i1 = min(m0, i0 + chunk);
    const int64_t t0 = 2 * k, t1 = t0 + 1;
    const bool has1 = t1 < n1;
    const int64_t t1r = (t1 + 1 < n1) ? t1 + 1 : t0;  // right corner column of t1
    double a1l = 0.0, a1r = 0.0;
    if (kNu && has1) a1l = nu.ax[1].wl[t1], a1r = nu.ax[1].wr[t1];
    const int64_t p_lo = i0 > 0 ? 2 * i0 - 2 : 0;
    const int64_t p_hi = min(n0 - 1, 2 * i1);
    Roll0 A0, A1;
    for (int64_t p = p_lo; p <= p_hi; ++p) {
      const bool owned = p >= 2 * i0 && p < 2 * i1;
      const int64_t r = p >> 1;
      double c0, c1 = 0.0;
      if (!(p & 1)) {
        const int64_t sp = r * (n1 - m1) + k;  // (even row, odd column)
        if (kRec) {
          c0 = 0.0;
          if (has1) c1 = double(blk[sp]);
        } else {
          const T x0 = blk[p * n1 + t0];
          if (owned) coarse[r * m1 + k] = x0;
          c0 = 0.0;
          if (has1) {
            const double v0 = double(x0), v1 = double(blk[p * n1 + t1r]);
            const double pred = kNu ? add_(add_(0.0, mul_(a1l, v0)), mul_(a1r, v1))
                                    : mul_(add_(add_(0.0, v0), v1), 0.5);
            const T v = to_t<T>(sub_(double(blk[p * n1 + t1]), pred));
            if (owned) shell[sp] = v;
            c1 = double(v);
          }
        }
      } else {
        const int64_t sp = (m0 + r) * n1 - m0 * m1 + k;  // (odd row, even column); odd column at + m1
        if (kRec) {
          c0 = double(blk[sp]);
          if (has1) c1 = double(blk[sp + m1]);
        } else {
          const int64_t pl = p - 1, pr = (p + 1 < n0) ? p + 1 : p - 1;
          double a0l = 0.0, a0r = 0.0;
          if (kNu) a0l = nu.ax[0].wl[p], a0r = nu.ax[0].wr[p];
          const double u00 = double(blk[pl * n1 + t0]), u10 = double(blk[pr * n1 + t0]);
          const double pred0 = kNu ? add_(add_(0.0, mul_(a0l, u00)), mul_(a0r, u10))
                                   : mul_(add_(add_(0.0, u00), u10), 0.5);
          const T v0 = to_t<T>(sub_(double(blk[p * n1 + t0]), pred0));
          if (owned) shell[sp] = v0;
          c0 = double(v0);
          if (has1) {
            const double u01 = double(blk[pl * n1 + t1r]), u11 = double(blk[pr * n1 + t1r]);
            double pred1;
            if (kNu) {
              pred1 = add_(0.0, mul_(mul_(a0l, a1l), u00));
              pred1 = add_(pred1, mul_(mul_(a0r, a1l), u10));
              pred1 = add_(pred1, mul_(mul_(a0l, a1r), u01));
              pred1 = add_(pred1, mul_(mul_(a0r, a1r), u11));
            } else {
              pred1 = mul_(add_(add_(add_(add_(0.0, u00), u10), u01), u11), 0.25);
            }
            const T v1 = to_t<T>(sub_(double(blk[p * n1 + t1]), pred1));
            if (owned) shell[sp + m1] = v1;
            c1 = double(v1);
          }
        }
      }
      roll0<kNu>(A0, c0, p, p_hi, n0, m0, i0, i1, s5, f0 + t0, n1);
      if (has1) roll0<kNu>(A1, c1, p, p_hi, n0, m0, i0, i1, s5, f0 + t1, n1);
    }
  }
}

// k_rec_interp for rank 2 (32-bit node counts), one column pair (2k, 2k+1)
// of one fine row per thread.
template <typename T, bool kNu>
__global__ void __launch_bounds__(256) k2_rec_interp(const T* __restrict__ shell, const T* __restrict__ coarse,
                                                     T* __restrict__ fine, const LevelGeom g, const NuLevel nu) {
  const uint32_t n0 = uint32_t(g.n[0]), m0 = uint32_t(g.m[0]), n1 = uint32_t(g.n[1]), m1 = uint32_t(g.m[1]);
  const uint32_t total = n0 * m1;
  const FastDiv dm1 = g.fn[0];  // set up by the caller as a divider by m1
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += gridDim.x * blockDim.x) {
    const uint32_t p = dm1.div(q), k = q - p * m1, r = p >> 1;
    const uint32_t t0 = 2 * k, t1 = t0 + 1;
    const bool has1 = t1 < n1;
    const uint32_t kr = (t1 + 1 < n1) ? k + 1 : k;
    T* fr = fine + p * n1;
    if (!(p & 1)) {
      const T x0 = coarse[r * m1 + k];
      fr[t0] = x0;
      if (has1) {
        const double v0 = double(x0), v1 = double(coarse[r * m1 + kr]);
        const double pred = kNu ? add_(add_(0.0, mul_(nu.ax[1].wl[t1], v0)), mul_(nu.ax[1].wr[t1], v1))
                                : mul_(add_(add_(0.0, v0), v1), 0.5);
        fr[t1] = to_t<T>(add_(double(shell[r * (n1 - m1) + k]), pred));
      }
    } else {
      const uint32_t rr = (p + 1 < n0) ? r + 1 : r;
      const uint32_t sp = (m0 + r) * n1 - m0 * m1 + k;
      double a0l = 0.0, a0r = 0.0;
      if (kNu) a0l = nu.ax[0].wl[p], a0r = nu.ax[0].wr[p];
      const double u00 = double(coarse[r * m1 + k]), u10 = double(coarse[rr * m1 + k]);
      const double pred0 = kNu ? add_(add_(0.0, mul_(a0l, u00)), mul_(a0r, u10)) : mul_(add_(add_(0.0, u00), u10), 0.5);
      fr[t0] = to_t<T>(add_(double(shell[sp]), pred0));
      if (has1) {
        const double u01 = double(coarse[r * m1 + kr]), u11 = double(coarse[rr * m1 + kr]);
        double pred1;
        if (kNu) {
          const double a1l = nu.ax[1].wl[t1], a1r = nu.ax[1].wr[t1];
          pred1 = add_(0.0, mul_(mul_(a0l, a1l), u00));
          pred1 = add_(pred1, mul_(mul_(a0r, a1l), u10));
          pred1 = add_(pred1, mul_(mul_(a0l, a1r), u01));
          pred1 = add_(pred1, mul_(mul_(a0r, a1r), u11));
        } else {
          pred1 = mul_(add_(add_(add_(add_(0.0, u00), u10), u01), u11), 0.25);
        }
        fr[t1] = to_t<T>(add_(double(shell[sp + m1]), pred1));
      }
    }
  }
}

// ---- rank 3-4 column-pair kernels (path "auto"): the last axis is walked
// in pairs (2k, 2k+1), the leading axes' corner set is built once per pair
// and shared: predict<T, kNu, D> enumerates corners in cmask order with the
// last axis as the highest bit, so the odd column's corner sum is the even
// column's sum continued over the right-hand corners (uniform case) —
// bit-identical with far fewer instructions than the per-node corner loop.
// The corner loop is specialised on the parity pattern OM of the leading
// axes (pair_predict dispatches; a lane's pattern is constant along a row):
// only the subsets of the odd axes are enumerated, in ascending mask order —
// a mask's odd-axis bits in ascending order are exactly predict's cmask, so
// the order is unchanged.  32-bit offsets (N < 2^32).
// pred0 at column cl (meaningful unless the even node is nodal), pred1 at
// the odd column between cl and cr (has1); w3l/w3r: nonuniform last-axis
// weights of the odd column.  Returns the all-left corner offset.
template <typename T, bool kNu, int D, unsigned OM>
__device__ __forceinline__ uint32_t pair_predict_m(const T* __restrict__ src, const LevelGeom& g, const NuLevel& nu,
                                                   const int64_t* j, bool coarse, uint32_t cl, uint32_t cr, bool has1,
                                                   double w3l, double w3r, double& pred0, double& pred1) {
  // OM: the odd axes among 0..D-2 (compile time: only the corner subsets of
  // the odd axes are enumerated, in ascending cmask order as before)
  constexpr int A = D - 1;
  uint32_t base = 0, dl[A];
  double wl[A], wr[A];
  int nodd = 0;
#pragma unroll
  for (int i = 0; i < A; ++i) {
    constexpr unsigned one = 1u;
    const bool odd = (OM >> i) & one;
    const uint32_t ji = uint32_t(j[i]);
    base += coarse ? (ji >> 1) * uint32_t(g.cst[i]) : (odd ? ji - 1 : ji) * uint32_t(g.st[i]);
    dl[i] = (odd && j[i] + 1 < g.n[i]) ? (coarse ? uint32_t(g.cst[i]) : 2 * uint32_t(g.st[i])) : 0;
    wl[i] = wr[i] = 1.0;
    if (kNu && odd) {
      wl[i] = nu.ax[i].wl[ji];
      wr[i] = nu.ax[i].wr[ji];
    }
    nodd += odd ? 1 : 0;
  }
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (uint32_t fm = 0; fm < (1u << A); ++fm) {
    if (fm & ~OM) continue;
    uint32_t off = base;
    double wp = 1.0;
#pragma unroll
    for (int i = 0; i < A; ++i) {
      if (!((OM >> i) & 1u)) continue;
      if ((fm >> i) & 1) off += dl[i];
      if (kNu) wp = mul_(wp, ((fm >> i) & 1) ? wr[i] : wl[i]);
    }
    const double L = double(src[off + cl]);
    if (kNu) {
      s0 = add_(s0, mul_(wp, L));
      s1 = add_(s1, mul_(mul_(wp, w3l), L));
    } else {
      s0 = add_(s0, L);
    }
  }
  // 2^-nodd, exactly
  const double sc0 = __longlong_as_double(int64_t(1023 - nodd) << 52);
  pred0 = kNu ? s0 : mul_(s0, sc0);
  if (has1) {
    if (!kNu) s1 = s0;
#pragma unroll
    for (uint32_t fm = 0; fm < (1u << A); ++fm) {
      if (fm & ~OM) continue;
      uint32_t off = base;
      double wp = 1.0;
#pragma unroll
      for (int i = 0; i < A; ++i) {
        if (!((OM >> i) & 1u)) continue;
        if ((fm >> i) & 1) off += dl[i];
        if (kNu) wp = mul_(wp, ((fm >> i) & 1) ? wr[i] : wl[i]);
      }
      const double R = double(src[off + cr]);
      s1 = kNu ? add_(s1, mul_(mul_(wp, w3r), R)) : add_(s1, R);
    }
    pred1 = kNu ? s1 : mul_(s1, 0.5 * sc0);
  }
  return base;
}

// Dispatch on the parity pattern of the leading axes (warp-uniform along a
// row of the last axis).
template <typename T, bool kNu, int D>
__device__ __forceinline__ uint32_t pair_predict(const T* __restrict__ src, const LevelGeom& g, const NuLevel& nu,
                                                 const int64_t* j, bool coarse, uint32_t cl, uint32_t cr, bool has1,
                                                 double w3l, double w3r, double& pred0, double& pred1) {
  unsigned om = 0;
#pragma unroll
  for (int i = 0; i < D - 1; ++i) om |= unsigned(j[i] & 1) << i;
#define PP_(M) \
  case M:      \
    return pair_predict_m<T, kNu, D, (M) & ((1u << (D - 1)) - 1)>(src, g, nu, j, coarse, cl, cr, has1, w3l, w3r, pred0, pred1)
  switch (om) {
    PP_(0);
    PP_(1);
    PP_(2);
    PP_(3);
    PP_(4);
    PP_(5);
    PP_(6);
    default:
      return pair_predict_m<T, kNu, D, 7u & ((1u << (D - 1)) - 1)>(src, g, nu, j, coarse, cl, cr, has1, w3l, w3r, pred0,
                                                                   pred1);
  }
#undef PP_
}

// k_coef_load0 for rank D = 3, 4: a thread owns a column pair of one row of
// the middle axes and a chunk of coarse rows along axis 0.
template <typename T, bool kRec, bool kNu, int D>
__global__ void __launch_bounds__(256) kN_coef_load0(const T* __restrict__ blk, T* __restrict__ shell,
                                                     T* __restrict__ coarse, double* __restrict__ f0,
                                                     const LevelGeom g, const NuLevel nu, int64_t inner, int chunk) {
  constexpr int E = D - 1;  // last axis
  const int64_t n0 = g.n[0], m0 = g.m[0], nl = g.n[E], ml = g.m[E];
  const int64_t rmid = inner / nl;
  const int64_t total = ((m0 + chunk - 1) / chunk) * rmid * ml;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const double* s5 = kNu ? nu.ax[0].s : nullptr;
  // 32-bit index decomposition (the caller guarantees < 2^32 work items):
  // g.fn[E] divides by ml, g.fn[0] by rmid (neither is otherwise used here)
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += stride) {
    const uint32_t q32 = uint32_t(q);
    const uint32_t rest = g.fn[E].div(q32);
    const int64_t k = q32 - rest * uint32_t(ml);
    const uint32_t ch32 = g.fn[0].div(rest);
    const int64_t row = rest - ch32 * uint32_t(rmid), ch = ch32;
    const int64_t i0 = ch * chunk, i1 = min(m0, i0 + chunk);
    int64_t j[kMaxD];
    bool mid_even = true;
    int64_t cmid = 0;  // coarse offset of the middle axes
    {
      uint32_t r = uint32_t(row);
#pragma unroll
      for (int i = D - 2; i >= 1; --i) {
        const uint32_t rq = g.fn[i].div(r);
        j[i] = r - rq * uint32_t(g.n[i]);
        r = rq;
        mid_even &= !(j[i] & 1);
        cmid += (j[i] >> 1) * g.cst[i];
      }
    }
    const int64_t t0 = 2 * k, t1 = t0 + 1;
    const bool has1 = t1 < nl;
    const int64_t t1r = (t1 + 1 < nl) ? t1 + 1 : t0;
    const int64_t tp0 = row * nl + t0;  // inner positions of the pair
    double w3l = 0.0, w3r = 0.0;
    if (kNu && has1) w3l = nu.ax[E].wl[t1], w3r = nu.ax[E].wr[t1];
    const int64_t p_lo = i0 > 0 ? 2 * i0 - 2 : 0;
    const int64_t p_hi = min(n0 - 1, 2 * i1);
    Roll0 A0, A1;
    for (int64_t p = p_lo; p <= p_hi; ++p) {
      const bool owned = p >= 2 * i0 && p < 2 * i1;
      const bool nodal0 = !(p & 1) && mid_even;
      j[0] = p;
      j[E] = t0;
      const int64_t sp0 = shell_pos<D>(g, j);  // odd column at sp0 + ml
      double c0 = 0.0, c1 = 0.0;
      if (kRec) {
        if (!nodal0) c0 = double(blk[sp0]);
        if (has1) c1 = double(blk[sp0 + ml]);
      } else {
        const T* xr = blk + p * inner + tp0;
        if (nodal0 && owned) coarse[(p >> 1) * g.cst[0] + cmid + k] = xr[0];
        double pred0 = 0.0, pred1 = 0.0;
        pair_predict<T, kNu, D>(blk, g, nu, j, false, uint32_t(t0), uint32_t(t1r), has1, w3l, w3r, pred0, pred1);
        if (!nodal0) {
          const T v = to_t<T>(sub_(double(xr[0]), pred0));
          if (owned) shell[sp0] = v;
          c0 = double(v);
        }
        if (has1) {
          const T v = to_t<T>(sub_(double(xr[1]), pred1));
          if (owned) shell[sp0 + ml] = v;
          c1 = double(v);
        }
      }
      roll0<kNu>(A0, c0, p, p_hi, n0, m0, i0, i1, s5, f0 + tp0, inner);
      if (has1) roll0<kNu>(A1, c1, p, p_hi, n0, m0, i0, i1, s5, f0 + tp0 + 1, inner);
    }
  }
}

// k_rec_interp for rank D = 3, 4, one column pair per thread.
template <typename T, bool kNu, int D>
__global__ void __launch_bounds__(256) kN_rec_interp(const T* __restrict__ shell, const T* __restrict__ coarse,
                                                     T* __restrict__ fine, const LevelGeom g, const NuLevel nu) {
  constexpr int E = D - 1;
  const int64_t nl = g.n[E], ml = g.m[E];
  const int64_t rows = g.N / nl;
  const int64_t total = rows * ml;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  // 32-bit index decomposition (N < 2^32); g.fn[E] divides by ml
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += stride) {
    const uint32_t q32 = uint32_t(q);
    const uint32_t row32 = g.fn[E].div(q32);
    const int64_t k = q32 - row32 * uint32_t(ml), row = row32;
    int64_t j[kMaxD];
    bool lead_even = true;
    {
      uint32_t r = row32;
#pragma unroll
      for (int i = D - 2; i >= 1; --i) {
        const uint32_t rq = g.fn[i].div(r);
        j[i] = r - rq * uint32_t(g.n[i]);
        r = rq;
        lead_even &= !(j[i] & 1);
      }
      j[0] = r;
      lead_even &= !(r & 1);
    }
    const int64_t t0 = 2 * k, t1 = t0 + 1;
    const bool has1 = t1 < nl;
    const int64_t kr = (t1 + 1 < nl) ? k + 1 : k;
    j[E] = t0;
    const int64_t sp0 = shell_pos<D>(g, j);
    double w3l = 0.0, w3r = 0.0;
    if (kNu && has1) w3l = nu.ax[E].wl[t1], w3r = nu.ax[E].wr[t1];
    double pred0 = 0.0, pred1 = 0.0;
    const uint32_t cb =
        pair_predict<T, kNu, D>(coarse, g, nu, j, true, uint32_t(k), uint32_t(kr), has1, w3l, w3r, pred0, pred1);
    T* fr = fine + row * nl + t0;
    fr[0] = lead_even ? coarse[cb + k] : to_t<T>(add_(double(shell[lead_even ? 0 : sp0]), pred0));
    if (has1) fr[1] = to_t<T>(add_(double(shell[sp0 + ml]), pred1));
  }
}

// ---- rank 3-4 axis-0 walkers (uniform weights, N < 2^32): a thread owns a
// column pair (2k, 2k+1) of one row of the middle axes and walks a chunk of
// fine planes along axis 0.  The corner values of the last even plane stay
// in registers: an odd plane's corner set is the left even plane's (cached)
// interleaved with the right one's (loaded once, then cached for the next
// even plane), so every corner value is loaded once per plane pair instead
// of three times.  Shell positions are linear in p for each parity (even
// planes: +Nmid nl - pm0 ml per plane pair, odd: +Nmid nl), so the per-node
// index math is a few additions.  Sums run in predict's cmask order (axis 0
// lowest, then the middle axes ascending, the last axis highest) as in
// pair_predict_m — bit-identical to kN_coef_load0 / kN_rec_interp.

// Corner offsets (inside one plane, without the column) of the middle-axis
// subsets of this row, and the row's parity pattern / odd count.
#ifndef MGRX_WALK_MINB
#define MGRX_WALK_MINB 2
#endif
#ifndef MGRX_WALK_MINB_I
#define MGRX_WALK_MINB_I 3
#endif
template <int D>
struct MidCorners {
  static constexpr int NC = 1 << (D - 2);
  uint32_t off[NC];  // fine (coarse = false) or coarse (coarse = true) offsets
  unsigned M;        // odd middle axes (bit i-1 for axis i)
  int nodd;
};

template <int D>
__device__ __forceinline__ MidCorners<D> mid_corners(const LevelGeom& g, const int64_t* j, bool coarse) {
  MidCorners<D> mc;
  mc.M = 0;
  mc.nodd = 0;
  uint32_t base = 0, dl[D > 2 ? D - 2 : 1];
#pragma unroll
  for (int i = 1; i <= D - 2; ++i) {
    const bool odd = j[i] & 1;
    const uint32_t ji = uint32_t(j[i]);
    base += coarse ? (ji >> 1) * uint32_t(g.cst[i]) : (odd ? ji - 1 : ji) * uint32_t(g.st[i]);
    dl[i - 1] = (odd && j[i] + 1 < g.n[i]) ? (coarse ? uint32_t(g.cst[i]) : 2 * uint32_t(g.st[i])) : 0;
    mc.M |= unsigned(odd) << (i - 1);
    mc.nodd += odd ? 1 : 0;
  }
#pragma unroll
  for (int fm = 0; fm < MidCorners<D>::NC; ++fm) {
    uint32_t o = base;
#pragma unroll
    for (int i = 0; i < D - 2; ++i)
      if ((fm >> i) & 1) o += dl[i];
    mc.off[fm] = o;
  }
  return mc;
}

// Corner values of one plane at columns cl / cr (only the subsets of M are loaded).
template <typename T, int D>
__device__ __forceinline__ void load_corners(const T* __restrict__ pl, const MidCorners<D>& mc, uint32_t cl,
                                             uint32_t cr, bool has1, double* vl, double* vr) {
#pragma unroll
  for (int fm = 0; fm < MidCorners<D>::NC; ++fm) {
    vl[fm] = vr[fm] = 0.0;
    if (fm & ~mc.M) continue;
    vl[fm] = double(pl[mc.off[fm] + cl]);
    if (has1) vr[fm] = double(pl[mc.off[fm] + cr]);
  }
}

// Even plane: predict over the plane's own corners (scale 2^-nodd).
template <int D>
__device__ __forceinline__ void pred_even(const MidCorners<D>& mc, const double* el, const double* er, double& p0,
                                          double& p1) {
  double s = 0.0;
#pragma unroll
  for (int fm = 0; fm < MidCorners<D>::NC; ++fm)
    if (!(fm & ~mc.M)) s = add_(s, el[fm]);
  const double sc = __longlong_as_double(int64_t(1023 - mc.nodd) << 52);
  p0 = mul_(s, sc);
#pragma unroll
  for (int fm = 0; fm < MidCorners<D>::NC; ++fm)
    if (!(fm & ~mc.M)) s = add_(s, er[fm]);
  p1 = mul_(s, 0.5 * sc);
}

// Odd plane: left / right planes interleaved per middle subset (scale 2^-(nodd+1)).
template <int D>
__device__ __forceinline__ void pred_odd(const MidCorners<D>& mc, const double* el, const double* er,
                                         const double* nl_, const double* nr_, double& p0, double& p1) {
  double s = 0.0;
#pragma unroll
  for (int fm = 0; fm < MidCorners<D>::NC; ++fm)
    if (!(fm & ~mc.M)) {
      s = add_(s, el[fm]);
      s = add_(s, nl_[fm]);
    }
  const double sc = __longlong_as_double(int64_t(1023 - mc.nodd - 1) << 52);
  p0 = mul_(s, sc);
#pragma unroll
  for (int fm = 0; fm < MidCorners<D>::NC; ++fm)
    if (!(fm & ~mc.M)) {
      s = add_(s, er[fm]);
      s = add_(s, nr_[fm]);
    }
  p1 = mul_(s, 0.5 * sc);
}

// roll0 split by plane parity (the same arithmetic).
__device__ __forceinline__ void roll_even(Roll0& A, double c, int k, int p, int n0, int m0, int i0, int i1,
                                          double* __restrict__ f0col, int64_t ld) {
  if (k >= 1) {
    A.prev = add_(A.prev, mul_(kW12, c));
    if (k - 1 >= i0 && k - 1 < i1) f0col[int64_t(k - 1) * ld] = A.prev;
  }
  A.cur = add_(A.cur, mul_((k == 0 || k + 1 == m0) ? kW5_12 : kW5_6, c));
  A.next = (k + 1 < m0) ? add_(0.0, mul_(kW12, c)) : 0.0;
  if (p == n0 - 1 && k >= i0 && k < i1) f0col[int64_t(k) * ld] = A.cur;
}
__device__ __forceinline__ void roll_odd(Roll0& A, double c, int k, int p, int p_hi, int n0, int m0, int i0, int i1,
                                         double* __restrict__ f0col, int64_t ld) {
  A.cur = add_(A.cur, mul_(0.5, c));
  if (k + 1 < m0) A.next = add_(A.next, mul_(0.5, c));
  if (p == n0 - 1 && k >= i0 && k < i1) f0col[int64_t(k) * ld] = A.cur;
  if (p < p_hi) {
    A.prev = A.cur;
    A.cur = A.next;
    A.next = 0.0;
  }
}

// Row of the middle axes -> j[1..D-2], their even-ness and coarse offset.
template <int D>
__device__ __forceinline__ void mid_unravel(const LevelGeom& g, uint32_t row, int64_t* j, bool& even, int64_t& cmid) {
  even = true;
  cmid = 0;
#pragma unroll
  for (int i = D - 2; i >= 1; --i) {
    const uint32_t rq = g.fn[i].div(row);
    j[i] = row - rq * uint32_t(g.n[i]);
    row = rq;
    even &= !(j[i] & 1);
    cmid += (j[i] >> 1) * g.cst[i];
  }
}

// Raw values one plane pair ahead (registers): the loop body works on the
// pair fetched one iteration earlier, so each thread keeps two pairs' loads
// in flight instead of waiting a full memory latency per pair.
template <typename T, int NC>
struct PairRaw {
  T e0, e1, o0, o1;   // even / odd plane values (coefficient walk: the node pair; kRec / interp: shell)
  T cl[NC], cr[NC];   // corners of the next even plane at columns cl / cr
};

template <typename T, int D>
__device__ __forceinline__ void fetch_corners(const T* __restrict__ pl, const MidCorners<D>& mc, uint32_t cl,
                                              uint32_t cr, bool has1, T* vl, T* vr) {
#pragma unroll
  for (int fm = 0; fm < MidCorners<D>::NC; ++fm) {
    vl[fm] = vr[fm] = T(0);
    if (fm & ~mc.M) continue;
    vl[fm] = pl[mc.off[fm] + cl];
    if (has1) vr[fm] = pl[mc.off[fm] + cr];
  }
}

// coefficients (kRec: the component read from the shell) + the axis-0 load
// vector, as kN_coef_load0 (uniform weights).
template <typename T, bool kRec, int D>
__global__ void __launch_bounds__(256, MGRX_WALK_MINB) kN_coef_load0w(const T* __restrict__ blk, T* __restrict__ shell,
                                                      T* __restrict__ coarse, double* __restrict__ f0,
                                                      const LevelGeom g, int64_t inner, int chunk) {
  constexpr int E = D - 1;
  constexpr int NC = MidCorners<D>::NC;
  const int n0 = int(g.n[0]), m0 = int(g.m[0]), nl = int(g.n[E]), ml = int(g.m[E]);
  const int64_t rmid = inner / nl;
  const int64_t total = ((m0 + chunk - 1) / chunk) * rmid * ml;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t nmid = 1;
#pragma unroll
  for (int i = 1; i <= D - 2; ++i) nmid *= g.n[i];
  const int64_t dsp_e = nmid * nl - g.pm[0] * ml, dsp_o = nmid * nl;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += stride) {
    const uint32_t q32 = uint32_t(q);
    const uint32_t rest = g.fn[E].div(q32);
    const int k = int(q32 - rest * uint32_t(ml));
    const uint32_t ch = g.fn[0].div(rest);
    const uint32_t row = rest - ch * uint32_t(rmid);
    const int i0 = int(ch) * chunk, i1 = min(m0, i0 + chunk);
    int64_t j[kMaxD];
    bool mid_even;
    int64_t cmid;
    mid_unravel<D>(g, row, j, mid_even, cmid);
    const int t0 = 2 * k, t1 = t0 + 1;
    const bool has1 = t1 < nl;
    const uint32_t cr = (t1 + 1 < nl) ? uint32_t(t1 + 1) : uint32_t(t0);
    const int64_t tp0 = int64_t(row) * nl + t0;
    const int p_lo = i0 > 0 ? 2 * i0 - 2 : 0;
    const int p_hi = min(n0 - 1, 2 * i1);
    j[E] = t0;
    j[0] = p_lo;
    int64_t sp_e = shell_pos<D>(g, j);
    j[0] = p_lo + 1;
    int64_t sp_o = shell_pos<D>(g, j);
    MidCorners<D> mc;
    if (!kRec) mc = mid_corners<D>(g, j, false);
    // fetch(p): the raw values of the plane pair (p, p + 1) and the corners
    // of the odd plane's right neighbour (p + 2, or p at a degenerate end)
    auto fetch = [&](int p, int64_t spe, int64_t spo, PairRaw<T, NC>& r) {
      const bool odd = p + 1 <= p_hi;
      if (kRec) {
        r.e0 = mid_even ? T(0) : blk[spe];
        r.e1 = has1 ? blk[spe + ml] : T(0);
        r.o0 = odd ? blk[spo] : T(0);
        r.o1 = (odd && has1) ? blk[spo + ml] : T(0);
      } else {
        const T* pl = blk + int64_t(p) * inner + tp0;
        r.e0 = pl[0];
        r.e1 = has1 ? pl[1] : T(0);
        r.o0 = odd ? pl[inner] : T(0);
        r.o1 = (odd && has1) ? pl[inner + 1] : T(0);
        if (odd) {
          const T* prt = blk + int64_t(p + 2 < n0 ? p + 2 : p) * inner;
          fetch_corners<T, D>(prt, mc, uint32_t(t0), cr, has1, r.cl, r.cr);
        }
      }
    };
    double el[NC], er[NC];
    if (!kRec) {
      T vl[NC], vr[NC];
      fetch_corners<T, D>(blk + int64_t(p_lo) * inner, mc, uint32_t(t0), cr, has1, vl, vr);
#pragma unroll
      for (int fm = 0; fm < NC; ++fm) {
        el[fm] = double(vl[fm]);
        er[fm] = double(vr[fm]);
      }
    }
    T* cp = coarse + int64_t(p_lo >> 1) * g.cst[0] + cmid + k;
    Roll0 A0, A1;
    double* f0c = f0 + tp0;
    PairRaw<T, NC> cur;
    fetch(p_lo, sp_e, sp_o, cur);
    for (int p = p_lo; p <= p_hi; p += 2, sp_e += dsp_e, sp_o += dsp_o, cp += g.cst[0]) {
      PairRaw<T, NC> nx;
      if (p + 2 <= p_hi) fetch(p + 2, sp_e + dsp_e, sp_o + dsp_o, nx);
      const int kk = p >> 1;
      {  // even plane p
        const bool owned = p >= 2 * i0 && p < 2 * i1;
        double c0 = 0.0, c1 = 0.0;
        if (kRec) {
          c0 = double(cur.e0);
          c1 = double(cur.e1);
        } else {
          double pred0, pred1;
          pred_even<D>(mc, el, er, pred0, pred1);
          if (mid_even) {
            if (owned) *cp = cur.e0;
          } else {
            const T v = to_t<T>(sub_(double(cur.e0), pred0));
            if (owned) shell[sp_e] = v;
            c0 = double(v);
          }
          if (has1) {
            const T v = to_t<T>(sub_(double(cur.e1), pred1));
            if (owned) shell[sp_e + ml] = v;
            c1 = double(v);
          }
        }
        roll_even(A0, c0, kk, p, n0, m0, i0, i1, f0c, inner);
        if (has1) roll_even(A1, c1, kk, p, n0, m0, i0, i1, f0c + 1, inner);
      }
      if (p + 1 <= p_hi) {  // odd plane p + 1
        const int po = p + 1;
        const bool owned = po >= 2 * i0 && po < 2 * i1;
        double c0, c1 = 0.0;
        if (kRec) {
          c0 = double(cur.o0);
          c1 = double(cur.o1);
        } else {
          double nl_[NC], nr_[NC];
#pragma unroll
          for (int fm = 0; fm < NC; ++fm) {
            nl_[fm] = double(cur.cl[fm]);
            nr_[fm] = double(cur.cr[fm]);
          }
          double pred0, pred1;
          pred_odd<D>(mc, el, er, nl_, nr_, pred0, pred1);
          {
            const T v = to_t<T>(sub_(double(cur.o0), pred0));
            if (owned) shell[sp_o] = v;
            c0 = double(v);
          }
          if (has1) {
            const T v = to_t<T>(sub_(double(cur.o1), pred1));
            if (owned) shell[sp_o + ml] = v;
            c1 = double(v);
          }
#pragma unroll
          for (int fm = 0; fm < NC; ++fm) {
            el[fm] = nl_[fm];
            er[fm] = nr_[fm];
          }
        }
        roll_odd(A0, c0, kk, po, p_hi, n0, m0, i0, i1, f0c, inner);
        if (has1) roll_odd(A1, c1, kk, po, p_hi, n0, m0, i0, i1, f0c + 1, inner);
      }
      cur = nx;
    }
  }
}

// add_interpolant + unpack (kN_rec_interp, uniform weights) walking chunks
// of `chunk` fine planes (even) along axis 0 with the coarse corner values
// of the current coarse plane cached and the next pair's loads in flight.
template <typename T, int D>
__global__ void __launch_bounds__(256, MGRX_WALK_MINB_I) kN_rec_interpw(const T* __restrict__ shell, const T* __restrict__ coarse,
                                                      T* __restrict__ fine, const LevelGeom g, int64_t inner,
                                                      int chunk) {
  constexpr int E = D - 1;
  constexpr int NC = MidCorners<D>::NC;
  const int n0 = int(g.n[0]), nl = int(g.n[E]), ml = int(g.m[E]);
  const int64_t rmid = inner / nl;
  const int64_t total = ((n0 + chunk - 1) / chunk) * rmid * ml;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t nmid = 1;
#pragma unroll
  for (int i = 1; i <= D - 2; ++i) nmid *= g.n[i];
  const int64_t dsp_e = nmid * nl - g.pm[0] * ml, dsp_o = nmid * nl;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += stride) {
    const uint32_t q32 = uint32_t(q);
    const uint32_t rest = g.fn[E].div(q32);
    const int k = int(q32 - rest * uint32_t(ml));
    const uint32_t ch = g.fn[0].div(rest);
    const uint32_t row = rest - ch * uint32_t(rmid);
    const int pa = int(ch) * chunk, pb = min(n0, pa + chunk);  // fine planes [pa, pb), pa even
    int64_t j[kMaxD];
    bool mid_even;
    int64_t cmid;
    mid_unravel<D>(g, row, j, mid_even, cmid);
    const int t0 = 2 * k, t1 = t0 + 1;
    const bool has1 = t1 < nl;
    const uint32_t kr = (t1 + 1 < nl) ? uint32_t(k + 1) : uint32_t(k);
    j[E] = t0;
    j[0] = pa;
    int64_t sp_e = shell_pos<D>(g, j);
    j[0] = pa + 1;
    int64_t sp_o = shell_pos<D>(g, j);
    const MidCorners<D> mc = mid_corners<D>(g, j, true);
    auto fetch = [&](int p, int64_t spe, int64_t spo, PairRaw<T, NC>& r) {
      const bool odd = p + 1 < pb;
      r.e0 = mid_even ? T(0) : shell[spe];
      r.e1 = has1 ? shell[spe + ml] : T(0);
      r.o0 = odd ? shell[spo] : T(0);
      r.o1 = (odd && has1) ? shell[spo + ml] : T(0);
      if (odd) {
        const int kc = (p + 2 < n0) ? (p >> 1) + 1 : (p >> 1);
        fetch_corners<T, D>(coarse + int64_t(kc) * g.cst[0], mc, uint32_t(k), kr, has1, r.cl, r.cr);
      }
    };
    double el[NC], er[NC];
    {
      T vl[NC], vr[NC];
      fetch_corners<T, D>(coarse + int64_t(pa >> 1) * g.cst[0], mc, uint32_t(k), kr, has1, vl, vr);
#pragma unroll
      for (int fm = 0; fm < NC; ++fm) {
        el[fm] = double(vl[fm]);
        er[fm] = double(vr[fm]);
      }
    }
    T* fr = fine + int64_t(pa) * inner + int64_t(row) * nl + t0;
    PairRaw<T, NC> cur;
    fetch(pa, sp_e, sp_o, cur);
    for (int p = pa; p < pb; p += 2, fr += 2 * inner, sp_e += dsp_e, sp_o += dsp_o) {
      PairRaw<T, NC> nx;
      if (p + 2 < pb) fetch(p + 2, sp_e + dsp_e, sp_o + dsp_o, nx);
      {  // even plane
        double pred0, pred1;
        pred_even<D>(mc, el, er, pred0, pred1);
        fr[0] = mid_even ? T(el[0]) : to_t<T>(add_(double(cur.e0), pred0));
        if (has1) fr[1] = to_t<T>(add_(double(cur.e1), pred1));
      }
      if (p + 1 < pb) {  // odd plane
        double nl_[NC], nr_[NC];
#pragma unroll
        for (int fm = 0; fm < NC; ++fm) {
          nl_[fm] = double(cur.cl[fm]);
          nr_[fm] = double(cur.cr[fm]);
        }
        double pred0, pred1;
        pred_odd<D>(mc, el, er, nl_, nr_, pred0, pred1);
        T* fo = fr + inner;
        fo[0] = to_t<T>(add_(double(cur.o0), pred0));
        if (has1) fo[1] = to_t<T>(add_(double(cur.o1), pred1));
#pragma unroll
        for (int fm = 0; fm < NC; ++fm) {
          el[fm] = nl_[fm];
          er[fm] = nr_[fm];
        }
      }
      cur = nx;
    }
  }
}

// Serial Thomas along axis-0-style lines over a precomputed load vector, in
// place: the same operations as k_sweep after its load (bit-identical).
template <bool kNu>
__global__ void __launch_bounds__(128) k_axis_thomas(double* __restrict__ y, int64_t lines, int64_t inner, int64_t m,
                                                     const double* __restrict__ w, const double* __restrict__ inv_d,
                                                     const NuAxis nu) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t0 < lines; t0 += stride) {
    const int64_t o = t0 / inner, t = t0 - o * inner;
    double* f = y + o * m * inner + t;
    double prev = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double acc = f[i * inner];
      if (i > 0) acc = sub_(acc, mul_(kNu ? nu.tw[i] : w[i], prev));
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

// Tiled variant for strided lines (path "auto"): LB consecutive lines per
// CTA staged whole in shared memory with the factor tables, so the four
// segment passes of k_axis_solve touch HBM once (one read, one write).
template <int LB>
__global__ void __launch_bounds__(256) k_axis_solve_tile(double* __restrict__ y, int64_t nlines, int m, int64_t inner,
                                                         const double* __restrict__ gw,
                                                         const double* __restrict__ gid,
                                                         const double* __restrict__ goff) {
  extern __shared__ double ts[];
  __shared__ double A[32][LB], B[32][LB];
  double* w = ts;
  double* inv_d = w + m;
  double* off = goff ? inv_d + m : nullptr;
  double* t = inv_d + (goff ? 2 : 1) * m;  // [m][LB]
  const int c = threadIdx.x % LB, s = threadIdx.x / LB, S = blockDim.x / LB;
  const int64_t line = int64_t(blockIdx.x) * LB + c;
  const bool valid = line < nlines;
  double* p = y + (valid ? (line / inner) * m * inner + line % inner : 0);
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    w[i] = gw[i];
    inv_d[i] = gid[i];
    if (goff) off[i] = goff[i];
  }
  // asynchronous 8-byte copies: the whole tile in flight at once (a plain
  // load loop keeps only a few rows per warp outstanding at 1 CTA per SM)
  for (int i = s; i < m; i += S) {
    if (valid) {
      const uint32_t dst = uint32_t(__cvta_generic_to_shared(t + i * LB + c));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(p + i * inner) : "memory");
    } else {
      t[i * LB + c] = 0.0;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int seg = (m + S - 1) / S;
  const int s0 = min(m, s * seg), s1 = min(m, s0 + seg);
  double ya = 0.0, yb = 1.0;
  for (int i = s0; i < s1; ++i) {
    const double wi = w[i];
    ya = t[i * LB + c] - wi * ya;
    yb = -wi * yb;
  }
  A[s][c] = ya;
  B[s][c] = yb;
  __syncthreads();
  double cy = 0.0;
  for (int q = 0; q < s; ++q) cy = A[q][c] + B[q][c] * cy;
  __syncthreads();
  for (int i = s0; i < s1; ++i) {
    cy = t[i * LB + c] - w[i] * cy;
    t[i * LB + c] = cy;
  }
  double za = 0.0, zb = 1.0;
  for (int i = s1 - 1; i >= s0; --i) {
    const double id = inv_d[i], oi = off ? off[i] : kOff;
    za = (t[i * LB + c] - oi * za) * id;
    zb = -oi * id * zb;
  }
  A[s][c] = za;
  B[s][c] = zb;
  __syncthreads();
  double z = 0.0;
  for (int q = S - 1; q > s; --q) z = A[q][c] + B[q][c] * z;
  for (int i = s1 - 1; i >= s0; --i) {
    z = (t[i * LB + c] - (off ? off[i] : kOff) * z) * inv_d[i];
    t[i * LB + c] = z;
  }
  __syncthreads();
  if (valid)
    for (int i = s; i < m; i += S) p[i * inner] = t[i * LB + c];
}

// Strided-line solve dispatch: tiled when LB lines fit in shared memory.
static void launch_axis_solve(double* y, int64_t lines, int64_t m, int64_t inner, const double* w, const double* id,
                              const double* of, const Exec& ex) {
  constexpr int LB = 8;
  const size_t sm = size_t(LB + (of ? 3 : 2)) * size_t(m) * 8;
  if (sm <= size_t(200) * 1024) {
    cudaFuncSetAttribute(k_axis_solve_tile<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    MGRX_LAUNCH(ex, "gen_solve", k_axis_solve_tile<LB><<<unsigned((lines + LB - 1) / LB), 256, sm, ex.s>>>(y, lines, int(m), inner, w, id, of));
  } else {
    const int SY = int(std::max<int64_t>(1, std::min<int64_t>(32, (m + 31) / 32)));
    MGRX_LAUNCH(ex, "gen_solve", k_axis_solve<<<unsigned((lines + 15) / 16), dim3(32, SY), 0, ex.s>>>(y, lines, m, inner, w, id, of));
  }
}

// Short contiguous lines (m <= kShortRow): one thread per line, the
// block's lines staged in shared memory with coalesced loads / stores; the
// serial Thomas recurrences of k_sweep (transform.hpp:116-130 order,
// bit-identical).
constexpr int kShortRow = 64;
constexpr int kShortRowThreads = 128;
__global__ void __launch_bounds__(kShortRowThreads) k_rows_thomas(double* __restrict__ y, int64_t nlines, int m,
                                                                  const double* __restrict__ w,
                                                                  const double* __restrict__ inv_d) {
  extern __shared__ double sb[];
  double* tw = sb;
  double* td = sb + kShortRow;
  double* x = sb + 2 * kShortRow;
  const int tid = threadIdx.x;
  for (int i = tid; i < m; i += kShortRowThreads) {
    tw[i] = w[i];
    td[i] = inv_d[i];
  }
  const int64_t l0 = int64_t(blockIdx.x) * kShortRowThreads;
  const int nl = int(min(int64_t(kShortRowThreads), nlines - l0));
  const int cnt = nl * m;
  double* gl = y + l0 * m;
  for (int e = tid; e < cnt; e += kShortRowThreads) x[e] = gl[e];
  __syncthreads();
  if (tid < nl) {
    double* f = x + tid * m;
    double prev = f[0];
    for (int i = 1; i < m; ++i) {
      prev = sub_(f[i], mul_(tw[i], prev));
      f[i] = prev;
    }
    double nxt = mul_(prev, td[m - 1]);
    f[m - 1] = nxt;
    for (int i = m - 2; i >= 0; --i) {
      const double v = mul_(sub_(f[i], mul_(kOff, nxt)), td[i]);
      f[i] = v;
      nxt = v;
    }
  }
  __syncthreads();
  for (int e = tid; e < cnt; e += kShortRowThreads) gl[e] = x[e];
}

static void launch_rows_thomas(double* y, int64_t lines, int m, const double* w, const double* id, const Exec& ex) {
  const size_t sm = size_t(2 * kShortRow + kShortRowThreads * m) * 8;
  cudaFuncSetAttribute(k_rows_thomas, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  MGRX_LAUNCH(ex, "gen_rows", k_rows_thomas<<<unsigned((lines + kShortRowThreads - 1) / kShortRowThreads),
                                              kShortRowThreads, sm, ex.s>>>(y, lines, m, w, id));
}

// Last-axis variant (contiguous lines): one warp per line, the line staged
// in shared memory, lanes own contiguous segments (affine carries combined
// with a warp shuffle scan, then exact reruns).
__global__ void __launch_bounds__(256) k_axis_solve_rows(double* __restrict__ y, int64_t nlines, int m,
                                                         const double* __restrict__ gw,
                                                         const double* __restrict__ gid,
                                                         const double* __restrict__ goff) {
  // the factor tables are staged too: lanes read them at a stride of one
  // segment, which would split every global load into 32 transactions
  extern __shared__ double rowbuf[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* w = rowbuf;
  double* inv_d = w + m;
  double* off = goff ? inv_d + m : nullptr;
  double* x = inv_d + (goff ? 2 : 1) * m + int64_t(warp) * m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    w[i] = gw[i];
    inv_d[i] = gid[i];
    if (goff) off[i] = goff[i];
  }
  __syncthreads();
  const int seg = ((m + 31) >> 5) | 1;  // odd: lanes' segments start in distinct shared-memory banks
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

// The tail's level geometry in registers with 32-bit indices (a tail level
// fits in shared memory): loaded once per level instead of re-reading the
// 64-bit LevelGeom from global memory for every node.  Same index maps as
// unravel / shell_pos / predict above.
template <int D>
struct TailGeo {
  static constexpr int R = D > 0 ? D : kMaxD;
  int d, N, Nc;
  int n[R], m[R], st[R], cst[R], pm[R];
  FastDiv fn[R];
};
#define TAIL_ND(G) (D > 0 ? D : (G).d)

template <int D>
__device__ __forceinline__ TailGeo<D> tail_geo(const LevelGeom& g) {
  TailGeo<D> G;
  G.d = g.d;
  G.N = int(g.N);
  G.Nc = int(g.Nc);
#pragma unroll
  for (int i = 0; i < TailGeo<D>::R; ++i) {
    if (i < TAIL_ND(G)) {
      G.n[i] = int(g.n[i]);
      G.m[i] = int(g.m[i]);
      G.st[i] = int(g.st[i]);
      G.cst[i] = int(g.cst[i]);
      G.pm[i] = int(g.pm[i]);
      G.fn[i] = g.fn[i];
    }
  }
  return G;
}

template <int D>
__device__ __forceinline__ void tail_unravel(int p, const TailGeo<D>& G, int* j) {
  uint32_t q = uint32_t(p);
#pragma unroll
  for (int i = TAIL_ND(G) - 1; i > 0; --i) {
    const uint32_t qq = G.fn[i].div(q);
    j[i] = int(q - qq * uint32_t(G.n[i]));
    q = qq;
  }
  j[0] = int(q);
}

template <int D>
__device__ __forceinline__ int tail_shell_pos(const TailGeo<D>& G, const int* j) {
  const int d = TAIL_ND(G);
  int row = 0, before = 0;
  bool inside = true;
#pragma unroll
  for (int i = 0; i + 1 < d; ++i) {
    const int r = (j[i] & 1) ? G.m[i] + (j[i] >> 1) : (j[i] >> 1);
    row = row * G.n[i] + r;
    if (inside) {
      if (r < G.m[i]) {
        before += r * G.pm[i];
      } else {
        before += G.m[i] * G.pm[i];
        inside = false;
      }
    }
  }
  const int jl = j[d - 1];
  const int rl = (jl & 1) ? G.m[d - 1] + (jl >> 1) : (jl >> 1);
  return row * G.n[d - 1] - before * G.m[d - 1] + (inside ? rl - G.m[d - 1] : rl);
}

// predict<T, kNu, D>: corners in cmask order, summed in that order.
template <typename T, bool kNu, int D>
__device__ __forceinline__ double tail_predict(const T* __restrict__ src, bool coarse, const TailGeo<D>& G,
                                               const NuLevel& nu, const int* j) {
  int k = 0, base = 0;
  int dl[TailGeo<D>::R];
  int bit[TailGeo<D>::R];
#pragma unroll
  for (int i = 0; i < TAIL_ND(G); ++i) {
    const int stride = coarse ? G.cst[i] : G.st[i];
    const bool odd = j[i] & 1;
    dl[i] = (odd && j[i] + 1 < G.n[i]) ? (coarse ? G.cst[i] : 2 * G.st[i]) : 0;
    bit[i] = odd ? k : -1;
    k += odd ? 1 : 0;
    base += (coarse ? (odd ? (j[i] - 1) >> 1 : j[i] >> 1) : (odd ? j[i] - 1 : j[i])) * stride;
  }
  double sum = 0.0;
#pragma unroll
  for (unsigned cm = 0; cm < (D > 0 ? (1u << D) : (1u << kMaxD)); ++cm) {
    if (cm >= (1u << k)) break;
    int off = base;
    double wprod = 1.0;
#pragma unroll
    for (int i = 0; i < TAIL_ND(G); ++i) {
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
    // (1) the restriction value of every (line, i), block-wide: y is laid out
    // [outer][m][inner], so e walks y in order.
    const int mi = m * inner;
    for (int e = threadIdx.x; e < outer * mi; e += blockDim.x) {
      const int o = e / mi, r = e - o * mi;
      const int i = r / inner, t = r - i * inner;
      const double* c = x + o * n * inner + t;
      double acc = 0.0;
      if (kNu) {  // same arithmetic as k_sweep<true>
        const double* sk = nu.ax[a].s + 5 * i;
        for (int k = 0; k < 5; ++k) {
          const int jj = 2 * i + k - 2;
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
      y[e] = acc;
    }
    __syncthreads();
    // (2) the two Thomas recurrences, one thread per line (the only serial part)
    for (int t0 = threadIdx.x; t0 < outer * inner; t0 += blockDim.x) {
      const int o = t0 / inner, t = t0 - o * inner;
      double* f = y + o * mi + t;
      double prev = f[0];
#pragma unroll 4
      for (int i = 1; i < m; ++i) {
        prev = sub_(f[i * inner], mul_(kNu ? nu.ax[a].tw[i] : w[i], prev));
        f[i * inner] = prev;
      }
      double nxt = mul_(prev, kNu ? nu.ax[a].tid[m - 1] : inv_d[m - 1]);
      f[(m - 1) * inner] = nxt;
#pragma unroll 4
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
    const TailGeo<D> G = tail_geo<D>(g);
    for (int p = threadIdx.x; p < G.N; p += blockDim.x) {
      int j[TailGeo<D>::R];
      tail_unravel<D>(p, G, j);
      bool nodal = true;
#pragma unroll
      for (int i = 0; i < TAIL_ND(G); ++i) nodal &= !(j[i] & 1);
      if (nodal) {
        int cc = 0;
#pragma unroll
        for (int i = 0; i < TAIL_ND(G); ++i) cc += (j[i] >> 1) * G.cst[i];
        nxt[cc] = cur[p];
        comp[p] = 0.0;
      } else {
        const double pred = tail_predict<T, kNu, D>(cur, false, G, nu, j);
        const T v = to_t<T>(sub_(double(cur[p]), pred));
        comp[p] = double(v);
        shell[tail_shell_pos<D>(G, j)] = v;
      }
    }
    __syncthreads();
    double* z = nullptr;
    tail_sweeps<D, kNu>(comp, tmp, g, lv[k].th, nu, &z);
    for (int p = threadIdx.x; p < G.Nc; p += blockDim.x) nxt[p] = to_t<T>(add_(double(nxt[p]), mul_(1.0, z[p])));
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
    const TailGeo<D> G = tail_geo<D>(g);
    for (int p = threadIdx.x; p < G.N; p += blockDim.x) {
      int j[TailGeo<D>::R];
      tail_unravel<D>(p, G, j);
      bool nodal = true;
#pragma unroll
      for (int i = 0; i < TAIL_ND(G); ++i) nodal &= !(j[i] & 1);
      comp[p] = nodal ? 0.0 : double(shell[tail_shell_pos<D>(G, j)]);
    }
    __syncthreads();
    double* z = nullptr;
    tail_sweeps<D, kNu>(comp, tmp, g, lv[k].th, nu, &z);
    for (int p = threadIdx.x; p < G.Nc; p += blockDim.x) cur[p] = to_t<T>(add_(double(cur[p]), mul_(-1.0, z[p])));
    __syncthreads();
    T* dst = (k == nlev - 1) ? fine_out : fin;
    for (int p = threadIdx.x; p < G.N; p += blockDim.x) {
      int j[TailGeo<D>::R];
      tail_unravel<D>(p, G, j);
      bool nodal = true;
#pragma unroll
      for (int i = 0; i < TAIL_ND(G); ++i) nodal &= !(j[i] & 1);
      if (nodal) {
        int cc = 0;
#pragma unroll
        for (int i = 0; i < TAIL_ND(G); ++i) cc += (j[i] >> 1) * G.cst[i];
        dst[p] = cur[cc];
      } else {
        const double pred = tail_predict<T, kNu, D>(cur, true, G, nu, j);
        dst[p] = to_t<T>(add_(double(shell[tail_shell_pos<D>(G, j)]), pred));
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

// Rank-specialised tails for 1-4 dimensions (the common cases), runtime
// rank otherwise; d_nu: per-level nonuniform tables (same order as the
// levels) or null for uniform coordinates.
template <typename T>
cudaError_t tail_decompose(const T* blk, T* out, T* coarse_out, const void* d_levels, const void* d_nu, int nlev,
                           int64_t nmax, int d, const Exec& ex) {
  switch (d) {
    case 1: return tail_dec_t<T, 1>(blk, out, coarse_out, d_levels, d_nu, nlev, nmax, ex);
    case 2: return tail_dec_t<T, 2>(blk, out, coarse_out, d_levels, d_nu, nlev, nmax, ex);
    case 3: return tail_dec_t<T, 3>(blk, out, coarse_out, d_levels, d_nu, nlev, nmax, ex);
    case 4: return tail_dec_t<T, 4>(blk, out, coarse_out, d_levels, d_nu, nlev, nmax, ex);
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
    case 4: return tail_rec_t<T, 4>(coeffs, coarse_in, fine_out, d_levels, d_nu, nlev, nmax, ex);
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
// a0 = 1: axis 0 is already done (comp holds its solved m0 x ... result).
static void run_sweeps(double* comp, double* tmp, const LevelGeom& g, const ThomasLevel* th, const NuLevel* nu,
                       double** result, const Exec& ex, bool fast, int a0 = 0) {
  int64_t cur[kMaxD];
  for (int i = 0; i < g.d; ++i) cur[i] = i < a0 ? g.m[i] : g.n[i];
  double* x = comp;
  double* y = tmp;
  for (int a = a0; a < g.d; ++a) {
    int64_t outer = 1, inner = 1;
    for (int i = 0; i < a; ++i) outer *= cur[i];
    for (int i = a + 1; i < g.d; ++i) inner *= cur[i];
    const int64_t lines = outer * inner;
    const int grid = grid_for(lines, 128, 32);
    // the serial per-line sweep saturates the GPU when there are many lines;
    // few long lines (2-D levels) need the segmented solve
    const int64_t outs_all = outer * g.m[a] * inner;
    static const bool seg_all = std::getenv("MGRX_SEG_BIG_ONLY") == nullptr;
    if (fast && !nu && (seg_all || lines >= (int64_t(1) << 17)) && g.m[a] <= 640 && outs_all < (int64_t(1) << 32)) {
      // many lines: the restriction (32-bit index math), then the segmented
      // column pass (or the row pass for the contiguous axis) on y
      MGRX_LAUNCH(ex, "gen_load", k_axis_load32<<<grid_for(outs_all, 256), 256, 0, ex.s>>>(
                                      x, y, uint32_t(outs_all), uint32_t(inner), uint32_t(g.n[a]), uint32_t(g.m[a]),
                                      FastDiv(uint32_t(inner)), FastDiv(uint32_t(g.m[a]))));
      if (inner == 1 && g.m[a] <= kShortRow)
        launch_rows_thomas(y, outer, int(g.m[a]), th->w[a], th->inv_d[a], ex);
      else if (f3_axis_solve(y, outer, g.m[a], inner, th->w[a], th->inv_d[a], ex) != cudaSuccess)
        cudaGetLastError();
    } else if (fast && lines < (int64_t(1) << 17)) {
      const int64_t outs = outer * g.m[a] * inner;
      if (nu)
        MGRX_LAUNCH(ex, "gen_load", k_axis_load<true><<<grid_for(outs, 256), 256, 0, ex.s>>>(x, y, outer, inner, g.n[a], g.m[a], nu->ax[a].s));
      else
        MGRX_LAUNCH(ex, "gen_load", k_axis_load<false><<<grid_for(outs, 256), 256, 0, ex.s>>>(x, y, outer, inner, g.n[a], g.m[a], nullptr));
      const int SY = int(std::max<int64_t>(1, std::min<int64_t>(32, (g.m[a] + 31) / 32)));
      const double* w = nu ? nu->ax[a].tw : th->w[a];
      const double* id = nu ? nu->ax[a].tid : th->inv_d[a];
      const double* of = nu ? nu->ax[a].off : nullptr;
      (void)SY;
      int nw = 8;
      while (nw > 1 && size_t(nw + (of ? 3 : 2)) * size_t(g.m[a]) * 8 > size_t(200) * 1024) nw >>= 1;
      const size_t row_smem = size_t(nw + (of ? 3 : 2)) * size_t(g.m[a]) * 8;
      if (inner == 1 && row_smem <= size_t(200) * 1024) {
        cudaFuncSetAttribute(k_axis_solve_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, int(row_smem));
        const int64_t blocks = std::min<int64_t>((lines + nw - 1) / nw, int64_t(kNumSMs) * 8);
        MGRX_LAUNCH(ex, "gen_solve", k_axis_solve_rows<<<unsigned(blocks), 32 * nw, row_smem, ex.s>>>(y, lines, int(g.m[a]), w, id, of));
      } else {
        launch_axis_solve(y, lines, g.m[a], inner, w, id, of, ex);
      }
    } else if (inner == 1 && size_t(128) * size_t((g.n[a] | 1) + (g.m[a] | 1)) * 8 <= size_t(160) * 1024) {
      // contiguous lines: staged in shared memory (same arithmetic as k_sweep)
      const size_t sm = size_t(128) * size_t((g.n[a] | 1) + (g.m[a] | 1)) * 8;
      const unsigned blocks = unsigned((lines + 127) / 128);
      if (nu) {
        cudaFuncSetAttribute(k_sweep_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        MGRX_LAUNCH(ex, "gen_sweep", k_sweep_rows<true><<<blocks, 128, sm, ex.s>>>(x, y, lines, int(g.n[a]), int(g.m[a]), nullptr, nullptr, nu->ax[a]));
      } else {
        cudaFuncSetAttribute(k_sweep_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        MGRX_LAUNCH(ex, "gen_sweep", k_sweep_rows<false><<<blocks, 128, sm, ex.s>>>(x, y, lines, int(g.n[a]), int(g.m[a]), th->w[a], th->inv_d[a], NuAxis{}));
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

// MGRX_NO_WALK: the per-node rank 3-4 kernels instead of the axis-0 walkers (A/B).
static bool walk_off() {
  static const bool off = std::getenv("MGRX_NO_WALK") != nullptr;
  return off;
}

// Path "auto", rank >= 2: coefficients (kRec: the component) fused with the
// axis-0 load into comp (m0 x inner), then the axis-0 solve in place.
template <typename T, bool kRec>
static void coef_load0_axis0(const T* src, T* shell, T* coarse, double* comp, const LevelGeom& g,
                             const ThomasLevel* th, const NuLevel* nu, const Exec& ex) {
  const int64_t inner = g.N / g.n[0], m0 = g.m[0];
  const int chunk = int(std::max<int64_t>(1, std::min<int64_t>(64, m0 * inner / (int64_t(600) << 10))));
  const int64_t work = ((m0 + chunk - 1) / chunk) * (g.d <= 4 ? inner / g.n[g.d - 1] * g.m[g.d - 1] : inner);
  const int grid = grid_for(work, 256);
  const NuLevel z = nu ? *nu : NuLevel{};
  LevelGeom gp = g;  // rank 3-4 pair kernels: dividers by m_last and by the middle row count
  gp.fn[g.d - 1] = FastDiv(uint32_t(g.m[g.d - 1]));
  gp.fn[0] = FastDiv(uint32_t(inner / g.n[g.d - 1]));
#define L_(NU, D)                                                                                         \
  MGRX_LAUNCH(ex, kRec ? "gen_comp_load0" : "gen_coef_load0",                                             \
              (k_coef_load0<T, kRec, NU, D><<<grid, 256, 0, ex.s>>>(src, shell, coarse, comp, g, z, inner, chunk)))
#define R_(NU)                                                                                             \
  if (g.d == 2)                                                                                            \
    MGRX_LAUNCH(ex, kRec ? "gen_comp_load0" : "gen_coef_load0",                                            \
                (k2_coef_load0<T, kRec, NU><<<grid, 256, 0, ex.s>>>(src, shell, coarse, comp, g, z, chunk))); \
  else if (g.d == 3 && g.N < (int64_t(1) << 32))                                                          \
    MGRX_LAUNCH(ex, kRec ? "gen_comp_load0" : "gen_coef_load0",                                            \
                (kN_coef_load0<T, kRec, NU, 3><<<grid, 256, 0, ex.s>>>(src, shell, coarse, comp, gp, z, inner, chunk))); \
  else if (g.d == 4 && g.N < (int64_t(1) << 32))                                                          \
    MGRX_LAUNCH(ex, kRec ? "gen_comp_load0" : "gen_coef_load0",                                            \
                (kN_coef_load0<T, kRec, NU, 4><<<grid, 256, 0, ex.s>>>(src, shell, coarse, comp, gp, z, inner, chunk))); \
  else                                                                                                     \
    L_(NU, 0);
  if (nu) {
    R_(true)
  } else if ((g.d == 3 || g.d == 4) && g.N < (int64_t(1) << 32) && !walk_off()) {
    if (g.d == 3)
      MGRX_LAUNCH(ex, kRec ? "gen_comp_load0" : "gen_coef_load0",
                  (kN_coef_load0w<T, kRec, 3><<<grid, 256, 0, ex.s>>>(src, shell, coarse, comp, gp, inner, chunk)));
    else
      MGRX_LAUNCH(ex, kRec ? "gen_comp_load0" : "gen_coef_load0",
                  (kN_coef_load0w<T, kRec, 4><<<grid, 256, 0, ex.s>>>(src, shell, coarse, comp, gp, inner, chunk)));
  } else {
    R_(false)
  }
#undef R_
#undef L_
  const double* w = nu ? nu->ax[0].tw : th->w[0];
  const double* id = nu ? nu->ax[0].tid : th->inv_d[0];
  const double* of = nu ? nu->ax[0].off : nullptr;
  static const bool seg_all = std::getenv("MGRX_SEG_BIG_ONLY") == nullptr;
  if (!nu && seg_all && f3_axis0_solve(comp, m0, inner, w, id, ex) == cudaSuccess) {
    // segmented column pass (any number of columns)
  } else if (inner < (int64_t(1) << 17)) {
    cudaGetLastError();
    launch_axis_solve(comp, inner, m0, inner, w, id, of, ex);
  } else if (nu) {
    MGRX_LAUNCH(ex, "gen_thomas", k_axis_thomas<true><<<grid_for(inner, 128, 32), 128, 0, ex.s>>>(comp, inner, inner, m0, nullptr, nullptr, nu->ax[0]));
  } else if (f3_axis0_solve(comp, m0, inner, w, id, ex) != cudaSuccess) {
    cudaGetLastError();
    MGRX_LAUNCH(ex, "gen_thomas", k_axis_thomas<false><<<grid_for(inner, 128, 32), 128, 0, ex.s>>>(comp, inner, inner, m0, w, id, NuAxis{}));
  }
}

template <typename T>
cudaError_t general_decompose_level(const T* blk, T* shell, T* coarse, double* comp, double* tmp, const LevelGeom& g,
                                    const ThomasLevel* th, const NuLevel* nu, const Exec& ex, bool fast) {
  double* z = nullptr;
  if (fast && g.d >= 2) {
    coef_load0_axis0<T, false>(blk, shell, coarse, comp, g, th, nu, ex);
    run_sweeps(comp, tmp, g, th, nu, &z, ex, fast, 1);
  } else {
    launch_dec_coef<T>(blk, shell, coarse, comp, g, nu, ex);
    run_sweeps(comp, tmp, g, th, nu, &z, ex, fast);
  }
  MGRX_LAUNCH(ex, "gen_apply", k_apply<T><<<grid_for(g.Nc, 256), 256, 0, ex.s>>>(coarse, z, g.Nc, 1.0));
  return cudaGetLastError();
}

template <typename T>
cudaError_t general_recompose_level(const T* shell, T* coarse, T* fine, double* comp, double* tmp, const LevelGeom& g,
                                    const ThomasLevel* th, const NuLevel* nu, const Exec& ex, bool fast) {
  double* z = nullptr;
  if (fast && g.d >= 2) {
    coef_load0_axis0<T, true>(shell, nullptr, nullptr, comp, g, th, nu, ex);
    run_sweeps(comp, tmp, g, th, nu, &z, ex, fast, 1);
  } else {
    launch_rec_comp<T>(shell, comp, g, ex);
    run_sweeps(comp, tmp, g, th, nu, &z, ex, fast);
  }
  MGRX_LAUNCH(ex, "gen_apply", k_apply<T><<<grid_for(g.Nc, 256), 256, 0, ex.s>>>(coarse, z, g.Nc, -1.0));
  if (fast && g.d == 2 && g.N < (int64_t(1) << 32)) {
    LevelGeom g2 = g;
    g2.fn[0] = FastDiv(uint32_t(g.m[1]));
    const int grid = grid_for(g.n[0] * g.m[1], 256);
    if (nu)
      MGRX_LAUNCH(ex, "gen_rec_interp", k2_rec_interp<T, true><<<grid, 256, 0, ex.s>>>(shell, coarse, fine, g2, *nu));
    else
      MGRX_LAUNCH(ex, "gen_rec_interp", k2_rec_interp<T, false><<<grid, 256, 0, ex.s>>>(shell, coarse, fine, g2, NuLevel{}));
    return cudaGetLastError();
  }
  if (fast && !nu && (g.d == 3 || g.d == 4) && g.N < (int64_t(1) << 32) && !walk_off()) {
    const int64_t inner = g.N / g.n[0];
    const int64_t pairs = inner / g.n[g.d - 1] * g.m[g.d - 1];
    int chunk = int(std::max<int64_t>(1, std::min<int64_t>(32, g.n[0] * pairs / (int64_t(600) << 10))));
    chunk += chunk & 1;
    LevelGeom gp = g;
    gp.fn[g.d - 1] = FastDiv(uint32_t(g.m[g.d - 1]));
    gp.fn[0] = FastDiv(uint32_t(inner / g.n[g.d - 1]));
    const int grid = grid_for(((g.n[0] + chunk - 1) / chunk) * pairs, 256);
    if (g.d == 3)
      MGRX_LAUNCH(ex, "gen_rec_interp", (kN_rec_interpw<T, 3><<<grid, 256, 0, ex.s>>>(shell, coarse, fine, gp, inner, chunk)));
    else
      MGRX_LAUNCH(ex, "gen_rec_interp", (kN_rec_interpw<T, 4><<<grid, 256, 0, ex.s>>>(shell, coarse, fine, gp, inner, chunk)));
    return cudaGetLastError();
  }
  if (fast && (g.d == 3 || g.d == 4) && g.N < (int64_t(1) << 32)) {
    const int grid = grid_for(g.N / g.n[g.d - 1] * g.m[g.d - 1], 256);
    const NuLevel z = nu ? *nu : NuLevel{};
    LevelGeom gp = g;
    gp.fn[g.d - 1] = FastDiv(uint32_t(g.m[g.d - 1]));
#define I_(NU, D) MGRX_LAUNCH(ex, "gen_rec_interp", (kN_rec_interp<T, NU, D><<<grid, 256, 0, ex.s>>>(shell, coarse, fine, gp, z)))
    if (g.d == 3) {
      if (nu) I_(true, 3); else I_(false, 3);
    } else {
      if (nu) I_(true, 4); else I_(false, 4);
    }
#undef I_
    return cudaGetLastError();
  }
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

// coarse[p] <- T(double(coarse[p]) + sign z[p]) over n values (slab mode's
// apply after the axis-0 transpose back; apply_correction, transform.hpp:435-477).
template <typename T>
cudaError_t apply_correction(T* coarse, const double* z, int64_t n, double sign, const Exec& ex) {
  if (n <= 0) return cudaSuccess;
  MGRX_LAUNCH(ex, "gen_apply", k_apply<T><<<grid_for(n, 256), 256, 0, ex.s>>>(coarse, z, n, sign));
  return cudaGetLastError();
}
template cudaError_t apply_correction<float>(float*, const double*, int64_t, double, const Exec&);
template cudaError_t apply_correction<double>(double*, const double*, int64_t, double, const Exec&);

template cudaError_t tail_decompose<float>(const float*, float*, float*, const void*, const void*, int, int64_t, int,
                                           const Exec&);
template cudaError_t tail_decompose<double>(const double*, double*, double*, const void*, const void*, int, int64_t,
                                            int, const Exec&);
template cudaError_t tail_recompose<float>(const float*, const float*, float*, const void*, const void*, int, int64_t,
                                           int, const Exec&);
template cudaError_t tail_recompose<double>(const double*, const double*, double*, const void*, const void*, int,
                                            int64_t, int, const Exec&);

}  // namespace mgrx_b200
