// Second-generation fused 3-D level pass (see p2.h) for sm_100a.
//
// Replaces, on fp32 3-D levels with odd extents, the reference's per-level
// sequence (reorder_level, reorder.hpp:131; compute_coefficients,
// transform.hpp:310; compute_correction, :331-431; apply_correction,
// :435-477; pack_level_centric, reorder.hpp:162) with two passes over the
// level (plus a small carry kernel):
//
//   k_p2_plane  one CTA per (chunk of coarse planes, tile of T coarse rows);
//               the tile's fine rows stream plane by plane through a TMA
//               ring.  Thread = one coarse column (pair of fine columns),
//               warps of 30 owned + 2 halo columns.  Per fine row: the
//               coefficients (decompose; corner sums of update_coefficients,
//               transform.hpp:216-304) or the component read from the shell
//               (recompose), the axis-1 load stencil accumulated in registers
//               (load_entry, transform.hpp:84-96, in stencil order); per
//               finished coarse row the axis-2 stencil through shuffles and
//               the axis-0 stencil into two running accumulators per coarse
//               row.  A finished coarse plane (the load vector L0 L1 L2 c) is
//               solved along axis 2 by one warp per row (segmented Thomas,
//               batched_solve :116-130), run through the axis-0 forward
//               elimination of the chunk (f_i -= w_i f_{i-1}, carry 0 at the
//               chunk start) and stored; the CTA that stores a plane's last
//               row solves the plane along axis 1 in place (it is in L2).
//               The chunk's first/last fine planes' shares of the
//               neighbouring chunks' coarse planes are exported instead of
//               being recomputed by the neighbour.
//   k_p2_carry  per (row, column): the axis-0 forward carries across chunks
//               and the back-substitution values at the chunk boundaries.
//   k_p2_col    per (row, column, chunk): axis-0 back substitution
//               z_i = (g_i - z_{i+1}/3) / d_i and coarse = T(coarse +/- z).
//
// The correction z = T0 T1 T2 L0 L1 L2 c is the reference's tensor-product
// S0 S1 S2 c (S_a = Thomas_a o Load_a, transform.hpp:392-428) with the
// operators reordered (they act on different axes and commute exactly) and
// the recurrences split into segments joined by exact affine carries: only
// rounding differs from the reference (parity tests: 1e-5 of the range for
// fp32, labels bit-exact up to bin-edge ties).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "p2.h"

namespace mgrx_b200 {

namespace {

constexpr int kT = 4;          // coarse rows per tile
constexpr int kNS = 3;         // ring slots
constexpr int kMaxThreads = 576;  // 18 warps of 30 owned columns (m2 <= 540)
constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(su32(bar)), "r"(parity), "r"(100000u)
      : "memory");
  return ok != 0;
}
// A wait that never completes (a bug) traps after ~4 s instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!mbar_try(bar, parity)) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) asm volatile("trap;");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 16-byte rounded span of [a, a + bytes): start, length, lead (bytes)
struct Span {
  const char* src;
  uint32_t bytes;
  int lead;
};
__device__ __forceinline__ Span span16(const void* p, int64_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t a0 = a & ~uintptr_t(15), a1 = (a + uintptr_t(bytes) + 15) & ~uintptr_t(15);
  return Span{reinterpret_cast<const char*>(a0), uint32_t(a1 - a0), int(a - a0)};
}

// Shell offset of reordered row (r0, r1) of a 3-D level block
// (pack_level_centric, reorder.hpp:180-215).
__device__ __forceinline__ int64_t shell_row(const P2Geom& g, int64_t r0, int64_t r1) {
  const int64_t before = (r0 < g.m0) ? r0 * g.m1 + min(r1, int64_t(g.m1)) : int64_t(g.m0) * g.m1;
  return (r0 * g.n1 + r1) * g.n2 - before * g.m2;
}

// ------------------------------------------------------------ shared memory
struct Pipe {
  uint64_t full[4];
  int cnt[4];
};
static_assert(sizeof(Pipe) <= 256, "pipe state");

__host__ __device__ inline int hpitch(int m2, int cpl) { return ((m2 + m2 / cpl + 2) + 1) & ~1; }
__device__ __forceinline__ int hidx(int k, int cpl) { return k + k / cpl; }

struct Layout {
  size_t slot, evb, ring, pipe, hbuf, gprev, sacc, total;
};
__host__ __device__ inline Layout layout(const P2Geom& g, int mode, int cpl) {
  Layout L{};
  const int T = kT;
  if (mode == 0) {
    L.slot = ((size_t(2 * T + 2) * size_t(g.in_sr) + size_t(g.n2)) * 4 + 32 + 127) / 128 * 128;
    L.evb = 0;
  } else {
    L.evb = (size_t(T + 2) * size_t(g.n2) * 4 + 32 + 127) / 128 * 128;
    L.slot = (L.evb + size_t(T + 1) * size_t(g.n2) * 4 + 32 + 127) / 128 * 128;
  }
  L.ring = 0;
  L.pipe = kNS * L.slot;
  L.hbuf = L.pipe + 256;
  L.gprev = L.hbuf + size_t(2) * (T + 1) * hpitch(g.m2, cpl) * 8;
  L.sacc = L.gprev + size_t(T + 1) * g.m2 * 8;
  L.total = L.sacc + size_t(T + 1) * g.m2 * 8;
  return L;
}

// ----------------------------------------------------------- axis-2 solve
// Thomas solve (ThomasAux factors; batched_solve, transform.hpp:116-130) of
// one row of m2 = 32 CPL + 1 values held in shared memory at hidx(k): lane
// q owns [CPL q, CPL q + CPL) (lane 31 also the last value); the segments'
// affine carries are combined by a shuffle scan, then every segment reruns
// the exact recurrence from its true carry.
template <int CPL>
__device__ __forceinline__ void warp_t2(double* hb, int m2, const double* __restrict__ w2,
                                        const double* __restrict__ id2) {
  const int lane = threadIdx.x & 31;
  const int s0 = lane * CPL;
  const bool tail = lane == 31;
  // value r of this lane's segment: index s0 + r (r < CPL), the tail m2 - 1
  auto kof = [&](int r) { return r < CPL ? s0 + r : m2 - 1; };
  double v[CPL + 1];
#pragma unroll
  for (int r = 0; r < CPL; ++r) v[r] = hb[s0 + r + lane];
  v[CPL] = tail ? hb[hidx(m2 - 1, CPL)] : 0.0;
  // forward y_k = f_k - w_k y_{k-1}
  double a = 0.0, b = 1.0;
#pragma unroll
  for (int r = 0; r <= CPL; ++r)
    if (r < CPL || tail) {
      const double wk = __ldg(w2 + kof(r));
      a = fma(-wk, a, v[r]);
      b = -wk * b;
    }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double ao = __shfl_up_sync(kFull, a, off), bo = __shfl_up_sync(kFull, b, off);
    if (lane >= off) {
      a = fma(b, ao, a);
      b *= bo;
    }
  }
  double y = __shfl_up_sync(kFull, a, 1);
  if (lane == 0) y = 0.0;
#pragma unroll
  for (int r = 0; r <= CPL; ++r)
    if (r < CPL || tail) {
      y = fma(-__ldg(w2 + kof(r)), y, v[r]);
      v[r] = y;
    }
  // back substitution x_k = (y_k - x_{k+1}/3) / d_k
  a = 0.0;
  b = 1.0;
#pragma unroll
  for (int r = CPL; r >= 0; --r)
    if (r < CPL || tail) {
      const double idk = __ldg(id2 + kof(r));
      a = (v[r] - kOff * a) * idk;
      b = -kOff * idk * b;
    }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double ao = __shfl_down_sync(kFull, a, off), bo = __shfl_down_sync(kFull, b, off);
    if (lane + off < 32) {
      a = fma(b, ao, a);
      b *= bo;
    }
  }
  double x = __shfl_down_sync(kFull, a, 1);
  if (lane == 31) x = 0.0;
#pragma unroll
  for (int r = CPL; r >= 0; --r)
    if (r < CPL || tail) {
      x = (v[r] - kOff * x) * __ldg(id2 + kof(r));
      v[r] = x;
    }
#pragma unroll
  for (int r = 0; r < CPL; ++r) hb[s0 + r + lane] = v[r];
  if (tail) hb[hidx(m2 - 1, CPL)] = v[CPL];
}

// ------------------------------------------------------------ plane pass
enum EmitKind { kNone = 0, kReg = 1, kExpU = 2, kExpD = 3 };

template <int MODE, int CPL, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT <= 288 ? 2 : 1)
    k_p2_plane(const float* __restrict__ src, float* __restrict__ shell, float* __restrict__ coarse, const P2Geom g,
               const P2Bufs bf, const P2Tabs tb) {
  constexpr int T = kT;
  constexpr int NR = 2 * T + 3;  // fine rows of a tile (local row i <-> fine row 2 b0 - 2 + i)
  constexpr int NE = T + 2;      // even rows
  extern __shared__ __align__(128) unsigned char smem[];
  const Layout LY = layout(g, MODE, CPL);
  Pipe* pp = reinterpret_cast<Pipe*>(smem + LY.pipe);
  double* hbuf = reinterpret_cast<double*>(smem + LY.hbuf);
  double* gprev = reinterpret_cast<double*>(smem + LY.gprev);
  double* sacc = reinterpret_cast<double*>(smem + LY.sacc);
  const int HP = hpitch(g.m2, CPL);

  const int tile = int(blockIdx.x) % g.ntile, chunk = int(blockIdx.x) / g.ntile;
  const bool last_tile = tile == g.ntile - 1, last_chunk = chunk == g.nchunk - 1;
  const int b0 = tile * T;
  const int TR = last_tile ? T + 1 : T;
  const int a0 = chunk * g.C, a1 = last_chunk ? g.m0 : a0 + g.C;
  const int p0 = 2 * a0;
  const int pend = last_chunk ? g.n0 : 2 * a1;      // processed planes [p0, pend)
  const int D = (last_chunk ? g.n0 - 1 : 2 * a1) - p0;  // loaded planes p0 + [0, D]
  const int rbase = 2 * b0 - 2;
  const int rlo = max(0, rbase), rhi = 2 * (b0 + T);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  const int c = 30 * warp - 1 + lane;
  const bool valid = c >= 0 && c < g.m2;
  const bool owned = valid && lane >= 1 && lane <= 30;
  const int cc = valid ? c : 0;
  const bool has_o = valid && c < g.m2 - 1;
  const double w2c = (c == 0 || c == g.m2 - 1) ? kW5_12 : kW5_6;
  // axis-1 load weight of the tile's coarse row q (5/12 on the grid's first and last row)
  const bool first_tile = b0 == 0;
  auto w1q = [&](int q) { return ((q == 0 && first_tile) || (q == T && last_tile)) ? kW5_12 : kW5_6; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s) {
      mbar_init(&pp->full[s], 1);
      pp->cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();

  // ---- TMA ring: slot d % kNS holds the tile's rows of plane p0 + d
  auto plane_src = [&](int d, Span* sp0, Span* sp1) {
    const int p = p0 + d;
    if (MODE == 0) {
      const float* s = src + int64_t(p) * g.in_sp + int64_t(rlo) * g.in_sr;
      *sp0 = span16(s, (int64_t(rhi - rlo) * g.in_sr + g.n2) * 4);
      sp1->bytes = 0;
      sp1->lead = 0;
    } else {
      const int64_t r0 = (p & 1) ? g.m0 + (p >> 1) : (p >> 1);
      const int64_t elo = rlo >> 1, ehi = rhi >> 1, olo = (rlo + 1) >> 1, ohi = (rhi - 1) >> 1;
      const int64_t se = shell_row(g, r0, elo), so = shell_row(g, r0, g.m1 + olo);
      *sp0 = span16(src + se, (shell_row(g, r0, ehi + 1) - se) * 4);
      *sp1 = span16(src + so, (ohi - olo + 1) * int64_t(g.n2) * 4);
    }
  };
  auto issue = [&](int d) {  // one thread
    Span a, b;
    plane_src(d, &a, &b);
    const int s = d % kNS;
    unsigned char* dst = smem + size_t(s) * LY.slot;
    fence_proxy_async();
    mbar_expect_tx(&pp->full[s], a.bytes + b.bytes);
    bulk_g2s(dst, a.src, a.bytes, &pp->full[s]);
    if (MODE == 1 && b.bytes) bulk_g2s(dst + LY.evb, b.src, b.bytes, &pp->full[s]);
  };
  auto wait_slot = [&](int d) { mbar_wait(&pp->full[d % kNS], uint32_t((d / kNS) & 1)); };
  auto release = [&](int d) {
    __syncwarp();
    if (lane == 0) {
      const int s = d % kNS;
      __threadfence_block();
      const int old = atomicAdd(&pp->cnt[s], 1);
      if (old == nwarp - 1) {
        pp->cnt[s] = 0;
        if (d + kNS <= D) issue(d + kNS);
      }
    }
  };
  if (threadIdx.x == 0)
    for (int d = 0; d <= min(D, kNS - 1); ++d) issue(d);

  // ---- per-thread state
  double Le[T + 1], Lo[T + 1];  // axis-1 accumulators (fine resolution: the column pair)
  double A[T + 1], B[T + 1];    // axis-0 accumulators (coarse planes k, k+1 or k-1, k)
  double P[NE];                 // decompose: nodal values of the last even plane's even rows
#pragma unroll
  for (int q = 0; q <= T; ++q) Le[q] = Lo[q] = A[q] = B[q] = 0.0;
#pragma unroll
  for (int e = 0; e < NE; ++e) P[e] = 0.0;

  int ecount = 0;  // emissions so far (their Hbuf buffer alternates)
  // solver phase of one emission: warp q < TR solves row q of the buffer
  auto solve_row = [&](int kind, int k, int buf, int q) {
    double* hb = hbuf + (size_t(buf) * (T + 1) + q) * HP;
    warp_t2<CPL>(hb, g.m2, tb.w2, tb.id2);
    __syncwarp();
    const int64_t row = int64_t(b0 + q) * g.PG;
    if (kind == kReg) {
      const double w0k = tb.w0[k], gk = tb.gam0[k];
      const bool first = k == a0, lastk = k == a1 - 1;
      double* gp = gprev + q * g.m2;
      double* sp = sacc + q * g.m2;
      double* Gk = bf.G + int64_t(k) * g.GP + row;
      double* Sc = bf.S + int64_t(chunk) * g.GP + row;
#pragma unroll
      for (int t = 0; t <= CPL; ++t) {
        const int kk = lane + 32 * t;
        if (kk < g.m2) {
          const double y = hb[hidx(kk, CPL)];
          const double gl = first ? y : fma(-w0k, gp[kk], y);
          gp[kk] = gl;
          const double s = first ? gk * gl : fma(gk, gl, sp[kk]);
          sp[kk] = s;
          __stcg(Gk + kk, gl);
          if (lastk) __stcg(Sc + kk, s);
        }
      }
    } else {
      double* E = (kind == kExpU ? bf.EU : bf.ED) + int64_t(chunk) * g.GP + row;
#pragma unroll
      for (int t = 0; t <= CPL; ++t) {
        const int kk = lane + 32 * t;
        if (kk < g.m2) __stcg(E + kk, hb[hidx(kk, CPL)]);
      }
    }
  };
  auto solve = [&](int kind, int k, int buf) {
    for (int q = warp; q < TR; q += nwarp) solve_row(kind, k, buf, q);
  };

  // ---- decompose: nodal values of the first plane's even rows
  if (MODE == 0) {
    wait_slot(0);
    Span a, b;
    plane_src(0, &a, &b);
    const float* s0 = reinterpret_cast<const float*>(smem + a.lead) + 2 * cc;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int r = rbase + 2 * e;
      if (r >= 0) P[e] = double(s0[int64_t(r - rlo) * g.in_sr]);
    }
  }

  for (int d = 0; d + p0 < pend; ++d) {
    const int p = p0 + d;
    const int k = p >> 1;
    const bool podd = p & 1;
    wait_slot(d);
    if (MODE == 0 && podd) wait_slot(d + 1);
    // emissions of this plane (uniform)
    int e1 = kNone, e1k = -1, e2 = kNone, e2k = -1;
    if (!podd) {
      if (k > a0) {
        e1 = kReg;
        e1k = k - 1;
      } else if (chunk > 0) {
        e1 = kExpU;
      }
      if (p == g.n0 - 1) {
        e2 = kReg;
        e2k = k;
      }
    } else if (!last_chunk && p == 2 * a1 - 1) {
      e1 = kReg;
      e1k = k;
      e2 = kExpD;
    }
    const int buf1 = ecount & 1, buf2 = (ecount + (e1 != kNone ? 1 : 0)) & 1;
    // a second emission reuses the buffer of the previous plane's emission:
    // wait until every warp has finished solving it
    if (e1 != kNone && e2 != kNone) __syncthreads();
    const double w0k = (k == 0 || k == g.m0 - 1) ? kW5_12 : kW5_6;

    Span sa, sb;
    plane_src(d, &sa, &sb);
    const unsigned char* slot = smem + size_t(d % kNS) * LY.slot;
    // decompose: this plane's and (odd planes) the next plane's row rlo of the slot at column 2 cc
    const float* rs = reinterpret_cast<const float*>(slot + sa.lead) + 2 * cc;
    const float* rn = rs;
    if (MODE == 0 && podd) {
      Span na, nb;
      plane_src(d + 1, &na, &nb);
      rn = reinterpret_cast<const float*>(smem + size_t((d + 1) % kNS) * LY.slot + na.lead) + 2 * cc;
    }
    // shell rows of this plane (decompose stores): even fine row 2e at
    // seb + e * ses, odd fine row 2e + 1 at sob + e * n2
    // (32-bit offsets: a level block has < 2^31 elements)
    const int64_t r0s = podd ? g.m0 + k : k;
    const int seb = int(shell_row(g, r0s, 0)) + c;
    const int sob = int(shell_row(g, r0s, g.m1)) + c;
    const int ses = podd ? g.n2 : g.m2 - 1;
    const int cob = int(int64_t(k) * g.co_sp) + c;
    // recompose runs: even rows 2e (e >= elo) and odd rows 2e + 1 (e >= olo)
    const float* evr = reinterpret_cast<const float*>(slot + sa.lead) + cc;
    const float* odr = reinterpret_cast<const float*>(slot + LY.evb + sb.lead) + cc;
    const int elo = rlo >> 1, olo = (rlo + 1) >> 1;
    // emission targets of this lane (row q at + q * HP)
    const int hb1 = buf1 * (T + 1) * HP + hidx(cc, CPL);
    const int hb2 = buf2 * (T + 1) * HP + hidx(cc, CPL);
    const bool w1e = owned && e1 != kNone, w2e = owned && e2 != kNone;

    // One plane, row by row, with the plane parity a compile-time constant:
    // every row runs the same instruction stream (rows missing at the grid
    // edge read a valid row and contribute zeros), so the shuffles stay in
    // converged code.
    auto body = [&](auto ppc) {
      constexpr bool PODD = decltype(ppc)::value;
      auto complete = [&](int q) {  // coarse row q of the tile: axis-2 stencil, axis-0 accumulation
        const double x = fma(0.5, Lo[q], kW12 * Le[q]);
        const double xl = __shfl_up_sync(kFull, x, 1);
        const double er = __shfl_down_sync(kFull, Le[q], 1);
        const double H = fma(kW12, er, fma(0.5, Lo[q], fma(w2c, Le[q], xl)));
        Le[q] = 0.0;
        Lo[q] = 0.0;
        if (!PODD) {
          const double ev = fma(kW12, H, A[q]);
          A[q] = fma(w0k, H, B[q]);
          B[q] = kW12 * H;
          if (w1e) hbuf[hb1 + q * HP] = ev;
          if (w2e) hbuf[hb2 + q * HP] = A[q];
        } else {
          A[q] = fma(0.5, H, A[q]);
          B[q] = fma(0.5, H, B[q]);
          if (w1e) {
            hbuf[hb1 + q * HP] = A[q];
            hbuf[hb2 + q * HP] = B[q];
          }
        }
      };
      double PSc = 0.0, PSn = 0.0, NXn = 0.0;  // odd planes: plane-pair sums of the even rows around row i
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const bool oddr = i & 1;
        const int e = i >> 1;
        const bool ex = i >= 2 || !first_tile;  // the fine row exists (uniform)
        const int off = ex ? rbase + i - rlo : 0;  // its row in the slot (a valid row otherwise)
        double ce = 0.0, co = 0.0;
        if (MODE == 0) {
          const float* row = rs + int64_t(off) * g.in_sr;
          const float fe = row[0];
          const double vo = double(row[1]);
          double E, se, so_;
          if (!PODD) {
            if (!oddr) {
              E = P[e];
              se = 0.0;
              so_ = 0.5;
            } else {
              E = P[e] + P[e + 1];
              se = 0.5;
              so_ = 0.25;
            }
          } else {
            // odd plane: the nodal values of planes p-1 (P) and p+1 at the even
            // rows; P[e] becomes plane p+1's value once row 2e is done
            if (!oddr) {
              if (i >= 3 || (i == 2 && !first_tile)) {  // computed by the odd row before
                E = PSn;
                P[e] = NXn;
              } else {
                const double nx = double(rn[int64_t(off) * g.in_sr]);
                E = P[e] + nx;
                P[e] = nx;
              }
              PSc = E;
              se = 0.5;
              so_ = 0.25;
            } else {
              NXn = double(rn[int64_t(off + 1) * g.in_sr]);
              PSn = P[e + 1] + NXn;
              E = PSc + PSn;
              se = 0.25;
              so_ = 0.125;
            }
          }
          const double Er = __shfl_down_sync(kFull, E, 1);
          const float to = __double2float_rn(fma(-(E + Er), so_, vo));
          const bool nodal = !PODD && !oddr;
          const float te = nodal ? fe : __double2float_rn(fma(-E, se, double(fe)));
          const bool store = owned && i >= 2 && (i < NR - 1 || last_tile);
          const int er_ = (rbase + i) >> 1;  // even row index of r (even r) / odd row index (odd r)
          if (store) {
            if (nodal) {
              coarse[cob + er_ * int(g.co_sr)] = fe;
              if (has_o) shell[seb + er_ * ses] = to;
            } else if (!oddr) {
              shell[seb + er_ * ses] = te;
              if (has_o) shell[seb + er_ * ses + g.m2] = to;
            } else {
              shell[sob + er_ * g.n2] = te;
              if (has_o) shell[sob + er_ * g.n2 + g.m2] = to;
            }
          }
          ce = (ex && valid && !nodal) ? double(te) : 0.0;
          co = (ex && has_o) ? double(to) : 0.0;
        } else {
          if (!oddr) {
            const int ro = ex ? e + (rbase >> 1) - elo : 0;
            const float* row = evr + int64_t(ro) * (PODD ? g.n2 : g.m2 - 1);
            if (PODD) {
              ce = (ex && valid) ? double(row[0]) : 0.0;
              co = (ex && has_o) ? double(row[g.m2]) : 0.0;
            } else {
              co = (ex && has_o) ? double(row[0]) : 0.0;
            }
          } else {
            const int ro = ex ? e + (rbase >> 1) - olo : 0;
            const float* row = odr + int64_t(ro) * g.n2;
            ce = (ex && valid) ? double(row[0]) : 0.0;
            co = (ex && has_o) ? double(row[g.m2]) : 0.0;
          }
        }
        // axis-1 stencil of coarse rows q (load_entry order: rows ascending)
        if (!oddr) {
          const int qj = e - 1;
          if (qj - 1 >= 0) {
            Le[qj - 1] = fma(kW12, ce, Le[qj - 1]);
            Lo[qj - 1] = fma(kW12, co, Lo[qj - 1]);
          }
          if (qj >= 0 && qj <= T) {
            Le[qj] = fma(w1q(qj), ce, Le[qj]);
            Lo[qj] = fma(w1q(qj), co, Lo[qj]);
          }
          if (qj + 1 <= T) {
            Le[qj + 1] = fma(kW12, ce, Le[qj + 1]);
            Lo[qj + 1] = fma(kW12, co, Lo[qj + 1]);
          }
        } else {
          const int qj = e - 1;
          if (qj >= 0 && qj <= T) {
            Le[qj] = fma(0.5, ce, Le[qj]);
            Lo[qj] = fma(0.5, co, Lo[qj]);
          }
          if (qj + 1 <= T) {
            Le[qj + 1] = fma(0.5, ce, Le[qj + 1]);
            Lo[qj + 1] = fma(0.5, co, Lo[qj + 1]);
          }
        }
        if (!oddr && i >= 4) complete(e - 2);
        if (i == NR - 1) complete(T);  // the last tile's extra row (harmless elsewhere)
      }
    };
    if (podd) body(std::true_type{});
    else body(std::false_type{});
    release(d);
    if (e1 != kNone || e2 != kNone) {
      __syncthreads();
      if (e1 != kNone) solve(e1, e1k, buf1);
      if (e2 != kNone) solve(e2, e2k, buf2);
      ecount += (e1 != kNone ? 1 : 0) + (e2 != kNone ? 1 : 0);
    }
  }
  pdl_trigger();
}

// ------------------------------------------------------------ carries
// Per (row, column): the axis-0 forward carry X_c entering each chunk and the
// back-substitution value XB_c just above it (constants: see p2_plan).  The
// loads of a batch of chunks are issued before its recurrence steps.
__global__ void __launch_bounds__(256) k_p2_carry(const P2Geom g, const P2Bufs bf, const P2Tabs tb) {
  pdl_wait();
  const int64_t pos = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pos >= int64_t(g.m1) * g.m2) return;
  const int j = int(pos / g.m2), k = int(pos - int64_t(j) * g.m2);
  const int64_t gi = int64_t(j) * g.PG + k;
  const int NC = g.nchunk;
  const double* ch = tb.ch;
  constexpr int BT = 8;
  double Xc = 0.0;
  for (int c0 = 0; c0 < NC; c0 += BT) {
    double ge[BT], eu[BT], ed[BT];
#pragma unroll
    for (int u = 0; u < BT; ++u) {
      const int c = c0 + u;
      ge[u] = eu[u] = ed[u] = 0.0;
      if (c + 1 < NC) {
        ge[u] = __ldcg(bf.G + int64_t((c + 1) * g.C - 1) * g.GP + gi);
        eu[u] = __ldcg(bf.EU + int64_t(c + 1) * g.GP + gi);
        ed[u] = __ldcg(bf.ED + int64_t(c) * g.GP + gi);
      }
    }
#pragma unroll
    for (int u = 0; u < BT; ++u) {
      const int c = c0 + u;
      if (c < NC) {
        bf.X[int64_t(c) * g.GP + gi] = Xc;
        if (c + 1 < NC) {
          const double gend = ge[u] + ch[5 * c + 0] * Xc + eu[u];
          Xc = fma(-ch[5 * c + 4], gend, ed[u]);
        }
      }
    }
  }
  double xn = 0.0;
  for (int c1 = NC - 1; c1 >= 0; c1 -= BT) {
    double sv[BT], xv[BT], eu[BT];
#pragma unroll
    for (int u = 0; u < BT; ++u) {
      const int c = c1 - u;
      sv[u] = xv[u] = eu[u] = 0.0;
      if (c >= 0) {
        sv[u] = __ldcg(bf.S + int64_t(c) * g.GP + gi);
        xv[u] = bf.X[int64_t(c) * g.GP + gi];
        if (c + 1 < NC) eu[u] = __ldcg(bf.EU + int64_t(c + 1) * g.GP + gi);
      }
    }
#pragma unroll
    for (int u = 0; u < BT; ++u) {
      const int c = c1 - u;
      if (c >= 0) {
        bf.XB[int64_t(c) * g.GP + gi] = xn;
        xn = sv[u] + ch[5 * c + 1] * xv[u] + ch[5 * c + 2] * eu[u] + ch[5 * c + 3] * xn;
      }
    }
  }
  pdl_trigger();
}

// ------------------------------------------------------------ strip pass
// One CTA of 16 warps per (chunk, strip of 16 coarse columns); thread =
// (column, segment of RPS rows): lanes 0-15 segment 2w, lanes 16-31 segment
// 2w + 1 of warp w (segment 31 also owns the last row).  Planes of the chunk
// descending:
//   axis 0  g_i = G_i + A_i X_c (+ the next chunk's export on the chunk's top
//           plane), z_i = (g_i - z_{i+1}/3) / d_i (transform.hpp:121-129)
//   axis 1  Thomas along the column (batched_solve, :116-130): segments from a
//           zero carry, the segments' carries by a shuffle scan in the warp
//           that owns the column (data-independent segment factors), then
//           the carries' contributions added per row
//   apply   coarse = T(double(coarse) + sign z) (transform.hpp:461)
// The next plane's G and coarse values are loaded into registers while the
// current plane is solved.
constexpr int kSW = 16;  // columns per strip

template <int RPS>
__global__ void __launch_bounds__(512, 1) k_p2_strip(float* __restrict__ coarse, const P2Geom g, const P2Bufs bf,
                                                    const P2Tabs tb, double sign) {
  constexpr int NV = RPS + 1;
  __shared__ double F[32 * 17];  // [segment][column]
  const int nstrip = (g.m2 + kSW - 1) / kSW;
  const int chunk = int(blockIdx.x) / nstrip, strip = int(blockIdx.x) - chunk * nstrip;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cl = lane & 15, seg = 2 * w + (lane >> 4);
  const int col = kSW * strip + cl;
  const bool vc = col < g.m2;
  const int cc = vc ? col : g.m2 - 1;
  const int a0 = chunk * g.C, a1 = (chunk == g.nchunk - 1) ? g.m0 : a0 + g.C;
  const bool tail = seg == 31;
  auto row = [&](int jv) { return jv < RPS ? RPS * seg + jv : g.m1 - 1; };
  auto has = [&](int jv) { return jv < RPS || tail; };
  pdl_wait();
  double Xc[NV], XS[NV], gv[NV];
  float cv[NV];
#pragma unroll
  for (int jv = 0; jv < NV; ++jv) {
    Xc[jv] = XS[jv] = gv[jv] = 0.0;
    cv[jv] = 0.f;
    if (has(jv)) {
      const int64_t gi = int64_t(row(jv)) * g.PG + cc;
      Xc[jv] = __ldcg(bf.X + int64_t(chunk) * g.GP + gi);
      XS[jv] = __ldcg(bf.XB + int64_t(chunk) * g.GP + gi);
      gv[jv] = __ldcs(bf.G + int64_t(a1 - 1) * g.GP + gi);
      cv[jv] = coarse[int64_t(a1 - 1) * g.co_sp + int64_t(row(jv)) * g.co_sr + cc];
    }
  }
  for (int i = a1 - 1; i >= a0; --i) {
    double gn[NV];
    float cn[NV];
#pragma unroll
    for (int jv = 0; jv < NV; ++jv) {
      gn[jv] = 0.0;
      cn[jv] = 0.f;
      if (i > a0 && has(jv)) {
        const int r = row(jv);
        gn[jv] = __ldcs(bf.G + int64_t(i - 1) * g.GP + int64_t(r) * g.PG + cc);
        cn[jv] = coarse[int64_t(i - 1) * g.co_sp + int64_t(r) * g.co_sr + cc];
      }
    }
    const double Ai = __ldg(tb.A0 + i), idi = __ldg(tb.id0 + i);
    const bool top = i == a1 - 1 && chunk + 1 < g.nchunk;
    double v[NV];
#pragma unroll
    for (int jv = 0; jv < NV; ++jv) {
      v[jv] = 0.0;
      if (has(jv)) {
        double gg = fma(Ai, Xc[jv], gv[jv]);
        if (top) gg += __ldcg(bf.EU + int64_t(chunk + 1) * g.GP + int64_t(row(jv)) * g.PG + cc);
        const double x = (gg - kOff * XS[jv]) * idi;
        XS[jv] = x;
        v[jv] = x;
      }
    }
    // axis 1, forward: local segment from a zero carry
    double y = 0.0;
#pragma unroll
    for (int jv = 0; jv < NV; ++jv)
      if (has(jv)) {
        y = fma(-__ldg(tb.w1 + row(jv)), y, v[jv]);
        v[jv] = y;
      }
    F[seg * 17 + cl] = y;
    __syncthreads();
    if (w < kSW) {  // warp w: the 32 segments of column w (lane = segment)
      double a = F[lane * 17 + w];
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const double ao = __shfl_up_sync(kFull, a, 1 << s);
        if (lane >= (1 << s)) a = fma(__ldg(tb.sf + 32 * s + lane), ao, a);
      }
      double cin = __shfl_up_sync(kFull, a, 1);
      if (lane == 0) cin = 0.0;
      F[lane * 17 + w] = cin;
    }
    __syncthreads();
    const double cf = F[seg * 17 + cl];
    double x = 0.0;
#pragma unroll
    for (int jv = NV - 1; jv >= 0; --jv)
      if (has(jv)) {
        const int r = row(jv);
        const double yt = fma(__ldg(tb.af1 + r), cf, v[jv]);
        x = (yt - kOff * x) * __ldg(tb.id1 + r);
        v[jv] = x;
      }
    __syncthreads();  // every thread has read its forward carry
    F[seg * 17 + cl] = x;
    __syncthreads();
    if (w < kSW) {
      double a = F[lane * 17 + w];
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const double ao = __shfl_down_sync(kFull, a, 1 << s);
        if (lane + (1 << s) < 32) a = fma(__ldg(tb.sb + 32 * s + lane), ao, a);
      }
      double cin = __shfl_down_sync(kFull, a, 1);
      if (lane == 31) cin = 0.0;
      F[lane * 17 + w] = cin;
    }
    __syncthreads();
    const double cb = F[seg * 17 + cl];
#pragma unroll
    for (int jv = 0; jv < NV; ++jv)
      if (has(jv) && vc) {
        const int r = row(jv);
        const double z = fma(__ldg(tb.bb1 + r), cb, v[jv]);
        coarse[int64_t(i) * g.co_sp + int64_t(r) * g.co_sr + col] = __double2float_rn(fma(sign, z, double(cv[jv])));
      }
    __syncthreads();  // every thread has read its backward carry before F is reused
#pragma unroll
    for (int jv = 0; jv < NV; ++jv) {
      gv[jv] = gn[jv];
      cv[jv] = cn[jv];
    }
  }
  pdl_trigger();
}

template <int MODE>
cudaError_t launch_plane(const float* src, float* shell, float* coarse, const P2Plan& p, const P2Bufs& b,
                         const P2Tabs& t, const Exec& ex) {
  const P2Geom& g = p.g;
  const int cpl = (g.m2 - 1) / 32;
  const size_t smem = layout(g, MODE, cpl).total;
  const dim3 grid(unsigned(g.ntile * g.nchunk)), block(unsigned(g.nw * 32));
  cudaError_t e = cudaSuccess;
#define P2_LAUNCH(CPLV, MT)                                                                                \
  do {                                                                                                     \
    e = cudaFuncSetAttribute(k_p2_plane<MODE, CPLV, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
    if (e != cudaSuccess) return e;                                                                        \
    MGRX_LAUNCH(ex, MODE == 0 ? "p2_dec_plane" : "p2_rec_plane",                                          \
                pdl_launch(k_p2_plane<MODE, CPLV, MT>, grid, block, smem, ex.s, !ex.prof, src, shell, coarse, g, b, t)); \
  } while (0)
  switch (cpl) {
    case 1: P2_LAUNCH(1, 288); break;
    case 2: P2_LAUNCH(2, 288); break;
    case 4: P2_LAUNCH(4, 288); break;
    case 8: P2_LAUNCH(8, 288); break;
    case 16: P2_LAUNCH(16, kMaxThreads); break;
    default: return cudaErrorInvalidValue;
  }
#undef P2_LAUNCH
  return cudaGetLastError();
}

void launch_carry(const P2Plan& p, const P2Bufs& b, const P2Tabs& t, const Exec& ex) {
  const P2Geom& g = p.g;
  const int64_t n = int64_t(g.m1) * g.m2;
  MGRX_LAUNCH(ex, "p2_carry", pdl_launch(k_p2_carry, dim3(unsigned((n + 255) / 256)), dim3(256), 0, ex.s, !ex.prof, g, b, t));
}

size_t strip_smem(int) { return 0; }

cudaError_t launch_col(float* coarse, double sign, const P2Plan& p, const P2Bufs& b, const P2Tabs& t, const Exec& ex) {
  const P2Geom& g = p.g;
  const int rps = (g.m1 - 1) / 32;
  const size_t smem = strip_smem(rps);
  const dim3 grid(unsigned(g.nchunk * ((g.m2 + kSW - 1) / kSW)));
  cudaError_t e = cudaSuccess;
#define P2_STRIP(R)                                                                                      \
  do {                                                                                                   \
    MGRX_LAUNCH(ex, "p2_strip", pdl_launch(k_p2_strip<R>, grid, dim3(512), smem, ex.s, !ex.prof, coarse, g, b, t, sign)); \
  } while (0)
  switch (rps) {
    case 1: P2_STRIP(1); break;
    case 2: P2_STRIP(2); break;
    case 4: P2_STRIP(4); break;
    case 8: P2_STRIP(8); break;
    default: return cudaErrorInvalidValue;
  }
#undef P2_STRIP
  return cudaGetLastError();
}

// ThomasAux::build (transform.hpp:29-43), the same constant expressions.
void thomas(int m, double* w, double* id) {
  double dd = kDiagB;
  w[0] = 0.0;
  id[0] = 1.0 / dd;
  for (int i = 1; i < m; ++i) {
    const double wi = kOff / dd;
    w[i] = wi;
    dd = (i + 1 == m ? kDiagB : kDiagI) - wi * kOff;
    id[i] = 1.0 / dd;
  }
}

}  // namespace

P2Plan p2_plan(const LevelGeom& lg, int esize) {
  P2Plan p;
  // opt-in until it beats the fused3d passes (MGRX_P2=1)
  {
    const char* e = std::getenv("MGRX_P2");
    if (!e || std::atoi(e) == 0) return p;
  }
  if (lg.d != 3 || esize != 4) return p;
  P2Geom& g = p.g;
  g.n0 = int(lg.n[0]);
  g.n1 = int(lg.n[1]);
  g.n2 = int(lg.n[2]);
  g.m0 = int(lg.m[0]);
  g.m1 = int(lg.m[1]);
  g.m2 = int(lg.m[2]);
  if (!(g.n0 & 1) || !(g.n1 & 1) || !(g.n2 & 1)) return p;
  if (g.m0 < 3 || g.m1 < 33 || (g.m1 - 1) % 32 != 0 || g.m1 > 257) return p;
  if (g.m2 < 33 || (g.m2 - 1) % 32 != 0 || g.m2 > 257) return p;
  const int cpl = (g.m2 - 1) / 32, rps = (g.m1 - 1) / 32;
  if (cpl != 1 && cpl != 2 && cpl != 4 && cpl != 8) return p;
  if (rps != 1 && rps != 2 && rps != 4 && rps != 8) return p;
  g.T = kT;
  g.ntile = (g.m1 - 1) / kT;
  int C = 8;
  if (const char* e = std::getenv("MGRX_P2_CHUNK")) C = std::max(1, std::atoi(e));
  C = std::min(C, g.m0 - 1);
  g.C = C;
  g.nchunk = std::max(1, (g.m0 - 1) / C);
  g.nw = (g.m2 + 29) / 30;
  g.in_sr = g.n2;
  g.in_sp = int64_t(g.n1) * g.n2;
  g.co_sr = g.m2;
  g.co_sp = int64_t(g.m1) * g.m2;
  g.PG = (g.m2 + 7) & ~7;
  g.GP = int64_t(g.m1) * g.PG;
  const size_t smem = std::max(std::max(layout(g, 0, cpl).total, layout(g, 1, cpl).total), strip_smem(rps));
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (optin <= 0) optin = 227 * 1024;
  if (smem > size_t(optin)) return p;
  // scratch: G + S, EU, ED, X, XB
  const size_t plane = size_t(g.GP) * 8;
  p.scratch_bytes = size_t(g.m0) * plane + 5 * size_t(g.nchunk) * plane + 256;
  // tables
  std::vector<double>& tb = p.tabs;
  auto take = [&](size_t n) {
    const size_t o = tb.size();
    tb.resize(o + n, 0.0);
    return o;
  };
  p.o_w0 = take(g.m0);
  p.o_id0 = take(g.m0);
  p.o_gam0 = take(g.m0);
  p.o_A0 = take(g.m0);
  p.o_w1 = take(g.m1);
  p.o_id1 = take(g.m1);
  p.o_w2 = take(g.m2);
  p.o_id2 = take(g.m2);
  p.o_ch = take(5 * size_t(g.nchunk));
  p.o_af1 = take(g.m1);
  p.o_bb1 = take(g.m1);
  p.o_sf = take(5 * 32);
  p.o_sb = take(5 * 32);
  thomas(g.m0, &tb[p.o_w0], &tb[p.o_id0]);
  thomas(g.m1, &tb[p.o_w1], &tb[p.o_id1]);
  thomas(g.m2, &tb[p.o_w2], &tb[p.o_id2]);
  const double* w0 = &tb[p.o_w0];
  const double* id0 = &tb[p.o_id0];
  // axis-0 chunk constants: A_i = prod_{a0 < k <= i} (-w_k) (forward carry
  // weight), Gamma_i = (1/d_i) prod_{a0 <= k < i} (-(1/3)/d_k) (weight of g_i
  // in z_{a0}), Delta = prod_{a0 <= k < a1} (-(1/3)/d_k) (weight of z_{a1})
  for (int c = 0; c < g.nchunk; ++c) {
    const int a0 = c * C, a1 = (c == g.nchunk - 1) ? g.m0 : a0 + C;
    double Aprod = 1.0, Gprod = 1.0, SG = 0.0;
    for (int i = a0; i < a1; ++i) {
      if (i > a0) Aprod *= -w0[i];
      tb[p.o_A0 + i] = Aprod;
      const double gam = id0[i] * Gprod;
      tb[p.o_gam0 + i] = gam;
      SG += gam * Aprod;
      Gprod *= -kOff * id0[i];
    }
    double* ch = &tb[p.o_ch + 5 * size_t(c)];
    ch[0] = tb[p.o_A0 + a1 - 1];
    ch[1] = SG;
    ch[2] = tb[p.o_gam0 + a1 - 1];
    ch[3] = Gprod;
    ch[4] = (c + 1 < g.nchunk) ? w0[a1] : 0.0;
  }
  // axis-1 segments of the strip pass: 32 segments of rps rows (the last
  // also row m1 - 1); af1_r = prod_{lo <= k <= r} (-w_k) (weight of the
  // carry y_{lo-1} in y_r), bb1_r = prod_{r <= k < hi} (-(1/3)/d_k) (weight
  // of z_hi in z_r); scan factors of the segments' affine maps per step
  {
    const double* w1 = &tb[p.o_w1];
    const double* id1 = &tb[p.o_id1];
    double bf[32], bbk[32];
    for (int sg = 0; sg < 32; ++sg) {
      const int lo = rps * sg, hi = sg == 31 ? g.m1 : lo + rps;
      double pr = 1.0;
      for (int r = lo; r < hi; ++r) {
        pr *= -w1[r];
        tb[p.o_af1 + r] = pr;
      }
      bf[sg] = pr;
      pr = 1.0;
      for (int r = hi - 1; r >= lo; --r) {
        pr *= -kOff * id1[r];
        tb[p.o_bb1 + r] = pr;
      }
      bbk[sg] = pr;
    }
    for (int st = 0; st < 5; ++st) {
      const int off = 1 << st;
      double nf[32], nb[32];
      for (int L = 0; L < 32; ++L) {
        tb[p.o_sf + 32 * st + L] = bf[L];
        tb[p.o_sb + 32 * st + L] = bbk[L];
        nf[L] = L >= off ? bf[L] * bf[L - off] : bf[L];
        nb[L] = L + off < 32 ? bbk[L] * bbk[L + off] : bbk[L];
      }
      for (int L = 0; L < 32; ++L) {
        bf[L] = nf[L];
        bbk[L] = nb[L];
      }
    }
  }
  p.enabled = true;
  return p;
}

void p2_bind(const P2Plan& p, void* scratch, const double* d_tabs, P2Bufs* b, P2Tabs* t) {
  const P2Geom& g = p.g;
  char* s = static_cast<char*>(scratch);
  const size_t plane = size_t(g.GP) * 8;
  b->G = reinterpret_cast<double*>(s);
  s += size_t(g.m0) * plane;
  b->S = reinterpret_cast<double*>(s);
  s += size_t(g.nchunk) * plane;
  b->EU = reinterpret_cast<double*>(s);
  s += size_t(g.nchunk) * plane;
  b->ED = reinterpret_cast<double*>(s);
  s += size_t(g.nchunk) * plane;
  b->X = reinterpret_cast<double*>(s);
  s += size_t(g.nchunk) * plane;
  b->XB = reinterpret_cast<double*>(s);
  s += size_t(g.nchunk) * plane;
  const double* d = d_tabs + p.tab_off;
  t->w0 = d + p.o_w0;
  t->id0 = d + p.o_id0;
  t->gam0 = d + p.o_gam0;
  t->A0 = d + p.o_A0;
  t->w1 = d + p.o_w1;
  t->id1 = d + p.o_id1;
  t->w2 = d + p.o_w2;
  t->id2 = d + p.o_id2;
  t->ch = d + p.o_ch;
  t->af1 = d + p.o_af1;
  t->bb1 = d + p.o_bb1;
  t->sf = d + p.o_sf;
  t->sb = d + p.o_sb;
}

cudaError_t p2_init(const P2Plan&, void*, cudaStream_t) { return cudaSuccess; }

cudaError_t p2_decompose_level(const float* blk, float* shell, float* coarse, const P2Plan& p, const P2Bufs& b,
                               const P2Tabs& t, const Exec& ex) {
  cudaError_t e = launch_plane<0>(blk, shell, coarse, p, b, t, ex);
  if (e != cudaSuccess) return e;
  launch_carry(p, b, t, ex);
  e = launch_col(coarse, 1.0, p, b, t, ex);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t p2_recompose_correction(const float* shell, const P2Plan& p, const P2Bufs& b, const P2Tabs& t,
                                    const Exec& ex) {
  cudaError_t e = launch_plane<1>(shell, nullptr, nullptr, p, b, t, ex);
  if (e != cudaSuccess) return e;
  launch_carry(p, b, t, ex);
  return cudaGetLastError();
}

cudaError_t p2_recompose_apply(float* coarse, const P2Plan& p, const P2Bufs& b, const P2Tabs& t, const Exec& ex) {
  const cudaError_t e = launch_col(coarse, -1.0, p, b, t, ex);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace mgrx_b200
