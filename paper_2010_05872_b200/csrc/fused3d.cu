// Fused 3-D level pass for sm_100a.
//
// Replaces the reference's per-level sequence (reorder_level, reorder.hpp:131;
// compute_coefficients, transform.hpp:310; compute_correction, :331;
// apply_correction, :435; pack_level_centric, reorder.hpp:162 — and the
// inverse chain of recompose, transform.hpp:517) on large 3-D levels with
// three or four kernels whose HBM traffic is close to one read and one write
// of the level block:
//
//   decompose  f3_dec_plane  streams fine planes (TMA bulk copies into a
//                            3- or 4-slot shared-memory ring), computes every
//                            coefficient (same corner order as
//                            update_coefficients), writes the shell straight
//                            into its level-centric position and the nodal
//                            values into the compact coarse block, and
//                            accumulates the load vector L0 L1 L2 c of the
//                            fp64 component in registers; a finished coarse
//                            plane's rows go to the fp64 volume G (optionally
//                            also check_finite of every value it reads).
//              f3_row        solve along axis 2 on G, in place (a warp per row).
//              f3_col (axis 1)  solve along axis 1 on G, in place.
//              f3_col (axis 0)  solve along axis 0 + coarse += z.
//                            (lines of >= 40 unknowns in Toeplitz form —
//                            constant Thomas factors + end corrections, see
//                            "Toeplitz solves" — k_f3_row_ring, k_f3_col_toep;
//                            shorter lines with the ThomasAux tables)
//   recompose  f3_rec_plane  same load-vector accumulation, reading the
//                            component from the shell;
//              f3_row, f3_col x2  as above, coarse -= z;
//              f3_rec_interp fine block = coarse nodes + shell + prediction.
//
// Measured and removed (slower at 513^3; commit 48aabc0 has
// them): an in-plane cluster solve of axes 2 + 1 through DSMEM and a
// one-launch dataflow solve of all three axes.
//
// The tensor-product correction z = S2 S1 S0 c (S_a = Thomas_a o Load_a,
// transform.hpp:392-428) is evaluated as (T0 T1 T2)(L0 L1 L2) c: the
// operators act on different axes and commute exactly, so only rounding
// differs from the reference (pinned by the parity tests at 1e-12 / 1e-5 of
// the range).  The Thomas factors are the reference's ThomasAux; the
// recurrences are split into per-lane / per-thread segments joined by an
// affine scan (exact algebra, rounding-level differences).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "fused3d.h"

namespace mgrx_b200 {

namespace {

constexpr int kPlaneMaxThreads = 288;  // plane passes: up to 9 strips of 30 coarse columns, 2 CTAs per SM
constexpr int kWideThreads = 576;      // wide rows (n2 <= 1079): up to 18 strips, 1 CTA per SM
// register budget of the wide variants: launch bounds of 640 threads keep
// ptxas at <= 96 registers (18 warps = 5 on some SM sub-partitions)
constexpr int kWideBound = 640;
constexpr int kColMaxM = 640;       // column passes: register-resident columns up to this length
// column-pass block: 16 columns x S segments of up to LS registers, two
// segments per warp row; LS = 16 for m <= 320, 32 for m <= 640
constexpr int kColThreads = 16 * 20;
constexpr int kColThreads12 = 32 * 11;  // 12-value segments, up to 11 warp rows (m <= 264)

// ------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// try_wait suspends the waiting warp (up to this many ns) instead of
// returning at once, so a waiting warp does not spin on issue slots.
constexpr uint32_t kMbarSuspendNs = 100000;

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(kMbarSuspendNs)
      : "memory");
  return ok != 0;
}

#ifndef MGRX_WAIT_MODE
#define MGRX_WAIT_MODE 0
#endif
#ifndef MGRX_MBAR_SPIN_LIMIT
#define MGRX_MBAR_SPIN_LIMIT 0  // > 0: trap with a message after that many failed polls (debug)
#endif

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Wait for the phase of `bar` with the given parity.  With
// MGRX_MBAR_SPIN_LIMIT (ns) set at build time a stuck wait traps instead of
// hanging the device (debug builds).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if MGRX_MBAR_SPIN_LIMIT > 0
  uint64_t t0 = 0;
  while (!mbar_try(bar, parity)) {
    if (t0 == 0) t0 = global_ns();
    if (global_ns() - t0 > uint64_t(MGRX_MBAR_SPIN_LIMIT)) asm volatile("trap;");
  }
#elif MGRX_WAIT_MODE == 1
  // plain try_wait (no suspend-time hint)
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) break;
  }
#elif MGRX_WAIT_MODE == 2
  while (!mbar_try(bar, parity)) __nanosleep(200);
#else
  while (!mbar_try(bar, parity)) {
  }
#endif
}

// 1-D bulk copy global -> shared (TMA engine), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}


// L2 residency hints for the fp64 volume G (136 MB at 513^3, next to a
// 126 MB L2): its producer stores it with evict_last so the row / column
// passes that follow find it in L2, while the streamed field reads are
// marked evict_first (A/B on the B200: decompose -10 us, recompose -7 us,
// mostly the axis-0 pass).
__device__ __forceinline__ uint64_t pol_keep() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_stream() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_pol(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_pol(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
// bulk copy global -> shared with an L2 policy
__device__ __forceinline__ void bulk_g2s_pol(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Shared-memory load the compiler may not hoist (keeps table reads out of
// the register budget of the register-resident column segments).
__device__ __forceinline__ double ld_volatile(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
  return v;
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Weight of fine index j = 2i + k in the load-vector stencil of coarse i
// along an axis of n fine / m coarse points (load_entry, transform.hpp:84-96).
__device__ __forceinline__ double load_w(int k, int64_t i, int64_t m) {
  if (k == 0) return (i == 0 || i + 1 == m) ? kW5_12 : kW5_6;
  return (k == 1 || k == -1) ? 0.5 : kW12;
}

// Bytes of a [start, start+len) element range rounded out to 16-byte bulk
// granularity; returns the element offset of `start` inside the copy.
template <typename T>
__device__ __forceinline__ void bulk_span(const T* base, int64_t start, int64_t len, const char** src,
                                          uint32_t* bytes, int* lead) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(base + start);
  const uintptr_t a0 = a & ~uintptr_t(15);
  const uintptr_t a1 = (a + uintptr_t(len) * sizeof(T) + 15) & ~uintptr_t(15);
  *src = reinterpret_cast<const char*>(a0);
  *bytes = uint32_t(a1 - a0);
  *lead = int((a - a0) / sizeof(T));
}

// Affine map y -> a + b y: the carry of the Thomas recurrences over a
// segment, combined across lanes by the segmented solves below.
struct Aff {
  double a, b;
};

__device__ __forceinline__ Aff aff_then(Aff first, Aff second) {  // apply first, then second
  return Aff{second.a + second.b * first.a, second.b * first.b};
}

// Shell offset of reordered row (r0, r1) of a 3-D level block
// (pack_level_centric, reorder.hpp:180-215).
__device__ __forceinline__ int64_t shell_row_start(const F3Geom& g, int64_t r0, int64_t r1) {
  const int64_t before = (r0 < g.m0) ? r0 * g.m1 + min(r1, g.m1) : g.m0 * g.m1;
  return (r0 * g.n1 + r1) * g.n2 - before * g.m2;
}

__device__ __forceinline__ int64_t reord(int64_t j, int64_t m) { return (j & 1) ? m + (j >> 1) : (j >> 1); }

// shell_row_start(reord(p), r1) is linear in k = p / 2 for each parity of p:
// b[p & 1] + k * s[p & 1] (per-CTA tables in shared memory).
struct ShellLin {
  int64_t b[2], s[2];
};

__device__ __forceinline__ ShellLin shell_lin(const F3Geom& g, int64_t r1) {
  ShellLin l;
  l.b[0] = shell_row_start(g, 0, r1);
  l.s[0] = g.n1 * g.n2 - g.m1 * g.m2;  // r0 = k < m0: one more nodal row of m1 entries per plane
  l.b[1] = shell_row_start(g, g.m0, r1) + g.odd_shift;
  l.s[1] = g.n1 * g.n2;
  return l;
}

__device__ __forceinline__ int64_t lin_at(const ShellLin* l, int par, int64_t k) {
  const volatile int64_t* b = l->b;
  const volatile int64_t* s = l->s;
  return b[par] + k * s[par];
}

struct UnitRange {
  int64_t a0, a1, b0, b1;  // coarse planes [a0,a1), coarse rows [b0,b1)
  int64_t plo, phi;        // fine planes touched, inclusive
  int64_t rlo, rhi;        // fine rows touched, inclusive
};

__device__ __forceinline__ UnitRange unit_range(const F3Geom& g, int u) {
  UnitRange r;
  const int chunk = u / g.ntile1, tile = u - chunk * g.ntile1;
  r.a0 = g.a_base + int64_t(chunk) * g.chunk;
  r.a1 = min(g.a_end < 0 ? g.m0 : g.a_end, r.a0 + g.chunk);
  r.b0 = int64_t(tile) * g.tile_rows;
  r.b1 = min(g.m1, r.b0 + g.tile_rows);
  r.plo = max(int64_t(0), 2 * r.a0 - 2);
  r.phi = min(g.n0 - 1, 2 * r.a1);
  r.rlo = max(int64_t(0), 2 * r.b0 - 2);
  r.rhi = min(g.n1 - 1, 2 * r.b1);
  return r;
}

// --------------------------------------------------------- plane kernels
// Thread layout of the plane and interpolation passes: warp w owns coarse
// columns c = 30 w .. 30 w + 29 on lanes 1..30; lanes 0 and 31 are halo
// lanes that recompute the neighbouring columns so every cross-column
// value (the odd node's right corners, the axis-2 restriction stencil) moves
// through warp shuffles.  A thread walks all rows of its tile for its column
// keeping the fp64 nodal values and the axis-1 restriction in registers.
struct StripLane {
  int lane, c;
  bool valid, owned;
};

__device__ __forceinline__ StripLane strip_lane(int m2) {
  StripLane s;
  s.lane = threadIdx.x & 31;
  s.c = 30 * int(threadIdx.x >> 5) - 1 + s.lane;
  s.valid = s.c >= 0 && s.c < m2;
  s.owned = s.valid && s.lane >= 1 && s.lane <= 30;
  return s;
}

// Shared memory of the plane passes.  Decompose: a 4-slot ring of tile
// planes (2 TI1 + 3 fine rows; an odd plane reads its two even neighbours in
// place).  Recompose: a 3-slot ring of shell runs (even + odd rows).
template <typename T, int TI1, int NSD = 4, int NSR = 4>
struct PlaneSmem {
  static constexpr int kRows = 2 * TI1 + 3;
  static constexpr int kDecRows = 2 * TI1 + 3;
  static constexpr int kDecSlots = NSD, kRecSlots = NSR;
  static __host__ __device__ size_t raw_bytes(int64_t n2) {
    return (size_t(kRows) * size_t(n2) * sizeof(T) + 256 + 127) / 128 * 128;
  }
  static __host__ __device__ size_t dec_raw_bytes(int64_t n2) {
    return (size_t(kDecRows) * size_t(n2) * sizeof(T) + 32 + 127) / 128 * 128;
  }
  static __host__ __device__ size_t ring_bytes(int64_t n2) {
    const size_t d = kDecSlots * dec_raw_bytes(n2), r = kRecSlots * raw_bytes(n2);
    return d > r ? d : r;  // the 3-CTA variants size one direction only (the other's slots = 0)
  }
  static __host__ __device__ size_t bytes(int64_t n2, int64_t m2) {
    size_t b = ring_bytes(n2);      // TMA ring of fine plane tiles / shell runs
    b += 256;                       // pipeline state (PlanePipe)
    b += size_t(TI1 + 2) * size_t((m2 + 29) / 30 * 32) * sizeof(T);  // per-thread nodal values of the last even plane
    return b;
  }
};

// Axis-2 load-vector restriction at column c from the pair values of this
// lane and its neighbours: H(c) = w(c) e(c) + o(c)/2 + [e(c-1)/12 + o(c-1)/2]
// + e(c+1)/12 (load_entry, transform.hpp:84-96; missing nodes carry 0).
// The weights are per-lane constants (StripW): a lane outside the grid
// (xe = 0) or without an odd node (xo = 0) contributes nothing, and the
// right neighbour's even node only exists for c + 1 < m2 (er = 0), so the
// lanes' values need no zeroing selects (they only have to be finite).
struct StripW {
  double wc, xe, xo, er;
};
__device__ __forceinline__ StripW strip_w(int c, int m2, bool valid, bool has_odd) {
  StripW w;
  w.wc = (c == 0 || c + 1 == m2) ? kW5_12 : kW5_6;
  w.xe = valid ? kW12 : 0.0;
  w.xo = has_odd ? 0.5 : 0.0;
  w.er = (c + 1 < m2) ? kW12 : 0.0;
  return w;
}
__device__ __forceinline__ double strip_restrict(double cE, double cO, const StripW& w) {
  const double x = w.xe * cE + w.xo * cO;  // this column's share of H(c+1)
  const double xl = __shfl_up_sync(0xffffffffu, x, 1);
  const double er = __shfl_down_sync(0xffffffffu, cE, 1);
  return w.wc * cE + w.xo * cO + xl + w.er * er;
}

// The same with the weights of column c (the recompose plane pass zeroes its
// lanes' values instead: fewer live registers).
__device__ __forceinline__ double strip_restrict(double cE, double cO, int c, int m2) {
  const double x = kW12 * cE + 0.5 * cO;  // this column's share of H(c+1)
  const double xl = __shfl_up_sync(0xffffffffu, x, 1);
  const double er = __shfl_down_sync(0xffffffffu, cE, 1);
  const double wc = (c == 0 || c + 1 == m2) ? kW5_12 : kW5_6;
  return wc * cE + 0.5 * cO + xl + kW12 * er;
}

// Predicated global store (no branch; the address is not dereferenced
// when p is false).  No memory clobber: nothing in these kernels reads
// what they store, so other accesses may move across it.
__device__ __forceinline__ void st_if(float* a, float v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f32 [%0], %1;\n\t}" ::"l"(a), "f"(v),
               "r"(int(p)));
}
__device__ __forceinline__ void st_if(double* a, double v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f64 [%0], %1;\n\t}" ::"l"(a), "d"(v),
               "r"(int(p)));
}

// Shuffle source of the right neighbour's corner sum: a degenerate right
// end (2c + 2 >= n2) uses its own (transform.hpp:231-266).
__device__ __forceinline__ int right_src(bool right_degen) {
  const int lane = threadIdx.x & 31;
  return right_degen ? lane : min(lane + 1, 31);
}

// Thomas solve of one row x[0..m) in shared memory by one warp: lane
// segments get their affine maps from a zero carry, a shuffle scan gives
// each segment its true carry, and the segment reruns the exact recurrence
// (ThomasAux factors, transform.hpp:25-44; batched_solve :116-130).
__device__ __forceinline__ void warp_row_thomas(double* x, int m, const double* __restrict__ w,
                                                const double* __restrict__ inv_d) {
  const int lane = threadIdx.x & 31;
  const int seg = ((m + 31) >> 5) | 1;  // odd: lanes' segments start in distinct shared-memory banks
  const int s0 = min(m, lane * seg), s1 = min(m, s0 + seg);
  Aff f{0.0, 1.0};
  for (int i = s0; i < s1; ++i) {
    const double wi = w[i];
    f.a = x[i] - wi * f.a;
    f.b = -wi * f.b;
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Aff o{__shfl_up_sync(0xffffffffu, f.a, off), __shfl_up_sync(0xffffffffu, f.b, off)};
    if (lane >= off) f = aff_then(o, f);
  }
  double y = __shfl_up_sync(0xffffffffu, f.a, 1);
  if (lane == 0) y = 0.0;
  for (int i = s0; i < s1; ++i) {
    y = x[i] - w[i] * y;
    x[i] = y;
  }
  Aff g{0.0, 1.0};
  for (int i = s1 - 1; i >= s0; --i) {
    const double id = inv_d[i];
    g.a = (x[i] - kOff * g.a) * id;
    g.b = -kOff * id * g.b;
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Aff o{__shfl_down_sync(0xffffffffu, g.a, off), __shfl_down_sync(0xffffffffu, g.b, off)};
    if (lane + off < 32) g = aff_then(o, g);
  }
  double z = __shfl_down_sync(0xffffffffu, g.a, 1);
  if (lane == 31) z = 0.0;
  for (int i = s1 - 1; i >= s0; --i) {
    z = (x[i] - kOff * z) * inv_d[i];
    x[i] = z;
  }
  __syncwarp();
}

// The same solve with the lane's segment (<= SEG values) held in registers:
// one shared-memory read and one write per value instead of four of each.
template <int SEG>
__device__ __forceinline__ void warp_row_thomas_reg(double* x, int m, const double* __restrict__ w,
                                                    const double* __restrict__ inv_d) {
  const int lane = threadIdx.x & 31;
  const int seg = ((m + 31) >> 5) | 1;  // odd: lanes' segments start in distinct shared-memory banks
  const int s0 = min(m, lane * seg), len = min(m, s0 + seg) - s0;
  double v[SEG];
#pragma unroll
  for (int k = 0; k < SEG; ++k) v[k] = k < len ? x[s0 + k] : 0.0;
  Aff f{0.0, 1.0};
#pragma unroll
  for (int k = 0; k < SEG; ++k)
    if (k < len) {
      const double wi = w[s0 + k];
      f.a = v[k] - wi * f.a;
      f.b = -wi * f.b;
    }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Aff o{__shfl_up_sync(0xffffffffu, f.a, off), __shfl_up_sync(0xffffffffu, f.b, off)};
    if (lane >= off) f = aff_then(o, f);
  }
  double y = __shfl_up_sync(0xffffffffu, f.a, 1);
  if (lane == 0) y = 0.0;
#pragma unroll
  for (int k = 0; k < SEG; ++k)
    if (k < len) {
      y = v[k] - w[s0 + k] * y;
      v[k] = y;
    }
  Aff g{0.0, 1.0};
#pragma unroll
  for (int k = SEG - 1; k >= 0; --k)
    if (k < len) {
      const double id = inv_d[s0 + k];
      g.a = (v[k] - kOff * g.a) * id;
      g.b = -kOff * id * g.b;
    }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Aff o{__shfl_down_sync(0xffffffffu, g.a, off), __shfl_down_sync(0xffffffffu, g.b, off)};
    if (lane + off < 32) g = aff_then(o, g);
  }
  double z = __shfl_down_sync(0xffffffffu, g.a, 1);
  if (lane == 31) z = 0.0;
#pragma unroll
  for (int k = SEG - 1; k >= 0; --k)
    if (k < len) {
      z = (v[k] - kOff * z) * inv_d[s0 + k];
      x[s0 + k] = z;
    }
  __syncwarp();
}

// ------------------------------------------------------- Toeplitz solves
// The correction matrix tridiag(1/3; 2/3, 4/3 ... 4/3, 2/3; 1/3) is Toeplitz
// except for its two corner entries, and the ThomasAux factors converge to
// the constants w = 2 - sqrt(3), 1/d = 1/(4/3 - w/3) within ~16 rows.  Solve
// with the CONSTANT factors (the matrix T' = L' U' equals T except
// T'(0,0) = d and T'(m-1,m-1) = 4/3) and correct the two ends
// (Sherman-Morrison): x = z + z_0 Gt + z_{m-1} Ht, z = T'^-1 f, where Gt / Ht
// (host tables, api.cu:toeplitz_end_tables) decay by w per row from their end
// — 32 entries each reach 2e-18 — and the ends decouple for m >= 40.  Exact
// algebra, rounding-level differences from batched_solve
// (transform.hpp:116-130), like the segmented solves; no factor tables are
// read in the recurrences and every segment's affine map has the same
// multiplier, so the scans move one value instead of two.
template <int N>
struct PowTab {
  double v[N + 1];
  constexpr PowTab(double x) : v() {
    v[0] = 1.0;
    for (int i = 1; i <= N; ++i) v[i] = v[i - 1] * x;
  }
};
constexpr double kTc = kOff * kTid;  // back-substitution multiplier

// Row x[0..m) in shared memory by one warp: lane = SEG consecutive values
// (zero past the end), carries by a shuffle scan of one value per lane.
template <int SEG>
__device__ __forceinline__ void warp_row_toep(double* x, int m, const double* __restrict__ gt,
                                              const double* __restrict__ ht) {
  constexpr PowTab<SEG> PF(-kTw), PB(-kTc);
  const int lane = threadIdx.x & 31;
  const int s0 = lane * SEG;
  double v[SEG];
#pragma unroll
  for (int k = 0; k < SEG; ++k) v[k] = (s0 + k < m) ? x[s0 + k] : 0.0;
  // forward y_i = f_i - w y_{i-1} from a zero carry
  double a = 0.0;
#pragma unroll
  for (int k = 0; k < SEG; ++k) {
    a = v[k] - kTw * a;
    v[k] = a;
  }
  {
    double b = PF.v[SEG];  // (-w)^SEG, squared at every doubling step
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double o = __shfl_up_sync(0xffffffffu, a, off);
      if (lane >= off) a = a + b * o;
      b = b * b;
    }
  }
  double c = __shfl_up_sync(0xffffffffu, a, 1);
  if (lane == 0) c = 0.0;
#pragma unroll
  for (int k = 0; k < SEG; ++k) v[k] = (s0 + k < m) ? v[k] + PF.v[k + 1] * c : 0.0;  // zero past the end again
  // back substitution z_i = (y_i - z_{i+1} / 3) / d from a zero carry
  double g = 0.0;
#pragma unroll
  for (int k = SEG - 1; k >= 0; --k) {
    g = (v[k] - kOff * g) * kTid;
    v[k] = g;
  }
  {
    double b = PB.v[SEG];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double o = __shfl_down_sync(0xffffffffu, g, off);
      if (lane + off < 32) g = g + b * o;
      b = b * b;
    }
  }
  double z = __shfl_down_sync(0xffffffffu, g, 1);
  if (lane == 31) z = 0.0;
#pragma unroll
  for (int k = 0; k < SEG; ++k) v[k] = v[k] + PB.v[SEG - k] * z;
  // end corrections
  const int last = m - 1;
  double zl = 0.0;
#pragma unroll
  for (int k = 0; k < SEG; ++k)
    if (s0 + k == last) zl = v[k];
  const double z0 = __shfl_sync(0xffffffffu, v[0], 0);
  const double zm = __shfl_sync(0xffffffffu, zl, last / SEG);
  if (s0 < kToepEnds) {
#pragma unroll
    for (int k = 0; k < SEG; ++k)
      if (s0 + k < kToepEnds) v[k] = v[k] + z0 * gt[s0 + k];
  }
  if (s0 + SEG > m - kToepEnds) {
#pragma unroll
    for (int k = 0; k < SEG; ++k) {
      const int rev = last - (s0 + k);
      if (rev >= 0 && rev < kToepEnds) v[k] = v[k] + zm * ht[rev];
    }
  }
#pragma unroll
  for (int k = 0; k < SEG; ++k)
    if (s0 + k < m) x[s0 + k] = v[k];
  __syncwarp();
}

// The same row solve on a RIGHT-ALIGNED buffer of 32 SEG values: element i of
// the row sits at position i + P0, P0 = 32 SEG - m, and the positions before
// it hold zeros.  The last element is then the last value of lane 31, so the
// back substitution starts from a zero carry without a test, and leading zeros
// are harmless in both recurrences (forward: they stay zero; backward: what
// they become is never stored): no per-value bounds tests or selects.  The
// end corrections read z_0 / z_{m-1} back from the buffer and lane l fixes
// elements l and m - 1 - l (gl = Gt[l], hl = Ht[l]).  Needs m >= 32.
template <int SEG>
struct ScanPow {  // B^(2^j), j = 0..4, for B = x^SEG
  double v[5];
  constexpr ScanPow(double x) : v() {
    double b = 1.0;
    for (int i = 0; i < SEG; ++i) b *= x;
    for (int j = 0; j < 5; ++j) {
      v[j] = b;
      if (j < 4) b *= b;
    }
  }
};

template <int SEG>
__device__ __forceinline__ void warp_row_toep_ra(double* x, int m, double gl, double hl) {
  constexpr PowTab<SEG> PF(-kTw), PB(-kTc);
  constexpr ScanPow<SEG> SF(-kTw), SB(-kTc);
  const int lane = threadIdx.x & 31;
  const int s0 = lane * SEG;
  const int P0 = 32 * SEG - m;
  double v[SEG];
#pragma unroll
  for (int k = 0; k < SEG; ++k) v[k] = x[s0 + k];
  double a = 0.0;
#pragma unroll
  for (int k = 0; k < SEG; ++k) {
    a = v[k] - kTw * a;
    v[k] = a;
  }
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const double o = __shfl_up_sync(0xffffffffu, a, 1 << j);
    if (lane >= (1 << j)) a = a + SF.v[j] * o;
  }
  double c = __shfl_up_sync(0xffffffffu, a, 1);
  if (lane == 0) c = 0.0;
#pragma unroll
  for (int k = 0; k < SEG; ++k) v[k] = v[k] + PF.v[k + 1] * c;
  double g = 0.0;
#pragma unroll
  for (int k = SEG - 1; k >= 0; --k) {
    g = (v[k] - kOff * g) * kTid;
    v[k] = g;
  }
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const double o = __shfl_down_sync(0xffffffffu, g, 1 << j);
    if (lane + (1 << j) < 32) g = g + SB.v[j] * o;
  }
  double z = __shfl_down_sync(0xffffffffu, g, 1);
  if (lane == 31) z = 0.0;
#pragma unroll
  for (int k = 0; k < SEG; ++k) {
    v[k] = v[k] + PB.v[SEG - k] * z;
    if (s0 + k >= P0) x[s0 + k] = v[k];
  }
  __syncwarp();
  const double z0 = x[P0], zm = x[32 * SEG - 1];
  __syncwarp();
  x[P0 + lane] = x[P0 + lane] + z0 * gl;
  __syncwarp();
  x[32 * SEG - 1 - lane] = x[32 * SEG - 1 - lane] + zm * hl;
  __syncwarp();
}

// L0 (axis-0 load-vector restriction) on registers: the coarse planes
// k-1, k, k+1 around fine plane p (k = p/2) accumulate the plane's
// restricted rows Q in stencil order (load_entry, transform.hpp:84-96);
// a finished coarse plane is staged in shared memory, solved along axis 2
// (one warp per row) and stored to G.
template <int TI1>
struct L0Planes {
  double prev[TI1], cur[TI1], next[TI1];
};

// Pipeline state of a plane-pass CTA (shared memory):
//   full[s]     TMA completion of ring slot s (count 1 + transaction bytes)
//   cnt[s]      warps done reading slot s; the last one refills it
struct PlanePipe {
  uint64_t full[4];
  int cnt[4];
  ShellLin lin[4];  // recompose: shell run bounds of the unit's rows
  int lead[4][4];   // interpolation: 16-byte leads of the runs in slot s (written by the issuing thread)
};
static_assert(sizeof(PlanePipe) <= 256, "PlaneSmem reserves 256 bytes for the pipeline state");

// A finished coarse plane (the j-th of this CTA): every owned lane stores
// its rows of the axis-0/1/2 load vector to G.  The axis-2 solve of these
// rows runs in the row pass (k_f3_row) after the plane pass, so the plane
// pass needs no CTA-wide barrier.
template <int TI1>
__device__ __forceinline__ void l0_complete(const F3Geom& g, const UnitRange& ur, const StripLane& S,
                                            const double* v, int64_t i0, int& j, double* __restrict__ G) {
  const int TR = int(ur.b1 - ur.b0);
  if (S.owned) {
    double* gp = G + (i0 * g.m1 + ur.b0) * g.m2 + S.c;
    const uint64_t pol = pol_keep();
#pragma unroll
    for (int ir = 0; ir < TI1; ++ir)
      if (ir < TR) st_pol(gp + int64_t(ir) * g.m2, v[ir], pol);
  }
  ++j;
}

template <int TI1>
__device__ __forceinline__ void l0_plane(const F3Geom& g, const UnitRange& ur, const StripLane& S, int64_t p,
                                         const double* Q, L0Planes<TI1>& A, int& j, double* __restrict__ G) {
  const int64_t k = p >> 1;
  const bool last = p == g.n0 - 1;
  if (!(p & 1)) {
    const double wc = (k == 0 || k + 1 == g.m0) ? kW5_12 : kW5_6;
#pragma unroll
    for (int ir = 0; ir < TI1; ++ir) {
      A.prev[ir] += kW12 * Q[ir];
      A.cur[ir] += wc * Q[ir];
      A.next[ir] += kW12 * Q[ir];
    }
    if (k - 1 >= ur.a0 && k - 1 < ur.a1) l0_complete<TI1>(g, ur, S, A.prev, k - 1, j, G);
    if (last && k >= ur.a0 && k < ur.a1) l0_complete<TI1>(g, ur, S, A.cur, k, j, G);
  } else {
#pragma unroll
    for (int ir = 0; ir < TI1; ++ir) {
      A.cur[ir] += 0.5 * Q[ir];
      A.next[ir] += 0.5 * Q[ir];
    }
    if (last && k >= ur.a0 && k < ur.a1) l0_complete<TI1>(g, ur, S, A.cur, k, j, G);
#pragma unroll
    for (int ir = 0; ir < TI1; ++ir) {
      A.prev[ir] = A.cur[ir];
      A.cur[ir] = A.next[ir];
      A.next[ir] = 0.0;
    }
  }
}

// Pipeline helpers: ring slot of the d-th plane of a unit and the parity of
// its use (NS slots).
template <int NS>
__device__ __forceinline__ int pipe_slot(int d) { return d % NS; }
template <int NS>
__device__ __forceinline__ uint32_t pipe_parity(int d) { return uint32_t((d / NS) & 1); }

// Called by every warp when it has finished reading the d-th plane's slot;
// the last warp refills the slot with plane d + NS via `issue` (d <= dmax).
template <int NS, typename Issue>
__device__ __forceinline__ void pipe_release(PlanePipe* pp, int d, int dmax, Issue&& issue) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    const int s = pipe_slot<NS>(d);
    __threadfence_block();
    const int old = atomicAdd(&pp->cnt[s], 1);
    if (old == int(blockDim.x >> 5) - 1) {
      pp->cnt[s] = 0;
      if (d + NS <= dmax) issue(d + NS);
    }
  }
}

// Per-plane, per-thread context of the decompose row loop.
// Order-preserving image of an fp64 value in 64-bit unsigned integers
// (x < y  <=>  ordered_bits(x) < ordered_bits(y) for non-NaN values).
__device__ __forceinline__ unsigned long long ordered_bits(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <typename T>
struct DecRows {
  const T* rp;        // tile row 0 (= fine row rlo), at column 2c
  T* se;              // shell slot of even tile row e = 0 (fine row jbase), at column c
  T* so;              // shell slot of odd tile row e = 0 (fine row jbase + 1), at column c
  T* cpe;             // coarse row of even tile row e = 0, at column c
  int st_e;           // shell stride between consecutive even rows
  int n2l;            // shell stride between consecutive odd rows
  int n2, m2, n1, m1; // extents
  int jbase, rlo, rhi, b0, TR, jlo_own, jhi_own;
  int oofs;           // odd-node offset inside an even row's shell slot
  bool own;           // owned lane and owned plane
  bool valid, has_odd, right_degen, has_right;
  int c;
  int oi;      // offset of the odd node's raw value (0 without an odd node: a finite stand-in)
  int rsrc;    // shuffle source of the right neighbour's corner sum
  StripW sw;   // restriction weights of this lane
};

// Rows of one fine plane (decompose): for every fine row and this lane's
// column pair, the coefficients (corner sets of update_coefficients,
// transform.hpp:216-304; the odd node's sum is the own column's sum plus the
// right column's, shuffled in), the shell / coarse writes, the axis-2
// restriction (shuffles) and the axis-1 restriction into Q (registers).
// PODD: plane parity; FULL: interior tile (all rows present, no degenerate
// row, interior axis-1 weights) — every row test is then compile-time.
// CF: also fold every raw value into `nf` as nf + v * 0 (stays 0 unless a
// value is inf / NaN): check_finite (pipeline.hpp:113-118) on the read the
// pass makes anyway.
template <typename T, int TI1, bool PODD, bool FULL, bool CF = false>
__device__ __forceinline__ void dec_rows(const DecRows<T>& x, const T* nl, const T* nr, T* nb, int nbs, double* Q,
                                         T& nf, T& lo, T& hi) {
  constexpr int RMAX = 2 * TI1 + 3;
  const int n2 = x.n2;
  const T* rr = x.rp + (x.jbase - x.rlo) * n2;  // tile row of jr = 0 (may precede the tile when not FULL)
  // nodal values (own column, even tile rows) of the left / right even
  // plane, read from their ring slots: nl / nr point at tile row jr = 0
  auto ns = [&](const T* base, int e) -> double {
    const int j1 = x.jbase + 2 * e;
    if (!FULL && (j1 < x.rlo || j1 > x.rhi)) return 0.0;
    return double(base[2 * e * n2]);
  };
  // left nodal values: an even plane reads its own slot and keeps them in
  // this thread's private buffer nb (stride nbs) for the odd plane after it
  auto nsl = [&](int e) -> double {
    if (PODD) return double(nb[e * nbs]);
    const double v = ns(nl, e);
    nb[e * nbs] = T(v);
    return v;
  };
  double aLc = nsl(0), aRc = (PODD && x.has_right) ? ns(nr, 0) : aLc;
  double aLn = 0.0, aRn = 0.0;
#pragma unroll
  for (int jr = 0; jr < RMAX; ++jr, rr += n2) {
    const int j1 = x.jbase + jr;
    const bool o1 = jr & 1;
    const int ea = jr >> 1;
    if (!o1 && jr + 1 < RMAX) {
      aLn = nsl(ea + 1);
      aRn = (PODD && x.has_right) ? ns(nr, ea + 1) : aLn;
    }
    if (!FULL && (j1 < x.rlo || j1 > x.rhi)) {  // uniform
      if (o1) {
        aLc = aLn;
        aRc = aRn;
      }
      continue;
    }
    const bool rdeg = !FULL && o1 && (j1 + 1 >= x.n1);
    const T rE = rr[0], rO = rr[x.oi];
    if (CF) {  // finiteness + range of every value read (NaN is ignored by fmin / fmax)
      nf = rE * T(0) + (rO * T(0) + nf);
      lo = fmin(lo, fmin(rE, rO));
      hi = fmax(hi, fmax(rE, rO));
    }
    const double rawE = double(rE);
    const double rawO = double(rO);
    const double aL = aLc;
    const double bL = o1 ? (rdeg ? aL : aLn) : aL;
    double se;
    int ke;
    if (!PODD) {
      se = o1 ? aL + bL : aL;
      ke = o1 ? 1 : 0;
    } else {
      const double aR = aRc;
      const double bR = o1 ? (rdeg ? aR : aRn) : aR;
      se = aL + aR;
      if (o1) {
        se += bL;
        se += bR;
      }
      ke = o1 ? 2 : 1;
    }
    const double sn = __shfl_sync(0xffffffffu, se, x.rsrc);
    const double so = se + sn;
    const double sc_e = ke == 1 ? 0.5 : 0.25;
    const double sc_o = ke == 0 ? 0.5 : (ke == 1 ? 0.25 : 0.125);
    const T tE = to_t<T>(rawE - se * sc_e);
    const T tO = to_t<T>(rawO - so * sc_o);
    const double cE = ke == 0 ? 0.0 : double(tE);  // finite on every lane (clamped columns)
    const double cO = double(tO);
    const bool own_row = FULL ? (jr >= 2 && jr < 2 * TI1 + 2) : (j1 >= x.jlo_own && j1 < x.jhi_own);
    if (x.own && own_row) {
      if (o1) {
        T* sr = x.so + ea * x.n2l;
        sr[0] = tE;
        if (x.has_odd) sr[x.m2] = tO;
      } else {
        T* sr = x.se + ea * x.st_e;
        if (ke == 0)
          x.cpe[ea * x.m2] = rr[0];
        else
          sr[0] = tE;
        if (x.has_odd) sr[x.oofs] = tO;
      }
    }
    const double h = strip_restrict(cE, cO, x.sw);
#pragma unroll
    for (int k = -2; k <= 2; ++k) {
      if (((jr - 2 - k) & 1) != 0) continue;
      const int ir = (jr - 2 - k) / 2;
      if (ir < 0 || ir >= TI1) continue;
      if (FULL)
        Q[ir] += (k == 0 ? kW5_6 : ((k & 1) ? 0.5 : kW12)) * h;
      else if (ir < x.TR)
        Q[ir] += load_w(k, x.b0 + ir, x.m1) * h;
    }
    if (o1) {
      aLc = aLn;
      aRc = aRn;
    }
  }
}

// Decompose plane pass: one CTA per (axis-0 chunk, axis-1 tile) unit; the
// unit's fine planes stream through a 3-deep TMA ring.
// NB = 3: the 3-CTAs-per-SM variant with a 3-slot ring (F3Geom::dec3)
template <typename T, int TI1, int MAXT, int NB = 0, bool CF = false>
__global__ void __launch_bounds__(MAXT, NB ? NB : (MAXT == kPlaneMaxThreads ? 2 : 1))
    k_f3_dec_plane(const T* __restrict__ blk, T* __restrict__ shell, T* __restrict__ coarse, double* __restrict__ G,
                   const F3Geom g) {
  using SM = PlaneSmem<T, TI1, NB == 3 ? 3 : 4, NB == 3 ? 0 : 4>;
  constexpr int RMAX = SM::kRows;
  constexpr int NS = SM::kDecSlots;
  extern __shared__ __align__(128) unsigned char smem[];
  const int m2 = int(g.m2), n2 = int(g.n2), n1 = int(g.n1), m1 = int(g.m1);
  const size_t rawb = SM::dec_raw_bytes(g.n2);
  unsigned char* raw = smem;
  PlanePipe* pp = reinterpret_cast<PlanePipe*>(smem + SM::ring_bytes(g.n2));
  T* nb = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(pp) + 256) + threadIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const StripLane S = strip_lane(m2);
  const int c = S.c;
  const UnitRange ur = unit_range(g, int(blockIdx.x));
  if (tid == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(&pp->full[b], 1);
      pp->cnt[b] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();

  const int R = int(ur.rhi - ur.rlo + 1);
  DecRows<T> x;
  x.n2 = n2;
  x.m2 = m2;
  x.n1 = n1;
  x.m1 = m1;
  x.rlo = int(ur.rlo);
  x.rhi = int(ur.rhi);
  x.jbase = int(2 * ur.b0) - 2;
  x.b0 = int(ur.b0);
  x.TR = int(ur.b1 - ur.b0);
  x.jlo_own = int(2 * ur.b0);
  x.jhi_own = int(min(2 * ur.b1, g.n1));
  x.valid = S.valid;
  x.has_odd = S.valid && 2 * c + 1 < n2;
  x.right_degen = 2 * c + 2 >= n2;
  x.c = c;
  x.oi = x.has_odd ? 1 : 0;
  x.rsrc = right_src(x.right_degen);
  x.sw = strip_w(c, m2, x.valid, x.has_odd);
  x.n2l = int(g.n2);
  const bool full = ur.b0 >= 1 && 2 * ur.b1 <= g.n1 - 1;
  const int cc = S.valid ? c : 0;  // clamp halo columns for addressing
  const int D = int(ur.phi - ur.plo);  // planes of the unit: plo + [0, D]
  auto tile_src = [&](int d) { return blk + ((ur.plo + d) * g.n1 + ur.rlo) * g.n2; };
  auto issue = [&](int d) {  // one thread
    const char* src;
    uint32_t bytes;
    int ld;
    const int sl = pipe_slot<NS>(d);
    bulk_span<T>(tile_src(d), 0, int64_t(R) * n2, &src, &bytes, &ld);
    fence_proxy_async();
    mbar_expect_tx(&pp->full[sl], bytes);
    bulk_g2s_pol(raw + size_t(sl) * rawb, src, bytes, &pp->full[sl], pol_stream());
  };
  // tile row jbase of plane d, column 2 cc (the row may precede the slot
  // when not FULL; never read then); the 16-byte lead of a plane's bulk copy
  // advances by a constant per plane
  const int row_off = (x.jbase - x.rlo) * n2 + 2 * cc;
  const int lead0 = int(reinterpret_cast<uintptr_t>(tile_src(0)) & 15);
  const int lead_inc = int((g.n1 * g.n2 * int64_t(sizeof(T))) & 15);
  auto row0 = [&](int d) {
    return reinterpret_cast<const T*>(raw + pipe_slot<NS>(d) * int(rawb) + ((lead0 + d * lead_inc) & 15)) + row_off;
  };
  if (tid == 0)
    for (int d = 0; d <= min(D, NS - 1); ++d) issue(d);
  L0Planes<TI1> A;
#pragma unroll
  for (int ir = 0; ir < TI1; ++ir) A.prev[ir] = A.cur[ir] = A.next[ir] = 0.0;
  int jdone = 0;  // coarse planes finished by this CTA
  T nf = T(0);    // CF: 0 unless a raw value was inf / NaN
  T lo = T(INFINITY), hi = T(-INFINITY);  // CF: range of the values read
  // Shell / coarse pointers of the unit's first even and odd plane, advanced
  // by a constant per plane pair (shell_row_start is linear in k = p / 2 for
  // each parity: +n1 n2 - m1 m2 for even planes, +n1 n2 for odd ones).
  const int e0 = x.jbase >> 1;  // even tile row 0 <-> coarse row e0
  const int64_t k0 = ur.plo >> 1;
  T* se_e = shell + (shell_row_start(g, k0, e0 + 1) - (g.n2 - g.m2)) + cc;
  T* so_e = shell + (shell_row_start(g, k0, g.m1 + e0 + 1) - g.n2) + cc;
  T* se_o = shell + (shell_row_start(g, g.m0 + k0, e0 + 1) - g.n2 + g.odd_shift) + cc;
  T* so_o = shell + (shell_row_start(g, g.m0 + k0, g.m1 + e0 + 1) - g.n2 + g.odd_shift) + cc;
  T* cpe = coarse + (k0 * g.m1 + e0) * g.m2 + cc;
  const int64_t step_e = g.n1 * g.n2 - g.m1 * g.m2, step_o = g.n1 * g.n2, step_c = g.m1 * g.m2;
  const int plo = int(ur.plo), n0 = int(g.n0), a0x2 = int(2 * ur.a0), a1x2 = int(2 * ur.a1);
  for (int d = 0; d <= D; d += 2) {
    {  // even plane p = plo + d
      const int p = plo + d;
      mbar_wait(&pp->full[pipe_slot<NS>(d)], pipe_parity<NS>(d));
      x.has_right = false;
      x.st_e = int(g.n2 - g.m2);
      x.oofs = 0;
      x.se = se_e;
      x.so = so_e;
      x.cpe = cpe;
      x.own = S.owned && p >= a0x2 && p < a1x2;
      const T* r_own = row0(d);
      x.rp = r_own - (x.jbase - x.rlo) * n2;
      double Q[TI1];
#pragma unroll
      for (int ir = 0; ir < TI1; ++ir) Q[ir] = 0.0;
      if (full) dec_rows<T, TI1, false, true, CF>(x, r_own, r_own, nb, nt, Q, nf, lo, hi);
      else dec_rows<T, TI1, false, false, CF>(x, r_own, r_own, nb, nt, Q, nf, lo, hi);
      pipe_release<NS>(pp, d, D, issue);  // this warp is done with plane d's slot
      l0_plane<TI1>(g, ur, S, p, Q, A, jdone, G);
      se_e += step_e;
      so_e += step_e;
      cpe += step_c;
    }
    if (d + 1 <= D) {  // odd plane p = plo + d + 1
      const int p = plo + d + 1;
      x.has_right = p + 1 <= n0 - 1;
      mbar_wait(&pp->full[pipe_slot<NS>(d + 1)], pipe_parity<NS>(d + 1));
      if (x.has_right) mbar_wait(&pp->full[pipe_slot<NS>(d + 2)], pipe_parity<NS>(d + 2));
      x.st_e = int(g.n2);
      x.oofs = m2;
      x.se = se_o;
      x.so = so_o;
      x.own = S.owned && p >= a0x2 && p < a1x2;
      const T* r_own = row0(d + 1);
      x.rp = r_own - (x.jbase - x.rlo) * n2;
      double Q[TI1];
#pragma unroll
      for (int ir = 0; ir < TI1; ++ir) Q[ir] = 0.0;
      const T* nr = x.has_right ? row0(d + 2) : r_own;
      if (full) dec_rows<T, TI1, true, true, CF>(x, r_own, nr, nb, nt, Q, nf, lo, hi);
      else dec_rows<T, TI1, true, false, CF>(x, r_own, nr, nb, nt, Q, nf, lo, hi);
      pipe_release<NS>(pp, d + 1, D, issue);
      l0_plane<TI1>(g, ur, S, p, Q, A, jdone, G);
      se_o += step_o;
      so_o += step_o;
    }
  }
  if (CF) {
    if (!(nf == T(0))) atomicOr(g.nonfinite, 1u);
    // range: warp minimum / maximum, one atomic per warp on the
    // order-preserving 64-bit image of the fp64 value
    double dl = double(lo), dh = double(hi);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dl = fmin(dl, __shfl_xor_sync(0xffffffffu, dl, o));
      dh = fmax(dh, __shfl_xor_sync(0xffffffffu, dh, o));
    }
    if ((threadIdx.x & 31) == 0) {
      unsigned long long* mm = reinterpret_cast<unsigned long long*>(g.nonfinite + 2);
      atomicMin(mm, ordered_bits(dl));
      atomicMax(mm + 1, ordered_bits(dh));
    }
  }
  pdl_trigger();
}

// Rows of one fine plane (recompose plane pass): component from the shell
// slot (coefficients; 0 on nodal points), axis-2 restriction through
// shuffles, axis-1 restriction into Q.  FULL as in dec_rows.
template <typename T, int TI1, bool PODD, bool FULL>
__device__ __forceinline__ void rec_rows(const T* ev, const T* od, int st_e, int n2, int m2, int jbase, int rlo,
                                         int rhi, int b0, int TR, int m1, int c, bool valid, bool has_odd, double* Q) {
  constexpr int RMAX = 2 * TI1 + 3;
#pragma unroll
  for (int jr = 0; jr < RMAX; ++jr) {
    const int j1 = jbase + jr;
    if (!FULL && (j1 < rlo || j1 > rhi)) continue;  // uniform
    const bool o1 = jr & 1;
    const int ea = jr >> 1;
    double cE, cO;
    if (o1) {
      const T* r = od + ea * n2;
      cE = valid ? double(r[0]) : 0.0;
      cO = has_odd ? double(r[m2]) : 0.0;
    } else {
      const T* r = ev + ea * st_e;
      cE = (PODD && valid) ? double(r[0]) : 0.0;
      cO = has_odd ? double(r[PODD ? m2 : 0]) : 0.0;
    }
    const double h = strip_restrict(cE, cO, c, m2);
#pragma unroll
    for (int k = -2; k <= 2; ++k) {
      if (((jr - 2 - k) & 1) != 0) continue;
      const int ir = (jr - 2 - k) / 2;
      if (ir < 0 || ir >= TI1) continue;
      if (FULL)
        Q[ir] += (k == 0 ? kW5_6 : ((k & 1) ? 0.5 : kW12)) * h;
      else if (ir < TR)
        Q[ir] += load_w(k, b0 + ir, m1) * h;
    }
  }
}

// Recompose plane pass: the same load-vector accumulation with the
// component read from the level's shell.  Per fine plane the tile's shell
// rows form two contiguous runs (even fine rows, odd fine rows), fetched
// with two bulk copies into one ring slot.
template <typename T, int TI1, int MAXT, int NB = 0>
__global__ void __launch_bounds__(MAXT, NB ? NB : (MAXT == kPlaneMaxThreads ? 2 : 1))
    k_f3_rec_plane(const T* __restrict__ shell, double* __restrict__ G, const F3Geom g) {
  using SM = PlaneSmem<T, TI1, NB == 3 ? 0 : 4, NB == 3 ? 3 : 4>;
  constexpr int RMAX = SM::kRows;
  extern __shared__ __align__(128) unsigned char smem[];
  const int m2 = int(g.m2), n2 = int(g.n2), m1 = int(g.m1);
  const size_t rawb = SM::raw_bytes(g.n2);
  unsigned char* raw = smem;
  constexpr int NS = SM::kRecSlots;
  PlanePipe* pp = reinterpret_cast<PlanePipe*>(smem + SM::ring_bytes(g.n2));

  const int tid = threadIdx.x, nt = blockDim.x;
  const StripLane S = strip_lane(m2);
  const int c = S.c;
  const int cc = S.valid ? c : 0;
  const bool has_odd = S.valid && 2 * c + 1 < n2;
  const UnitRange ur = unit_range(g, int(blockIdx.x));
  if (tid == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(&pp->full[b], 1);
      pp->cnt[b] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pp->lin[0] = shell_lin(g, ur.rlo >> 1);
    pp->lin[1] = shell_lin(g, (ur.rhi >> 1) + 1);
    pp->lin[2] = shell_lin(g, g.m1 + ((ur.rlo + 1) >> 1));
    pp->lin[3] = shell_lin(g, g.m1 + ((ur.rhi - 1) >> 1) + 1);
  }
  __syncthreads();
  pdl_wait();

  const int rlo = int(ur.rlo), rhi = int(ur.rhi);
  const int jbase = int(2 * ur.b0) - 2;
  const int TR = int(ur.b1 - ur.b0), b0 = int(ur.b0);
  const bool full = ur.b0 >= 1 && 2 * ur.b1 <= g.n1 - 1;
  // even fine rows: r1 in [rlo/2, rhi/2]; odd: r1 = m1 + [(rlo+1)/2, (rhi-1)/2]
  const int64_t e_lo = ur.rlo >> 1, e_hi = ur.rhi >> 1;
  const int64_t o_lo = (ur.rlo + 1) >> 1, o_hi = (ur.rhi - 1) >> 1;
  struct Runs {
    int64_t se, le, so, lo;
  };
  auto runs = [&](int64_t p) {
    const int par = int(p & 1);
    const int64_t k = p >> 1;
    Runs x;
    x.se = lin_at(&pp->lin[0], par, k);
    x.le = lin_at(&pp->lin[1], par, k) - x.se;
    x.so = o_hi >= o_lo ? lin_at(&pp->lin[2], par, k) : 0;
    x.lo = o_hi >= o_lo ? lin_at(&pp->lin[3], par, k) - x.so : 0;
    return x;
  };
  auto odd_slot_off = [&](const Runs& x) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(shell + x.se) & ~uintptr_t(15);
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(shell + x.se + x.le) + 15) & ~uintptr_t(15);
    return (uint32_t(a1 - a0) + 127u) & ~127u;
  };
  const int D = int(ur.phi - ur.plo);
  auto issue = [&](int d) {  // one thread
    const Runs x = runs(ur.plo + d);
    const char *src0, *src1 = nullptr;
    uint32_t b0b, b1b = 0;
    int ld;
    const int sl = pipe_slot<NS>(d);
    bulk_span<T>(shell, x.se, x.le, &src0, &b0b, &ld);
    if (x.lo > 0) bulk_span<T>(shell, x.so, x.lo, &src1, &b1b, &ld);
    unsigned char* dst = raw + size_t(sl) * rawb;
    const uint32_t oso = odd_slot_off(x);
    pp->lead[sl][0] = int(reinterpret_cast<uintptr_t>(shell + x.se) & 15);
    pp->lead[sl][1] = int(oso + (reinterpret_cast<uintptr_t>(shell + x.so) & 15));
    fence_proxy_async();
    mbar_expect_tx(&pp->full[sl], b0b + b1b);  // release: the leads are visible to the waiters
    bulk_g2s(dst, src0, b0b, &pp->full[sl]);
    if (x.lo > 0) bulk_g2s(dst + oso, src1, b1b, &pp->full[sl]);
  };
  if (tid == 0)
    for (int d = 0; d <= min(D, NS - 1); ++d) issue(d);
  L0Planes<TI1> A;
#pragma unroll
  for (int ir = 0; ir < TI1; ++ir) A.prev[ir] = A.cur[ir] = A.next[ir] = 0.0;
  int jdone = 0;
  for (int d = 0; d <= D; ++d) {
    const int64_t p = ur.plo + d;
    mbar_wait(&pp->full[pipe_slot<NS>(d)], pipe_parity<NS>(d));
    const bool p_odd = p & 1;
    const int sl = pipe_slot<NS>(d);
    const unsigned char* slot = raw + sl * int(rawb);
    const volatile int* ld = pp->lead[sl];
    // slot positions of even tile row e = 0 (fine row jbase) and odd e = 0 (jbase + 1)
    const int st_e = int(p_odd ? g.n2 : g.n2 - g.m2);
    const T* evrun = reinterpret_cast<const T*>(slot + ld[0]);
    const T* odrun = reinterpret_cast<const T*>(slot + ld[1]);
    // even run starts at fine row 2 e_lo = rlo (rlo is even); jbase may be rlo - 2
    const T* ev = evrun + (int64_t((jbase - rlo) >> 1)) * st_e + cc;
    // odd run starts at fine row 2 o_lo + 1; tile odd row e = 0 is fine row jbase + 1
    const T* od = odrun + (int64_t(((jbase + 1) - (2 * o_lo + 1)) >> 1)) * g.n2 + cc;
    double Q[TI1];
#pragma unroll
    for (int ir = 0; ir < TI1; ++ir) Q[ir] = 0.0;
    if (p_odd) {
      if (full) rec_rows<T, TI1, true, true>(ev, od, st_e, n2, m2, jbase, rlo, rhi, b0, TR, m1, c, S.valid, has_odd, Q);
      else rec_rows<T, TI1, true, false>(ev, od, st_e, n2, m2, jbase, rlo, rhi, b0, TR, m1, c, S.valid, has_odd, Q);
    } else {
      if (full) rec_rows<T, TI1, false, true>(ev, od, st_e, n2, m2, jbase, rlo, rhi, b0, TR, m1, c, S.valid, has_odd, Q);
      else rec_rows<T, TI1, false, false>(ev, od, st_e, n2, m2, jbase, rlo, rhi, b0, TR, m1, c, S.valid, has_odd, Q);
    }
    pipe_release<NS>(pp, d, D, issue);
    l0_plane<TI1>(g, ur, S, p, Q, A, jdone, G);
  }
  pdl_trigger();
}

// ----------------------------------------------------------- interpolate
// add_interpolant (transform.hpp:317) + inverse_reorder_level
// (reorder.hpp:138) + unpack of the shell: fine block of level l from the
// corrected coarse block and the shell.  One CTA per (chunk of fine planes,
// tile of TRI fine rows) unit; each fine plane's shell runs (even rows, odd
// rows) and the coarse rows it interpolates from stream through a 3-slot
// TMA ring (no CTA barrier: the last warp done with a slot refills it).
// Strip lanes as the plane passes; every computed row is owned.
template <typename T, int TRI>
struct InterpSmem {
  static constexpr int NS = 3;
  static constexpr int NE = TRI / 2 + 1;  // coarse rows of a tile
  static __host__ __device__ size_t run_bytes(int64_t rows, int64_t len) {
    return (size_t(rows) * size_t(len) * sizeof(T) + 32 + 127) / 128 * 128;
  }
  static __host__ __device__ size_t ev_bytes(int64_t n2) { return run_bytes(TRI / 2, n2); }
  static __host__ __device__ size_t co_bytes(int64_t m2) { return run_bytes(NE, m2); }
  static __host__ __device__ size_t slot_bytes(int64_t n2, int64_t m2) { return 2 * ev_bytes(n2) + co_bytes(m2); }
  static __host__ __device__ size_t bytes(int64_t n2, int64_t m2) { return NS * slot_bytes(n2, m2) + sizeof(PlanePipe); }
};

template <typename T, int TRI, bool PODD, bool FULL>
__device__ __forceinline__ void interp_rows(const T* ev, const T* od, int64_t st_e, int oofs, T* __restrict__ out,
                                            const double* CL, const double* CR, int j1lo, int n1, int64_t n2l,
                                            int m2, bool owned, bool has_odd, bool right_degen) {
  const int rsrc = right_src(right_degen);
#pragma unroll
  for (int jr = 0; jr < TRI; ++jr) {
    const int j1 = j1lo + jr;
    if (!FULL && j1 >= n1) break;  // uniform
    const bool o1 = jr & 1;
    const int ea = jr >> 1;
    const T* sr = o1 ? od + ea * n2l : ev + ea * st_e;
    const bool rdeg = !FULL && o1 && (j1 + 1 >= n1);
    const double aL = CL[ea];
    const double bL = o1 ? (rdeg ? aL : CL[ea + 1]) : aL;
    double se;
    int ke;
    if (!PODD) {
      se = o1 ? aL + bL : aL;
      ke = o1 ? 1 : 0;
    } else {
      const double aR = CR[ea];
      const double bR = o1 ? (rdeg ? aR : CR[ea + 1]) : aR;
      se = aL + aR;
      if (o1) {
        se += bL;
        se += bR;
      }
      ke = o1 ? 2 : 1;
    }
    const double sn = __shfl_sync(0xffffffffu, se, rsrc);
    const double so = se + sn;
    {  // predicated stores (owned lanes; the odd node where it exists)
      const double sc_e = ke == 1 ? 0.5 : 0.25;
      const double sc_o = ke == 0 ? 0.5 : (ke == 1 ? 0.25 : 0.125);
      T* o = out + int64_t(jr) * n2l;
      st_if(o, ke == 0 ? to_t<T>(aL) : to_t<T>(double(sr[0]) + se * sc_e), owned);
      st_if(o + 1, to_t<T>(double(sr[o1 ? (has_odd ? m2 : 0) : (has_odd ? oofs : 0)]) + so * sc_o), owned && has_odd);
    }
  }
}

template <typename T, int TRI, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT == kPlaneMaxThreads ? 3 : 1)
    k_f3_rec_interp(const T* __restrict__ shell, const T* __restrict__ coarse, T* __restrict__ fine, const F3Geom g,
                    int ich, int ntile) {
  using SM = InterpSmem<T, TRI>;
  constexpr int NS = SM::NS, NE = SM::NE;
  extern __shared__ __align__(128) unsigned char smem[];
  const size_t evb = SM::ev_bytes(g.n2), slotb = SM::slot_bytes(g.n2, g.m2);
  PlanePipe* pp = reinterpret_cast<PlanePipe*>(smem + NS * slotb);
  const int m2 = int(g.m2), n2 = int(g.n2), n1 = int(g.n1), m1 = int(g.m1);
  const StripLane S = strip_lane(m2);
  const int c = S.c;
  const int cc = S.valid ? c : 0;
  const bool has_odd = S.valid && 2 * c + 1 < n2;
  const bool right_degen = 2 * c + 2 >= n2;
  const int chunk = int(blockIdx.x) / ntile, tile = int(blockIdx.x) - chunk * ntile;
  const int64_t p0 = g.p_base + int64_t(chunk) * ich;  // even
  const int D = int(min(g.p_end < 0 ? g.n0 : g.p_end, p0 + ich) - 1 - p0);
  const int j1lo = tile * TRI;  // even
  const int nrows = min(TRI, n1 - j1lo);
  const int e0 = j1lo >> 1;
  const int ne = (nrows + 1) >> 1, no = nrows >> 1, nc = min(NE, m1 - e0);
  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(&pp->full[b], 1);
      pp->cnt[b] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  struct Src {
    int64_t se, le, so, lo, cs;
  };
  auto src = [&](int d) {
    const int64_t p = p0 + d;
    const int64_t r0 = reord(p, g.m0);
    Src x;
    x.se = shell_row_start(g, r0, e0);
    x.le = shell_row_start(g, r0, e0 + ne) - x.se;
    x.so = shell_row_start(g, r0, g.m1 + e0);
    x.lo = shell_row_start(g, r0, g.m1 + e0 + no) - x.so;
    if (p & 1) {  // slab-sized buffers: the odd planes' region
      x.se += g.odd_shift;
      x.so += g.odd_shift;
    }
    const int64_t k = ((p & 1) && p + 1 < g.n0) ? (p >> 1) + 1 : (p >> 1);
    x.cs = (k * g.m1 + e0) * g.m2;
    return x;
  };
  auto issue = [&](int d) {  // one thread
    const Src x = src(d);
    const char *s0, *s1 = nullptr, *s2;
    uint32_t b0 = 0, b1 = 0, b2 = 0;
    int ld;
    bulk_span<T>(shell, x.se, x.le, &s0, &b0, &ld);
    if (x.lo > 0) bulk_span<T>(shell, x.so, x.lo, &s1, &b1, &ld);
    bulk_span<T>(coarse, x.cs, int64_t(nc) * g.m2, &s2, &b2, &ld);
    const int sl = pipe_slot<NS>(d);
    unsigned char* dst = smem + size_t(sl) * slotb;
    pp->lead[sl][0] = int(reinterpret_cast<uintptr_t>(shell + x.se) & 15);
    pp->lead[sl][1] = int(reinterpret_cast<uintptr_t>(shell + x.so) & 15);
    pp->lead[sl][2] = int(reinterpret_cast<uintptr_t>(coarse + x.cs) & 15);
    fence_proxy_async();
    mbar_expect_tx(&pp->full[sl], b0 + b1 + b2);  // release: the leads are visible to the waiters
    bulk_g2s(dst, s0, b0, &pp->full[sl]);
    if (x.lo > 0) bulk_g2s(dst + evb, s1, b1, &pp->full[sl]);
    bulk_g2s(dst + 2 * evb, s2, b2, &pp->full[sl]);
  };
  if (threadIdx.x == 0)
    for (int d = 0; d <= min(D, NS - 1); ++d) issue(d);
  const bool full = j1lo + TRI + 1 <= n1 - 1;
  double Cp[NE];  // coarse rows of the last even plane
#pragma unroll
  for (int e = 0; e < NE; ++e) Cp[e] = 0.0;
  for (int d = 0; d <= D; ++d) {
    const int64_t p = p0 + d;
    const bool p_odd = d & 1;
    const int sl = pipe_slot<NS>(d);
    mbar_wait(&pp->full[sl], pipe_parity<NS>(d));
    const unsigned char* slot = smem + sl * int(slotb);
    const volatile int* ld = pp->lead[sl];
    const T* ev = reinterpret_cast<const T*>(slot + ld[0]) + cc;
    const T* od = reinterpret_cast<const T*>(slot + evb + ld[1]) + cc;
    const T* co = reinterpret_cast<const T*>(slot + 2 * evb + ld[2]) + cc;
    double C[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) C[e] = (e < nc) ? double(co[e * m2]) : 0.0;
    T* out = fine + (p * g.n1 + j1lo) * g.n2 + 2 * cc;
    const int64_t st_e = p_odd ? g.n2 : g.n2 - g.m2;
    if (p_odd) {
      const double* CR = (p + 1 < g.n0) ? C : Cp;
      if (full) interp_rows<T, TRI, true, true>(ev, od, st_e, m2, out, Cp, CR, j1lo, n1, g.n2, m2, S.owned, has_odd, right_degen);
      else interp_rows<T, TRI, true, false>(ev, od, st_e, m2, out, Cp, CR, j1lo, n1, g.n2, m2, S.owned, has_odd, right_degen);
    } else {
      if (full) interp_rows<T, TRI, false, true>(ev, od, st_e, 0, out, C, C, j1lo, n1, g.n2, m2, S.owned, has_odd, right_degen);
      else interp_rows<T, TRI, false, false>(ev, od, st_e, 0, out, C, C, j1lo, n1, g.n2, m2, S.owned, has_odd, right_degen);
#pragma unroll
      for (int e = 0; e < NE; ++e) Cp[e] = C[e];
    }
    pipe_release<NS>(pp, d, D, issue);
  }
  pdl_trigger();
}

// --------------------------------------------------------------- row pass
// Thomas along axis 2 (batched_solve, transform.hpp:116-130) of every row of
// the coarse fp64 volume G, in place: one warp per row, the row staged in
// shared memory for the segmented solve (warp_row_thomas).  The next row's
// NC coalesced 256-byte chunks are loaded into registers while the current
// row is solved, so each warp keeps a whole row of loads in flight (the
// pass is bound by HBM latency x bytes in flight, not by the solve).
__host__ __device__ constexpr int kRowCtas(int nc) { return nc <= 5 ? 4 : (nc <= 9 ? 3 : (nc <= 17 ? 2 : 1)); }

template <int NC, bool TOEP = false>
__global__ void __launch_bounds__(256, kRowCtas(NC)) k_f3_row(double* __restrict__ G, int64_t rows, int m,
                                                const double* __restrict__ w, const double* __restrict__ inv_d) {
  extern __shared__ double rs[];
  double* tw = rs;
  double* tid = rs + m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* buf = tid + m + warp * m;
  if (TOEP) {  // only the end-correction tables (they follow inv_d: api.cu get_plan)
    for (int i = threadIdx.x; i < 2 * kToepEnds; i += blockDim.x) tw[i] = inv_d[m + i];
  } else {
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      tw[i] = w[i];
      tid[i] = inv_d[i];
    }
  }
  __syncthreads();
  pdl_wait();
  const int64_t step = int64_t(gridDim.x) * nw;
  int64_t r = int64_t(blockIdx.x) * nw + warp;
  const uint64_t pkeep = pol_keep(), pstream = pol_stream();
  double t[NC];
  // rows are walked from the last one down: the producer of G (plane pass)
  // wrote the high planes last, so they are the likeliest L2 hits
  auto load = [&](int64_t rr) {
    const int64_t row = rows - 1 - rr;
    const double* gr = G + row * m + lane;
#pragma unroll
    for (int k = 0; k < NC; ++k) t[k] = (lane + 32 * k < m) ? ld_pol(gr + 32 * k, pstream) : 0.0;
  };
  if (r < rows) load(r);
  for (; r < rows; r += step) {
#pragma unroll
    for (int k = 0; k < NC; ++k)
      if (lane + 32 * k < m) buf[lane + 32 * k] = t[k];
    __syncwarp();
    if (r + step < rows) load(r + step);
    if (TOEP) warp_row_toep<NC>(buf, m, tw, tw + kToepEnds);
    else warp_row_thomas_reg<NC>(buf, m, tw, tid);
    double* gr = G + (rows - 1 - r) * m;
#pragma unroll
    for (int k = 0; k < NC; ++k)
      if (lane + 32 * k < m) st_pol(gr + lane + 32 * k, buf[lane + 32 * k], pkeep);
    __syncwarp();
  }
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Row pass in Toeplitz form with a deeper prefetch: every warp owns a ring of
// kRowRing row buffers filled by cp.async (8-byte copies: rows are only
// 8-byte aligned), two rows in flight while one is solved; no registers are
// spent on the prefetch.
constexpr int kRowRing = 3;
template <int NC>
__global__ void __launch_bounds__(256, kRowCtas(NC)) k_f3_row_ring(double* __restrict__ G, int64_t rows, int m,
                                                                    const double* __restrict__ gh) {
  extern __shared__ double rs[];
  constexpr int W = 32 * NC;  // buffer width: the row right-aligned, zeros before it (warp_row_toep_ra)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* ring = rs + size_t(warp) * kRowRing * W;
  const int P0 = W - m;
  for (int i = lane; i < kRowRing * W; i += 32)
    if (i % W < P0) ring[i] = 0.0;
  const double gl = gh[lane], hl = gh[kToepEnds + lane];
  __syncwarp();
  pdl_wait();
  const int64_t step = int64_t(gridDim.x) * nw;
  const int64_t r0 = int64_t(blockIdx.x) * nw + warp;
  const uint64_t pkeep = pol_keep();
  // rows are walked from the last one down (the producer wrote the high planes last)
  auto issue = [&](int64_t rr, int slot) {
    if (rr < rows) {
      const double* gr = G + (rows - 1 - rr) * m + lane;
      double* dst = ring + slot * W + P0 + lane;
#pragma unroll
      for (int k = 0; k < NC; ++k)
        if (lane + 32 * k < m) cp_async8(dst + 32 * k, gr + 32 * k);
    }
    cp_async_commit();  // a group per step, empty past the end
  };
  issue(r0, 0);
  issue(r0 + step, 1);
  int slot = 0;
  for (int64_t r = r0; r < rows; r += step) {
    issue(r + 2 * step, slot >= 1 ? slot - 1 : kRowRing - 1);  // (slot + 2) % 3
    cp_async_wait<2>();
    __syncwarp();
    double* buf = ring + slot * W;
    warp_row_toep_ra<NC>(buf, m, gl, hl);
    double* gr = G + (rows - 1 - r) * m + lane;
    const double* src = buf + P0 + lane;
#pragma unroll
    for (int k = 0; k < NC; ++k)
      if (lane + 32 * k < m) st_pol(gr + 32 * k, src[32 * k], pkeep);
    __syncwarp();
    slot = slot == kRowRing - 1 ? 0 : slot + 1;
  }
}

// MGRX_NO_TOEP keeps the table-driven Thomas solves (A/B switch)
bool toep_enabled() {
  static const bool off = std::getenv("MGRX_NO_TOEP") != nullptr;
  return !off;
}

bool ring_enabled() {
  static const bool off = std::getenv("MGRX_NO_ROW_RING") != nullptr;
  return !off;
}

void launch_row(double* G, const F3Geom& g, const double* w, const double* id, const Exec& ex, bool toep = false) {
  const int m = int(g.m2);
  const int64_t rows = g.m0 * g.m1;
  const int threads = 256;
  const size_t smem = size_t(2 + threads / 32) * m * 8;
  // lanes solve segments of an ODD number of values (warp_row_thomas_reg): an
  // even segment length puts the lanes' strided shared-memory accesses on a
  // few banks (m2 = 251: 47 -> 13 us at 51 x 251 rows)
  const int nc = ((m + 31) / 32) | 1;
  const int64_t blocks = std::min<int64_t>((rows + 7) / 8, int64_t(kNumSMs) * kRowCtas(nc));
#define ROW_(NC)                                                                                           \
  do {                                                                                                     \
    if (toep && m >= kToepMinM && ring_enabled()) {                                                        \
      /* at least so much shared memory that one block more than kRowCtas(NC) cannot be resident: the  \
         grid is kRowCtas blocks per SM, and a register allocation that lets a 4th block in measured   \
         48 -> 58 us (uneven blocks per SM) */                                                           \
      const size_t rsm = std::max(size_t((threads / 32) * kRowRing * 32 * NC) * 8,                         \
                                  size_t(228 * 1024) / (kRowCtas(NC) + 1) + 1024);                         \
      cudaFuncSetAttribute(k_f3_row_ring<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(rsm));      \
      MGRX_LAUNCH(ex, "f3_row", pdl_launch(k_f3_row_ring<NC>, dim3(unsigned(blocks)), dim3(threads), rsm, ex.s, \
                                           !ex.prof, G, rows, m, id + m));                                 \
    } else if (toep && m >= kToepMinM) {                                                                   \
      cudaFuncSetAttribute(k_f3_row<NC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));    \
      MGRX_LAUNCH(ex, "f3_row", pdl_launch(k_f3_row<NC, true>, dim3(unsigned(blocks)), dim3(threads), smem, ex.s, \
                                           !ex.prof, G, rows, m, w, id));                                  \
    } else {                                                                                               \
      cudaFuncSetAttribute(k_f3_row<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));          \
      MGRX_LAUNCH(ex, "f3_row", pdl_launch(k_f3_row<NC>, dim3(unsigned(blocks)), dim3(threads), smem, ex.s, \
                                           !ex.prof, G, rows, m, w, id));                                  \
    }                                                                                                      \
  } while (0)
  if (nc <= 1) ROW_(1);
  else if (nc <= 3) ROW_(3);
  else if (nc <= 5) ROW_(5);
  else if (nc <= 9) ROW_(9);
  else if (nc <= 17) ROW_(17);
  else ROW_(33);  // plane-pass CTAs (<= 1024 threads, 30 coarse columns per warp) cap m2 at 960
#undef ROW_
}

// ------------------------------------------------------------ column pass
// Thomas along axis 0 or 1 of the coarse fp64 volume G (m0 x m1 x m2).
// 16 consecutive columns per block; each column is split into S segments
// (two per warp row) of up to LS values kept in registers.  A segment runs
// the recurrence from a zero carry to get its affine map, the maps are
// folded through shared memory, and the segment reruns the exact recurrence
// from its true carry.  With `coarse` set the result is applied:
// coarse += sign * z (apply_correction, transform.hpp:435-477); otherwise it
// is written back to G.
template <typename T, int LS, bool APPLY, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT == kColThreads ? 3 : (MAXT == kColThreads12 ? 3 : 1))
    k_f3_col(double* __restrict__ G, T* __restrict__ coarse, double sign, int64_t ncols, int m, int64_t stride,
             int64_t outer_stride, int64_t inner, const double* __restrict__ w, const double* __restrict__ inv_d) {
  extern __shared__ double sc[];
  const int lane = threadIdx.x, S = 2 * blockDim.y;
  const int c16 = lane & 15, s = 2 * threadIdx.y + (lane >> 4);
  double* tw = sc;
  double* tid = sc + m;
  double* A = tid + m;  // [S][16]
  double* B = A + S * 16;
  for (int i = threadIdx.y * 32 + lane; i < m; i += blockDim.y * 32) {
    tw[i] = w[i];
    tid[i] = inv_d[i];
  }
  // tiles from the last one down (the previous pass wrote the high planes last)
  const int64_t col = int64_t(gridDim.x - 1 - blockIdx.x) * 16 + c16;
  const bool valid = col < ncols;
  const int64_t base = valid ? (col / inner) * outer_stride + (col % inner) : 0;
  const int seg = (m + S - 1) / S;
  const int s0 = min(m, s * seg), s1 = min(m, s0 + seg);
  const int len = s1 - s0;
  double v[LS];
  pdl_wait();
  {
    const double* gp = G + base + int64_t(s0) * stride;
    // the axis-0 pass reads G for the last time (evict first)
#pragma unroll
    for (int k = 0; k < LS; ++k) {
      v[k] = (valid && k < len) ? (APPLY ? __ldcs(gp) : *gp) : 0.0;
      gp += stride;
    }
  }
  __syncthreads();
  // forward y_i = f_i - w_i y_{i-1} (batched_solve, transform.hpp:117-120)
  double ya = 0.0, yb = 1.0;
#pragma unroll
  for (int k = 0; k < LS; ++k)
    if (k < len) {
      const double wi = ld_volatile(tw + s0 + k);
      ya = v[k] - wi * ya;
      yb = -wi * yb;
    }
  A[s * 16 + c16] = ya;
  B[s * 16 + c16] = yb;
  __syncthreads();
  double y = 0.0;
  for (int q = 0; q < s; ++q) y = A[q * 16 + c16] + B[q * 16 + c16] * y;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < LS; ++k)
    if (k < len) {
      y = v[k] - ld_volatile(tw + s0 + k) * y;
      v[k] = y;
    }
  // back substitution z_i = (y_i - z_{i+1}/3) / d_i (transform.hpp:121-129)
  double za = 0.0, zb = 1.0;
#pragma unroll
  for (int k = LS - 1; k >= 0; --k)
    if (k < len) {
      const double id = ld_volatile(tid + s0 + k);
      za = (v[k] - kOff * za) * id;
      zb = -kOff * id * zb;
    }
  A[s * 16 + c16] = za;
  B[s * 16 + c16] = zb;
  __syncthreads();
  double z = 0.0;
  for (int q = S - 1; q > s; --q) z = A[q * 16 + c16] + B[q * 16 + c16] * z;
#pragma unroll
  for (int k = LS - 1; k >= 0; --k)
    if (k < len) {
      z = (v[k] - kOff * z) * ld_volatile(tid + s0 + k);
      v[k] = z;
    }
  pdl_trigger();
  if (!valid) return;
  if (APPLY) {  // coarse values loaded only now, four at a time: fewer live registers
    T* c = coarse + base + int64_t(s0) * stride;
#pragma unroll
    for (int k0 = 0; k0 < LS; k0 += 4) {
      T cv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) cv[u] = (k0 + u < LS && k0 + u < len) ? c[int64_t(k0 + u) * stride] : T(0);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k0 + u < LS && k0 + u < len) c[int64_t(k0 + u) * stride] = to_t<T>(double(cv[u]) + sign * v[k0 + u]);
    }
  } else {
    double* gp = G + base + int64_t(s0) * stride;
    const uint64_t pol = pol_keep();
#pragma unroll
    for (int k = 0; k < LS; ++k) {
      if (k < len) st_pol(gp, v[k], pol);
      gp += stride;
    }
  }
}

// The column pass in Toeplitz form (see "Toeplitz solves"): segments of
// exactly LS values (zero past the end), no factor tables in the recurrences,
// one folded value per segment; the two end corrections need the column's
// z_0 and z_{m-1}, passed through shared memory.
template <typename T, int LS, bool APPLY, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT == kColThreads ? 3 : (MAXT == kColThreads12 ? 3 : 1))
    k_f3_col_toep(double* __restrict__ G, T* __restrict__ coarse, double sign, int64_t ncols, int m, int64_t stride,
                  int64_t outer_stride, int64_t inner, const double* __restrict__ gh) {
  constexpr PowTab<LS> PF(-kTw), PB(-kTc);
  extern __shared__ double sc[];
  const int lane = threadIdx.x, S = 2 * blockDim.y;
  const int c16 = lane & 15, s = 2 * threadIdx.y + (lane >> 4);
  double* gt = sc;               // [kToepEnds]
  double* ht = sc + kToepEnds;   // [kToepEnds]
  double* A = ht + kToepEnds;    // [S][16]
  double* E = A + S * 16;        // [2][16]: z_0 and z_{m-1} of the 16 columns
  T* cbuf = reinterpret_cast<T*>(E + 32);  // APPLY: [S * LS][16] the coarse values, prefetched under the solve
  // the end-correction tables: loaded now, stored after this thread's G loads are in flight
  const int gi = threadIdx.y * 32 + lane;
  const double ghv = gi < 2 * kToepEnds ? gh[gi] : 0.0;
  const int64_t col = int64_t(gridDim.x - 1 - blockIdx.x) * 16 + c16;
  const bool valid = col < ncols;
  const int64_t base = valid ? (col / inner) * outer_stride + (col % inner) : 0;
  const int s0 = s * LS;
  const int len = max(0, min(m, s0 + LS) - s0);
  double v[LS];
  pdl_wait();
  {
    const double* gp = G + base + int64_t(s0) * stride;
#pragma unroll
    for (int k = 0; k < LS; ++k) {
      v[k] = (valid && k < len) ? (APPLY ? __ldcs(gp) : *gp) : 0.0;
      gp += stride;
    }
  }
  if (gi < 2 * kToepEnds) sc[gi] = ghv;
  if (APPLY) {  // this thread's coarse values into its own slots of cbuf (4- or 8-byte cp.async)
    const T* c = coarse + base + int64_t(s0) * stride;
    T* mine = cbuf + s0 * 16 + c16;
#pragma unroll
    for (int k = 0; k < LS; ++k) {
      if (valid && k < len) {
        if (sizeof(T) == 4) cp_async4(mine + k * 16, c);
        else cp_async8(mine + k * 16, c);
      }
      c += stride;
    }
    cp_async_commit();
  }
  // forward from a zero carry; v[k] keeps the zero-carry values
  double a = 0.0;
#pragma unroll
  for (int k = 0; k < LS; ++k) {
    a = v[k] - kTw * a;
    v[k] = a;
  }
  A[s * 16 + c16] = a;
  __syncthreads();
  double y = 0.0;
  for (int q = 0; q < s; ++q) y = A[q * 16 + c16] + PF.v[LS] * y;
#pragma unroll
  for (int k = 0; k < LS; ++k) v[k] = (k < len) ? v[k] + PF.v[k + 1] * y : 0.0;
  // back substitution from a zero carry
  double g = 0.0;
#pragma unroll
  for (int k = LS - 1; k >= 0; --k) {
    g = (v[k] - kOff * g) * kTid;
    v[k] = g;
  }
  __syncthreads();  // the forward folds have read A
  A[s * 16 + c16] = g;
  __syncthreads();
  double z = 0.0;
  for (int q = S - 1; q > s; --q) z = A[q * 16 + c16] + PB.v[LS] * z;
#pragma unroll
  for (int k = 0; k < LS; ++k) v[k] = v[k] + PB.v[LS - k] * z;
  // end corrections: x = z + z_0 Gt + z_{m-1} Ht
  const int last = m - 1;
  if (s == 0) E[c16] = v[0];
  if (s == last / LS) {
    double zl = 0.0;
#pragma unroll
    for (int k = 0; k < LS; ++k)
      if (s0 + k == last) zl = v[k];
    E[16 + c16] = zl;
  }
  __syncthreads();
  if (s0 < kToepEnds) {
    const double z0 = E[c16];
#pragma unroll
    for (int k = 0; k < LS; ++k)
      if (s0 + k < kToepEnds) v[k] = v[k] + z0 * gt[s0 + k];
  }
  if (s0 + LS > m - kToepEnds) {
    const double zm = E[16 + c16];
#pragma unroll
    for (int k = 0; k < LS; ++k) {
      const int rev = last - (s0 + k);
      if (rev >= 0 && rev < kToepEnds) v[k] = v[k] + zm * ht[rev];
    }
  }
  pdl_trigger();
  if (!valid) return;
  if (APPLY) {  // the coarse values were prefetched into this thread's slots of cbuf
    cp_async_wait<0>();
    T* c = coarse + base + int64_t(s0) * stride;
    const T* mine = cbuf + s0 * 16 + c16;
#pragma unroll
    for (int k = 0; k < LS; ++k) {
      if (k < len) *c = to_t<T>(double(mine[k * 16]) + sign * v[k]);
      c += stride;
    }
  } else {
    double* gp = G + base + int64_t(s0) * stride;
    const uint64_t pol = pol_keep();
#pragma unroll
    for (int k = 0; k < LS; ++k) {
      if (k < len) st_pol(gp, v[k], pol);
      gp += stride;
    }
  }
}

// ------------------------------------------------------------ host side

template <typename T, int TI1>
size_t plane_smem(const F3Geom& g) {
  return PlaneSmem<T, TI1>::bytes(g.n2, g.m2);
}
template <typename T>
size_t plane_smem3r(const F3Geom& g) {
  return PlaneSmem<T, 4, 0, 3>::bytes(g.n2, g.m2);
}
template <typename T>
size_t plane_smem3(const F3Geom& g) {
  return PlaneSmem<T, 4, 3, 0>::bytes(g.n2, g.m2);
}

// Row tile of the plane passes: maximise resident warps x useful-row
// fraction (2 TI1 owned rows of 2 TI1 + 3 computed) within shared memory and
// the register budget of __launch_bounds__(kPlaneMaxThreads, 2).
template <typename T>
bool pick_tile(F3Geom& g, size_t optin, size_t per_sm) {
  const int warps = int((g.m2 + 29) / 30);
  const int cands[2] = {4, 2};
  double best = -1.0;
  for (int c : cands) {
    size_t need = 0;
    if (c == 4) need = plane_smem<T, 4>(g);
    if (c == 2) need = plane_smem<T, 2>(g);
    if (need > optin) continue;
    int ctas = int(per_sm / (need + 1024));
    // registers: <= 96 per thread (launch bounds 288 x 2) -> 5 warps per SM sub-partition
    ctas = std::min(ctas, std::max(1, 20 / warps));
    ctas = std::max(ctas, 1);
    const int resident = std::min(ctas * warps, 32);
    const double score = resident * (2.0 * c) / (2.0 * c + 3.0);
    if (score > best + 1e-9) {
      best = score;
      g.tile_rows = c;
      g.ctas_per_sm = ctas;
    }
  }
  // wide levels (8-9 warps per CTA, 4 coarse rows per tile): the decompose
  // plane pass runs 3 CTAs per SM on a 3-slot ring (72 registers) — more
  // independent plane streams per SM (MGRX_NO_DEC3 disables)
  g.dec3 = 0;
  static const bool no3 = std::getenv("MGRX_NO_DEC3") != nullptr;
  if (!no3 && g.tile_rows == 4 && warps >= 8 && warps <= 9 && 3 * (plane_smem3<T>(g) + 1024) <= per_sm) g.dec3 = 1;
  return best > 0.0;
}

template <typename T>
void launch_col(double* G, T* coarse, double sign, const F3Geom& g, int axis, const double* w, const double* id,
                const Exec& ex, bool toep = false) {
  int64_t stride, outer_stride, inner, ncols;
  int m;
  if (axis == 1) {
    m = int(g.m1);
    stride = g.m2;
    inner = g.m2;
    outer_stride = g.m1 * g.m2;
    ncols = g.m0 * g.m2;
  } else {
    m = int(g.m0);
    stride = g.m1 * g.m2;
    inner = g.m1 * g.m2;
    outer_stride = 0;
    ncols = g.m1 * g.m2;
  }
  const unsigned blocks = unsigned((ncols + 15) / 16);
  const char* tag = axis == 1 ? "f3_col1" : "f3_col0";
// segments of <= 16 values: up to 10 warp rows (320 threads, 3 blocks/SM)
  // for m <= 320, up to 20 (640 threads, 1 block/SM) for m <= 640
#define MGRX_COL(AP, MT) MGRX_COLL(16, AP, MT)
#define MGRX_COLL(LS, AP, MT)                                                                             \
  {                                                                                                       \
    const int SY = (m + 2 * LS - 1) / (2 * LS);                                                          \
    MGRX_LAUNCH(ex, tag, pdl_launch(k_f3_col<T, LS, AP, MT>, dim3(blocks), dim3(32, SY),                      \
                                    size_t(2 * m + 2 * 2 * SY * 16) * 8, ex.s, !ex.prof, G, coarse, sign, ncols, m,       \
                                    stride, outer_stride, inner, w, id));                                       \
  }
#define MGRX_COLT(LS, AP, MT)                                                                            \
  {                                                                                                       \
    const int SY = (m + 2 * LS - 1) / (2 * LS);                                                          \
    const size_t csm = size_t(2 * kToepEnds + 2 * SY * 16 + 32) * 8 +                                     \
                       (AP ? size_t(2 * SY * LS * 16) * sizeof(T) : size_t(0)); /* + the prefetched coarse values */ \
    cudaFuncSetAttribute(k_f3_col_toep<T, LS, AP, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(csm)); \
    MGRX_LAUNCH(ex, tag, pdl_launch(k_f3_col_toep<T, LS, AP, MT>, dim3(blocks), dim3(32, SY), csm, ex.s, !ex.prof, \
                                    G, coarse, sign, ncols, m, stride, outer_stride, inner, id + m));     \
  }
  if (toep && m >= kToepMinM) {  // the end-correction tables follow inv_d (api.cu get_plan)
    if (m <= 264) {
      if (coarse) MGRX_COLT(12, true, kColThreads12) else MGRX_COLT(12, false, kColThreads12)
    } else if (m <= 320) {
      if (coarse) MGRX_COLT(16, true, kColThreads) else MGRX_COLT(16, false, kColThreads)
    } else {
      if (coarse) MGRX_COLT(16, true, 2 * kColThreads) else MGRX_COLT(16, false, 2 * kColThreads)
    }
  } else if (m <= 264) {
    if (coarse) MGRX_COLL(12, true, kColThreads12) else MGRX_COLL(12, false, kColThreads12)
  } else if (m <= 320) {
    if (coarse) MGRX_COL(true, kColThreads) else MGRX_COL(false, kColThreads)
  } else {
    if (coarse) MGRX_COL(true, 2 * kColThreads) else MGRX_COL(false, 2 * kColThreads)
  }
#undef MGRX_COL
#undef MGRX_COLL
#undef MGRX_COLT
}

// Axis-2 then axis-1 solves of G: the row pass and the axis-1 column pass.
static void row_col1(double* G, const F3Geom& g, const ThomasLevel& th, const Exec& ex) {
  launch_row(G, g, th.w[2], th.inv_d[2], ex, toep_enabled());
  launch_col<float>(G, static_cast<float*>(nullptr), 0.0, g, 1, th.w[1], th.inv_d[1], ex, toep_enabled());
}

}  // namespace

Fused3DPlan fused3d_plan(const LevelGeom& lg, int esize) {
  Fused3DPlan fp;
  if (lg.d != 3) return fp;
  F3Geom& g = fp.g;
  g.n0 = lg.n[0];
  g.n1 = lg.n[1];
  g.n2 = lg.n[2];
  g.m0 = lg.m[0];
  g.m1 = lg.m[1];
  g.m2 = lg.m[2];
  if (g.n2 < 33 || g.m1 > kColMaxM || g.m0 > kColMaxM || g.n1 < 5 || g.n0 < 5) return fp;
  if ((g.m2 + 29) / 30 * 32 > kWideThreads) return fp;
  // small levels stay on the general kernels (launch-latency bound either way)
  {
    int64_t min_elems = int64_t(1) << 15;
    if (const char* env = std::getenv("MGRX_FUSED_MIN_ELEMS")) min_elems = std::atoll(env);
    if (int64_t(g.n0) * g.n1 * g.n2 < min_elems) return fp;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  int optin = 0, nsm = 0, per_sm = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  if (optin <= 0) optin = 227 * 1024;
  if (per_sm <= 0) per_sm = 228 * 1024;
  if (nsm <= 0) nsm = kNumSMs;
  const bool ok = esize == 4 ? pick_tile<float>(g, size_t(optin), size_t(per_sm))
                             : pick_tile<double>(g, size_t(optin), size_t(per_sm));
  if (!ok) return fp;
  g.threads = int((g.m2 + 29) / 30) * 32;
  const int ctas = nsm * g.ctas_per_sm;
  // Small levels are latency bound (a unit streams its planes serially):
  // shrink the row tile until single-plane-pair units give two waves.
  const bool shrink = std::getenv("MGRX_NO_TILE_SHRINK") == nullptr;
  while (shrink && g.tile_rows > 2 && ((g.m1 + g.tile_rows - 1) / g.tile_rows) * g.m0 < 2 * int64_t(ctas))
    g.tile_rows = g.tile_rows == 8 ? 6 : (g.tile_rows == 6 ? 4 : 2);
  g.ntile1 = int((g.m1 + g.tile_rows - 1) / g.tile_rows);
  // axis-0 chunk of a unit: a unit of c coarse planes streams 2c + 3 fine
  // planes (two halo planes are recomputed by the neighbour) plus a fixed
  // pipeline fill; pick c minimising waves x per-unit time.
  double fill_planes = 3.0;  // pipeline fill of a unit, in plane-times (MGRX_FILL_PLANES overrides)
  if (const char* env = std::getenv("MGRX_FILL_PLANES")) fill_planes = std::atof(env);
  auto pick_chunk = [&](int64_t slots) {
    int64_t ch = 1;
    double best = 1e300;
    for (int64_t c = 1; c <= 32 && c <= g.m0; ++c) {
      const int64_t units = ((g.m0 + c - 1) / c) * g.ntile1;
      const int64_t waves = (units + slots - 1) / slots;
      const double cost = double(waves) * double(2 * c + 3 + fill_planes);
      if (cost < best - 1e-9) {
        best = cost;
        ch = c;
      }
    }
    return ch;
  };
  int64_t chunk = pick_chunk(ctas);
  if (g.dec3) g.dec_chunk = pick_chunk(int64_t(nsm) * 3);
  if (const char* env = std::getenv("MGRX_CHUNK")) chunk = std::max<int64_t>(1, std::min<int64_t>(g.m0, std::atoll(env)));
  const int64_t nchunk = (g.m0 + chunk - 1) / chunk;
  g.chunk = chunk;
  g.units = int(nchunk * g.ntile1);
  g.grid = g.units;  // one CTA per unit; the hardware scheduler balances
  fp.enabled = true;
  fp.scratch_bytes = size_t(g.m0) * g.m1 * g.m2 * 8 + 256;
  return fp;
}

// Interpolation pass: TRI = 8 fine rows per tile (4 for fp64, keeping three
// CTAs per SM); an even number of fine planes per unit, sized for about
// eight units per resident CTA slot.
template <typename T, int TRI, int MAXT>
static cudaError_t launch_interp_t(const T* shell, const T* coarse, T* fine, const F3Geom& g, const Exec& ex) {
  const size_t smem = InterpSmem<T, TRI>::bytes(g.n2, g.m2);
  cudaError_t e =
      cudaFuncSetAttribute(k_f3_rec_interp<T, TRI, MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ntile = int((g.n1 + TRI - 1) / TRI);
  int64_t per_slot = 8;  // units per resident CTA slot (MGRX_INTERP_UNITS overrides)
  if (const char* env = std::getenv("MGRX_INTERP_UNITS")) per_slot = std::max(1, std::atoi(env));
  const int64_t want = int64_t(sms) * 3 * per_slot;
  const int64_t np = (g.p_end < 0 ? g.n0 : g.p_end) - g.p_base;  // fine planes of this launch
  int64_t ich = (np * ntile) / want;
  ich = std::max<int64_t>(2, std::min<int64_t>(32, ich & ~int64_t(1)));
  const int64_t chunks = (np + ich - 1) / ich;
  MGRX_LAUNCH(ex, "f3_rec_interp",
              pdl_launch(k_f3_rec_interp<T, TRI, MAXT>, dim3(unsigned(chunks * ntile)), dim3(g.threads), smem, ex.s, !ex.prof,
                         shell, coarse, fine, g, int(ich), ntile));
  return cudaSuccess;
}

template <typename T>
static cudaError_t launch_interp(const T* shell, const T* coarse, T* fine, const F3Geom& g, const Exec& ex) {
  if (g.threads > kPlaneMaxThreads) {
    if (sizeof(T) == 4) return launch_interp_t<T, 8, kWideBound>(shell, coarse, fine, g, ex);
    return launch_interp_t<T, 4, kWideBound>(shell, coarse, fine, g, ex);
  }
  if (sizeof(T) == 4) return launch_interp_t<T, 8, kPlaneMaxThreads>(shell, coarse, fine, g, ex);
  return launch_interp_t<T, 4, kPlaneMaxThreads>(shell, coarse, fine, g, ex);
}

// The recompose plane pass's 3-CTA / 3-slot variant on the levels that use
// the decompose one (MGRX_NO_REC3 disables; ~5 us per recompose at 513^3).
static bool rec3_enabled() {
  static const bool on = std::getenv("MGRX_NO_REC3") == nullptr;
  return on;
}

// The decompose plane pass's chunking for its 3-CTA variant.
static F3Geom dec3_geom(const F3Geom& g) {
  F3Geom gd = g;
  if (g.dec_chunk > 0 && g.a_end < 0) {
    gd.chunk = g.dec_chunk;
    gd.units = int(((g.m0 + gd.chunk - 1) / gd.chunk) * g.ntile1);
    gd.grid = gd.units;
  }
  return gd;
}

template <typename T>
static cudaError_t set_attrs(const F3Geom& g, size_t* smem) {
  cudaError_t e = cudaSuccess;
#define MGRX_ATTR(TI, MT)                                                                                      \
  if (g.tile_rows == TI && (MT == kWideBound) == (g.threads > kPlaneMaxThreads)) {                        \
    *smem = plane_smem<T, TI>(g);                                                                           \
    e = cudaFuncSetAttribute(k_f3_dec_plane<T, TI, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(*smem)); \
    if (e == cudaSuccess)                                                                                   \
      e = cudaFuncSetAttribute(k_f3_rec_plane<T, TI, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                               int(*smem));                                                                 \
  }
  MGRX_ATTR(4, kPlaneMaxThreads)
  MGRX_ATTR(2, kPlaneMaxThreads)
  MGRX_ATTR(4, kWideBound)
  MGRX_ATTR(2, kWideBound)
#undef MGRX_ATTR
  if (e == cudaSuccess && g.dec3)
    e = cudaFuncSetAttribute(k_f3_dec_plane<T, 4, kPlaneMaxThreads, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(plane_smem3<T>(g)));
  if (e == cudaSuccess && g.dec3 && rec3_enabled())
    e = cudaFuncSetAttribute(k_f3_rec_plane<T, 4, kPlaneMaxThreads, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(plane_smem3r<T>(g)));
  return e;
}

template <typename T>
cudaError_t fused3d_decompose_level(const T* blk, T* shell, T* coarse, void* scratch, const LevelGeom&,
                                    const Fused3DPlan& fp, const ThomasLevel& th, const Exec& ex) {
  const F3Geom& g = fp.g;
  double* G = static_cast<double*>(scratch);
  size_t ds = 0;
  cudaError_t e = set_attrs<T>(g, &ds);
  if (e != cudaSuccess) return e;
  // ex.nonfinite: the finiteness check rides on this pass (the variant with CF)
  const bool cf = ex.nonfinite != nullptr;
  F3Geom gc = g;
  gc.nonfinite = ex.nonfinite;
#define MGRX_DEC(TI, MT)                                                                                      \
  if (!g.dec3 && g.tile_rows == TI && (MT == kWideBound) == (g.threads > kPlaneMaxThreads)) {               \
    if (cf) {                                                                                                 \
      e = cudaFuncSetAttribute(k_f3_dec_plane<T, TI, MT, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               int(ds));                                                                      \
      if (e != cudaSuccess) return e;                                                                         \
      MGRX_LAUNCH(ex, "f3_dec_plane", pdl_launch(k_f3_dec_plane<T, TI, MT, 0, true>, dim3(g.grid), dim3(g.threads), \
                                                 ds, ex.s, !ex.prof, blk, shell, coarse, G, gc));             \
    } else {                                                                                                  \
      MGRX_LAUNCH(ex, "f3_dec_plane", pdl_launch(k_f3_dec_plane<T, TI, MT>, dim3(g.grid), dim3(g.threads), ds,  \
                                                 ex.s, !ex.prof, blk, shell, coarse, G, g));                  \
    }                                                                                                         \
  }
  MGRX_DEC(4, kPlaneMaxThreads)
  MGRX_DEC(2, kPlaneMaxThreads)
  MGRX_DEC(4, kWideBound)
  MGRX_DEC(2, kWideBound)
#undef MGRX_DEC
  if (g.dec3) {
    F3Geom gd = dec3_geom(g);
    if (cf) {
      gd.nonfinite = ex.nonfinite;
      e = cudaFuncSetAttribute(k_f3_dec_plane<T, 4, kPlaneMaxThreads, 3, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(plane_smem3<T>(g)));
      if (e != cudaSuccess) return e;
      MGRX_LAUNCH(ex, "f3_dec_plane", pdl_launch(k_f3_dec_plane<T, 4, kPlaneMaxThreads, 3, true>, dim3(gd.grid),
                                                 dim3(gd.threads), plane_smem3<T>(gd), ex.s, !ex.prof, blk, shell,
                                                 coarse, G, gd));
    } else {
      MGRX_LAUNCH(ex, "f3_dec_plane", pdl_launch(k_f3_dec_plane<T, 4, kPlaneMaxThreads, 3>, dim3(gd.grid),
                                                 dim3(gd.threads), plane_smem3<T>(gd), ex.s, !ex.prof, blk, shell,
                                                 coarse, G, gd));
    }
  }
  if (ex.after_plane) {
    e = cudaEventRecord(ex.after_plane, ex.s);
    if (e != cudaSuccess) return e;
  }
  row_col1(G, g, th, ex);
  launch_col<T>(G, coarse, 1.0, g, 0, th.w[0], th.inv_d[0], ex, toep_enabled());
  return cudaGetLastError();
}

// Recompose correction of a level (rec plane + row + axis-1 column pass,
// into the level's G): depends only on the level's shell, so the levels'
// corrections may run concurrently (transform.hpp:343-366: the component
// is zero on the coarse nodes).
template <typename T>
cudaError_t fused3d_recompose_correction(const T* shell, void* scratch, const Fused3DPlan& fp, const ThomasLevel& th,
                                         const Exec& ex) {
  const F3Geom& g = fp.g;
  double* G = static_cast<double*>(scratch);
  size_t ds = 0;
  cudaError_t e = set_attrs<T>(g, &ds);
  if (e != cudaSuccess) return e;
  const bool r3 = g.dec3 && rec3_enabled();
#define MGRX_REC(TI, MT)                                                                               \
  if (!r3 && g.tile_rows == TI && (MT == kWideBound) == (g.threads > kPlaneMaxThreads))              \
    MGRX_LAUNCH(ex, "f3_rec_plane", pdl_launch(k_f3_rec_plane<T, TI, MT>, dim3(g.grid), dim3(g.threads), ds, \
                                               ex.s, !ex.prof, shell, G, g));
  MGRX_REC(4, kPlaneMaxThreads)
  MGRX_REC(2, kPlaneMaxThreads)
  MGRX_REC(4, kWideBound)
  MGRX_REC(2, kWideBound)
#undef MGRX_REC
  if (r3) {
    const F3Geom gd = dec3_geom(g);
    MGRX_LAUNCH(ex, "f3_rec_plane", pdl_launch(k_f3_rec_plane<T, 4, kPlaneMaxThreads, 3>, dim3(gd.grid),
                                               dim3(gd.threads), plane_smem3r<T>(gd), ex.s, !ex.prof, shell, G, gd));
  }
  row_col1(G, g, th, ex);
  return cudaGetLastError();
}

// The sequential part: axis-0 solve + coarse -= z, then interpolation.
template <typename T>
cudaError_t fused3d_recompose_finish(const T* shell, T* coarse, T* fine, void* scratch, const Fused3DPlan& fp,
                                     const ThomasLevel& th, const Exec& ex) {
  const F3Geom& g = fp.g;
  double* G = static_cast<double*>(scratch);
  launch_col<T>(G, coarse, -1.0, g, 0, th.w[0], th.inv_d[0], ex, toep_enabled());
  cudaError_t e = launch_interp<T>(shell, coarse, fine, g, ex);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <typename T>
cudaError_t fused3d_recompose_level(const T* shell, T* coarse, T* fine, void* scratch, const LevelGeom&,
                                    const Fused3DPlan& fp, const ThomasLevel& th, const Exec& ex) {
  cudaError_t e = fused3d_recompose_correction<T>(shell, scratch, fp, th, ex);
  if (e != cudaSuccess) return e;
  return fused3d_recompose_finish<T>(shell, coarse, fine, scratch, fp, th, ex);
}

// ------------------------------------------------------------ slab mode
// Chunking of a slab of K coarse planes (the cost model of fused3d_plan).
static F3Geom slab_geom(const F3Geom& g0, int64_t k0, int64_t k1) {
  F3Geom g = g0;
  g.a_base = k0;
  g.a_end = k1;
  const int64_t K = k1 - k0;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (nsm <= 0) nsm = kNumSMs;
  const int64_t ctas = int64_t(nsm) * g.ctas_per_sm;
  int64_t chunk = 1;
  double best = 1e300;
  for (int64_t c = 1; c <= 32 && c <= K; ++c) {
    const int64_t units = ((K + c - 1) / c) * g.ntile1;
    const double cost = double((units + ctas - 1) / ctas) * double(2 * c + 6);
    if (cost < best - 1e-9) {
      best = cost;
      chunk = c;
    }
  }
  g.chunk = chunk;
  g.units = int(((K + chunk - 1) / chunk) * g.ntile1);
  g.grid = g.units;
  return g;
}

template <typename T>
cudaError_t fused3d_slab_dec_plane(const T* blk, T* shell, T* coarse, double* G, const Fused3DPlan& fp, int64_t k0,
                                   int64_t k1, const Exec& ex) {
  if (k1 <= k0) return cudaSuccess;
  const F3Geom g = slab_geom(fp.g, k0, k1);
  size_t ds = 0;
  cudaError_t e = set_attrs<T>(g, &ds);
  if (e != cudaSuccess) return e;
  // ex.nonfinite: the finiteness check rides on this pass (the variant with CF)
  const bool cf = ex.nonfinite != nullptr;
  F3Geom gc = g;
  gc.nonfinite = ex.nonfinite;
#define MGRX_DEC(TI, MT)                                                                                      \
  if (!g.dec3 && g.tile_rows == TI && (MT == kWideBound) == (g.threads > kPlaneMaxThreads)) {               \
    if (cf) {                                                                                                 \
      e = cudaFuncSetAttribute(k_f3_dec_plane<T, TI, MT, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               int(ds));                                                                      \
      if (e != cudaSuccess) return e;                                                                         \
      MGRX_LAUNCH(ex, "f3_dec_plane", pdl_launch(k_f3_dec_plane<T, TI, MT, 0, true>, dim3(g.grid), dim3(g.threads), \
                                                 ds, ex.s, !ex.prof, blk, shell, coarse, G, gc));             \
    } else {                                                                                                  \
      MGRX_LAUNCH(ex, "f3_dec_plane", pdl_launch(k_f3_dec_plane<T, TI, MT>, dim3(g.grid), dim3(g.threads), ds,  \
                                                 ex.s, !ex.prof, blk, shell, coarse, G, g));                  \
    }                                                                                                         \
  }
  MGRX_DEC(4, kPlaneMaxThreads)
  MGRX_DEC(2, kPlaneMaxThreads)
  MGRX_DEC(4, kWideBound)
  MGRX_DEC(2, kWideBound)
#undef MGRX_DEC
  if (g.dec3)
    MGRX_LAUNCH(ex, "f3_dec_plane", pdl_launch(k_f3_dec_plane<T, 4, kPlaneMaxThreads, 3>, dim3(g.grid), dim3(g.threads),
                                               plane_smem3<T>(g), ex.s, !ex.prof, blk, shell, coarse, G, g));
  return cudaGetLastError();
}

template <typename T>
cudaError_t fused3d_slab_rec_plane(const T* shell, double* G, const Fused3DPlan& fp, int64_t k0, int64_t k1,
                                   const Exec& ex) {
  if (k1 <= k0) return cudaSuccess;
  const F3Geom g = slab_geom(fp.g, k0, k1);
  size_t ds = 0;
  cudaError_t e = set_attrs<T>(g, &ds);
  if (e != cudaSuccess) return e;
#define MGRX_REC(TI, MT)                                                                               \
  if (g.tile_rows == TI && (MT == kWideBound) == (g.threads > kPlaneMaxThreads))                      \
    MGRX_LAUNCH(ex, "f3_rec_plane", pdl_launch(k_f3_rec_plane<T, TI, MT>, dim3(g.grid), dim3(g.threads), ds, \
                                               ex.s, !ex.prof, shell, G, g));
  MGRX_REC(4, kPlaneMaxThreads)
  MGRX_REC(2, kPlaneMaxThreads)
  MGRX_REC(4, kWideBound)
  MGRX_REC(2, kWideBound)
#undef MGRX_REC
  return cudaGetLastError();
}

cudaError_t fused3d_slab_inplane(double* G, const Fused3DPlan& fp, const ThomasLevel& th, int64_t k0, int64_t k1,
                                 const Exec& ex) {
  if (k1 <= k0) return cudaSuccess;
  F3Geom gs = fp.g;
  gs.m0 = k1 - k0;
  double* Gs = G + k0 * fp.g.m1 * fp.g.m2;
  launch_row(Gs, gs, th.w[2], th.inv_d[2], ex, toep_enabled());
  launch_col<float>(Gs, static_cast<float*>(nullptr), 0.0, gs, 1, th.w[1], th.inv_d[1], ex, toep_enabled());
  return cudaGetLastError();
}

// Thomas (uniform ThomasAux) along the middle axis of a [outer][m][inner]
// fp64 array (inner > 1: the segmented column pass) or along the rows of a
// [outer][m] array (inner == 1: the row pass), in place.
cudaError_t f3_axis_solve(double* y, int64_t outer, int64_t m, int64_t inner, const double* w, const double* id,
                          const Exec& ex) {
  if (m > kColMaxM || m < 2 || outer <= 0 || inner <= 0) return cudaErrorNotSupported;
  F3Geom g;
  if (inner == 1) {
    g.m0 = outer;
    g.m1 = 1;
    g.m2 = m;
    launch_row(y, g, w, id, ex, toep_enabled());
  } else {
    g.m0 = outer;
    g.m1 = m;
    g.m2 = inner;
    launch_col<float>(y, static_cast<float*>(nullptr), 0.0, g, 1, w, id, ex, toep_enabled());
  }
  return cudaGetLastError();
}

// Axis-0 Thomas (uniform ThomasAux) of every column of a [m0][inner] fp64
// array, in place, by the segmented column pass (general path, auto mode):
// one read and one write instead of the per-line recurrence's two of each.
cudaError_t f3_axis0_solve(double* y, int64_t m0, int64_t inner, const double* w, const double* id,
                           const Exec& ex) {
  if (m0 > kColMaxM || m0 < 2 || inner <= 0) return cudaErrorNotSupported;
  F3Geom g;
  g.m0 = m0;
  g.m1 = 1;
  g.m2 = inner;
  launch_col<float>(y, static_cast<float*>(nullptr), 0.0, g, 0, w, id, ex, toep_enabled());
  return cudaGetLastError();
}

cudaError_t fused3d_slab_axis0(double* Gt, int64_t width, const Fused3DPlan& fp, const ThomasLevel& th,
                               const Exec& ex) {
  if (width <= 0) return cudaSuccess;
  // a [m0][width] block is the axis-0 layout of a volume with m1 = 1, m2 = width
  F3Geom gs = fp.g;
  gs.m1 = 1;
  gs.m2 = width;
  launch_col<float>(Gt, static_cast<float*>(nullptr), 0.0, gs, 0, th.w[0], th.inv_d[0], ex, toep_enabled());
  return cudaGetLastError();
}

template <typename T>
cudaError_t fused3d_slab_interp(const T* shell, const T* coarse, T* fine, const Fused3DPlan& fp, int64_t p0, int64_t p1,
                                const Exec& ex) {
  if (p1 <= p0) return cudaSuccess;
  F3Geom g = fp.g;
  g.p_base = p0;
  g.p_end = p1;
  return launch_interp<T>(shell, coarse, fine, g, ex);
}


// ------------------------------------------------------------- slab K-pack
// Column blocks of a rows x pitch fp64 array, back to back (block q is rows
// x (cb[q+1] - cb[q]) row-major at rows * (cb[q] - cb[0])): the send buffer
// of slab mode's transpose (all-to-all), and its inverse for the way back.
struct PackParts {
  int64_t cb[257];
  int n;
};
template <bool UNPACK>
__global__ void __launch_bounds__(256) k_slab_pack(const double* __restrict__ src, double* __restrict__ dst,
                                                   int64_t rows, int64_t pitch, const PackParts pp) {
  const int64_t c0 = pp.cb[0], width = pp.cb[pp.n] - c0;
  const int64_t total = rows * width;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / width, c = c0 + (i - r * width);  // (row, column) of the strided array
    int q = 0;
    while (c >= pp.cb[q + 1]) ++q;
    const int64_t w = pp.cb[q + 1] - pp.cb[q];
    const int64_t pk = rows * (pp.cb[q] - c0) + r * w + (c - pp.cb[q]);
    if (UNPACK)
      dst[r * pitch + c] = src[pk];
    else
      dst[pk] = src[r * pitch + c];
  }
}

cudaError_t slab_pack(const double* src, int64_t rows, int64_t pitch, const uint64_t* cb, int nparts, double* dst,
                      bool unpack, const Exec& ex) {
  PackParts pp;
  pp.n = nparts;
  for (int q = 0; q <= nparts; ++q) pp.cb[q] = int64_t(cb[q]);
  const int64_t total = rows * (pp.cb[nparts] - pp.cb[0]);
  if (total <= 0) return cudaSuccess;
  const int grid = grid_for(total, 256, 8);
  if (unpack)
    MGRX_LAUNCH(ex, "slab_unpack", k_slab_pack<true><<<grid, 256, 0, ex.s>>>(src, dst, rows, pitch, pp));
  else
    MGRX_LAUNCH(ex, "slab_pack", k_slab_pack<false><<<grid, 256, 0, ex.s>>>(src, dst, rows, pitch, pp));
  return cudaGetLastError();
}

#define MGRX_INST(T)                                                                                     \
  template cudaError_t fused3d_decompose_level<T>(const T*, T*, T*, void*, const LevelGeom&, const Fused3DPlan&, \
                                                  const ThomasLevel&, const Exec&);                      \
  template cudaError_t fused3d_recompose_level<T>(const T*, T*, T*, void*, const LevelGeom&, const Fused3DPlan&, \
                                                  const ThomasLevel&, const Exec&);                      \
  template cudaError_t fused3d_recompose_correction<T>(const T*, void*, const Fused3DPlan&, const ThomasLevel&,   \
                                                       const Exec&);                                     \
  template cudaError_t fused3d_recompose_finish<T>(const T*, T*, T*, void*, const Fused3DPlan&, const ThomasLevel&, \
                                                   const Exec&);
MGRX_INST(float)
MGRX_INST(double)
#define MGRX_INST_SLAB(T)                                                                                        \
  template cudaError_t fused3d_slab_dec_plane<T>(const T*, T*, T*, double*, const Fused3DPlan&, int64_t, int64_t, \
                                                 const Exec&);                                                   \
  template cudaError_t fused3d_slab_rec_plane<T>(const T*, double*, const Fused3DPlan&, int64_t, int64_t,         \
                                                 const Exec&);                                                   \
  template cudaError_t fused3d_slab_interp<T>(const T*, const T*, T*, const Fused3DPlan&, int64_t, int64_t, const Exec&);
MGRX_INST_SLAB(float)
MGRX_INST_SLAB(double)
#undef MGRX_INST_SLAB
#undef MGRX_INST

}  // namespace mgrx_b200
