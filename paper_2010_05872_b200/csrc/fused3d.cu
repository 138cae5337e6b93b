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
//                            3-deep shared-memory ring), computes every
//                            coefficient (same corner order as
//                            update_coefficients), writes the shell straight
//                            into its level-centric position and the nodal
//                            values into the compact coarse block, and
//                            accumulates the load vector L0 L1 L2 c of the
//                            fp64 component in registers/shared memory; once
//                            a coarse plane is complete its rows are solved
//                            along axis 2 (warp-parallel Thomas) and written
//                            to the fp64 volume G.
//              f3_col (axis 1)  Thomas along axis 1 on G, in place.
//              f3_col (axis 0)  Thomas along axis 0 + coarse += z.
//   recompose  f3_rec_plane  same load-vector accumulation, reading the
//                            component from the shell;
//              f3_col x2     as above, coarse -= z;
//              f3_rec_interp fine block = coarse nodes + shell + prediction.
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

#include "fused3d.h"

namespace mgrx_b200 {

namespace {

constexpr int kF3MaxThreads = 640;  // plane passes: one thread per coarse column (m2 <= 640)
constexpr int kColMaxM = 640;       // column passes: register-resident columns up to this length
// column-pass block: 32 columns x ceil(m / LS) segments of LS registers;
// LS = 16 for m <= 320 and LS = 32 for m <= 640, so at most 20 segments
template <int LS>
constexpr int kColMaxThreads = 640;

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

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
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

// ---------------------------------------------- warp-parallel Thomas (row)
// Solves M z = f in place for one row x[0..m) held in shared memory with the
// reference's factors (ThomasAux, transform.hpp:25-44): lane segments run the
// forward / backward recurrences locally, an affine scan across lanes joins
// them (exact algebra; rounding differs from the sequential sweep).
__device__ void warp_thomas_row(double* x, int m, const double* __restrict__ w, const double* __restrict__ inv_d) {
  const int lane = threadIdx.x & 31;
  const int seg = (m + 31) >> 5;
  const int s0 = min(m, lane * seg), s1 = min(m, s0 + seg);
  // forward: y_i = x_i - w_i y_{i-1}
  double yl = 0.0, mu = 1.0;
  for (int i = s0; i < s1; ++i) {
    const double wi = w[i];
    yl = x[i] - wi * yl;
    mu = -wi * mu;
    x[i] = yl;
  }
  double A = (s1 > s0) ? yl : 0.0, B = (s1 > s0) ? mu : 1.0;  // y_end = A + B * y_in
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double a2 = __shfl_up_sync(0xffffffffu, A, off);
    const double b2 = __shfl_up_sync(0xffffffffu, B, off);
    if (lane >= off) {
      A = A + B * a2;
      B = B * b2;
    }
  }
  double cin = __shfl_up_sync(0xffffffffu, A, 1);
  if (lane == 0) cin = 0.0;
  mu = 1.0;
  for (int i = s0; i < s1; ++i) {
    mu = -w[i] * mu;
    x[i] = x[i] + mu * cin;
  }
  // backward: z_i = (y_i - kOff z_{i+1}) inv_d_i, z_m = 0
  double xl = 0.0, nu = 1.0;
  for (int i = s1 - 1; i >= s0; --i) {
    const double id = inv_d[i];
    xl = (x[i] - kOff * xl) * id;
    nu = -kOff * id * nu;
    x[i] = xl;
  }
  A = (s1 > s0) ? xl : 0.0;
  B = (s1 > s0) ? nu : 1.0;  // z_start = A + B * z_in(right)
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double a2 = __shfl_down_sync(0xffffffffu, A, off);
    const double b2 = __shfl_down_sync(0xffffffffu, B, off);
    if (lane + off < 32) {
      A = A + B * a2;
      B = B * b2;
    }
  }
  double cr = __shfl_down_sync(0xffffffffu, A, 1);
  if (lane == 31) cr = 0.0;
  nu = 1.0;
  for (int i = s1 - 1; i >= s0; --i) {
    nu = -kOff * inv_d[i] * nu;
    x[i] = x[i] + nu * cr;
  }
}

// Shell offset of reordered row (r0, r1) of a 3-D level block
// (pack_level_centric, reorder.hpp:180-215).
__device__ __forceinline__ int64_t shell_row_start(const F3Geom& g, int64_t r0, int64_t r1) {
  const int64_t before = (r0 < g.m0) ? r0 * g.m1 + min(r1, g.m1) : g.m0 * g.m1;
  return (r0 * g.n1 + r1) * g.n2 - before * g.m2;
}

__device__ __forceinline__ int64_t reord(int64_t j, int64_t m) { return (j & 1) ? m + (j >> 1) : (j >> 1); }

struct UnitRange {
  int64_t a0, a1, b0, b1;  // coarse planes [a0,a1), coarse rows [b0,b1)
  int64_t plo, phi;        // fine planes touched, inclusive
  int64_t rlo, rhi;        // fine rows touched, inclusive
};

__device__ __forceinline__ UnitRange unit_range(const F3Geom& g, int u) {
  UnitRange r;
  const int chunk = u / g.ntile1, tile = u - chunk * g.ntile1;
  r.a0 = int64_t(chunk) * g.chunk;
  r.a1 = min(g.m0, r.a0 + g.chunk);
  r.b0 = int64_t(tile) * g.tile_rows;
  r.b1 = min(g.m1, r.b0 + g.tile_rows);
  r.plo = max(int64_t(0), 2 * r.a0 - 2);
  r.phi = min(g.n0 - 1, 2 * r.a1);
  r.rlo = max(int64_t(0), 2 * r.b0 - 2);
  r.rhi = min(g.n1 - 1, 2 * r.b1);
  return r;
}

// --------------------------------------------------------- plane kernels
// Shared-memory layout shared by the decompose and recompose plane passes.
template <typename T, int TI1>
struct PlaneSmem {
  static constexpr int kRows = 2 * TI1 + 3;
  static __host__ __device__ size_t raw_bytes(int64_t n2) {
    return (size_t(kRows) * size_t(n2) * sizeof(T) + 256 + 127) / 128 * 128;
  }
  static __host__ __device__ size_t nsd_elems(int64_t m2) { return size_t(TI1 + 2) * size_t(m2); }
  static __host__ __device__ size_t acc_elems(int64_t m2) { return size_t(TI1) * size_t(m2); }
  static __host__ __device__ size_t bytes(int64_t n2, int64_t m2, bool dec) {
    size_t b = 3 * raw_bytes(n2);
    if (dec) b += 2 * nsd_elems(m2) * 8;
    b += 3 * acc_elems(m2) * 8;
    b += 2 * size_t(n2 + 8) * 8;  // crow double buffer
    b += 2 * size_t(m2) * 8;      // Thomas tables axis 2
    b += 64;                      // mbarriers + unit slot
    return b;
  }
};

// Component value of fine node (p, j1, j2) in decompose (coefficient of the
// reordered level block, transform.hpp:216-304, or 0 on a nodal point).
// Corners come from the fp64 nodal planes `nsA` (plane p-1 or p) and `nsB`
// (plane p+1); rows of ns* are the even fine rows from rlo, columns the
// coarse i2.  Returns the T-rounded coefficient (as double) and sets *nodal.
template <typename T>
__device__ __forceinline__ double dec_coef(const F3Geom& g, bool p_odd, bool p_has_right, const double* nsP,
                                           const double* nsN, int64_t m2s, int64_t j1, int64_t rlo, int64_t j2,
                                           double raw, bool* nodal) {
  const bool o1 = j1 & 1, o2 = j2 & 1;
  *nodal = !(p_odd || o1 || o2);
  if (*nodal) return 0.0;
  // corner index pieces
  const int64_t rl = ((o1 ? j1 - 1 : j1) - rlo) >> 1;            // left/own even row
  const int64_t rr = o1 ? ((j1 + 1 < g.n1) ? rl + 1 : rl) : rl;   // right even row
  const int64_t cl = o2 ? (j2 - 1) >> 1 : j2 >> 1;                // left/own coarse column
  const int64_t cr = o2 ? ((j2 + 1 < g.n2) ? cl + 1 : cl) : cl;   // right coarse column
  const double* pl = nsP;                                         // left plane (or own)
  const double* pr = p_odd ? (p_has_right ? nsN : nsP) : nsP;     // right plane
  double sum;
  // set axes ascending (0,1,2); cmask bit b <-> b-th set axis; cmask ascending
  if (p_odd) {
    if (o1) {
      if (o2) {  // k = 3
        sum = pl[rl * m2s + cl];
        sum += pr[rl * m2s + cl];
        sum += pl[rr * m2s + cl];
        sum += pr[rr * m2s + cl];
        sum += pl[rl * m2s + cr];
        sum += pr[rl * m2s + cr];
        sum += pl[rr * m2s + cr];
        sum += pr[rr * m2s + cr];
        sum *= 0.125;
      } else {  // axes 0,1
        sum = pl[rl * m2s + cl];
        sum += pr[rl * m2s + cl];
        sum += pl[rr * m2s + cl];
        sum += pr[rr * m2s + cl];
        sum *= 0.25;
      }
    } else if (o2) {  // axes 0,2
      sum = pl[rl * m2s + cl];
      sum += pr[rl * m2s + cl];
      sum += pl[rl * m2s + cr];
      sum += pr[rl * m2s + cr];
      sum *= 0.25;
    } else {  // axis 0
      sum = pl[rl * m2s + cl];
      sum += pr[rl * m2s + cl];
      sum *= 0.5;
    }
  } else {
    if (o1) {
      if (o2) {  // axes 1,2
        sum = pl[rl * m2s + cl];
        sum += pl[rr * m2s + cl];
        sum += pl[rl * m2s + cr];
        sum += pl[rr * m2s + cr];
        sum *= 0.25;
      } else {  // axis 1
        sum = pl[rl * m2s + cl];
        sum += pl[rr * m2s + cl];
        sum *= 0.5;
      }
    } else {  // axis 2
      sum = pl[rl * m2s + cl];
      sum += pl[rl * m2s + cr];
      sum *= 0.5;
    }
  }
  return double(to_t<T>(raw - sum));
}

// One fine row's contribution: L2 restriction of the component row in
// crow[0..n2) at coarse column i2 (load_entry along axis 2).
__device__ __forceinline__ double restrict_row(const double* crow, int64_t i2, const F3Geom& g) {
  const int64_t c = 2 * i2;
  double acc = 0.0;
  if (i2 >= 1) {
    acc += kW12 * crow[c - 2];
    acc += 0.5 * crow[c - 1];
  }
  acc += ((i2 == 0 || i2 + 1 == g.m2) ? kW5_12 : kW5_6) * crow[c];
  if (c + 1 < g.n2) acc += 0.5 * crow[c + 1];
  if (c + 2 < g.n2) acc += kW12 * crow[c + 2];
  return acc;
}

// Adds the plane's restricted rows Q[] into the coarse-plane accumulators
// (L0 along axis 0, terms in stencil order) and finishes coarse planes:
// Thomas along axis 2 per row, store to G.
template <int TI1>
__device__ __forceinline__ void plane_epilogue(const F3Geom& g, const UnitRange& ur, int64_t p, const double* Q,
                                               double* acc, const double* tw2, const double* tid2, double* G,
                                               int64_t i2, bool active) {
  const int64_t TR = ur.b1 - ur.b0;
  const size_t accsz = size_t(TI1) * size_t(g.m2);
  // target coarse planes i0 with |p - 2 i0| <= 2, i0 in [a0, a1)
  const int64_t ilo = max(ur.a0, (p - 1) >> 1), ihi = min(ur.a1 - 1, (p + 2) >> 1);
  if (active) {
    for (int64_t i0 = ilo; i0 <= ihi; ++i0) {
      const int k = int(p - 2 * i0);
      if (k < -2 || k > 2) continue;
      const double wt = load_w(k, i0, g.m0);
      double* a = acc + size_t(i0 % 3) * accsz;
      const bool first = (p == max(int64_t(0), 2 * i0 - 2));
#pragma unroll
      for (int r = 0; r < TI1; ++r)
        if (r < TR) {
          double* cell = a + size_t(r) * g.m2 + i2;
          *cell = first ? wt * Q[r] : *cell + wt * Q[r];
        }
    }
  }
  // coarse plane i0 = (p-2)/2 completes at p = 2 i0 + 2, or at the last fine plane
  int64_t done_lo = -1, done_hi = -2;
  if (p == g.n0 - 1) {
    done_lo = max(ur.a0, (p - 2 + 1) >> 1);
    done_hi = ur.a1 - 1;
  } else if (!(p & 1) && p >= 2) {
    done_lo = done_hi = (p - 2) >> 1;
  }
  done_lo = max(done_lo, ur.a0);
  done_hi = min(done_hi, ur.a1 - 1);
  if (done_lo > done_hi) return;
  __syncthreads();
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int64_t i0 = done_lo; i0 <= done_hi; ++i0) {
    double* a = acc + size_t(i0 % 3) * accsz;
    for (int r = warp; r < TR; r += nwarps) warp_thomas_row(a + size_t(r) * g.m2, int(g.m2), tw2, tid2);
  }
  __syncthreads();
  for (int64_t i0 = done_lo; i0 <= done_hi; ++i0) {
    const double* a = acc + size_t(i0 % 3) * accsz;
    if (active)
      for (int r = 0; r < TR; ++r) G[((i0 * g.m1) + ur.b0 + r) * g.m2 + i2] = a[size_t(r) * g.m2 + i2];
  }
}

// Decompose plane pass. One thread per coarse column i2 (its fine pair
// 2 i2, 2 i2 + 1); persistent CTAs take (axis-0 chunk, axis-1 tile) units.
template <typename T, int TI1>
__global__ void __launch_bounds__(kF3MaxThreads, 1)
    k_f3_dec_plane(const T* __restrict__ blk, T* __restrict__ shell, T* __restrict__ coarse, double* __restrict__ G,
                   const double* __restrict__ w2g, const double* __restrict__ id2g, int* __restrict__ counter,
                   const F3Geom g) {
  using SM = PlaneSmem<T, TI1>;
  extern __shared__ __align__(128) unsigned char smem[];
  const size_t rawb = SM::raw_bytes(g.n2);
  unsigned char* raw = smem;
  double* nsd = reinterpret_cast<double*>(smem + 3 * rawb);
  double* acc = nsd + 2 * SM::nsd_elems(g.m2);
  double* crow = acc + 3 * SM::acc_elems(g.m2);
  double* tw2 = crow + 2 * (g.n2 + 8);
  double* tid2 = tw2 + g.m2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(tid2 + g.m2);
  int* unit_slot = reinterpret_cast<int*>(bars + 4);

  const int tid = threadIdx.x;
  const int64_t i2 = tid;
  const bool active = i2 < g.m2;
  for (int64_t i = tid; i < g.m2; i += blockDim.x) {
    tw2[i] = w2g[i];
    tid2[i] = id2g[i];
  }
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&bars[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase[3] = {0, 0, 0};
  const int64_t m2s = g.m2;

  for (;;) {
    if (tid == 0) *unit_slot = atomicAdd(counter, 1);
    __syncthreads();
    const int u = *unit_slot;
    if (u >= g.units) break;
    const UnitRange ur = unit_range(g, u);
    const int64_t R = ur.rhi - ur.rlo + 1;
    int lead[3] = {0, 0, 0};
    // issue one plane into ring slot (p % 3)
    auto issue = [&](int64_t p) {
      if (tid == 0) {
        const char* src;
        uint32_t bytes;
        int ld;
        bulk_span<T>(blk, (p * g.n1 + ur.rlo) * g.n2, R * g.n2, &src, &bytes, &ld);
        uint64_t* bar = &bars[p % 3];
        fence_proxy_async();
        mbar_expect_tx(bar, bytes);
        bulk_g2s(raw + size_t(p % 3) * rawb, src, bytes, bar);
      }
    };
    auto lead_of = [&](int64_t p) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(blk + (p * g.n1 + ur.rlo) * g.n2);
      return int((a & 15) / sizeof(T));
    };
    issue(ur.plo);
    if (ur.plo + 1 <= ur.phi) issue(ur.plo + 1);
    for (int b = 0; b < 3; ++b) lead[b] = 0;

    int64_t ready = ur.plo - 1;  // planes waited for so far (in order)
    for (int64_t p = ur.plo; p <= ur.phi; ++p) {
      const bool p_odd = p & 1;
      const bool has_right = p_odd && (p + 1 <= g.n0 - 1);
      // wait for plane p (and p + 1 when p is odd)
      const int64_t need = has_right ? p + 1 : p;
      while (ready < need) {
        ++ready;
        mbar_wait(&bars[ready % 3], phase[ready % 3]);
        phase[ready % 3] ^= 1;
      }
      const T* rp = reinterpret_cast<const T*>(raw + size_t(p % 3) * rawb) + lead_of(p);
      // nodal fp64 copies of even planes: slot (plane/2) % 2
      auto extract = [&](int64_t q) {
        const T* rq = reinterpret_cast<const T*>(raw + size_t(q % 3) * rawb) + lead_of(q);
        double* ns = nsd + size_t((q >> 1) & 1) * SM::nsd_elems(g.m2);
        if (active)
          for (int64_t j1 = ur.rlo; j1 <= ur.rhi; j1 += 2) ns[((j1 - ur.rlo) >> 1) * m2s + i2] =
              double(rq[(j1 - ur.rlo) * g.n2 + 2 * i2]);
      };
      if (p == ur.plo) extract(p);  // first plane of the unit is even
      if (has_right) extract(p + 1);
      __syncthreads();
      // the slot of plane p-1 (odd) / p-2 is free: prefetch p + 2
      if (p + 2 <= ur.phi) issue(p + 2);
      const double* nsP = nsd + size_t(((p_odd ? p - 1 : p) >> 1) & 1) * SM::nsd_elems(g.m2);
      const double* nsN = nsd + size_t(((p + 1) >> 1) & 1) * SM::nsd_elems(g.m2);
      const bool own_p = p >= 2 * ur.a0 && p < 2 * ur.a1;
      const int64_t r0 = reord(p, g.m0);

      double Q[TI1];
#pragma unroll
      for (int r = 0; r < TI1; ++r) Q[r] = 0.0;
      // fine rows relative to 2 b0 - 2 (compile-time unrolled for static Q indexing)
#pragma unroll
      for (int jr = 0; jr < 2 * TI1 + 3; ++jr) {
        const int64_t j1 = 2 * ur.b0 - 2 + jr;
        if (j1 < ur.rlo || j1 > ur.rhi) continue;  // uniform across the CTA
        double* cr = crow + (jr & 1) * (g.n2 + 8);
        const bool own_row = own_p && j1 >= 2 * ur.b0 && j1 < 2 * ur.b1;
        if (active) {
          const T* rr = rp + (j1 - ur.rlo) * g.n2;
          const int64_t r1 = reord(j1, g.m1);
          const int64_t rs = own_row ? shell_row_start(g, r0, r1) : 0;
          const bool inside = r0 < g.m0 && r1 < g.m1;
          // even node 2 i2
          {
            const int64_t j2 = 2 * i2;
            const T rawv = rr[j2];
            bool nodal;
            const double c = dec_coef<T>(g, p_odd, has_right, nsP, nsN, m2s, j1, ur.rlo, j2, double(rawv), &nodal);
            cr[j2] = c;
            if (own_row) {
              if (nodal)
                coarse[((p >> 1) * g.m1 + (j1 >> 1)) * g.m2 + i2] = rawv;
              else
                shell[rs + i2] = to_t<T>(c);
            }
          }
          if (2 * i2 + 1 < g.n2) {
            const int64_t j2 = 2 * i2 + 1;
            bool nodal;
            const double c = dec_coef<T>(g, p_odd, has_right, nsP, nsN, m2s, j1, ur.rlo, j2, double(rr[j2]), &nodal);
            cr[j2] = c;
            if (own_row) shell[rs + (inside ? 0 : g.m2) + i2] = to_t<T>(c);
          }
        }
        __syncthreads();
        if (active) {
          const double h = restrict_row(cr, i2, g);
          // rows 2 i1 + k, k in [-2, 2], of coarse rows i1 in [b0, b1)
#pragma unroll
          for (int k = -2; k <= 2; ++k) {
            if (((jr - 2 - k) & 1) != 0) continue;
            const int ir = (jr - 2 - k) / 2;  // i1 - b0
            if (ir < 0 || ir >= TI1) continue;
            const int64_t i1 = ur.b0 + ir;
            if (i1 >= ur.b1) continue;
            Q[ir] += load_w(k, i1, g.m1) * h;
          }
        }
      }
      plane_epilogue<TI1>(g, ur, p, Q, acc, tw2, tid2, G, i2, active);
      // make sure every thread is done with slot p before it is refilled
      __syncthreads();
    }
  }
}

// Recompose plane pass: the same load-vector accumulation with the
// component read from the level's shell (coefficients; 0 on nodal points).
// Per fine plane the tile's shell rows form two contiguous runs (even fine
// rows, odd fine rows), fetched with two bulk copies.
template <typename T, int TI1>
__global__ void __launch_bounds__(kF3MaxThreads, 1)
    k_f3_rec_plane(const T* __restrict__ shell, double* __restrict__ G, const double* __restrict__ w2g,
                   const double* __restrict__ id2g, int* __restrict__ counter, const F3Geom g) {
  using SM = PlaneSmem<T, TI1>;
  extern __shared__ __align__(128) unsigned char smem[];
  const size_t rawb = SM::raw_bytes(g.n2);
  unsigned char* raw = smem;
  double* acc = reinterpret_cast<double*>(smem + 3 * rawb);
  double* crow = acc + 3 * SM::acc_elems(g.m2);
  double* tw2 = crow + 2 * (g.n2 + 8);
  double* tid2 = tw2 + g.m2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(tid2 + g.m2);
  int* unit_slot = reinterpret_cast<int*>(bars + 4);

  const int tid = threadIdx.x;
  const int64_t i2 = tid;
  const bool active = i2 < g.m2;
  for (int64_t i = tid; i < g.m2; i += blockDim.x) {
    tw2[i] = w2g[i];
    tid2[i] = id2g[i];
  }
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&bars[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase[3] = {0, 0, 0};

  for (;;) {
    if (tid == 0) *unit_slot = atomicAdd(counter, 1);
    __syncthreads();
    const int u = *unit_slot;
    if (u >= g.units) break;
    const UnitRange ur = unit_range(g, u);
    // even fine rows of the tile: r1 in [rlo/2, rhi/2]; odd: r1 in [m1 + rlo/2, m1 + (rhi-1)/2]
    const int64_t e_lo = ur.rlo >> 1, e_hi = ur.rhi >> 1;
    const int64_t o_lo = (ur.rlo + 1) >> 1, o_hi = (ur.rhi - 1) >> 1;  // (j1 - 1) / 2 range
    auto runs = [&](int64_t p, int64_t* s_even, int64_t* l_even, int64_t* s_odd, int64_t* l_odd) {
      const int64_t r0 = reord(p, g.m0);
      *s_even = shell_row_start(g, r0, e_lo);
      *l_even = shell_row_start(g, r0, e_hi + 1) - *s_even;
      if (o_hi >= o_lo) {
        *s_odd = shell_row_start(g, r0, g.m1 + o_lo);
        *l_odd = shell_row_start(g, r0, g.m1 + o_hi + 1) - *s_odd;
      } else {
        *s_odd = 0;
        *l_odd = 0;
      }
    };
    auto issue = [&](int64_t p) {
      if (tid == 0) {
        int64_t se, le, so, lo;
        runs(p, &se, &le, &so, &lo);
        const char *src0, *src1;
        uint32_t b0, b1 = 0;
        int ld0, ld1;
        bulk_span<T>(shell, se, le, &src0, &b0, &ld0);
        if (lo > 0) bulk_span<T>(shell, so, lo, &src1, &b1, &ld1);
        uint64_t* bar = &bars[p % 3];
        unsigned char* dst = raw + size_t(p % 3) * rawb;
        fence_proxy_async();
        mbar_expect_tx(bar, b0 + b1);
        bulk_g2s(dst, src0, b0, bar);
        if (lo > 0) bulk_g2s(dst + ((b0 + 127) & ~127u), src1, b1, bar);
      }
    };
    issue(ur.plo);
    if (ur.plo + 1 <= ur.phi) issue(ur.plo + 1);

    for (int64_t p = ur.plo; p <= ur.phi; ++p) {
      mbar_wait(&bars[p % 3], phase[p % 3]);
      phase[p % 3] ^= 1;
      if (p + 2 <= ur.phi) {
        // slot (p+2)%3 held plane p-1, finished at the end of the previous step
        issue(p + 2);
      }
      int64_t se, le, so, lo;
      runs(p, &se, &le, &so, &lo);
      const unsigned char* base = raw + size_t(p % 3) * rawb;
      const T* ev = reinterpret_cast<const T*>(base) + (reinterpret_cast<uintptr_t>(shell + se) & 15) / sizeof(T);
      uint32_t b0 = uint32_t(((reinterpret_cast<uintptr_t>(shell + se + le) + 15) & ~uintptr_t(15)) -
                             (reinterpret_cast<uintptr_t>(shell + se) & ~uintptr_t(15)));
      const T* od = reinterpret_cast<const T*>(base + ((b0 + 127) & ~127u)) +
                    (reinterpret_cast<uintptr_t>(shell + so) & 15) / sizeof(T);
      const bool p_odd = p & 1;
      const int64_t r0 = reord(p, g.m0);

      double Q[TI1];
#pragma unroll
      for (int r = 0; r < TI1; ++r) Q[r] = 0.0;
#pragma unroll
      for (int jr = 0; jr < 2 * TI1 + 3; ++jr) {
        const int64_t j1 = 2 * ur.b0 - 2 + jr;
        if (j1 < ur.rlo || j1 > ur.rhi) continue;
        double* cr = crow + (jr & 1) * (g.n2 + 8);
        if (active) {
          const bool o1 = j1 & 1;
          const int64_t r1 = reord(j1, g.m1);
          const bool inside = r0 < g.m0 && r1 < g.m1;
          // offset of this row inside its run
          const T* row = o1 ? od + (shell_row_start(g, r0, r1) - so) : ev + (shell_row_start(g, r0, r1) - se);
          const int64_t j2 = 2 * i2;
          cr[j2] = (p_odd || o1) ? double(row[i2]) : 0.0;  // even node: coefficient unless nodal
          if (j2 + 1 < g.n2) cr[j2 + 1] = double(row[(inside ? 0 : g.m2) + i2]);
        }
        __syncthreads();
        if (active) {
          const double h = restrict_row(cr, i2, g);
#pragma unroll
          for (int k = -2; k <= 2; ++k) {
            if (((jr - 2 - k) & 1) != 0) continue;
            const int ir = (jr - 2 - k) / 2;
            if (ir < 0 || ir >= TI1) continue;
            const int64_t i1 = ur.b0 + ir;
            if (i1 >= ur.b1) continue;
            Q[ir] += load_w(k, i1, g.m1) * h;
          }
        }
      }
      plane_epilogue<TI1>(g, ur, p, Q, acc, tw2, tid2, G, i2, active);
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------ column pass
// Thomas along axis 0 or 1 of the coarse fp64 volume G (m0 x m1 x m2).
// Columns are consecutive in memory across lanes (32 per block row); each
// column is split over blockDim.y segments of up to LS elements held in
// registers, joined by an affine scan through shared memory.  With `coarse`
// set (axis 0) the result is applied: coarse += sign * z (apply_correction,
// transform.hpp:435-477); otherwise written back to G.
template <typename T, int LS>
__global__ void __launch_bounds__(kColMaxThreads<LS>)
    k_f3_col(double* __restrict__ G, T* __restrict__ coarse, double sign, int64_t ncols, int64_t m, int64_t stride,
             int64_t outer_stride, int64_t inner, const double* __restrict__ w, const double* __restrict__ inv_d) {
  // shared: w[m], inv_d[m], then the scan exchange [2][S][32]
  extern __shared__ double sc[];
  const int lane = threadIdx.x, s = threadIdx.y, S = blockDim.y;
  double* tw = sc;
  double* tid = sc + m;
  double* A = tid + m;
  double* B = A + S * 32;
  for (int64_t i = s * 32 + lane; i < m; i += S * 32) {
    tw[i] = w[i];
    tid[i] = inv_d[i];
  }
  const int64_t col = int64_t(blockIdx.x) * 32 + lane;
  const bool valid = col < ncols;
  // column col -> base offset: (col / inner) * outer_stride + col % inner
  const int64_t base = valid ? (col / inner) * outer_stride + (col % inner) : 0;
  const int64_t seg = (m + S - 1) / S;
  const int s0 = int(min(m, int64_t(s) * seg)), s1 = int(min(m, int64_t(s0) + seg));
  const int len = s1 - s0;
  double v[LS];
  {
    const double* gp = G + base + int64_t(s0) * stride;
#pragma unroll
    for (int k = 0; k < LS; ++k) {
      v[k] = (valid && k < len) ? *gp : 0.0;
      gp += stride;
    }
  }
  __syncthreads();
  // Forward elimination y_i = f_i - w_i y_{i-1} (batched_solve,
  // transform.hpp:117-120): local run from 0 gives the segment's affine map.
  double yl = 0.0, mu = 1.0;
#pragma unroll
  for (int k = 0; k < LS; ++k)
    if (k < len) {
      const double wi = ld_volatile(tw + s0 + k);
      yl = v[k] - wi * yl;
      mu = -wi * mu;
    }
  A[s * 32 + lane] = len > 0 ? yl : 0.0;
  B[s * 32 + lane] = len > 0 ? mu : 1.0;
  __syncthreads();
  double y = 0.0;  // true y_{s0 - 1}
  for (int q = 0; q < s; ++q) y = A[q * 32 + lane] + B[q * 32 + lane] * y;
  __syncthreads();
  // rerun the recurrence from the true carry
#pragma unroll
  for (int k = 0; k < LS; ++k)
    if (k < len) {
      y = v[k] - ld_volatile(tw + s0 + k) * y;
      v[k] = y;
    }
  // Back substitution z_i = (y_i - z_{i+1}/3) / d_i (transform.hpp:121-129).
  double xl = 0.0, nu = 1.0;
#pragma unroll
  for (int k = LS - 1; k >= 0; --k)
    if (k < len) {
      const double id = ld_volatile(tid + s0 + k);
      xl = (v[k] - kOff * xl) * id;
      nu = -kOff * id * nu;
    }
  A[s * 32 + lane] = len > 0 ? xl : 0.0;
  B[s * 32 + lane] = len > 0 ? nu : 1.0;
  __syncthreads();
  double z = 0.0;  // true z_{s1}
  for (int q = S - 1; q > s; --q) z = A[q * 32 + lane] + B[q * 32 + lane] * z;
#pragma unroll
  for (int k = LS - 1; k >= 0; --k)
    if (k < len) {
      z = (v[k] - kOff * z) * ld_volatile(tid + s0 + k);
      v[k] = z;
    }
  if (!valid) return;
  if (coarse) {
    T* c = coarse + base + int64_t(s0) * stride;
#pragma unroll
    for (int k = 0; k < LS; ++k) {
      if (k < len) *c = to_t<T>(double(*c) + sign * v[k]);
      c += stride;
    }
  } else {
    double* gp = G + base + int64_t(s0) * stride;
#pragma unroll
    for (int k = 0; k < LS; ++k) {
      if (k < len) *gp = v[k];
      gp += stride;
    }
  }
}

// ----------------------------------------------------------- interpolate
// add_interpolant + inverse_reorder_level for one fine row tile: one thread
// per coarse column i2 (fine pair), blockIdx.x = fine plane, blockIdx.y =
// group of kRowsPerBlock fine rows.  Corner order as update_coefficients.
template <typename T>
__global__ void __launch_bounds__(1024)
    k_f3_rec_interp(const T* __restrict__ shell, const T* __restrict__ coarse, T* __restrict__ fine, const F3Geom g,
                    int rows_per_block) {
  const int64_t p = blockIdx.x;
  const int64_t i2 = threadIdx.x;
  if (i2 >= g.m2) return;
  const bool p_odd = p & 1;
  const int64_t cp = p >> 1;                                   // left/own coarse plane
  const int64_t cpr = p_odd ? ((p + 1 < g.n0) ? cp + 1 : cp) : cp;  // right coarse plane
  const int64_t r0 = reord(p, g.m0);
  const int64_t j1lo = int64_t(blockIdx.y) * rows_per_block;
  const int64_t j1hi = min(g.n1, j1lo + rows_per_block);
  const int64_t cl = i2, crc = (2 * i2 + 2 < g.n2) ? i2 + 1 : i2;
  const int64_t ps = g.m1 * g.m2;
  for (int64_t j1 = j1lo; j1 < j1hi; ++j1) {
    const bool o1 = j1 & 1;
    const int64_t rl = j1 >> 1, rr = o1 ? ((j1 + 1 < g.n1) ? rl + 1 : rl) : rl;
    const int64_t r1 = reord(j1, g.m1);
    const int64_t rs = shell_row_start(g, r0, r1);
    const bool inside = r0 < g.m0 && r1 < g.m1;
    const T* cL = coarse + cp * ps;
    const T* cR = coarse + cpr * ps;
    T* out = fine + (p * g.n1 + j1) * g.n2;
    // even node 2 i2
    {
      double pred;
      if (p_odd) {
        if (o1) {
          pred = double(__ldg(cL + rl * g.m2 + cl));
          pred += double(__ldg(cR + rl * g.m2 + cl));
          pred += double(__ldg(cL + rr * g.m2 + cl));
          pred += double(__ldg(cR + rr * g.m2 + cl));
          pred *= 0.25;
        } else {
          pred = double(__ldg(cL + rl * g.m2 + cl));
          pred += double(__ldg(cR + rl * g.m2 + cl));
          pred *= 0.5;
        }
        out[2 * i2] = to_t<T>(double(shell[rs + i2]) + pred);
      } else if (o1) {
        pred = double(__ldg(cL + rl * g.m2 + cl));
        pred += double(__ldg(cL + rr * g.m2 + cl));
        pred *= 0.5;
        out[2 * i2] = to_t<T>(double(shell[rs + i2]) + pred);
      } else {
        out[2 * i2] = __ldg(cL + rl * g.m2 + cl);
      }
    }
    if (2 * i2 + 1 < g.n2) {
      double pred;
      if (p_odd) {
        if (o1) {
          pred = double(__ldg(cL + rl * g.m2 + cl));
          pred += double(__ldg(cR + rl * g.m2 + cl));
          pred += double(__ldg(cL + rr * g.m2 + cl));
          pred += double(__ldg(cR + rr * g.m2 + cl));
          pred += double(__ldg(cL + rl * g.m2 + crc));
          pred += double(__ldg(cR + rl * g.m2 + crc));
          pred += double(__ldg(cL + rr * g.m2 + crc));
          pred += double(__ldg(cR + rr * g.m2 + crc));
          pred *= 0.125;
        } else {
          pred = double(__ldg(cL + rl * g.m2 + cl));
          pred += double(__ldg(cR + rl * g.m2 + cl));
          pred += double(__ldg(cL + rl * g.m2 + crc));
          pred += double(__ldg(cR + rl * g.m2 + crc));
          pred *= 0.25;
        }
      } else if (o1) {
        pred = double(__ldg(cL + rl * g.m2 + cl));
        pred += double(__ldg(cL + rr * g.m2 + cl));
        pred += double(__ldg(cL + rl * g.m2 + crc));
        pred += double(__ldg(cL + rr * g.m2 + crc));
        pred *= 0.25;
      } else {
        pred = double(__ldg(cL + rl * g.m2 + cl));
        pred += double(__ldg(cL + rl * g.m2 + crc));
        pred *= 0.5;
      }
      out[2 * i2 + 1] = to_t<T>(double(shell[rs + (inside ? 0 : g.m2) + i2]) + pred);
    }
  }
}

// ------------------------------------------------------------ host side

template <typename T, int TI1>
size_t plane_smem(const F3Geom& g, bool dec) {
  return PlaneSmem<T, TI1>::bytes(g.n2, g.m2, dec);
}

template <typename T>
bool pick_tile(F3Geom& g, size_t limit) {
  const int cands[3] = {8, 4, 2};
  for (int c : cands) {
    size_t need = 0;
    if (c == 8) need = plane_smem<T, 8>(g, true);
    if (c == 4) need = plane_smem<T, 4>(g, true);
    if (c == 2) need = plane_smem<T, 2>(g, true);
    if (need <= limit) {
      g.tile_rows = c;
      return true;
    }
  }
  return false;
}

template <int LS>
int col_segments(int64_t m) { return int((m + LS - 1) / LS); }

template <typename T>
void launch_col(double* G, T* coarse, double sign, const F3Geom& g, int axis, const double* w, const double* id,
                const Exec& ex) {
  int64_t m, stride, outer_stride, inner, ncols;
  if (axis == 1) {
    m = g.m1;
    stride = g.m2;
    inner = g.m2;
    outer_stride = g.m1 * g.m2;
    ncols = g.m0 * g.m2;
  } else {
    m = g.m0;
    stride = g.m1 * g.m2;
    inner = g.m1 * g.m2;
    outer_stride = 0;
    ncols = g.m1 * g.m2;
  }
  const unsigned blocks = unsigned((ncols + 31) / 32);
  const char* tag = axis == 1 ? "f3_col1" : "f3_col0";
  if (m <= 320) {
    const int S = col_segments<16>(m);
    MGRX_LAUNCH(ex, tag, k_f3_col<T, 16><<<blocks, dim3(32, S), (2 * S * 32 + 2 * m) * 8, ex.s>>>(
                             G, coarse, sign, ncols, m, stride, outer_stride, inner, w, id));
  } else {
    const int S = col_segments<32>(m);
    MGRX_LAUNCH(ex, tag, k_f3_col<T, 32><<<blocks, dim3(32, S), (2 * S * 32 + 2 * m) * 8, ex.s>>>(
                             G, coarse, sign, ncols, m, stride, outer_stride, inner, w, id));
  }
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
  // worth it only for sizeable rows; one thread per coarse column
  if (g.n2 < 33 || g.m2 > kF3MaxThreads || g.m1 > kColMaxM || g.m0 > kColMaxM || g.n1 < 5 || g.n0 < 5) return fp;
  if (int64_t(g.n0) * g.n1 * g.n2 < (int64_t(1) << 15)) return fp;
  int dev = 0;
  cudaGetDevice(&dev);
  int optin = 0, nsm = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (optin <= 0) optin = 227 * 1024;
  if (nsm <= 0) nsm = kNumSMs;
  const bool ok = esize == 4 ? pick_tile<float>(g, size_t(optin)) : pick_tile<double>(g, size_t(optin));
  if (!ok) return fp;
  g.ntile1 = int((g.m1 + g.tile_rows - 1) / g.tile_rows);
  // axis-0 chunks: about 6 units per SM so dynamic scheduling evens out
  const int64_t want_units = int64_t(nsm) * 6;
  int64_t nchunk = std::max<int64_t>(1, (want_units + g.ntile1 - 1) / g.ntile1);
  int64_t chunk = std::max<int64_t>(4, (g.m0 + nchunk - 1) / nchunk);
  nchunk = (g.m0 + chunk - 1) / chunk;
  g.chunk = chunk;
  g.units = int(nchunk * g.ntile1);
  g.threads = int((g.m2 + 31) / 32 * 32);
  g.grid = std::min<int>(g.units, nsm);
  fp.enabled = true;
  fp.scratch_bytes = size_t(g.m0) * g.m1 * g.m2 * 8 + 256;
  return fp;
}

template <typename T>
static cudaError_t set_attrs(const F3Geom& g, size_t* dec_smem, size_t* rec_smem) {
  cudaError_t e = cudaSuccess;
#define MGRX_ATTR(TI)                                                                                    \
  if (g.tile_rows == TI) {                                                                              \
    *dec_smem = plane_smem<T, TI>(g, true);                                                             \
    *rec_smem = plane_smem<T, TI>(g, false);                                                            \
    e = cudaFuncSetAttribute(k_f3_dec_plane<T, TI>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(*dec_smem)); \
    if (e == cudaSuccess)                                                                               \
      e = cudaFuncSetAttribute(k_f3_rec_plane<T, TI>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(*rec_smem)); \
  }
  MGRX_ATTR(8)
  MGRX_ATTR(4)
  MGRX_ATTR(2)
#undef MGRX_ATTR
  return e;
}

template <typename T>
cudaError_t fused3d_decompose_level(const T* blk, T* shell, T* coarse, void* scratch, const LevelGeom&,
                                    const Fused3DPlan& fp, const ThomasLevel& th, const Exec& ex) {
  const F3Geom& g = fp.g;
  double* G = static_cast<double*>(scratch);
  int* counter = reinterpret_cast<int*>(static_cast<char*>(scratch) + size_t(g.m0) * g.m1 * g.m2 * 8);
  size_t ds = 0, rs = 0;
  cudaError_t e = set_attrs<T>(g, &ds, &rs);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(int), ex.s);
  if (e != cudaSuccess) return e;
#define MGRX_DEC(TI)                                                                                   \
  if (g.tile_rows == TI)                                                                              \
    MGRX_LAUNCH(ex, "f3_dec_plane", k_f3_dec_plane<T, TI><<<g.grid, g.threads, ds, ex.s>>>(            \
                                        blk, shell, coarse, G, th.w[2], th.inv_d[2], counter, g));
  MGRX_DEC(8)
  MGRX_DEC(4)
  MGRX_DEC(2)
#undef MGRX_DEC
  launch_col<T>(G, nullptr, 0.0, g, 1, th.w[1], th.inv_d[1], ex);
  launch_col<T>(G, coarse, 1.0, g, 0, th.w[0], th.inv_d[0], ex);
  return cudaGetLastError();
}

template <typename T>
cudaError_t fused3d_recompose_level(const T* shell, T* coarse, T* fine, void* scratch, const LevelGeom&,
                                    const Fused3DPlan& fp, const ThomasLevel& th, const Exec& ex) {
  const F3Geom& g = fp.g;
  double* G = static_cast<double*>(scratch);
  int* counter = reinterpret_cast<int*>(static_cast<char*>(scratch) + size_t(g.m0) * g.m1 * g.m2 * 8);
  size_t ds = 0, rs = 0;
  cudaError_t e = set_attrs<T>(g, &ds, &rs);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(int), ex.s);
  if (e != cudaSuccess) return e;
#define MGRX_REC(TI)                                                                                   \
  if (g.tile_rows == TI)                                                                              \
    MGRX_LAUNCH(ex, "f3_rec_plane",                                                                   \
                k_f3_rec_plane<T, TI><<<g.grid, g.threads, rs, ex.s>>>(shell, G, th.w[2], th.inv_d[2], counter, g));
  MGRX_REC(8)
  MGRX_REC(4)
  MGRX_REC(2)
#undef MGRX_REC
  launch_col<T>(G, nullptr, 0.0, g, 1, th.w[1], th.inv_d[1], ex);
  launch_col<T>(G, coarse, -1.0, g, 0, th.w[0], th.inv_d[0], ex);
  const int rows = 4;
  MGRX_LAUNCH(ex, "f3_rec_interp", k_f3_rec_interp<T><<<dim3(unsigned(g.n0), unsigned((g.n1 + rows - 1) / rows)),
                                                         g.threads, 0, ex.s>>>(shell, coarse, fine, g, rows));
  return cudaGetLastError();
}

#define MGRX_INST(T)                                                                                     \
  template cudaError_t fused3d_decompose_level<T>(const T*, T*, T*, void*, const LevelGeom&, const Fused3DPlan&, \
                                                  const ThomasLevel&, const Exec&);                      \
  template cudaError_t fused3d_recompose_level<T>(const T*, T*, T*, void*, const LevelGeom&, const Fused3DPlan&, \
                                                  const ThomasLevel&, const Exec&);
MGRX_INST(float)
MGRX_INST(double)
#undef MGRX_INST

}  // namespace mgrx_b200
