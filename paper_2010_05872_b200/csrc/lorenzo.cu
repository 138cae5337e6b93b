// Lorenzo coder on the GPU: compress_lorenzo
// (lorenzo.hpp:87-128) of a block in HBM — the coarse block an adaptive
// decomposition stops at.  Every prediction reads reconstructed values of
// lexicographically earlier neighbours (index - e_S for the 2^d - 1 nonempty
// axis sets S), all on the hyperplanes sum(index) - |S| < sum(index): so the
// points of one hyperplane sum(index) = h are independent once the earlier
// hyperplanes are reconstructed.  One CTA walks the hyperplanes (host-built
// ordering), a barrier between them; per point the reference's arithmetic
// (inclusion-exclusion sum in its order, nearbyint((v - pred) / step), the
// stored-value bound check) with explicit round-to-nearest fp64 ops, so the
// labels, outliers and reconstruction are bit-identical.  A second pass
// compacts the outliers in position order.
#include <cuda_runtime.h>

#include "kernels.h"

namespace mgrx_b200 {
namespace {

struct LzGeom {
  int d;
  int64_t n[kMaxD];
  int64_t st[kMaxD];
};

template <typename T>
__global__ void __launch_bounds__(1024) k_lorenzo(const T* __restrict__ x, const LzGeom g,
                                                  const uint32_t* __restrict__ order, const uint32_t* __restrict__ hs,
                                                  int H, double e, int32_t* __restrict__ labels,
                                                  uint8_t* __restrict__ outl, T* __restrict__ recon) {
  const double step = 2.0 * e;
  const int d = g.d;
  for (int h = 0; h < H; ++h) {
    for (uint32_t k = hs[h] + threadIdx.x; k < hs[h + 1]; k += blockDim.x) {
      const int64_t p = order[k];
      int64_t idx[kMaxD];
      int64_t r = p;
      bool interior = true;
      for (int i = d - 1; i >= 0; --i) {
        idx[i] = r % g.n[i];
        r /= g.n[i];
        interior &= idx[i] != 0;
      }
      double pred = 0.0;
      for (unsigned s = 1; s < (1u << d); ++s) {
        int64_t off = p;
        int bits = 0;
        bool valid = true;
        for (int i = 0; i < d; ++i)
          if ((s >> i) & 1u) {
            if (!interior && idx[i] == 0) {
              valid = false;
              break;
            }
            off -= g.st[i];
            ++bits;
          }
        if (!valid) continue;
        const double v = double(recon[off]);
        pred = (bits & 1) ? __dadd_rn(pred, v) : __dadd_rn(pred, -v);
      }
      const double v = double(x[p]);
      const double q = rint(__ddiv_rn(__dsub_rn(v, pred), step));
      bool outlier = q < -32768.0 || q > 32767.0;
      T stored{};
      if (!outlier) {
        stored = T(__dadd_rn(pred, __dmul_rn(q, step)));
        if (fabs(__dsub_rn(double(stored), v)) > e) outlier = true;
      }
      if (outlier) {
        labels[p] = 0;
        outl[p] = 1;
        recon[p] = x[p];
      } else {
        labels[p] = int32_t(q);
        outl[p] = 0;
        recon[p] = stored;
      }
    }
    __syncthreads();
  }
}

// Outlier positions / values in position order (one CTA, chunks of 1024).
template <typename T>
__global__ void __launch_bounds__(1024) k_lz_compact(const T* __restrict__ x, const uint8_t* __restrict__ outl,
                                                     int64_t n, uint64_t* __restrict__ opos, T* __restrict__ oval,
                                                     uint64_t cap, unsigned long long* __restrict__ count) {
  __shared__ int wsum[32];
  __shared__ unsigned long long base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t c0 = 0; c0 < n; c0 += blockDim.x) {
    const int64_t p = c0 + threadIdx.x;
    const int f = (p < n && outl[p]) ? 1 : 0;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[w] = __popc(m);
    __syncthreads();
    int before = 0, total = 0;
    for (int k = 0; k < int(blockDim.x >> 5); ++k) {
      if (k < w) before += wsum[k];
      total += wsum[k];
    }
    const unsigned long long at = base + before + __popc(m & ((1u << lane) - 1u));
    if (f && at < cap) {
      opos[at] = uint64_t(p);
      oval[at] = x[p];
    }
    __syncthreads();
    if (threadIdx.x == 0) base += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base;
}

}  // namespace

template <typename T>
cudaError_t lorenzo_run(const T* x, int d, const int64_t* n, const uint32_t* order, const uint32_t* hs, int H,
                        double e, int32_t* labels, uint8_t* outl, T* recon, uint64_t* opos, T* oval, uint64_t cap,
                        unsigned long long* count, const Exec& ex) {
  LzGeom g{};
  g.d = d;
  int64_t s = 1, N = 1;
  for (int i = d - 1; i >= 0; --i) {
    g.n[i] = n[i];
    g.st[i] = s;
    s *= n[i];
  }
  N = s;
  MGRX_LAUNCH(ex, "lorenzo", k_lorenzo<T><<<1, 1024, 0, ex.s>>>(x, g, order, hs, H, e, labels, outl, recon));
  MGRX_LAUNCH(ex, "lorenzo_outliers", k_lz_compact<T><<<1, 1024, 0, ex.s>>>(x, outl, N, opos, oval, cap, count));
  return cudaGetLastError();
}
template cudaError_t lorenzo_run<float>(const float*, int, const int64_t*, const uint32_t*, const uint32_t*, int, double,
                                        int32_t*, uint8_t*, float*, uint64_t*, float*, uint64_t, unsigned long long*,
                                        const Exec&);
template cudaError_t lorenzo_run<double>(const double*, int, const int64_t*, const uint32_t*, const uint32_t*, int,
                                         double, int32_t*, uint8_t*, double*, uint64_t*, double*, uint64_t,
                                         unsigned long long*, const Exec&);

}  // namespace mgrx_b200
