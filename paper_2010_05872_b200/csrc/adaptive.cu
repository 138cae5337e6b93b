// Adaptive stop decision on the GPU: the sampled
// prediction-error estimate of choose_stop (adaptive.hpp:99-104) over a
// level block that is already in HBM, so compress(adaptive) needs no copy of
// the level block to the host.  One thread per sampled 3^d block (anchors
// every `step` nodes along each axis, accumulate_block_errors,
// adaptive.hpp:51-94); each block's two sums are estimate_block_errors
// (src/adaptive.cpp:74-138) with the same operation order and no
// contraction (explicit __dadd_rn / __dmul_rn / __ddiv_rn), and the caller
// adds the blocks up in anchor order on the host — the totals and the
// decision are bit-identical to the reference's.
#include <cuda_runtime.h>

#include "kernels.h"

namespace mgrx_b200 {
namespace {

struct StopGeom {
  int d;
  int step;
  int64_t nblocks;
  int64_t na[kMaxD];  // anchors per axis
  int64_t st[kMaxD];  // row-major strides of the level block
  double pen[kMaxD];  // model.interp[k - 1]
  double lpen;        // model.lorenzo
  double e;
};

template <typename T>
__global__ void __launch_bounds__(128) k_block_errors(const T* __restrict__ blk, const StopGeom sg,
                                                      double* __restrict__ out) {
  const int d = sg.d;
  const int64_t gstride = int64_t(gridDim.x) * blockDim.x;
  int n3 = 1;
  for (int i = 0; i < d; ++i) n3 *= 3;
  for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < sg.nblocks; b += gstride) {
    int64_t rem = b, base = 0;
    for (int i = d - 1; i >= 0; --i) {
      const int64_t a = rem % sg.na[i];
      rem /= sg.na[i];
      base += a * sg.step * sg.st[i];
    }
    double lz = 0.0, ip = 0.0;
    int t[kMaxD];
    for (int i = 0; i < d; ++i) t[i] = 0;
    for (int p = 0; p < n3; ++p) {
      int k = 0;
      bool lorenzo_ok = true;
      int64_t pos = base;
      for (int i = 0; i < d; ++i) {
        k += t[i] & 1;
        lorenzo_ok &= t[i] != 0;
        pos += t[i] * sg.st[i];
      }
      if (k > 0) {
        const double v = double(blk[pos]);
        double sum = 0.0;
        const unsigned corners = 1u << k;
        for (unsigned cm = 0; cm < corners; ++cm) {
          int64_t off = pos;
          unsigned bit = 0;
          for (int i = 0; i < d; ++i)
            if (t[i] & 1) {
              off += ((cm >> bit) & 1u) ? sg.st[i] : -sg.st[i];
              ++bit;
            }
          sum = __dadd_rn(sum, double(blk[off]));
        }
        ip = __dadd_rn(ip, __dadd_rn(fabs(__dsub_rn(v, __ddiv_rn(sum, double(corners)))), __dmul_rn(sg.pen[k - 1], sg.e)));
        if (lorenzo_ok) {
          double pred = 0.0;
          for (unsigned s = 1; s < (1u << d); ++s) {
            int64_t off = pos;
            for (int i = 0; i < d; ++i)
              if ((s >> i) & 1u) off -= sg.st[i];
            const double x = double(blk[off]);
            pred = (__popc(s) & 1) ? __dadd_rn(pred, x) : __dsub_rn(pred, x);
          }
          lz = __dadd_rn(lz, __dadd_rn(fabs(__dsub_rn(v, pred)), __dmul_rn(sg.lpen, sg.e)));
        }
      }
      for (int i = d - 1; i >= 0; --i) {
        if (++t[i] < 3) break;
        t[i] = 0;
      }
    }
    out[2 * b] = lz;
    out[2 * b + 1] = ip;
  }
}

}  // namespace

int64_t stop_blocks(int d, const int64_t* ext, int step) {
  int64_t n = 1;
  for (int i = 0; i < d; ++i) {
    if (ext[i] < 3) return 0;
    n *= (ext[i] - 3) / step + 1;
  }
  return n;
}

template <typename T>
cudaError_t block_errors(const T* blk, int d, const int64_t* ext, int step, double e, const double* interp_pen,
                         double lorenzo_pen, double* out, const Exec& ex) {
  StopGeom sg{};
  sg.d = d;
  sg.step = step;
  sg.nblocks = stop_blocks(d, ext, step);
  if (sg.nblocks == 0) return cudaSuccess;
  int64_t s = 1;
  for (int i = d - 1; i >= 0; --i) {
    sg.na[i] = (ext[i] - 3) / step + 1;
    sg.st[i] = s;
    s *= ext[i];
  }
  for (int i = 0; i < d; ++i) sg.pen[i] = interp_pen[i];
  sg.lpen = lorenzo_pen;
  sg.e = e;
  MGRX_LAUNCH(ex, "stop_blocks", k_block_errors<T><<<grid_for(sg.nblocks, 128, 8), 128, 0, ex.s>>>(blk, sg, out));
  return cudaGetLastError();
}

template cudaError_t block_errors<float>(const float*, int, const int64_t*, int, double, const double*, double, double*,
                                         const Exec&);
template cudaError_t block_errors<double>(const double*, int, const int64_t*, int, double, const double*, double,
                                          double*, const Exec&);

}  // namespace mgrx_b200

// ---- field statistics --------------------------------
// check_finite (pipeline.hpp:113-118) and the value range in one read of the
// field: per block the min / max of the finite values and the first
// non-finite offset; the host folds the blocks.
namespace mgrx_b200 {
namespace {
template <typename T>
__global__ void __launch_bounds__(256) k_field_stats(const T* __restrict__ x, int64_t n, double* __restrict__ bmin,
                                                     double* __restrict__ bmax, unsigned long long* __restrict__ bbad) {
  double lo = INFINITY, hi = -INFINITY;
  unsigned long long bad = ~0ull;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double v = double(x[i]);
    if (isfinite(v)) {
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    } else if (bad == ~0ull) {
      bad = (unsigned long long)i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, bad, o);
    bad = b < bad ? b : bad;
  }
  __shared__ double slo[8], shi[8];
  __shared__ unsigned long long sbad[8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    slo[w] = lo;
    shi[w] = hi;
    sbad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < int(blockDim.x >> 5); ++k) {
      lo = fmin(lo, slo[k]);
      hi = fmax(hi, shi[k]);
      bad = sbad[k] < bad ? sbad[k] : bad;
    }
    bmin[blockIdx.x] = lo;
    bmax[blockIdx.x] = hi;
    bbad[blockIdx.x] = bad;
  }
}
}  // namespace

int field_stats_blocks(int64_t n) { return grid_for(n, 256, 4); }

template <typename T>
cudaError_t field_stats(const T* x, int64_t n, double* bmin, double* bmax, unsigned long long* bbad, const Exec& ex) {
  MGRX_LAUNCH(ex, "field_stats", k_field_stats<T><<<field_stats_blocks(n), 256, 0, ex.s>>>(x, n, bmin, bmax, bbad));
  return cudaGetLastError();
}
template cudaError_t field_stats<float>(const float*, int64_t, double*, double*, unsigned long long*, const Exec&);
template cudaError_t field_stats<double>(const double*, int64_t, double*, double*, unsigned long long*, const Exec&);
}  // namespace mgrx_b200
