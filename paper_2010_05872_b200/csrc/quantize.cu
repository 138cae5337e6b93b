// Level-wise quantization and dequantization (reference quantize.hpp:39-150).
//
//   label = nearbyint(double(v) / q_l)   (IEEE fp64 division, ties to even)
//   |label| outside [-32768, 32767] -> outlier {position, value}, label 0
//   non-finite input                 -> nonfinite_data
//
// Outliers must come out in strictly increasing position order
// (read_outliers, pipeline.hpp:56-57).  The buffer is cut into fixed chunks;
// pass 1 writes every label and counts outliers per chunk, a single-CTA scan
// turns the counts into offsets, and pass 2 revisits only chunks that hold
// outliers and writes them in order with a block-wide prefix.  Labels are
// written exactly once, so the bulk cost is one read of the coefficients and
// one int32 write.
#include "common.cuh"
#include "kernels.h"

namespace mgrx_b200 {

constexpr int kQBlock = 256;
constexpr int kQPerThread = 16;
constexpr int64_t kQChunk = int64_t(kQBlock) * kQPerThread;

__device__ __forceinline__ int level_of(const QuantLevels& ql, int64_t pos) {
  int l = ql.first;
  while (l < ql.last && pos >= ql.end[l]) ++l;
  return l;
}

template <typename T>
__device__ __forceinline__ bool quant_one(T v, double q, int32_t* label, bool* nonfinite) {
  const double x = double(v);
  if (!isfinite(x)) {
    *nonfinite = true;
    *label = 0;
    return false;
  }
  const double r = rint(__ddiv_rn(x, q));
  if (r < -32768.0 || r > 32767.0) {
    *label = 0;
    return true;
  }
  *label = int32_t(r);
  return false;
}

// Pass 1: labels + per-chunk outlier counts.  Chunk c covers positions
// [base + c*kQChunk, ...); thread t of the block takes positions
// chunk + i*kQBlock + t for coalescing.
template <typename T>
__global__ void __launch_bounds__(kQBlock) k_quant_labels(const T* __restrict__ c, int32_t* __restrict__ labels,
                                                          uint32_t* __restrict__ chunk_counts,
                                                          int* __restrict__ flags, const QuantLevels ql) {
  const int64_t chunk0 = ql.base + int64_t(blockIdx.x) * kQChunk;
  int count = 0;
  bool nonfinite = false;
#pragma unroll 4
  for (int i = 0; i < kQPerThread; ++i) {
    const int64_t pos = chunk0 + int64_t(i) * kQBlock + threadIdx.x;
    if (pos < ql.total) {
      const int l = level_of(ql, pos);
      int32_t lab;
      count += quant_one<T>(c[pos], ql.q[l], &lab, &nonfinite);
      labels[pos - ql.base] = lab;
    }
  }
  if (nonfinite) atomicOr(flags, 1);
  // block reduction of counts
  __shared__ int warp_sums[kQBlock / 32];
  int v = count;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kQBlock / 32; ++w) s += warp_sums[w];
    chunk_counts[blockIdx.x] = uint32_t(s);
  }
}

// Exclusive scan of the chunk counts in one CTA; offsets[nchunks] = total.
__global__ void __launch_bounds__(1024) k_scan_counts(const uint32_t* __restrict__ counts,
                                                      uint64_t* __restrict__ offsets, int64_t nchunks) {
  __shared__ uint64_t carry;
  __shared__ uint64_t warp_tot[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b = 0; b < nchunks; b += blockDim.x) {
    const int64_t i = b + threadIdx.x;
    const uint64_t x = i < nchunks ? counts[i] : 0;
    uint64_t incl = x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      uint64_t t = lane < int(blockDim.x >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive warp prefix
    }
    __syncthreads();
    const uint64_t warp_prefix = wid ? warp_tot[wid - 1] : 0;
    if (i < nchunks) offsets[i] = carry + warp_prefix + incl - x;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += warp_prefix + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) offsets[nchunks] = carry;
}

// Pass 2: ordered outlier write for chunks that hold any.  Positions are
// visited in increasing order: round i covers chunk + i*kQBlock + [0, 256),
// and a block-wide prefix ranks the flagged lanes inside the round.
template <typename T>
__global__ void __launch_bounds__(kQBlock) k_quant_outliers(const T* __restrict__ c,
                                                            const uint32_t* __restrict__ chunk_counts,
                                                            const uint64_t* __restrict__ offsets,
                                                            uint64_t* __restrict__ opos, T* __restrict__ oval,
                                                            uint64_t capacity, const QuantLevels ql) {
  if (chunk_counts[blockIdx.x] == 0) return;
  __shared__ int warp_cnt[kQBlock / 32];
  uint64_t out = offsets[blockIdx.x];
  const int64_t chunk0 = ql.base + int64_t(blockIdx.x) * kQChunk;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = 0; i < kQPerThread; ++i) {
    const int64_t pos = chunk0 + int64_t(i) * kQBlock + threadIdx.x;
    bool is_out = false;
    T v{};
    if (pos < ql.total) {
      v = c[pos];
      int32_t lab;
      bool nf = false;
      is_out = quant_one<T>(v, ql.q[level_of(ql, pos)], &lab, &nf);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, is_out);
    if (lane == 0) warp_cnt[wid] = __popc(bal);
    __syncthreads();
    int before = 0, round_total = 0;
    for (int w = 0; w < kQBlock / 32; ++w) {
      if (w < wid) before += warp_cnt[w];
      round_total += warp_cnt[w];
    }
    if (is_out) {
      const uint64_t k = out + before + __popc(bal & ((1u << lane) - 1u));
      if (k < capacity) {
        opos[k] = uint64_t(pos);
        oval[k] = v;
      }
    }
    out += round_total;
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_dequant(const int32_t* __restrict__ labels, T* __restrict__ c,
                                                 const QuantLevels ql) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t pos = ql.base + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; pos < ql.total; pos += stride) {
    const int l = level_of(ql, pos);
    c[pos] = to_t<T>(__dmul_rn(double(labels[pos - ql.base]), ql.q[l]));
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_restore_outliers(const uint64_t* __restrict__ opos,
                                                          const T* __restrict__ oval, uint64_t n,
                                                          T* __restrict__ c) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) c[opos[i]] = oval[i];
}

int64_t quant_num_chunks(const QuantLevels& ql) { return (ql.total - ql.base + kQChunk - 1) / kQChunk; }

template <typename T>
cudaError_t quantize_pass1(const T* c, int32_t* labels, uint32_t* chunk_counts, uint64_t* offsets, int* flags,
                           const QuantLevels& ql, const Exec& ex) {
  const int64_t nch = quant_num_chunks(ql);
  if (nch > 0)
    MGRX_LAUNCH(ex, "quant_labels", k_quant_labels<T><<<unsigned(nch), kQBlock, 0, ex.s>>>(c, labels, chunk_counts, flags, ql));
  MGRX_LAUNCH(ex, "quant_scan", k_scan_counts<<<1, 1024, 0, ex.s>>>(chunk_counts, offsets, nch));
  return cudaGetLastError();
}

template <typename T>
cudaError_t quantize_pass2(const T* c, const uint32_t* chunk_counts, const uint64_t* offsets, uint64_t* opos, T* oval,
                           uint64_t capacity, const QuantLevels& ql, const Exec& ex) {
  const int64_t nch = quant_num_chunks(ql);
  if (nch > 0)
    MGRX_LAUNCH(ex, "quant_outliers",
                k_quant_outliers<T><<<unsigned(nch), kQBlock, 0, ex.s>>>(c, chunk_counts, offsets, opos, oval, capacity, ql));
  return cudaGetLastError();
}

template <typename T>
cudaError_t dequantize_run(const int32_t* labels, const uint64_t* opos, const T* oval, uint64_t n_out, T* c,
                           const QuantLevels& ql, const Exec& ex) {
  MGRX_LAUNCH(ex, "dequant", k_dequant<T><<<grid_for(ql.total - ql.base, 256), 256, 0, ex.s>>>(labels, c, ql));
  if (n_out > 0)
    MGRX_LAUNCH(ex, "dequant_outliers",
                k_restore_outliers<T><<<unsigned((n_out + 255) / 256), 256, 0, ex.s>>>(opos, oval, n_out, c));
  return cudaGetLastError();
}

#define MGRX_INST(T)                                                                                        \
  template cudaError_t quantize_pass1<T>(const T*, int32_t*, uint32_t*, uint64_t*, int*, const QuantLevels&, \
                                         const Exec&);                                                      \
  template cudaError_t quantize_pass2<T>(const T*, const uint32_t*, const uint64_t*, uint64_t*, T*, uint64_t, \
                                         const QuantLevels&, const Exec&);                                  \
  template cudaError_t dequantize_run<T>(const int32_t*, const uint64_t*, const T*, uint64_t, T*,            \
                                         const QuantLevels&, const Exec&);
MGRX_INST(float)
MGRX_INST(double)
#undef MGRX_INST

}  // namespace mgrx_b200
