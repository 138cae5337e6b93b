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

// r = nearbyint(x / q) exactly as the reference (IEEE division, ties to
// even): x * (1/q) is within 2 ulp of x / q, so its rounding can only differ
// when it lies within a few ulp of a half-integer; those rare values take
// the exact division.  So does a non-finite product (a subnormal bin width
// whose reciprocal overflows: 0 * inf, x * inf), where only x / q is right.
__device__ __forceinline__ double quant_round(double x, double q, double inv) {
  const double r1 = x * inv;
  const double n1 = rint(r1);
  if (!isfinite(r1) || fabs(fabs(r1 - n1) - 0.5) <= fabs(r1) * 0x1p-48) return rint(__ddiv_rn(x, q));
  return n1;
}

template <typename T>
__device__ __forceinline__ bool quant_one(T v, double q, double inv, int32_t* label, bool* nonfinite) {
  const double x = double(v);
  if (!isfinite(x)) {
    *nonfinite = true;
    *label = 0;
    return false;
  }
  const double r = quant_round(x, q, inv);
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
__global__ void __launch_bounds__(kQBlock, 4) k_quant_labels(const T* __restrict__ c, int32_t* __restrict__ labels,
                                                             uint32_t* __restrict__ chunk_counts,
                                                             int* __restrict__ flags, const QuantLevels ql) {
  const int64_t chunk0 = ql.base + int64_t(blockIdx.x) * kQChunk;
  const int n = int(min(int64_t(kQChunk), ql.total - chunk0));  // positions in this chunk
  const T* cp = c + chunk0 + threadIdx.x;
  int32_t* lp = labels + (chunk0 - ql.base) + threadIdx.x;
  int count = 0;
  bool nonfinite = false;
  // level of this chunk's first position and the chunk-relative end of it
  int l = level_of(ql, chunk0);
  int end = int(min(ql.end[l] - chunk0, int64_t(kQChunk)));
  double q = ql.q[l], inv = ql.inv[l];
  T v[kQPerThread];
#pragma unroll
  for (int i = 0; i < kQPerThread; ++i) v[i] = (i * kQBlock + int(threadIdx.x) < n) ? cp[i * kQBlock] : T(0);
#pragma unroll
  for (int i = 0; i < kQPerThread; ++i) {
    const int r = i * kQBlock + int(threadIdx.x);
    if (r < n) {
      while (r >= end) {  // level boundary inside the chunk (rare)
        ++l;
        end = int(min(ql.end[l] - chunk0, int64_t(kQChunk)));
        q = ql.q[l];
        inv = ql.inv[l];
      }
      int32_t lab;
      count += quant_one<T>(v[i], q, inv, &lab, &nonfinite);
      lp[i * kQBlock] = lab;
    }
  }
  if (nonfinite) atomicOr(flags, 1);
  // block reduction of counts
  __shared__ int warp_sums[kQBlock / 32];
  int wsum = count;
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kQBlock / 32; ++w) t += warp_sums[w];
    chunk_counts[blockIdx.x] = uint32_t(t);
  }
}

// Exclusive scan of the chunk counts in one CTA; offsets[nchunks] = total.
// Thread t owns a contiguous run of counts: local sums, one block-wide scan
// of the sums, then each thread writes its run's offsets.
__global__ void __launch_bounds__(1024) k_scan_counts(const uint32_t* __restrict__ counts,
                                                      uint64_t* __restrict__ offsets, int64_t nchunks) {
  __shared__ uint64_t warp_tot[32];
  const int t = threadIdx.x, nt = blockDim.x, lane = t & 31, wid = t >> 5;
  const int64_t per = (nchunks + nt - 1) / nt;
  const int64_t i0 = min(nchunks, int64_t(t) * per), i1 = min(nchunks, i0 + per);
  uint64_t sum = 0;
  for (int64_t i = i0; i < i1; ++i) sum += counts[i];
  uint64_t incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint64_t w = lane < (nt >> 5) ? warp_tot[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_tot[lane] = w;  // inclusive prefix over warps
  }
  __syncthreads();
  uint64_t run = (wid ? warp_tot[wid - 1] : 0) + incl - sum;
  for (int64_t i = i0; i < i1; ++i) {
    offsets[i] = run;
    run += counts[i];
  }
  if (t == nt - 1) offsets[nchunks] = warp_tot[(nt >> 5) - 1];
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
      const int l = level_of(ql, pos);
      is_out = quant_one<T>(v, ql.q[l], ql.inv[l], &lab, &nf);
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

// buf[pos] = T(double(label) * q_l) (dequantize, quantize.hpp:118-135): the
// same chunking as the quantizer, labels loaded first, level tracked per
// thread.
template <typename T>
__global__ void __launch_bounds__(kQBlock, 4) k_dequant(const int32_t* __restrict__ labels, T* __restrict__ c,
                                                        const QuantLevels ql) {
  const int64_t chunk0 = ql.base + int64_t(blockIdx.x) * kQChunk;
  const int n = int(min(int64_t(kQChunk), ql.total - chunk0));
  const int32_t* lp = labels + (chunk0 - ql.base) + threadIdx.x;
  T* cp = c + chunk0 + threadIdx.x;
  int l = level_of(ql, chunk0);
  int end = int(min(ql.end[l] - chunk0, int64_t(kQChunk)));
  double q = ql.q[l];
  int32_t lab[kQPerThread];
#pragma unroll
  for (int i = 0; i < kQPerThread; ++i) lab[i] = (i * kQBlock + int(threadIdx.x) < n) ? lp[i * kQBlock] : 0;
#pragma unroll
  for (int i = 0; i < kQPerThread; ++i) {
    const int r = i * kQBlock + int(threadIdx.x);
    if (r < n) {
      while (r >= end) {
        ++l;
        end = int(min(ql.end[l] - chunk0, int64_t(kQChunk)));
        q = ql.q[l];
      }
      cp[i * kQBlock] = to_t<T>(__dmul_rn(double(lab[i]), q));
    }
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
  const int64_t nch = quant_num_chunks(ql);
  if (nch > 0) MGRX_LAUNCH(ex, "dequant", k_dequant<T><<<unsigned(nch), kQBlock, 0, ex.s>>>(labels, c, ql));
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
