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
#include <algorithm>

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
constexpr double kRoundMagic = 6755399441055744.0;  // 1.5 * 2^52: r + M - M = nearbyint(r), ties to even

// Fast label of x = double(v) (quant_round without a conversion round trip):
// r = x * (1/q) rounded by the magic constant, the label read from the low
// word of r + M.  Returns false when the value must take the exact path
// (within a few ulp of a half-integer, or a non-finite / huge product).
__device__ __forceinline__ bool quant_fast(double x, double inv, int32_t* lab, bool* out) {
  const double r1 = x * inv;
  const double t = r1 + kRoundMagic;
  const double n1 = t - kRoundMagic;
  const bool ok = fabs(fabs(r1 - n1) - 0.5) > fabs(r1) * 0x1p-48;  // false for NaN / inf / |r| >= 2^51
  *out = !(r1 >= -32768.5 && r1 < 32767.5);
  *lab = *out ? 0 : __double2loint(t);
  return ok;
}

// Pass 1: labels + per-chunk outlier counts.  Chunk c covers positions
// [base + c*kQChunk, ...); thread t of the block takes positions
// chunk + i*kQBlock + t for coalescing.  A chunk inside one level (all but a
// few) runs the fast path; a thread that met a value needing the exact
// division (or a non-finite one) redoes its 16 values exactly.
template <typename T>
__device__ __forceinline__ void quant_chunk(const T* __restrict__ c, int32_t* __restrict__ labels,
                                            uint32_t* __restrict__ chunk_counts, int* __restrict__ flags,
                                            const QuantLevels& ql, const int64_t chunk, int* warp_sums) {
  const int64_t chunk0 = ql.base + chunk * kQChunk;
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
  for (int i = 0; i < kQPerThread; ++i) v[i] = (i * kQBlock + int(threadIdx.x) < n) ? __ldcs(cp + i * kQBlock) : T(0);
  bool exact = end < n;  // a level boundary inside the chunk (block-uniform)
  if (!exact) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < kQPerThread; ++i) {
      if (i * kQBlock + int(threadIdx.x) < n) {
        int32_t lab;
        bool o;
        ok &= quant_fast(double(v[i]), inv, &lab, &o);
        count += o;
        __stcs(lp + i * kQBlock, lab);
      }
    }
    exact = !ok;
    if (exact) count = 0;
  }
  if (exact) {
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
  }
  if (nonfinite) atomicOr(flags, 1);
  // block reduction of counts
  int wsum = count;
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kQBlock / 32; ++w) t += warp_sums[w];
    chunk_counts[chunk] = uint32_t(t);
  }
}

template <typename T>
__global__ void __launch_bounds__(kQBlock, 4) k_quant_labels(const T* __restrict__ c, int32_t* __restrict__ labels,
                                                             uint32_t* __restrict__ chunk_counts,
                                                             int* __restrict__ flags, const QuantLevels ql,
                                                             const int64_t chunk_begin) {
  __shared__ int warp_sums[kQBlock / 32];
  quant_chunk<T>(c, labels, chunk_counts, flags, ql, chunk_begin + int64_t(blockIdx.x), warp_sums);
}

// Exclusive scan of the chunk counts in one CTA; offsets[nchunks] = total.
// The counts are staged in (dynamic) shared memory with one round of
// coalesced loads per tile of up to kScanMax; thread t scans its contiguous
// run, one block-wide scan of the run sums, then each thread writes its run.
constexpr int kScanThreads = 1024;
constexpr int kScanMax = 48 * 1024;  // counts per tile (192 KB of shared memory)
__global__ void __launch_bounds__(kScanThreads) k_scan_counts(const uint32_t* __restrict__ counts,
                                                              uint64_t* __restrict__ offsets, int64_t nchunks) {
  extern __shared__ uint32_t tile[];
  __shared__ uint64_t warp_tot[32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  uint64_t carry = 0;
  for (int64_t base = 0; base < nchunks; base += kScanMax) {
    const int len = int(min(int64_t(kScanMax), nchunks - base));
#pragma unroll 8
    for (int i = t; i < len; i += kScanThreads) tile[i] = counts[base + i];
    __syncthreads();
    const int per = (len + kScanThreads - 1) / kScanThreads;
    const int i0 = min(len, t * per), i1 = min(len, i0 + per);
    uint64_t sum = 0;
    for (int i = i0; i < i1; ++i) sum += tile[i];
    uint64_t incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      uint64_t w = warp_tot[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;  // inclusive prefix over warps
    }
    __syncthreads();
    // tile-local exclusive offsets in place (a tile holds < 2^32 outliers),
    // then written out coalesced
    uint32_t run = uint32_t((wid ? warp_tot[wid - 1] : 0) + incl - sum);
    for (int i = i0; i < i1; ++i) {
      const uint32_t x = tile[i];
      tile[i] = run;
      run += x;
    }
    __syncthreads();
#pragma unroll 8
    for (int i = t; i < len; i += kScanThreads) offsets[base + i] = carry + tile[i];
    carry += warp_tot[31];
    __syncthreads();
  }
  if (t == 0) offsets[nchunks] = carry;
}

// Pass 2: ordered outlier write for chunks that hold any.  Positions are
// visited in increasing order: round i covers chunk + i*kQBlock + [0, 256),
// and a block-wide prefix ranks the flagged lanes inside the round.
// Pass 2: ordered outlier write for chunks that hold any.  A thread loads
// its 16 values of the chunk at once and flags its outliers; the per-(round,
// warp) ballots go to shared memory, one exclusive prefix over them (in
// position order: round-major, then warp, then lane) ranks every outlier.
template <typename T>
__global__ void __launch_bounds__(kQBlock) k_quant_outliers(const T* __restrict__ c,
                                                            const uint32_t* __restrict__ chunk_counts,
                                                            const uint64_t* __restrict__ offsets,
                                                            uint64_t* __restrict__ opos, T* __restrict__ oval,
                                                            uint64_t capacity, const QuantLevels ql, int64_t nch) {
  constexpr int NW = kQBlock / 32;
  __shared__ unsigned bal_s[kQPerThread * NW];  // ballot of outliers per (round, warp)
  __shared__ int pre_s[kQPerThread * NW];       // outliers before (round, warp) in position order
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  __shared__ unsigned todo_s;
  // chunks b, b + G, b + 2G, ... (G = grid): their counts are checked 32 at
  // a time (one coalesced load), then the non-empty ones are processed
  for (int64_t j0 = 0; int64_t(blockIdx.x) + j0 * gridDim.x < nch; j0 += 32) {
    if (wid == 0) {
      const int64_t chl = int64_t(blockIdx.x) + (j0 + lane) * gridDim.x;
      const unsigned b = __ballot_sync(0xffffffffu, chl < nch && chunk_counts[chl] != 0);
      if (lane == 0) todo_s = b;
    }
    __syncthreads();
    unsigned todo = todo_s;
    __syncthreads();
  while (todo) {
    const int64_t ch = int64_t(blockIdx.x) + (j0 + __ffs(todo) - 1) * gridDim.x;
    todo &= todo - 1;
    const uint64_t out = offsets[ch];
    const int64_t chunk0 = ql.base + ch * kQChunk;
    T v[kQPerThread];
#pragma unroll
    for (int i = 0; i < kQPerThread; ++i) {
      const int64_t pos = chunk0 + int64_t(i) * kQBlock + threadIdx.x;
      v[i] = pos < ql.total ? c[pos] : T(0);
    }
    unsigned mask = 0;
#pragma unroll
    for (int i = 0; i < kQPerThread; ++i) {
      const int64_t pos = chunk0 + int64_t(i) * kQBlock + threadIdx.x;
      bool is_out = false;
      if (pos < ql.total) {
        int32_t lab;
        bool nf = false;
        const int l = level_of(ql, pos);
        is_out = quant_one<T>(v[i], ql.q[l], ql.inv[l], &lab, &nf);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, is_out);
      if (lane == 0) bal_s[i * NW + wid] = bal;
      mask |= unsigned(is_out) << i;
    }
    __syncthreads();
    if (wid == 0) {  // exclusive prefix of the 16 x NW popcounts (<= 32 per lane pass)
      int run = 0;
      for (int k0 = 0; k0 < kQPerThread * NW; k0 += 32) {
        const int k = k0 + lane;
        const int x = k < kQPerThread * NW ? __popc(bal_s[k]) : 0;
        int incl = x;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (k < kQPerThread * NW) pre_s[k] = run + incl - x;
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kQPerThread; ++i)
      if (mask & (1u << i)) {
        const int slot = i * NW + wid;
        const uint64_t k = out + uint64_t(pre_s[slot]) + __popc(bal_s[slot] & lt);
        if (k < capacity) {
          opos[k] = uint64_t(chunk0 + int64_t(i) * kQBlock + threadIdx.x);
          oval[k] = v[i];
        }
      }
    __syncthreads();  // bal_s / pre_s are reused by the next chunk
  }
  }
}

// buf[pos] = T(double(label) * q_l) (dequantize, quantize.hpp:118-135): the
// same chunking as the quantizer, labels loaded first, level tracked per
// thread.
template <typename T>
__global__ void __launch_bounds__(kQBlock, 4) k_dequant(const int32_t* __restrict__ labels, T* __restrict__ c,
                                                        const QuantLevels ql, const int64_t chunk_begin) {
  const int64_t chunk0 = ql.base + (chunk_begin + int64_t(blockIdx.x)) * kQChunk;
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
                                                          T* __restrict__ c, uint64_t lo, uint64_t hi) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    const uint64_t p = opos[i];
    if (p >= lo && p < hi) c[p] = oval[i];
  }
}

int64_t quant_num_chunks(const QuantLevels& ql) { return (ql.total - ql.base + kQChunk - 1) / kQChunk; }

int64_t quant_chunk_of(const QuantLevels& ql, int64_t pos) { return (pos - ql.base + kQChunk - 1) / kQChunk; }

// Labels + outlier counts of chunks [chunk_begin, chunk_end) only (the
// overlapped decompose + quantize launches the finest shell's chunks as soon
// as that shell is final).
template <typename T>
cudaError_t quantize_labels_range(const T* c, int32_t* labels, uint32_t* chunk_counts, int* flags,
                                  const QuantLevels& ql, int64_t chunk_begin, int64_t chunk_end, const Exec& ex) {
  if (chunk_end > chunk_begin)
    MGRX_LAUNCH(ex, "quant_labels", k_quant_labels<T><<<unsigned(chunk_end - chunk_begin), kQBlock, 0, ex.s>>>(
                                        c, labels, chunk_counts, flags, ql, chunk_begin));
  return cudaGetLastError();
}

cudaError_t quantize_scan(const uint32_t* chunk_counts, uint64_t* offsets, const QuantLevels& ql, const Exec& ex) {
  const int64_t nch = quant_num_chunks(ql);
  const size_t ssm = size_t(std::min<int64_t>(std::max<int64_t>(nch, 1), kScanMax)) * 4;
  cudaFuncSetAttribute(k_scan_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ssm));
  MGRX_LAUNCH(ex, "quant_scan", k_scan_counts<<<1, kScanThreads, ssm, ex.s>>>(chunk_counts, offsets, nch));
  return cudaGetLastError();
}

template <typename T>
cudaError_t quantize_pass1(const T* c, int32_t* labels, uint32_t* chunk_counts, uint64_t* offsets, int* flags,
                           const QuantLevels& ql, const Exec& ex) {
  const int64_t nch = quant_num_chunks(ql);
  if (nch > 0)
    MGRX_LAUNCH(ex, "quant_labels", k_quant_labels<T><<<unsigned(nch), kQBlock, 0, ex.s>>>(c, labels, chunk_counts, flags, ql, 0));
  const size_t ssm = size_t(std::min<int64_t>(std::max<int64_t>(nch, 1), kScanMax)) * 4;
  cudaFuncSetAttribute(k_scan_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ssm));
  MGRX_LAUNCH(ex, "quant_scan", k_scan_counts<<<1, kScanThreads, ssm, ex.s>>>(chunk_counts, offsets, nch));
  return cudaGetLastError();
}

template <typename T>
cudaError_t quantize_pass2(const T* c, const uint32_t* chunk_counts, const uint64_t* offsets, uint64_t* opos, T* oval,
                           uint64_t capacity, const QuantLevels& ql, const Exec& ex) {
  const int64_t nch = quant_num_chunks(ql);
  if (nch > 0)
    MGRX_LAUNCH(ex, "quant_outliers",
                k_quant_outliers<T><<<unsigned(std::min<int64_t>(nch, int64_t(kNumSMs) * 8)), kQBlock, 0, ex.s>>>(
                    c, chunk_counts, offsets, opos, oval, capacity, ql, nch));
  return cudaGetLastError();
}

template <typename T>
cudaError_t dequantize_run(const int32_t* labels, const uint64_t* opos, const T* oval, uint64_t n_out, T* c,
                           const QuantLevels& ql, const Exec& ex) {
  const int64_t nch = quant_num_chunks(ql);
  if (nch > 0) MGRX_LAUNCH(ex, "dequant", k_dequant<T><<<unsigned(nch), kQBlock, 0, ex.s>>>(labels, c, ql, 0));
  if (n_out > 0)
    MGRX_LAUNCH(ex, "dequant_outliers",
                k_restore_outliers<T><<<unsigned((n_out + 255) / 256), 256, 0, ex.s>>>(opos, oval, n_out, c, 0,
                                                                                       ~uint64_t(0)));
  return cudaGetLastError();
}

// Labels -> coefficients of chunks [chunk_begin, chunk_end) only (no outlier
// restore): the overlapped dequantize + recompose.
template <typename T>
cudaError_t dequantize_range(const int32_t* labels, const uint64_t* opos, const T* oval, uint64_t n_out, T* c,
                             const QuantLevels& ql, int64_t chunk_begin, int64_t chunk_end, const Exec& ex) {
  if (chunk_end > chunk_begin)
    MGRX_LAUNCH(ex, "dequant", k_dequant<T><<<unsigned(chunk_end - chunk_begin), kQBlock, 0, ex.s>>>(labels, c, ql,
                                                                                                 chunk_begin));
  if (n_out > 0 && chunk_end > chunk_begin) {  // outliers of this chunk range only
    const uint64_t lo = uint64_t(ql.base + chunk_begin * kQChunk);
    const uint64_t hi = uint64_t(std::min<int64_t>(ql.total, ql.base + chunk_end * kQChunk));
    MGRX_LAUNCH(ex, "dequant_outliers",
                k_restore_outliers<T><<<unsigned((n_out + 255) / 256), 256, 0, ex.s>>>(opos, oval, n_out, c, lo, hi));
  }
  return cudaGetLastError();
}

#define MGRX_INST(T)                                                                                        \
  template cudaError_t quantize_pass1<T>(const T*, int32_t*, uint32_t*, uint64_t*, int*, const QuantLevels&, \
                                         const Exec&);                                                      \
  template cudaError_t quantize_pass2<T>(const T*, const uint32_t*, const uint64_t*, uint64_t*, T*, uint64_t, \
                                         const QuantLevels&, const Exec&);                                  \
  template cudaError_t dequantize_run<T>(const int32_t*, const uint64_t*, const T*, uint64_t, T*,            \
                                         const QuantLevels&, const Exec&);                                  \
  template cudaError_t quantize_labels_range<T>(const T*, int32_t*, uint32_t*, int*, const QuantLevels&,     \
                                                int64_t, int64_t, const Exec&);                                \
  template cudaError_t dequantize_range<T>(const int32_t*, const uint64_t*, const T*, uint64_t, T*,          \
                                           const QuantLevels&, int64_t, int64_t, const Exec&);
MGRX_INST(float)
MGRX_INST(double)
#undef MGRX_INST

}  // namespace mgrx_b200
