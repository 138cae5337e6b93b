// Label entropy coding on the GPU: the byte stream of
// the reference's encode_labels (src/huffman.cpp:209-255) — canonical
// Huffman over the label alphabet [min, max], code-length table, then the
// codes bit-reversed and packed LSB-first — produced from labels already in
// HBM, so only the encoded bytes cross PCIe.  The device computes min/max,
// the histogram and the bit packing (per label its code's bit offset from a
// chunked prefix sum of the code lengths, the bits OR-ed into 64-bit words);
// the host builds the code lengths from the histogram with the reference's
// heap order (code_lengths, :84-127) and canonicalises them (:138-160).
#include <cuda_runtime.h>

#include "kernels.h"

namespace mgrx_b200 {
namespace {

constexpr int kEncChunk = 4096;  // labels per chunk of the bit-offset scan

__global__ void __launch_bounds__(256) k_label_minmax(const int32_t* __restrict__ x, int64_t n, int* __restrict__ mm) {
  int lo = INT32_MAX, hi = INT32_MIN;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int v = x[i];
    lo = min(lo, v);
    hi = max(hi, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
}

// Histogram over [lo, lo + range): per-block shared counts when they fit.
__global__ void __launch_bounds__(256) k_label_hist(const int32_t* __restrict__ x, int64_t n, int lo, int range,
                                                    unsigned long long* __restrict__ freq, int smem_bins) {
  extern __shared__ unsigned int sh[];
  const bool local = range <= smem_bins;
  if (local)
    for (int i = threadIdx.x; i < range; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int s = x[i] - lo;
    if (local)
      atomicAdd(&sh[s], 1u);
    else
      atomicAdd(&freq[s], 1ull);
  }
  __syncthreads();
  if (local)
    for (int i = threadIdx.x; i < range; i += blockDim.x)
      if (sh[i]) atomicAdd(&freq[i], (unsigned long long)sh[i]);
}

// Bits of each chunk of kEncChunk labels.
__global__ void __launch_bounds__(256) k_chunk_bits(const int32_t* __restrict__ x, int64_t n, int lo,
                                                    const unsigned long long* __restrict__ code,
                                                    unsigned long long* __restrict__ chunk_bits) {
  const int64_t c0 = int64_t(blockIdx.x) * kEncChunk;
  const int64_t c1 = min(n, c0 + kEncChunk);
  unsigned long long b = 0;
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) b += code[x[i] - lo] & 63ull;
  for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
  __shared__ unsigned long long ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += ws[w];
    chunk_bits[blockIdx.x] = t;
  }
}

// Emit: block = chunk; labels in order, each thread a run of consecutive
// labels; block-wide exclusive scan of the runs' bits gives every code's
// bit offset (chunk base from the scanned chunk sums).
__global__ void __launch_bounds__(256) k_emit(const int32_t* __restrict__ x, int64_t n, int lo,
                                              const unsigned long long* __restrict__ code,
                                              const unsigned long long* __restrict__ chunk_off,
                                              unsigned long long* __restrict__ words) {
  constexpr int PER = kEncChunk / 256;
  const int64_t c0 = int64_t(blockIdx.x) * kEncChunk;
  const int64_t i0 = c0 + int64_t(threadIdx.x) * PER;
  unsigned long long mine = 0;
  for (int k = 0; k < PER; ++k)
    if (i0 + k < n) mine += code[x[i0 + k] - lo] & 63ull;
  // block exclusive scan of `mine`
  unsigned long long incl = mine;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __shared__ unsigned long long wsum[8];
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  unsigned long long before = 0;
  for (int w = 0; w < warp; ++w) before += wsum[w];
  unsigned long long off = chunk_off[blockIdx.x] + before + incl - mine;
  for (int k = 0; k < PER; ++k) {
    if (i0 + k >= n) break;
    const unsigned long long cw = code[x[i0 + k] - lo];
    const int len = int(cw & 63ull);
    const unsigned long long bits = cw >> 6;
    const unsigned long long w = off >> 6;
    const int sh = int(off & 63ull);
    atomicOr(&words[w], bits << sh);
    if (sh + len > 64) atomicOr(&words[w + 1], bits >> (64 - sh));
    off += len;
  }
}

}  // namespace

cudaError_t label_minmax(const int32_t* x, int64_t n, int* d_mm, const Exec& ex) {
  const int init[2] = {INT32_MAX, INT32_MIN};
  cudaError_t e = cudaMemcpyAsync(d_mm, init, sizeof(init), cudaMemcpyHostToDevice, ex.s);
  if (e != cudaSuccess) return e;
  MGRX_LAUNCH(ex, "enc_minmax", k_label_minmax<<<grid_for(n, 256, 4), 256, 0, ex.s>>>(x, n, d_mm));
  return cudaGetLastError();
}

cudaError_t label_hist(const int32_t* x, int64_t n, int lo, int range, unsigned long long* d_freq, const Exec& ex) {
  cudaError_t e = cudaMemsetAsync(d_freq, 0, size_t(range) * 8, ex.s);
  if (e != cudaSuccess) return e;
  const int smem_bins = 12 * 1024;  // 48 KB of per-block counts
  const size_t sm = range <= smem_bins ? size_t(range) * 4 : 0;
  MGRX_LAUNCH(ex, "enc_hist", k_label_hist<<<grid_for(n, 256, 4), 256, sm, ex.s>>>(x, n, lo, range, d_freq, smem_bins));
  return cudaGetLastError();
}

int64_t enc_chunks(int64_t n) { return (n + kEncChunk - 1) / kEncChunk; }

cudaError_t label_chunk_bits(const int32_t* x, int64_t n, int lo, const unsigned long long* d_code,
                             unsigned long long* d_chunk_bits, const Exec& ex) {
  MGRX_LAUNCH(ex, "enc_chunks", k_chunk_bits<<<unsigned(enc_chunks(n)), 256, 0, ex.s>>>(x, n, lo, d_code, d_chunk_bits));
  return cudaGetLastError();
}

cudaError_t label_emit(const int32_t* x, int64_t n, int lo, const unsigned long long* d_code,
                       const unsigned long long* d_chunk_off, unsigned long long* d_words, uint64_t nwords,
                       const Exec& ex) {
  cudaError_t e = cudaMemsetAsync(d_words, 0, size_t(nwords) * 8, ex.s);
  if (e != cudaSuccess) return e;
  MGRX_LAUNCH(ex, "enc_emit", k_emit<<<unsigned(enc_chunks(n)), 256, 0, ex.s>>>(x, n, lo, d_code, d_chunk_off, d_words));
  return cudaGetLastError();
}

}  // namespace mgrx_b200
