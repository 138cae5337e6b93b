// Internal launch interface between the C-ABI layer (api.cu) and the kernel
// translation units.  Not part of the public boundary.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mgrx_b200 {

// ---- general per-step path (general.cu) -----------------------------------
template <typename T>
// fast: parallel load + segmented Thomas sweeps (path "auto"); false: the
// serial per-line sweeps, bit-identical to the reference (path "general")
cudaError_t general_decompose_level(const T* blk, T* shell, T* coarse, double* comp, double* tmp,
                                    const LevelGeom& g, const ThomasLevel* th, const NuLevel* nu, const Exec& ex,
                                    bool fast);
template <typename T>
cudaError_t general_recompose_level(const T* shell, T* coarse, T* fine, double* comp, double* tmp,
                                    const LevelGeom& g, const ThomasLevel* th, const NuLevel* nu, const Exec& ex,
                                    bool fast);

template <typename T>
cudaError_t apply_correction(T* coarse, const double* z, int64_t n, double sign, const Exec& ex);

// ---- adaptive stop decision (adaptive.cu) -----------------------------------
// Sampled 3^d blocks of a level block (anchor step `step`): their count, and
// per block the (lorenzo, interp) sums of estimate_block_errors into out.
int64_t stop_blocks(int d, const int64_t* ext, int step);
template <typename T>
cudaError_t block_errors(const T* blk, int d, const int64_t* ext, int step, double e, const double* interp_pen,
                         double lorenzo_pen, double* out, const Exec& ex);

// ---- field statistics (adaptive.cu): per block min / max / first non-finite
int field_stats_blocks(int64_t n);
template <typename T>
cudaError_t field_stats(const T* x, int64_t n, double* bmin, double* bmax, unsigned long long* bbad, const Exec& ex);

// ---- Lorenzo coder (lorenzo.cu): hyperplane wavefront in one CTA -------------
template <typename T>
cudaError_t lorenzo_run(const T* x, int d, const int64_t* n, const uint32_t* order, const uint32_t* hs, int H,
                        double e, int32_t* labels, uint8_t* outl, T* recon, uint64_t* opos, T* oval, uint64_t cap,
                        unsigned long long* count, const Exec& ex);

// ---- label entropy coding (huffman.cu) ---------------------------------------
cudaError_t label_minmax(const int32_t* x, int64_t n, int* d_mm, const Exec& ex);
cudaError_t label_hist(const int32_t* x, int64_t n, int lo, int range, unsigned long long* d_freq, const Exec& ex);
int64_t enc_chunks(int64_t n);
// d_code[s] = (reversed code << 6) | length
cudaError_t label_chunk_bits(const int32_t* x, int64_t n, int lo, const unsigned long long* d_code,
                             unsigned long long* d_chunk_bits, const Exec& ex);
cudaError_t label_emit(const int32_t* x, int64_t n, int lo, const unsigned long long* d_code,
                       const unsigned long long* d_chunk_off, unsigned long long* d_words, uint64_t nwords,
                       const Exec& ex);

// ---- tail: all small levels in one CTA (general.cu) -------------------------
size_t tail_smem_bytes(int64_t nmax, int esize);
size_t tail_level_bytes();
void tail_fill_level(void* dst, const LevelGeom& g, const ThomasLevel& th, int64_t shell_off);
template <typename T>
cudaError_t tail_decompose(const T* blk, T* out, T* coarse_out, const void* d_levels, const void* d_nu, int nlev,
                           int64_t nmax, int d, const Exec& ex);
template <typename T>
cudaError_t tail_recompose(const T* coeffs, const T* coarse_in, T* fine_out, const void* d_levels, const void* d_nu,
                           int nlev, int64_t nmax, int d, const Exec& ex);

// ---- quantization (quantize.cu) --------------------------------------------
struct QuantLevels {
  int first, last;         // level range [first, last]
  int64_t base, total;     // quantized positions [base, total)
  int64_t end[kMaxLevels]; // end position (exclusive) of level l = node_count(l)
  double q[kMaxLevels];    // bin widths
  double inv[kMaxLevels];  // 1 / q (fast path of the division; exact fallback near ties)
};
int64_t quant_num_chunks(const QuantLevels& ql);
template <typename T>
cudaError_t quantize_pass1(const T* c, int32_t* labels, uint32_t* chunk_counts, uint64_t* offsets, int* flags,
                           const QuantLevels& ql, const Exec& ex);
template <typename T>
cudaError_t quantize_pass2(const T* c, const uint32_t* chunk_counts, const uint64_t* offsets, uint64_t* opos,
                           T* oval, uint64_t capacity, const QuantLevels& ql, const Exec& ex);
// chunk ranges (the overlapped decompose + quantize / dequantize + recompose):
// first chunk lying entirely at or after position pos
int64_t quant_chunk_of(const QuantLevels& ql, int64_t pos);
template <typename T>
cudaError_t quantize_labels_range(const T* c, int32_t* labels, uint32_t* chunk_counts, int* flags,
                                  const QuantLevels& ql, int64_t chunk_begin, int64_t chunk_end, const Exec& ex);
cudaError_t quantize_scan(const uint32_t* chunk_counts, uint64_t* offsets, const QuantLevels& ql, const Exec& ex);
template <typename T>
cudaError_t dequantize_range(const int32_t* labels, const uint64_t* opos, const T* oval, uint64_t n_out, T* c,
                             const QuantLevels& ql, int64_t chunk_begin, int64_t chunk_end, const Exec& ex);
template <typename T>
cudaError_t dequantize_run(const int32_t* labels, const uint64_t* opos, const T* oval, uint64_t n_out, T* c,
                           const QuantLevels& ql, const Exec& ex);

}  // namespace mgrx_b200
