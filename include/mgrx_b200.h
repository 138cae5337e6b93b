/* mgrx_b200 — C-ABI of the B200-native multilevel decompose / recompose and
 * level-wise quantization path (the hot path of the optimized multigrid
 * compressor, arXiv 2010.05872; reference: /root/reference/proj/core).
 *
 * This is the drop-in boundary.  Every entry point takes plain pointers and
 * sizes; no C++ or torch types cross it and nothing throws across it.  Each
 * function below names the reference interface it replaces (file:line is
 * relative to the reference's proj/core/).
 *
 * Conventions
 *  - Status: MGRX_OK (0) or 1 + the reference's mgrx::errc value
 *    (include/mgrx/error.hpp:9-36), so a host wrapper can rethrow the same
 *    mgrx::Error code.  CUDA failures and argument errors that the reference
 *    cannot produce get codes >= 100.  mgrx_gpu_last_error() returns the
 *    message of the last failure on that context.
 *  - dims: row-major extents, slowest axis first (TensorField, tensor.hpp:20).
 *  - levels: number of levels L, or -1 for the default depth
 *    (GridHierarchy::create, src/grid.cpp:22).
 *  - Device-pointer calls (mgrx_gpu_*) are asynchronous on the context's
 *    stream unless stated otherwise; host-buffer calls (mgrx_host_*) copy in,
 *    compute and copy out, and return after the stream has drained.
 *  - A context is the GPU analogue of SolverWorkspace (transform.hpp:46-75):
 *    it owns a stream, device scratch, uploaded per-level tables and cached
 *    launch plans.  It is not thread-safe; use one per host thread.  Calls on
 *    distinct contexts are independent.
 */
#ifndef MGRX_B200_H
#define MGRX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGRX_B200_ABI_VERSION 1
#define MGRX_MAX_DIMS 8 /* update_coefficients' corner table: offs[1u << 8] (transform.hpp:271) */

typedef struct mgrx_gpu_ctx mgrx_gpu_ctx;

typedef enum { MGRX_F32 = 0, MGRX_F64 = 1 } mgrx_dtype;

/* QuantMode (quantize.hpp:14) */
typedef enum { MGRX_QUANT_UNIFORM = 0, MGRX_QUANT_LEVELWISE = 1 } mgrx_quant_mode;

/* Status codes: 1 + mgrx::errc (error.hpp:9-36), then local codes. */
enum {
  MGRX_OK = 0,
  MGRX_INVALID_DIMS = 1,
  MGRX_DEPTH_EXCEEDED = 2,
  MGRX_INVALID_LEVEL = 3,
  MGRX_INVALID_AXIS = 4,
  MGRX_DEGENERATE_LINE = 5,
  MGRX_DEGENERATE_SYSTEM = 6,
  MGRX_SHAPE_ERROR = 7,
  MGRX_INVALID_BUDGET = 8,
  MGRX_NONFINITE_DATA = 9,
  MGRX_INVALID_INPUT = 15,
  MGRX_CUDA_ERROR = 100,
  MGRX_OUT_OF_MEMORY = 101,
  MGRX_INVALID_ARGUMENT = 102,
  MGRX_CAPACITY_EXCEEDED = 103
};

/* ---- library / context ------------------------------------------------ */

int mgrx_abi_version(void);

/* Creates a context on `device` with its own non-blocking stream.  Replaces
 * SolverWorkspace ws(batch); ws.prepare(h) (transform.hpp:50,58). */
int mgrx_gpu_ctx_create(int device, mgrx_gpu_ctx** out);
int mgrx_gpu_ctx_destroy(mgrx_gpu_ctx* ctx);
/* Run subsequent work on an external stream (cudaStream_t as void*), used
 * as-is: NULL is the legacy default stream (what torch's default stream is).
 * mgrx_gpu_get_stream right after creation returns the context's own stream,
 * which can be passed back here to restore it. */
int mgrx_gpu_set_stream(mgrx_gpu_ctx* ctx, void* stream);
void* mgrx_gpu_get_stream(mgrx_gpu_ctx* ctx);
int mgrx_gpu_synchronize(mgrx_gpu_ctx* ctx);
const char* mgrx_gpu_last_error(const mgrx_gpu_ctx* ctx);
/* Number of kernels this context has launched so far (launch accounting for
 * the benchmark's gpu_launches). */
uint64_t mgrx_gpu_launch_count(const mgrx_gpu_ctx* ctx);
/* Per-kernel CUDA-event timing for roofline reporting: between begin and
 * end every tagged kernel launch is bracketed by events on its stream.  end
 * synchronises and returns, per distinct kernel tag, the summed device
 * time (ms) and launch count; tags are written as 32-byte NUL-terminated
 * slots.  *n = number of distinct tags (rows beyond cap are dropped). */
int mgrx_gpu_profile_begin(mgrx_gpu_ctx* ctx);
int mgrx_gpu_profile_end(mgrx_gpu_ctx* ctx, char* tags, double* ms, uint64_t* counts, int cap, int* n);
/* Select the kernel family: 0 = auto (fused 3-D path where it applies),
 * 1 = general per-step kernels only (bitwise equal to the reference). */
int mgrx_gpu_set_path(mgrx_gpu_ctx* ctx, int path);

/* ---- host metadata (no device work) ------------------------------------ */

/* GridHierarchy::create / level_dims / delta_count (grid.hpp:30-56,
 * grid.cpp:9-49).  level_dims: (L+1) * ndims entries, level 0 (coarsest)
 * first; delta_counts: L+1 entries.  Either output may be NULL. */
int mgrx_hierarchy(int ndims, const uint64_t* dims, int levels, int* out_levels, uint64_t* level_dims,
                   uint64_t* delta_counts);

/* make_plan (quantize.cpp:7-24): bin_widths[L+1], level 0 first. */
int mgrx_make_plan(int mode, double budget, int ndims, const uint64_t* dims, int levels, double* bin_widths);

/* ---- device-pointer entry points ----------------------------------------- */

/* decompose (transform.hpp:509-515): d_field (N elements, row-major, not
 * modified) -> d_out, the level-centric buffer of MultilevelCoefficients
 * (transform.hpp:158-163, layout pack_level_centric reorder.hpp:162). */
int mgrx_gpu_decompose(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                       int stop_level, const void* d_field, void* d_out);

/* recompose (transform.hpp:517-530): level-centric d_coeffs -> d_field. */
int mgrx_gpu_recompose(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                       int stop_level, const void* d_coeffs, void* d_field);

/* Nonuniform-coordinate variants (no reference counterpart: SPEC.md:13,:73
 * normalise the spacing away).  coords[a] is a HOST array of dims[a]
 * strictly increasing coordinates for axis a; with equispaced coordinates
 * the result equals mgrx_gpu_decompose to rounding. */
int mgrx_gpu_decompose_nonuniform(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                                  int stop_level, const double* const* coords, const void* d_field,
                                  void* d_out);
int mgrx_gpu_recompose_nonuniform(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                                  int stop_level, const double* const* coords, const void* d_coeffs,
                                  void* d_field);

/* quantize (quantize.hpp:79-95) for stop_level == 0, quantize_tail
 * (quantize.hpp:99-114) for stop_level > 0.  bin_widths: HOST, L+1 entries.
 * d_labels receives the concatenated per-level LabelStream::labels (levels
 * stop+1..L for a tail, 0..L otherwise).  Outliers (|label| beyond the
 * 16-bit alphabet) are written in strictly increasing position order as
 * required by read_outliers (pipeline.hpp:56-57).  SYNCHRONOUS: returns
 * MGRX_NONFINITE_DATA like quantize_span (quantize.hpp:64), and
 * MGRX_CAPACITY_EXCEEDED (with *n_outliers set) when more than
 * outlier_capacity outliers exist. */
int mgrx_gpu_quantize(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                      int stop_level, const double* bin_widths, const void* d_coeffs, int32_t* d_labels,
                      uint64_t* d_outlier_pos, void* d_outlier_val, uint64_t outlier_capacity,
                      uint64_t* n_outliers);

/* dequantize / dequantize_tail (quantize.hpp:118-150): labels -> d_coeffs,
 * then outliers restored exactly.  For stop_level > 0 the coarse block
 * [0, node_count(stop)) of d_coeffs is left untouched. */
int mgrx_gpu_dequantize(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                        int stop_level, const double* bin_widths, const int32_t* d_labels,
                        const uint64_t* d_outlier_pos, const void* d_outlier_val, uint64_t n_outliers,
                        void* d_coeffs);

/* decompose (transform.hpp:485-506) followed by quantize / quantize_tail
 * (quantize.hpp:79-114) of its output — the ★ pair compress_field runs back
 * to back (pipeline.hpp:145-183) — as ONE call: d_coeffs receives decompose's
 * buffer, d_labels / outliers quantize's output, results identical to the
 * two calls.  The finest shell (7/8 of a 3-D field) is final after the first
 * plane pass, so its labels are produced on a low-priority side stream under
 * the rest of the decomposition (the solves and every coarser level), which
 * runs on a high-priority stream: the quantizer's read of the coefficients
 * leaves the critical path.  SYNCHRONOUS like mgrx_gpu_quantize (same
 * errors). */
int mgrx_gpu_decompose_quantize(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                                int stop_level, const void* d_field, const double* bin_widths, void* d_coeffs,
                                int32_t* d_labels, uint64_t* d_outlier_pos, void* d_outlier_val,
                                uint64_t outlier_capacity, uint64_t* n_outliers);

/* dequantize / dequantize_tail (quantize.hpp:118-150) followed by recompose
 * (transform.hpp:509-530) — the ★ pair of decompress_field
 * (pipeline.hpp:235-260) — as one call: d_coeffs receives the dequantized
 * buffer (for stop_level > 0 its coarse block must already hold the decoded
 * coarse values), d_field the reconstruction; identical to the two calls.
 * Without outliers the finest shell is dequantized on the stream of the finest
 * level's correction while the coarser levels recompose beside it. */
int mgrx_gpu_dequantize_recompose(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                                  int stop_level, const double* bin_widths, const int32_t* d_labels,
                                  const uint64_t* d_outlier_pos, const void* d_outlier_val, uint64_t n_outliers,
                                  void* d_coeffs, void* d_field);

/* ---- host-buffer entry points (end-to-end: H2D + compute + D2H) ---------- */

/* decompress_field's ★ pair (pipeline.hpp:235-260) from HOST buffers in one
 * device-resident pass: labels (+ outliers, + for stop_level > 0 the decoded
 * coarse block of node_count(stop) values, else NULL) go to the GPU,
 * mgrx_gpu_dequantize_recompose runs there, only the field comes back. */
int mgrx_host_decompress(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                         int stop_level, const double* bin_widths, const int32_t* h_labels,
                         const uint64_t* h_outlier_pos, const void* h_outlier_val, uint64_t n_outliers,
                         const void* h_coarse, void* h_field);

int mgrx_host_decompose(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                        int stop_level, const void* h_field, void* h_out);
int mgrx_host_recompose(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                        int stop_level, const void* h_coeffs, void* h_field);

/* quantize / dequantize on host buffers (same semantics as the device
 * versions; outliers written to host arrays of outlier_capacity entries). */
int mgrx_host_quantize(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels, int stop_level,
                       const double* bin_widths, const void* h_coeffs, int32_t* h_labels, uint64_t* h_outlier_pos,
                       void* h_outlier_val, uint64_t outlier_capacity, uint64_t* n_outliers);
int mgrx_host_dequantize(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels, int stop_level,
                         const double* bin_widths, const int32_t* h_labels, const uint64_t* h_outlier_pos,
                         const void* h_outlier_val, uint64_t n_outliers, void* h_coeffs);

/* Device scratch a decompose/recompose of this shape needs (bytes). */
int mgrx_gpu_workspace_size(int dtype, int ndims, const uint64_t* dims, int levels, int stop_level,
                            uint64_t* bytes);

/* ---- adaptive stop decision ---------------------------------------------
 * choose_stop (adaptive.hpp:99-104; anchor_step 8, choose_stop_full: 2) on a
 * level block already in device memory (natural row-major order,
 * level_dims extents): per sampled 3^d block estimate_block_errors
 * (src/adaptive.cpp:74-138) on the GPU, the blocks summed in anchor order on
 * the host.  interp_penalty[k - 1] (k = 1..ndims) and lorenzo_penalty are
 * the PenaltyModel's (adaptive.hpp:16-21); e the level's error bound.
 * *stop = 1 when the Lorenzo estimate is lower (or the block is too small to
 * sample), else 0; totals (optional) = {lorenzo, interp}.  Synchronous. */
int mgrx_gpu_choose_stop(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* level_dims, const void* d_block,
                         double e, const double* interp_penalty, double lorenzo_penalty, int anchor_step,
                         double* totals, int* stop);

/* decompose_with (transform.hpp:485-506) with the reference's adaptive
 * decider — compress(adaptive) (pipeline.hpp:148-156) — on host buffers,
 * the level blocks staying on the device: before level l (L..min_stop+1),
 * mgrx_gpu_choose_stop with e_per_level[l], interp_penalty[l * ndims ..]
 * and lorenzo_penalty[l] (arrays indexed by level, L + 1 entries; the
 * caller evaluates penalty_model_for per level, adaptive.cpp:55-72) decides
 * whether to stop there.  h_out receives the level-centric buffer of the
 * whole field (coarse block of the stop level first), *stop_level the stop. */
int mgrx_host_decompose_adaptive(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                                 const void* h_field, const double* e_per_level, const double* interp_penalty,
                                 const double* lorenzo_penalty, int anchor_step, int min_stop_level, void* h_out,
                                 int* stop_level);

/* ---- label entropy coding -------------------------------------------------
 * encode_labels (src/huffman.cpp:209-255) of n device-resident labels: the
 * reference's exact byte stream (min, range, code-length table, bit count,
 * canonical Huffman codes bit-reversed and packed LSB-first) written to the
 * host buffer h_out (capacity bytes; *out_size = the stream's size, also
 * when it does not fit: MGRX_CAPACITY_EXCEEDED).  Histogram and bit packing
 * run on the GPU, only the encoded bytes come back.  Synchronous. */
int mgrx_gpu_encode_labels(mgrx_gpu_ctx* ctx, const int32_t* d_labels, uint64_t n, uint8_t* h_out, uint64_t capacity,
                           uint64_t* out_size);

/* compress_lorenzo (lorenzo.hpp:87-128) of a row-major block (host buffer,
 * dims extents) with error bound e, on the GPU (hyperplane wavefront): the
 * labels come back already entropy-coded (encode_labels' byte stream in
 * h_enc, *enc_size bytes), the outliers in position order.  Bit-identical to
 * the reference.  MGRX_CAPACITY_EXCEEDED (with the needed size / count set)
 * when a buffer is too small.  Synchronous. */
int mgrx_host_lorenzo(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, const void* h_block, double e,
                      uint8_t* h_enc, uint64_t enc_capacity, uint64_t* enc_size, uint64_t* h_outlier_pos,
                      void* h_outlier_val, uint64_t outlier_capacity, uint64_t* n_outliers);

/* check_finite (pipeline.hpp:113-118) + the value range in one read of n
 * device values: min / max of the finite values (+inf / -inf when none) and
 * the offset of the first non-finite value (n when all are finite).
 * Synchronous. */
int mgrx_gpu_field_stats(mgrx_gpu_ctx* ctx, int dtype, uint64_t n, const void* d_field, double* min_value,
                         double* max_value, uint64_t* first_nonfinite);

/* decompose (as mgrx_gpu_decompose) with check_finite and the range of the
 * field (pipeline.hpp:113-118; the range gives the absolute bound of a
 * relative tolerance) computed in the same read: on the fused 3-D path the
 * finest level's plane pass folds them in; otherwise (or to locate the first
 * non-finite value) a field_stats pass runs.  Outputs as
 * mgrx_gpu_field_stats; MGRX_NONFINITE_DATA (the reference's message) when a
 * value is inf / NaN.  Synchronous. */
int mgrx_gpu_decompose_checked(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels,
                               int stop_level, const void* d_field, void* d_out, double* min_value,
                               double* max_value, uint64_t* first_nonfinite);

/* compress (pipeline.hpp:130-196) up to its sections, device-resident: the
 * field's check_finite runs on the device copy (MGRX_NONFINITE_DATA with the
 * reference's message); the field goes to the GPU once; the stop level is
 * force_stop (>= 0), else the
 * adaptive decision (adaptive != 0; e_per_level / interp_penalty /
 * lorenzo_penalty as for mgrx_host_decompose_adaptive), else 0; decompose,
 * quantize (bin_widths: make_plan's, L + 1 entries) and each level's
 * encode_labels run on the GPU.  Returns: *stop_level; for stop < L the
 * encoded label streams of levels (stop ? stop + 1 : 0)..L back to back in
 * h_sections with section_sizes[l] bytes each (L + 1 entries, 0 for absent
 * levels), the outliers (strictly increasing positions), and for stop > 0
 * the coarse block (node_count(stop) values) in h_coarse for the caller's
 * Lorenzo coder.  For stop == L nothing else is produced (Lorenzo only). */
int mgrx_host_compress(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels, const void* h_field,
                       const double* bin_widths, int adaptive, int force_stop, const double* e_per_level,
                       const double* interp_penalty, const double* lorenzo_penalty, uint8_t* h_sections,
                       uint64_t sections_capacity, uint64_t* section_sizes, uint64_t* h_outlier_pos,
                       void* h_outlier_val, uint64_t outlier_capacity, uint64_t* n_outliers, void* h_coarse,
                       int* stop_level);

/* ---- slab mode (one 3-D field sharded by slabs of axis-0 planes) -------
 * The reference has no distributed path; these are the per-pass pieces of
 * decompose_with / recompose (transform.hpp:485-530) for ONE fused 3-D level
 * restricted to a slab, so that a caller holding the slab on one GPU can run
 * a level with its neighbours: it exchanges halo planes, and transposes the
 * fp64 load-vector volume G (m0 x m1 x m2, row-major, global plane indexing)
 * for the axis-0 solve (NCCL all-to-all in paper_2010_05872_b200/slab.py).
 * All buffers are full-size and globally indexed (a rank touches its planes
 * only): the level block `blk` / coarse block / level-centric `out` of the
 * whole field.  `level` is the fine level l of the pass (1 <= l <= L).
 *
 * info[0..8] = n0, n1, n2 (level l), m0, m1, m2 (level l-1), fused (1 when
 * the level runs on the fused 3-D path, which slab mode needs),
 * node_count(l-1) (the level's shell offset), node_count(l). */
int mgrx_gpu_slab_level(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels, int level,
                        int64_t* info);
/* Decompose plane pass for coarse planes [k0, k1): coefficients of the fine
 * planes [2 k0, 2 k1) (and n0 - 1 when k1 = m0) into `out`'s shell, their
 * nodal values into `coarse`, the axis-0/1/2 load vector into G[k0, k1).
 * Reads fine planes [2 k0 - 2, 2 k1] of `blk`.
 *
 * All buffers are indexed globally (plane p of blk at p * n1 * n2, shell
 * entries at their level-centric position).  A rank may hold only its slab:
 * pass base pointers shifted back by the global offset of its first element
 * (only the planes named above are touched), and keep the shells of its even
 * and odd fine planes as two runs — odd_shift (elements) is added to the
 * position of every odd plane's shell entry (0 for one global buffer). */
int mgrx_gpu_slab_dec_plane(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels, int level,
                            uint64_t k0, uint64_t k1, const void* d_blk, void* d_out, void* d_coarse, double* d_G,
                            int64_t odd_shift);
/* Recompose plane pass: the load vector of the shell's coefficients (reads
 * the shells of fine planes [2 k0 - 2, 2 k1]) into G[k0, k1). */
int mgrx_gpu_slab_rec_plane(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels, int level,
                            uint64_t k0, uint64_t k1, const void* d_coeffs, double* d_G, int64_t odd_shift);
/* Axis-2 and axis-1 solves (batched_solve, transform.hpp:116-130) of G's
 * planes [k0, k1), in place. */
int mgrx_gpu_slab_inplane(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels, int level,
                          uint64_t k0, uint64_t k1, double* d_G);
/* Axis-0 solve of a transposed block Gt[m0][width] (full axis-0 columns),
 * in place. */
int mgrx_gpu_slab_axis0(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels, int level,
                        uint64_t width, double* d_Gt);
/* coarse[i] = T(double(coarse[i]) + sign * z[i]), i < n (apply_correction,
 * transform.hpp:435-477). */
int mgrx_gpu_slab_apply(mgrx_gpu_ctx* ctx, int dtype, void* d_coarse, const double* d_z, uint64_t n, double sign);
/* Recompose interpolation of the fine planes [p0, p1) (p0 even) from the
 * corrected coarse block (planes [p0 / 2, (p1 + 1) / 2]) and the shell. */
int mgrx_gpu_slab_interp(mgrx_gpu_ctx* ctx, int dtype, int ndims, const uint64_t* dims, int levels, int level,
                         uint64_t p0, uint64_t p1, const void* d_coeffs, const void* d_coarse, void* d_fine,
                         int64_t odd_shift);
/* K-pack for the all-to-all of slab mode: dst[q] = the rows x (c1 - c0)
 * block of src (row pitch `pitch` doubles) at columns [cb[q], cb[q+1]) for
 * q < nparts, packed back to back (unpack: the inverse scatter). */
int mgrx_gpu_slab_pack(mgrx_gpu_ctx* ctx, const double* d_src, uint64_t rows, uint64_t pitch, const uint64_t* cb,
                       int nparts, double* d_dst);
int mgrx_gpu_slab_unpack(mgrx_gpu_ctx* ctx, const double* d_src, uint64_t rows, uint64_t pitch, const uint64_t* cb,
                         int nparts, double* d_dst);

#ifdef __cplusplus
}
#endif
#endif /* MGRX_B200_H */
