/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the parity tests.
 *
 * Plain-C restatement of the reference's hot path (multilevel decompose /
 * recompose and level-wise quantization, /root/reference/proj/core).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it; the product library never links it.
 *
 * Parity pins (see tests/test_oracle.py): bitwise against the unmodified
 * reference built into oracle/_ref/libmgrx_ref.so on every shape the
 * reference's own tests use, plus the reference tests' stated known answers
 * (test_transform.cpp:35-154, test_reorder.cpp:32-67, test_grid.cpp:11-97,
 * test_quantize.cpp:19-93) committed as tests/golden/ fixtures.
 *
 * The nonuniform-coordinate functions (mo_*_nu) have no reference
 * counterpart: they are pinned by reduction to the uniform
 * path, by exact quadrature and by a dense solve.
 *
 * Return value: 0 or 1 + mgrx::errc (error.hpp:9-36). */
#ifndef MGRX_ORACLE_H
#define MGRX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int mo_max_levels(int nd, const uint64_t* dims, int* out);
int mo_hierarchy(int nd, const uint64_t* dims, int levels, int* out_levels, uint64_t* level_dims,
                 uint64_t* delta_counts);
int mo_make_plan(int mode, double budget, int nd, const uint64_t* dims, int levels, double* q);

int mo_load_vector_1d(const double* line, uint64_t n, double* out);
int mo_thomas_aux(uint64_t m, double* w, double* inv_d);
int mo_solve_correction_1d(double* f, uint64_t m);

int mo_decompose_f64(int nd, const uint64_t* dims, int levels, int stop, const double* in, double* out);
int mo_decompose_f32(int nd, const uint64_t* dims, int levels, int stop, const float* in, float* out);
int mo_recompose_f64(int nd, const uint64_t* dims, int levels, int stop, const double* in, double* out);
int mo_recompose_f32(int nd, const uint64_t* dims, int levels, int stop, const float* in, float* out);

/* coords: nd pointers, coords[a] has dims[a] strictly increasing entries. */
int mo_decompose_nu_f64(int nd, const uint64_t* dims, int levels, int stop, const double* const* coords,
                        const double* in, double* out);
int mo_recompose_nu_f64(int nd, const uint64_t* dims, int levels, int stop, const double* const* coords,
                        const double* in, double* out);
int mo_decompose_nu_f32(int nd, const uint64_t* dims, int levels, int stop, const double* const* coords,
                        const float* in, float* out);
int mo_recompose_nu_f32(int nd, const uint64_t* dims, int levels, int stop, const double* const* coords,
                        const float* in, float* out);
/* nonuniform 1-D load vector and mass solve for one line with coordinates x */
int mo_load_vector_nu_1d(const double* line, const double* x, uint64_t n, double* out);
int mo_solve_correction_nu_1d(double* f, const double* X, uint64_t m);

int mo_quantize_f64(int nd, const uint64_t* dims, int levels, int stop, const double* q, const double* c,
                    int32_t* labels, uint64_t* opos, double* oval, uint64_t cap, uint64_t* n_out);
int mo_quantize_f32(int nd, const uint64_t* dims, int levels, int stop, const double* q, const float* c,
                    int32_t* labels, uint64_t* opos, float* oval, uint64_t cap, uint64_t* n_out);
int mo_dequantize_f64(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                      const int32_t* labels, const uint64_t* opos, const double* oval, uint64_t n_out,
                      double* c);
int mo_dequantize_f32(int nd, const uint64_t* dims, int levels, int stop, const double* q,
                      const int32_t* labels, const uint64_t* opos, const float* oval, uint64_t n_out,
                      float* c);

#ifdef __cplusplus
}
#endif
#endif
