// Shared device-side definitions for the mgrx_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mgrx_b200.h"

namespace mgrx_b200 {

constexpr int kMaxD = MGRX_MAX_DIMS;
constexpr int kMaxLevels = 64;
constexpr int kNumSMs = 148;

// Mass-matrix constants with the common spacing cancelled
// (reference transform.hpp:17-21) and the load-vector stencil weights
// (transform.hpp:84-96).  Written as the same constant expressions so the
// rounded doubles are identical.
constexpr double kOff = 1.0 / 3.0;
constexpr double kDiagB = 2.0 / 3.0;
constexpr double kDiagI = 4.0 / 3.0;
// Toeplitz form of the correction solves (fused3d.cu "Toeplitz solves"): the
// limit of the ThomasAux factors, w = 2 - sqrt(3) (w^2 - 4 w + 1 = 0) and
// 1 / d with d = 4/3 - w / 3.
constexpr double kTw = 2.0 - 1.7320508075688772;
constexpr double kTid = 1.0 / (kDiagI - kTw * kOff);
constexpr int kToepEnds = 32;   // end-correction entries per side
constexpr int kToepMinM = 40;   // shortest line solved this way (the two ends decouple below 1e-22)
constexpr double kW12 = 1.0 / 12.0;
constexpr double kW5_12 = 5.0 / 12.0;
constexpr double kW5_6 = 5.0 / 6.0;

// Exact-order fp64 helpers: the reference is compiled with
// -ffp-contract=off (proj/CMakeLists.txt:12-14); the bitwise-parity kernels
// use the _rn intrinsics so nvcc cannot fuse a multiply into an add.
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }

// static_cast<T>(double) with round-to-nearest, like the host cast.
template <typename T> __device__ __forceinline__ T to_t(double v);
template <> __device__ __forceinline__ float to_t<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ double to_t<double>(double v) { return v; }

// Division by a run-time invariant 32-bit divisor (Granlund-Montgomery):
// exact for every 32-bit dividend.
struct FastDiv {
  uint32_t d, mul, shift;  // shift == 0 encodes d == 1
  __host__ __device__ FastDiv() : d(1), mul(0), shift(0) {}
  __host__ explicit FastDiv(uint32_t div) : d(div), mul(0), shift(0) {
    if (div <= 1) return;
    uint32_t l = 0;
    while ((uint64_t(1) << l) < div) ++l;  // ceil(log2(div))
    mul = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << l) - div)) / div + 1);
    shift = l;
  }
  __device__ __forceinline__ uint32_t div(uint32_t x) const {
    if (shift == 0) return x;
    const uint32_t t = __umulhi(mul, x);
    return (t + ((x - t) >> 1)) >> (shift - 1);
  }
};

// Geometry of one level pass: fine extents n (level l), coarse extents m
// (level l-1), natural row-major strides of the fine block, and the shell
// packing constants of pack_level_centric (reorder.hpp:180-215).
struct LevelGeom {
  int d;
  int64_t n[kMaxD], m[kMaxD];
  int64_t st[kMaxD];   // fine natural strides
  int64_t cst[kMaxD];  // coarse natural strides
  int64_t pm[kMaxD];   // prod_{i<k<d-1} m_k  (inside-row counting)
  int64_t N, Nc;       // fine / coarse element counts
  FastDiv fn[kMaxD];   // divisors by n[i] (32-bit index path)
};

// Per-axis nonuniform tables of one level (see nonuniform.cpp for the
// derivation); device pointers.  Unused on the uniform path.
struct NuAxis {
  const double* wl;   // [n] left interpolation weight at odd j
  const double* wr;   // [n] right interpolation weight at odd j
  const double* s;    // [5m] load stencil
  const double* tw;   // [m] Thomas w
  const double* tid;  // [m] Thomas 1/d
  const double* off;  // [m] super diagonal
};
struct NuLevel {
  NuAxis ax[kMaxD];
};

// Uniform Thomas factors (ThomasAux, transform.hpp:25-44) of one level.
struct ThomasLevel {
  const double* w[kMaxD];
  const double* inv_d[kMaxD];
};

// Launch context handed to the kernel translation units: the stream, the
// context's launch counter and (when profiling is on) the event profiler.
struct Profiler;
struct Exec {
  cudaStream_t s;
  uint64_t* launches;
  Profiler* prof;
  int level = -1;  // hierarchy level being processed (profiling key), -1 = none
  unsigned* nonfinite = nullptr;  // finest level of a compress: check_finite fused into its first pass
  cudaEvent_t after_plane = nullptr;  // recorded after a fused level's decompose plane pass (its shell is final)
};
// Records a CUDA event before/after a tagged launch when profiling
// (api.cu); no-op otherwise.
void prof_mark(const Exec& ex, const char* tag, bool begin);

#define MGRX_LAUNCH(ex, tag, ...)           \
  do {                                       \
    if ((ex).prof) prof_mark(ex, tag, true); \
    __VA_ARGS__;                             \
    ++*(ex).launches;                        \
    if ((ex).prof) prof_mark(ex, tag, false); \
  } while (0)

// Programmatic dependent launch: kernels of a level chain are launched with
// programmatic stream serialization, so the next kernel's CTAs are launched
// (and run their prologue) while the previous kernel drains; they call
// pdl_wait() before touching memory the previous kernel writes or reads
// (griddepcontrol.wait returns once the previous grid has completed and its
// memory is visible; a no-op when launched without the attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              bool pdl, Args... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;  // plain serialisation while profiling (per-kernel event times)
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

inline int grid_for(int64_t work, int block, int per_sm = 16) {
  int64_t g = (work + block - 1) / block;
  const int64_t cap = int64_t(kNumSMs) * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return int(g);
}

}  // namespace mgrx_b200
