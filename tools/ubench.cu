// Microbenchmarks of the B200 pipes the level passes lean on (fp64 FMA,
// f32<->f64 conversions, shuffles, shared loads) plus cluster occupancy and
// a plain streaming copy.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o tools/ubench tools/ubench.cu ; run on the B200 box.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = fma(x0, a, 1.0); x1 = fma(x1, a, 1.0); x2 = fma(x2, a, 1.0); x3 = fma(x3, a, 1.0);
    x4 = fma(x4, a, 1.0); x5 = fma(x5, a, 1.0); x6 = fma(x6, a, 1.0); x7 = fma(x7, a, 1.0);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_dadd(double* out, double a) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 += a; x1 += a; x2 += a; x3 += a; x4 += a; x5 += a; x6 += a; x7 += a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// float -> double conversions (independent): F2F.F64.F32
__global__ void k_f2d(double* out, float a) {
  float f[8];
  unsigned long long acc[8];
  for (int k = 0; k < 8; ++k) { f[k] = a * (threadIdx.x + k); acc[k] = 0; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double d = (double)f[k];
      asm volatile("" : "+d"(d));
      acc[k] ^= __double_as_longlong(d);  // keep live
      f[k] = __int_as_float(__float_as_int(f[k]) + 1);
    }
  }
  unsigned long long s = 0;
  for (int k = 0; k < 8; ++k) s ^= acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __longlong_as_double(s);
}

// double -> float conversions: F2F.F32.F64
__global__ void k_d2f(float* out, double a) {
  double d[8];
  unsigned acc[8];
  for (int k = 0; k < 8; ++k) { d[k] = a * (threadIdx.x + k); acc[k] = 0; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float f = __double2float_rn(d[k]);
      asm volatile("" : "+f"(f));
      acc[k] ^= __float_as_uint(f);
      d[k] = __longlong_as_double(__double_as_longlong(d[k]) + 1);
    }
  }
  unsigned s = 0;
  for (int k = 0; k < 8; ++k) s ^= acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(s);
}

__global__ void k_shfl(float* out, float a) {
  float x[8];
  for (int k = 0; k < 8; ++k) x[k] = a + threadIdx.x + k;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __shfl_down_sync(0xffffffffu, x[k], 1);
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lds(float* out, int stride) {
  __shared__ float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  float s = 0;
  int idx = threadIdx.x;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) s += sm[(idx + k * 1024) & 8191];
    idx += stride;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  const size_t st = size_t(gridDim.x) * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

__global__ void k_cl(int* p) { if (p) p[0] = 1; }

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  const int nsm = prop.multiProcessorCount;
  double* dout;
  CK(cudaMalloc(&dout, sizeof(double) * nsm * 8 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, double ops_per_thread) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double threads = double(nsm) * 8 * 256;
    const double per_sm_clk = ops_per_thread * threads / (ms * 1e-3) / nsm / (prop.clockRate * 1e3);
    printf("%-8s %.3f ms  %.1f thread-ops/clk/SM (at max clock)  err=%s\n", name, ms, per_sm_clk,
           cudaGetErrorString(cudaGetLastError()));
  };
  const int G = nsm * 8, B = 256;
  run("dfma", [&] { k_dfma<<<G, B>>>(dout, 0.999); }, 8.0 * ITERS);
  run("dadd", [&] { k_dadd<<<G, B>>>(dout, 0.999); }, 8.0 * ITERS);
  run("f2d", [&] { k_f2d<<<G, B>>>(dout, 0.5f); }, 8.0 * ITERS);
  run("d2f", [&] { k_d2f<<<G, B>>>((float*)dout, 0.5); }, 8.0 * ITERS);
  run("shfl", [&] { k_shfl<<<G, B>>>((float*)dout, 0.5f); }, 8.0 * ITERS);
  run("lds", [&] { k_lds<<<G, B>>>((float*)dout, 1); }, 8.0 * ITERS);

  // streaming copy bandwidth, 540 MB each way
  const size_t n = size_t(513) * 513 * 513 / 4;
  float4 *a, *b;
  CK(cudaMalloc(&a, n * 16));
  CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 2; ++rep) {
    for (int g : {nsm * 4, nsm * 8, nsm * 16}) {
      k_copy<<<g, 256>>>(a, b, n);
      cudaEventRecord(e0);
      k_copy<<<g, 256>>>(a, b, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("copy grid %d: %.3f ms  %.0f GB/s (r+w)\n", g, ms, 2.0 * n * 16 / (ms * 1e-3) / 1e9);
    }
  }

  // cluster occupancy: 1 CTA per SM with big shared memory
  for (int cs : {1, 2, 4, 8, 16}) {
    for (int smem : {100 * 1024, 200 * 1024}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 64);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaFuncSetAttribute(k_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      int ncl = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)k_cl, &cfg);
      printf("cluster %2d smem %3d KB: max active clusters %d (%d CTAs) %s\n", cs, smem / 1024, ncl, ncl * cs,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
