// Latency microbenchmarks for the small-block engine's Cholesky (dev tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sb_ubench tools/sb_ubench.cu && tools/sb_ubench
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

__global__ void k_dmma(long long *out, double *sink, int iters) {
  double d[2] = {threadIdx.x * 1e-3, 1.0};
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) dmma(d, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = d[0] + d[1];
}
__global__ void k_dfma(long long *out, double *sink, int iters) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999, 1e-3);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = x;
}
__global__ void k_shfl(long long *out, double *sink, int iters) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = x;
}
__global__ void k_rsqrt(long long *out, double *sink, int iters) {
  double x = 2.0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 + rsqrt_nr(x);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = x;
}
__global__ void k_rsqrt_lib(long long *out, double *sink, int iters) {
  double x = 2.0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 + rsqrt(x);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = x;
}
// one-thread 8 x 8 Cholesky + inverse in registers (the leaf the engine could use)
__global__ void k_leaf1(long long *out, double *sink, int iters) {
  double a[8][8], w[8][8];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) a[i][j] = (i == j ? 8.0 : 0.1) + threadIdx.x * 1e-6;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) w[i][j] = i == j ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double rs = rsqrt_nr(a[k][k]);
      a[k][k] *= rs;
#pragma unroll
      for (int i = k + 1; i < 8; ++i) a[i][k] *= rs;
#pragma unroll
      for (int i = k + 1; i < 8; ++i)
#pragma unroll
        for (int j = k + 1; j <= i; ++j) a[i][j] = fma(-a[i][k], a[j][k], a[i][j]);
#pragma unroll
      for (int j = 0; j <= k; ++j) w[k][j] *= rs;
#pragma unroll
      for (int i = k + 1; i < 8; ++i)
#pragma unroll
        for (int j = 0; j <= k; ++j) w[i][j] = fma(-a[i][k], w[k][j], w[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i][i] += w[i][i] * 1e-30 + 8.0 - a[i][i];  // restore (dependency)
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  double s = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) s += a[i][j] + w[i][j];
  sink[threadIdx.x] = s;
}

int main() {
  long long *d_out, h;
  double *sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&sink, 1024 * 8);
  const int it = 4096;
  auto run = [&](const char *name, void (*k)(long long *, double *, int), int threads) {
    k<<<1, threads>>>(d_out, sink, it);
    k<<<1, threads>>>(d_out, sink, it);
    cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %6lld cycles\n", name, h);
  };
  run("dmma dependent", k_dmma, 32);
  run("dfma dependent", k_dfma, 32);
  run("shfl.f64 dependent", k_shfl, 32);
  run("rsqrt_nr dependent", k_rsqrt, 32);
  run("rsqrt (libdevice) dependent", k_rsqrt_lib, 32);
  run("leaf 8x8 chol+inv 1 thread", k_leaf1, 1);
  run("leaf 8x8 chol+inv 32 thr", k_leaf1, 32);
  return 0;
}
