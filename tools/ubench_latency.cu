// Latency microbenchmarks for the POTRF critical path design (dev tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_latency tools/ubench_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_sync(long long *out, int iters) {
  __shared__ double buf[64];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  (void)buf;
}

__global__ void k_sync_lds_div(long long *out, int iters, double *sink) {
  __shared__ double buf[3][64];
  if (threadIdx.x < 64) buf[0][threadIdx.x] = 1.0 + threadIdx.x;
  __syncthreads();
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 16) buf[(i + 1) % 3][threadIdx.x] = acc + i;
    __syncthreads();
    double d = buf[i % 3][i & 63] + 2.0;
    acc += 1.0 / d;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = acc;
}

__global__ void k_sync_lds_rsqrt(long long *out, int iters, double *sink) {
  __shared__ double buf[3][64];
  if (threadIdx.x < 64) buf[0][threadIdx.x] = 1.0 + threadIdx.x;
  __syncthreads();
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 16) buf[(i + 1) % 3][threadIdx.x] = acc + i;
    __syncthreads();
    double d = buf[i % 3][i & 63] + 2.0;
    acc += rsqrt(d);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = acc;
}

__global__ void k_dep_div(long long *out, int iters, double *sink) {
  double x = 1.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 1.0);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = x;
}
__global__ void k_dep_dfma(long long *out, int iters, double *sink) {
  double x = 1.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999, 1e-3);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = x;
}
__global__ void k_dep_rsqrt(long long *out, int iters, double *sink) {
  double x = 1.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x + 1.0);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = x;
}
__global__ void k_dep_shfl(long long *out, int iters, double *sink) {
  double x = 1.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffff, x, (i + 1) & 31) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = x;
}
__global__ void k_dep_lds(long long *out, int iters, double *sink) {
  __shared__ double buf[64];
  buf[threadIdx.x & 63] = threadIdx.x & 63;
  __syncwarp();
  int idx = threadIdx.x & 63;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = (int)buf[idx];
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = idx;
}
__global__ void k_clock(long long *out) {
  long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  while (clock64() - t0 < 100000000LL) {}
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  out[0] = (long long)(g1 - g0);
}

int main() {
  long long *d, h;
  double *sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 4096);
  int it = 10000;
  auto run = [&](const char *name, auto f) {
    f(); cudaDeviceSynchronize(); f(); cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %lld cycles\n", name, h);
  };
  for (int nt : {32, 128, 256, 512}) {
    char buf[64];
    sprintf(buf, "syncthreads nt=%d", nt);
    run(buf, [&] { k_sync<<<1, nt>>>(d, it); });
    sprintf(buf, "sync+lds+div nt=%d", nt);
    run(buf, [&] { k_sync_lds_div<<<1, nt>>>(d, it, sink); });
    sprintf(buf, "sync+lds+rsqrt nt=%d", nt);
    run(buf, [&] { k_sync_lds_rsqrt<<<1, nt>>>(d, it, sink); });
  }
  run("dependent ddiv", [&] { k_dep_div<<<1, 32>>>(d, it, sink); });
  run("dependent dfma", [&] { k_dep_dfma<<<1, 32>>>(d, it, sink); });
  run("dependent rsqrt(double)", [&] { k_dep_rsqrt<<<1, 32>>>(d, it, sink); });
  run("dependent shfl+dadd", [&] { k_dep_shfl<<<1, 32>>>(d, it, sink); });
  run("dependent lds (f64->int)", [&] { k_dep_lds<<<1, 32>>>(d, it, sink); });
  k_clock<<<1, 1>>>(d);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("clock: 1e8 cycles = %lld ns -> %.0f MHz\n", h, 1e8 / h * 1e3);
  return 0;
}
