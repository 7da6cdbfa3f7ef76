// FP64 roofline denominators on the B200 box: DFMA, DMMA (mma.sync m8n8k4 f64),
// cuBLAS DGEMM (burst + sustained) and device copy bandwidth.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks tools/fp64_peaks.cu -lcublas
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
  double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
  const double m = 0.999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1234.5) out[0] = a0;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void dmma_kernel(double* out, int iters) {
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = 1e-3 * threadIdx.x, b = 2e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) dmma(acc[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1234.5) out[0] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  {
    int iters = 20000; int thr = 512, blocks = sms * 4;
    dfma_kernel<<<blocks, thr>>>(out, 100); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_kernel<<<blocks, thr>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    double flops = 2.0 * 8 * 16 * (double)iters * thr * blocks;
    printf(", \"dfma_tflops\": %.2f", flops / best / 1e9);
  }
  // DMMA
  for (int warps_per_block : {4, 8, 16}) {
    int iters = 20000; int thr = 32 * warps_per_block, blocks = sms * 2;
    dmma_kernel<8><<<blocks, thr>>>(out, 100); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dmma_kernel<8><<<blocks, thr>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    double flops = 2.0 * 256 * 8 * (double)iters * (thr / 32) * blocks;
    printf(", \"dmma_tflops_w%d\": %.2f", warps_per_block * 2, flops / best / 1e9);
  }
  // DMMA latency (1 warp, dependent chain)
  {
    int iters = 20000;
    dmma_kernel<1><<<1, 32>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_kernel<1><<<1, 32>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"dmma_dep_ns\": %.2f", ms * 1e6 / iters);
  }
  // cuBLAS DGEMM
  {
    cublasHandle_t h; cublasCreate(&h);
    for (int N : {2048, 4096, 8192}) {
      double *A, *B, *C;
      CK(cudaMalloc(&A, (size_t)N * N * 8)); CK(cudaMalloc(&B, (size_t)N * N * 8)); CK(cudaMalloc(&C, (size_t)N * N * 8));
      cudaMemset(A, 0, (size_t)N * N * 8); cudaMemset(B, 0, (size_t)N * N * 8);
      double al = 1, be = 0;
      cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, N, N, &al, A, N, B, N, &be, C, N);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, N, N, &al, A, N, B, N, &be, C, N);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
      }
      printf(", \"cublas_dgemm_%d_tflops\": %.2f", N, 2.0 * N * N * (double)N / best / 1e9);
      if (N == 8192) {  // sustained ~4 s
        int reps = 0; cudaEventRecord(e0);
        float tot = 0;
        while (tot < 4000.f) {
          for (int r = 0; r < 5; ++r) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, N, N, &al, A, N, B, N, &be, C, N);
          reps += 5; cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&tot, e0, e1);
        }
        printf(", \"cublas_dgemm_8192_sustained_tflops\": %.2f", 2.0 * N * N * (double)N * reps / tot / 1e9);
      }
      cudaFree(A); cudaFree(B); cudaFree(C);
    }
  }
  // copy bandwidth
  {
    size_t bytes = (size_t)4 << 30; void *a, *b;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    cudaMemcpy(b, a, bytes, cudaMemcpyDeviceToDevice); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); cudaMemcpy(b, a, bytes, cudaMemcpyDeviceToDevice); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    printf(", \"d2d_copy_gbs\": %.1f", 2.0 * bytes / best / 1e6);
  }
  printf("}\n");
  return 0;
}
