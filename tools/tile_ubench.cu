// Diagnostic: FP64 DMMA tile main loop throughput vs CTA tile shape (cp.async
// staging from L2-resident panels, [row][k] padded smem, 148 SMs).
//   BM x BN output per CTA, warps of WM x WN, STG stages of KC = 32, MINB CTAs/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tile_ubench tools/tile_ubench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
constexpr int KC = 32, LDMK = KC + 4;
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int R, int NTH>
__device__ __forceinline__ void load_chunk(double *s, const double *g, int ld, int k0) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int it = 0; it < (R * (KC / 2) + NTH - 1) / NTH; ++it) {
    int idx = tid + it * NTH;
    if (idx < R * KC / 2) {
      int r = idx >> 4, kk = (idx & 15) * 2;
      cp_async16(s + r * LDMK + kk, g + (size_t)r * ld + k0 + kk);
    }
  }
}

template <int BM, int BN, int WM, int WN, int NTH, int STG, int MINB>
__global__ void __launch_bounds__(NTH, MINB) kern(const double *A, const double *B, int K, int reps, double *out) {
  extern __shared__ double sm[];
  constexpr int FM = WM / 8, FN = WN / 8, WCOL = BN / WN;
  constexpr int STAGE = (BM + BN) * LDMK;
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = (warp / WCOL) * WM + (lane >> 2), c0 = (warp % WCOL) * WN + (lane >> 2), kq = lane & 3;
  const int nch = K / KC;
  const double *Ag = A + (size_t)(blockIdx.x % 32) * BM * K, *Bg = B + (size_t)((blockIdx.x + 7) % 32) * BN * K;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int j = 0; j < STG - 1; ++j) {
      double *As = sm + j * STAGE;
      load_chunk<BM, NTH>(As, Ag, K, j * KC); load_chunk<BN, NTH>(As + BM * LDMK, Bg, K, j * KC); cp_commit();
    }
    for (int j = 0; j < nch; ++j) {
      cp_wait<STG - 2>();
      __syncthreads();
      if (j + STG - 1 < nch) {
        double *As = sm + ((j + STG - 1) % STG) * STAGE;
        load_chunk<BM, NTH>(As, Ag, K, (j + STG - 1) * KC); load_chunk<BN, NTH>(As + BM * LDMK, Bg, K, (j + STG - 1) * KC);
      }
      cp_commit();
      const double *As = sm + (j % STG) * STAGE, *Bs = As + BM * LDMK;
#pragma unroll
      for (int ks = 0; ks < KC / 4; ++ks) {
        const int kk = ks * 4 + kq;
        double a[FM], b[FN];
#pragma unroll
        for (int mi = 0; mi < FM; ++mi) a[mi] = As[(r0 + mi * 8) * LDMK + kk];
#pragma unroll
        for (int ni = 0; ni < FN; ++ni) b[ni] = Bs[(c0 + ni * 8) * LDMK + kk];
#pragma unroll
        for (int mi = 0; mi < FM; ++mi)
#pragma unroll
          for (int ni = 0; ni < FN; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
      }
    }
    cp_wait<0>();
    __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1234.5) out[0] = s;
}

template <int BM, int BN, int WM, int WN, int NTH, int STG, int MINB>
void run(const double *A, const double *B, double *out, int K) {
  const int smem = STG * (BM + BN) * LDMK * 8;
  auto k = kern<BM, BN, WM, WN, NTH, STG, MINB>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int blocks = 148 * MINB, reps = 20;
  k<<<blocks, NTH, smem>>>(A, B, K, 1, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int t = 0; t < 5; ++t) {
    cudaEventRecord(e0); k<<<blocks, NTH, smem>>>(A, B, K, reps, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * BM * BN * (double)K * reps * blocks;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k);
  printf("BM=%d BN=%d warp %dx%d thr=%d stages=%d ctas/SM=%d smem=%dKB regs=%d K=%d: %.2f TF/s\n", BM, BN, WM, WN, NTH, STG, MINB,
         smem / 1024, fa.numRegs, K, flops / best / 1e9);
}

int main() {
  int K = 1024;
  double *A, *B, *out;
  CK(cudaMalloc(&A, 32ull * 128 * K * 8)); CK(cudaMalloc(&B, 32ull * 128 * K * 8)); CK(cudaMalloc(&out, 64));
  CK(cudaMemset(A, 0, 32ull * 128 * K * 8)); CK(cudaMemset(B, 0, 32ull * 128 * K * 8));
  run<64, 64, 16, 32, 256, 3, 2>(A, B, out, K);    // current engine shape
  run<64, 64, 32, 32, 128, 3, 3>(A, B, out, K);    // 4 warps, 3 CTAs/SM
  run<128, 64, 32, 32, 256, 2, 2>(A, B, out, K);
  run<128, 64, 32, 64, 128, 3, 2>(A, B, out, K);
  run<128, 128, 32, 32, 512, 3, 1>(A, B, out, K);
  run<128, 128, 32, 64, 256, 3, 1>(A, B, out, K);
  run<128, 128, 64, 32, 256, 3, 1>(A, B, out, K);
  run<128, 128, 32, 64, 256, 4, 1>(A, B, out, K);
  return 0;
}
