// Cycle-level breakdown of the small-block engine's 64 x 64 Cholesky + inverse (dev tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/sb_chol_ubench \
//   tools/sb_chol_ubench.cu paper_2503_17528_b200/csrc/graph.cpp && tools/sb_chol_ubench
#include "../paper_2503_17528_b200/csrc/sb.cu"

#include <cstdio>
#include <vector>

using namespace serinv::sb::dev;

__global__ void k_chol(const double *A, double *out, unsigned long long *st, int reps) {
  extern __shared__ __align__(16) double sm[];
  double *D = sm, *Wd = D + TD, *ldg = Wd + 8 * T, *Ps = ldg + T + 8;
  __shared__ int s_bad;
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < TD; i += NT) D[swz(i >> 6, i & 63)] = A[i];
    __syncthreads();
    unsigned long long t0 = gtimer();
    chol_inv64(D, Wd, Ps, ldg, &s_bad, r == reps - 1 ? st + 1 : nullptr);
    if (threadIdx.x == 0 && r == reps - 1) st[0] = t0;
  }
  for (int i = threadIdx.x; i < TD; i += NT) out[i] = D[swz(i >> 6, i & 63)];
}

int main() {
  std::vector<double> A(4096);
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) A[i * 64 + j] = (i == j ? 64.0 : 0.0) + 1.0 / (1.0 + i + j);
  double *dA, *dO;
  unsigned long long *dS;
  cudaMalloc(&dA, 4096 * 8);
  cudaMalloc(&dO, 4096 * 8);
  cudaMalloc(&dS, 32 * 8);
  cudaMemcpy(dA, A.data(), 4096 * 8, cudaMemcpyHostToDevice);
  const int smem = (TD + 8 * T + T + 8 + 8 * 512) * 8;
  cudaFuncSetAttribute(k_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_chol<<<1, NT, smem>>>(dA, dO, dS, 20);
  cudaDeviceSynchronize();
  unsigned long long s[17];
  cudaMemcpy(s, dS, 17 * 8, cudaMemcpyDeviceToHost);
  printf("chol_inv64 total %.2f us\n", (s[16] - s[0]) / 1e3);
  unsigned long long prev = s[0];
  for (int i = 1; i <= 16; ++i) {
    if (!s[i]) continue;
    printf("  stamp %2d  +%.3f us\n", i - 1, (s[i] - prev) / 1e3);
    prev = s[i];
  }
  // check W * L... : W A W^T = I
  std::vector<double> W(4096);
  cudaMemcpy(W.data(), dO, 4096 * 8, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) {
      double v = 0;
      for (int k = 0; k < 64; ++k)
        for (int m = 0; m < 64; ++m) v += W[i * 64 + k] * A[k * 64 + m] * W[j * 64 + m];
      err = fmax(err, fabs(v - (i == j)));
    }
  printf("max |W A W^T - I| = %.3e\n", err);
  return 0;
}

// ---- GEMM phase throughput: one CTA, 8 warps, mma64 on smem tiles (ideal 64^3: 4096 SM cycles)
__global__ void k_gemm(double *out, unsigned long long *st, int reps, int mode) {
  extern __shared__ __align__(16) double sm[];
  double *A = sm, *B = A + TD;
  for (int i = threadIdx.x; i < 2 * TD; i += NT) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const Frags<2, 4> F = lay64(threadIdx.x >> 5);
  double acc[2][4][2];
  acc_zero(acc);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (mode == 0) mma64<false, true, false>(acc, A, B, F);
    else if (mode == 1) mma64<false, false, false>(acc, A, B, F);
    else if (mode == 2) mma64<true, false, false>(acc, A, B, F);
    else if (mode == 3) mma64<false, true, false, B_LE>(acc, A, B, F);
    else if (mode == 4) mma64<true, false, true, K_FULL, true>(acc, A, B, F);
    else if (mode == 5) mma64<true, false, false, K_FULL, false, AR>(acc, A, B, F);
    else if (mode == 6) {
      double a2[1][2][2] = {};
      mma<1, 2, false, false, false>(a2, A, B, layA<16>(threadIdx.x >> 5), T);
      acc[0][0][0] += a2[0][0][0] + a2[0][1][1];
    } else mma64<true, false, false, B_GE, true>(acc, A, B, F);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) st[0] = (t1 - t0) / reps;
  acc_st_smem(A, acc, F, 1.0);
  __syncthreads();
  out[threadIdx.x] = A[threadIdx.x];
}

struct GemmBench {
  GemmBench() {
    double *o;
    unsigned long long *s, h;
    cudaMalloc(&o, 4096 * 8);
    cudaMalloc(&s, 8);
    cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TD * 8);
    const char *nm[8] = {"NT (A B^T)", "NN (A B)", "TN (A^T B)", "NT, B = W^T (B_LE)", "TN LOW (X_kk terms)",
                         "TN K=16 (arrow contraction)", "arrow out 16x64 K=64", "TN B_GE LOW (Lam)"};
    for (int m = 0; m < 8; ++m) {
      k_gemm<<<1, NT, 2 * TD * 8>>>(o, s, 200, m);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, s, 8, cudaMemcpyDeviceToHost);
      printf("gemm %-22s %6llu cycles per 64^3 (ideal 4096 full)\n", nm[m], h);
    }
  }
} g_gemm_bench;
