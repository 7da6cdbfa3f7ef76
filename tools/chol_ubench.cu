// Diagnostic: cycles of the POTRF building blocks (leaf_chol8, chol8_pipelined,
// leaf_chol16) on one CTA of 256 threads, with a correctness check of chol8.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          -I paper_2503_17528_b200/csrc -o tools/chol_ubench tools/chol_ubench.cu
#include "../paper_2503_17528_b200/csrc/exec.cu"
#include <cstdio>
#include <cmath>
#include <vector>
using namespace serinv::dev;
namespace serinv { namespace dev {
__device__ void chol8_dbg(double *St, double *Wt, double *S2, double *dv, int m, long long *ts, int mode) {
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int idx = tid; idx < SERINV_TILE * SERINV_TILE; idx += NT) {
    const int i = idx >> 6, j = idx & 63;
    if (i >= m || j >= m) St[i * LDT + j] = (i == j) ? 1.0 : 0.0;
  }
  double *scr = S2 + 8 * warp * LDT;  // per-warp 8 x 8 scratch
  auto blk = [](double *T, int i, int j) { return T + 8 * i * LDT + 8 * j; };
  // W(r,j) = -Z_r sum_{l=j}^{r-1} L(r,l) W(l,j), one block per call
  auto wblock = [&](int r, int j) {
    double t[2] = {0.0, 0.0};
    for (int l = j; l < r; ++l) blk_mma_nn(t, blk(St, r, l), blk(Wt, l, j));
    blk_store(scr, t);
    __syncwarp();
    double w[2] = {0.0, 0.0};
    {
      const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
      const double *Z = blk(Wt, r, r);
      dmma(w, -Z[g * LDT + q], scr[q * LDT + g]);
      dmma(w, -Z[g * LDT + 4 + q], scr[(4 + q) * LDT + g]);
    }
    __syncwarp();
    blk_store(blk(Wt, r, j), w);
  };
  for (int k = 0; k < 8; ++k) {
    __syncthreads();
    if ((threadIdx.x & 31) == 0) ts[(threadIdx.x >> 5) * 40 + 4 * k] = clock64();
    if (__all_sync(0xffffffffu, warp == 0)) {
      double *Akk = blk(St, k, k);
      if (k > 0) {
        double l[2] = {0.0, 0.0};
        blk_mma_nt(l, blk(St, k, k - 1), blk(Wt, k - 1, k - 1));
        blk_store(blk(St, k, k - 1), l);
        __syncwarp();
        asm volatile("bar.arrive 1, 256;" ::: "memory");
        double a[2];
        blk_load(Akk, a);
        blk_mma_nt_sub(a, blk(St, k, k - 1), blk(St, k, k - 1));
        leaf_chol8r(a[0], a[1], Akk, blk(Wt, k, k), dv + 8 * k);  // the updated block stays in registers
      } else {
        leaf_chol8(Akk, blk(Wt, k, k), dv + 8 * k);
      }
    } else if (k > 0) {
      const int wk = warp - 1;  // 0..6
      const int ip = k + 1 + wk;
      if (ip < 8) {  // panel block (ip, k-1)
        double l[2] = {0.0, 0.0};
        blk_mma_nt(l, blk(St, ip, k - 1), blk(Wt, k - 1, k - 1));
        blk_store(blk(St, ip, k - 1), l);
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      // trailing update by column k-1: blocks (i, j), k <= j <= i <= 7, except (k, k)
      // (entries off(k)+1 .. 35 of the column-major lower-triangle table); this warp
      // takes every 7th: all operands loaded, then all DMMAs, then the stores
      const int off = k * 8 - (k * (k - 1)) / 2;          // entries with j < k
      const int idx = 36 - off - 1;                        // blocks this step
      int bi[4], bj[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int e = off + 1 + wk + 7 * t;
        const int v = (e < 36) ? c_lower8[e] : 0;
        bi[t] = v >> 4;
        bj[t] = v & 15;
      }
      double acc[4][2];
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (wk + 7 * t < idx) blk_load(blk(St, bi[t], bj[t]), acc[t]);
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (wk + 7 * t < idx) blk_mma_nt_sub(acc[t], blk(St, bi[t], k - 1), blk(St, bj[t], k - 1));
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (wk + 7 * t < idx) blk_store(blk(St, bi[t], bj[t]), acc[t]);
      // block row k-1 of W (blocks j < k-1), round-robin after the updates
      for (int j = 0; j < k - 1; ++j)
        if ((idx + j) % 7 == wk) wblock(k - 1, j);
    }
  }
  __syncthreads();
  if (warp < 7) wblock(7, warp);  // last block row of W
  for (int idx = tid; idx < SERINV_TILE * SERINV_TILE; idx += NT) {  // strict-upper blocks of L
    const int i = idx >> 6, j = idx & 63;
    if ((j >> 3) > (i >> 3)) St[i * LDT + j] = 0.0;
  }
  __syncthreads();
}

}}


__global__ void __launch_bounds__(256, 2) kchol(const double *A, double *L, double *W, long long *cyc, int which) {
  extern __shared__ __align__(16) double smem[];
  double *St = smem, *Wt = St + 64 * LDT, *S2 = Wt + 64 * LDT, *dv = S2 + 64 * LDT;
  for (int i = threadIdx.x; i < 64 * 64; i += 256) { St[(i >> 6) * LDT + (i & 63)] = A[i]; Wt[(i >> 6) * LDT + (i & 63)] = 0.0; }
  __syncthreads();
  long long t0 = clock64();
  if (which == 0) {
    chol8_pipelined(St, Wt, S2, dv, 64);
  } else if (which >= 3) {
    chol8_dbg(St, Wt, S2, dv, 64, cyc + 1, which - 3);
  } else if (which == 1) {
    if (threadIdx.x < 32) leaf_chol8(St, Wt, dv);
    __syncthreads();
  } else {
    __shared__ int bad;
    if (threadIdx.x < 32) leaf_chol16(St, Wt, dv, 0, 64, &bad);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  for (int i = threadIdx.x; i < 64 * 64; i += 256) { L[i] = St[(i >> 6) * LDT + (i & 63)]; W[i] = Wt[(i >> 6) * LDT + (i & 63)]; }
}

int main() {
  std::vector<double> A(4096), L(4096), W(4096);
  unsigned s = 1;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) / 16777216.0 - 0.5; };
  std::vector<double> M(4096);
  for (auto &x : M) x = rnd();
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) {
      double t = 0;
      for (int k = 0; k < 64; ++k) t += M[i * 64 + k] * M[j * 64 + k];
      A[i * 64 + j] = t + (i == j ? 64.0 : 0.0);
    }
  double *dA, *dL, *dW; long long *dc;
  cudaMalloc(&dA, 32768); cudaMalloc(&dL, 32768); cudaMalloc(&dW, 32768); cudaMalloc(&dc, 8 * 400);
  cudaMemcpy(dA, A.data(), 32768, cudaMemcpyHostToDevice);
  int smem = 3 * 64 * LDT * 8 + 64 * 8;
  cudaFuncSetAttribute(kchol, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char *names[3] = {"chol8_pipelined (64x64 L + W)", "leaf_chol8 (one 8x8 block)", "leaf_chol16 (one 16x16 block)"};
  long long *hts = new long long[400];
  for (int mode : {0, 1, 2}) {
    cudaMemset(dc, 0, 8 * 400);
    kchol<<<1, 256, smem>>>(dA, dL, dW, dc, 3 + mode);
    kchol<<<1, 256, smem>>>(dA, dL, dW, dc, 3 + mode);
    cudaMemcpy(hts, dc, 8 * 400, cudaMemcpyDeviceToHost);
    printf("dbg mode %d (1: no leaf, 2: no worker phase B): total %lld\n", mode, hts[0]);
    long long t0 = hts[1];
    for (int k = 0; k < 8; ++k)
      printf("  step %d: warp0 start %6lld leaf %6lld..%6lld | warp1 start %6lld barB %6lld end %6lld\n", k, hts[1 + 4 * k] - t0,
             hts[2 + 4 * k] - t0, hts[3 + 4 * k] - t0, hts[1 + 40 + 4 * k] - t0, hts[2 + 40 + 4 * k] - t0, hts[3 + 40 + 4 * k] - t0);
  }
  for (int which = 0; which < 3; ++which) {
    long long best = 1LL << 60, c;
    for (int r = 0; r < 5; ++r) {
      kchol<<<1, 256, smem>>>(dA, dL, dW, dc, which);
      cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      if (c < best) best = c;
    }
    printf("%-32s %8lld cycles  (%s)\n", names[which], best, cudaGetErrorString(cudaGetLastError()));
    if (which == 0) {
      cudaMemcpy(L.data(), dL, 32768, cudaMemcpyDeviceToHost);
      cudaMemcpy(W.data(), dW, 32768, cudaMemcpyDeviceToHost);
      double e1 = 0, e2 = 0;
      for (int i = 0; i < 64; ++i)
        for (int j = 0; j < 64; ++j) {
          double t = 0, u = 0;
          for (int k = 0; k < 64; ++k) { t += L[i * 64 + k] * L[j * 64 + k]; u += W[i * 64 + k] * L[k * 64 + j]; }
          e1 = fmax(e1, fabs(t - A[i * 64 + j]));
          e2 = fmax(e2, fabs(u - (i == j)));
        }
      printf("   chol8 check: max|LL^T - A| = %.2e, max|WL - I| = %.2e\n", e1, e2);
    }
  }
  return 0;
}
