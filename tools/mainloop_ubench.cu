// Diagnostic: where does the 64x64 FP64 DMMA tile main loop lose throughput?
// Variants (all 8 warps x 2 CTAs/SM unless noted, 64x64 output tile per CTA):
//   0  registers only (DMMA peak)
//   1  fragments from smem (LDS.64), no barriers
//   2  1 + __syncthreads every KC/4 k-steps
//   3  2 + cp.async.cg staging of the next chunk from an L2-resident global panel (3 stages)
//   4  3 with vectorised fragments (LDS.128; k-pair permutation)
//   5  3 with 32x32 warp tiles, the two 4-warp groups splitting each chunk along k
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mainloop_ubench tools/mainloop_ubench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int T = 64, KC = 32, LDMK = KC + 4, STAGES = 3, OPSZ = T * LDMK;

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

// [row][k] stride LDMK for both A (64 rows) and B (64 cols)
__device__ __forceinline__ void steps_lds64(const double *As, const double *Bs, double (&acc)[2][4][2], int ksteps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = (warp >> 1) * 16 + (lane >> 2), c0 = (warp & 1) * 32 + (lane >> 2), kq = lane & 3;
#pragma unroll 4
  for (int ks = 0; ks < ksteps; ++ks) {
    const int kk = ks * 4 + kq;
    double a0 = As[r0 * LDMK + kk], a1 = As[(r0 + 8) * LDMK + kk], b[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(c0 + ni * 8) * LDMK + kk];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) { dmma(acc[0][ni], a0, b[ni]); dmma(acc[1][ni], a1, b[ni]); }
  }
}
// vectorised: thread q holds k = 8*s + 2q + {0,1}; one LDS.128 per row per 2 k-steps
__device__ __forceinline__ void steps_lds128(const double *As, const double *Bs, double (&acc)[2][4][2], int ksteps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = (warp >> 1) * 16 + (lane >> 2), c0 = (warp & 1) * 32 + (lane >> 2), kq = lane & 3;
#pragma unroll 2
  for (int ks = 0; ks < ksteps; ks += 2) {
    const int kk = ks * 4 + 2 * kq;
    double2 a0 = *(const double2 *)&As[r0 * LDMK + kk], a1 = *(const double2 *)&As[(r0 + 8) * LDMK + kk];
    double2 b[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = *(const double2 *)&Bs[(c0 + ni * 8) * LDMK + kk];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) { dmma(acc[0][ni], a0.x, b[ni].x); dmma(acc[1][ni], a1.x, b[ni].x); }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) { dmma(acc[0][ni], a0.y, b[ni].y); dmma(acc[1][ni], a1.y, b[ni].y); }
  }
}

// 32x32 warp tile, warp group g = warp>>2 takes k-steps [g*ksteps/2, (g+1)*ksteps/2) of the chunk
__device__ __forceinline__ void steps_ksplit(const double *As, const double *Bs, double (&acc)[4][4][2], int ksteps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, w = warp & 3, g = warp >> 2;
  const int r0 = (w >> 1) * 32 + (lane >> 2), c0 = (w & 1) * 32 + (lane >> 2), kq = lane & 3;
  const int h = ksteps / 2;
#pragma unroll 4
  for (int ks = g * h; ks < g * h + h; ++ks) {
    const int kk = ks * 4 + kq;
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = As[(r0 + mi * 8) * LDMK + kk];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(c0 + ni * 8) * LDMK + kk];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
  }
}

__device__ __forceinline__ void load_chunk(double *s, const double *g, int ld, int k0) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int it = 0; it < (T * (KC / 2)) / 256; ++it) {
    int idx = tid + it * 256, r = idx >> 4, kk = (idx & 15) * 2;
    cp_async16(s + r * LDMK + kk, g + (size_t)r * ld + k0 + kk);
  }
}

template <int V>
__global__ void __launch_bounds__(256, 2) kern(const double *A, const double *B, int K, int reps, double *out) {
  extern __shared__ double sm[];
  double acc[2][4][2], acc4[4][4][2];
  for (int i = 0; i < 2; ++i) for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) acc4[i][j][0] = acc4[i][j][1] = 0;
  for (int i = threadIdx.x; i < STAGES * 2 * OPSZ; i += 256) sm[i] = 1e-3 * (i % 17);
  __syncthreads();
  const int nch = K / KC;
  const double *Ag = A + (size_t)(blockIdx.x % 64) * T * K, *Bg = B + (size_t)(blockIdx.x % 64) * T * K;
  for (int r = 0; r < reps; ++r) {
    if (V == 0) {
      double a = 1e-3 * threadIdx.x, b = 2e-3;
      for (int j = 0; j < nch * KC / 4; ++j)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) { dmma(acc[0][ni], a, b); dmma(acc[1][ni], b, a); }
    } else if (V == 1 || V == 2) {
      for (int j = 0; j < nch; ++j) {
        if (V == 2) __syncthreads();
        const double *As = sm + (j % STAGES) * 2 * OPSZ;
        steps_lds64(As, As + OPSZ, acc, KC / 4);
      }
    } else {
      for (int j = 0; j < STAGES - 1; ++j) {
        double *As = sm + j * 2 * OPSZ;
        load_chunk(As, Ag, K, j * KC); load_chunk(As + OPSZ, Bg, K, j * KC); cp_commit();
      }
      for (int j = 0; j < nch; ++j) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        if (j + STAGES - 1 < nch) {
          double *As = sm + ((j + STAGES - 1) % STAGES) * 2 * OPSZ;
          load_chunk(As, Ag, K, (j + STAGES - 1) * KC); load_chunk(As + OPSZ, Bg, K, (j + STAGES - 1) * KC);
        }
        cp_commit();
        const double *As = sm + (j % STAGES) * 2 * OPSZ;
        if (V == 3) steps_lds64(As, As + OPSZ, acc, KC / 4);
        else if (V == 4) steps_lds128(As, As + OPSZ, acc, KC / 4);
        else steps_ksplit(As, As + OPSZ, acc4, KC / 4);
      }
      cp_wait<0>();
      __syncthreads();
    }
  }
  double s = 0;
  for (int i = 0; i < 2; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += acc4[i][j][0] + acc4[i][j][1];
  if (s == 1234.5) out[0] = s;
}

template <int V>
void run(const double *A, const double *B, double *out, int K, int blocks) {
  const int smem = STAGES * 2 * OPSZ * 8;
  CK(cudaFuncSetAttribute(kern<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int reps = 40;
  kern<V><<<blocks, 256, smem>>>(A, B, K, 2, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int t = 0; t < 5; ++t) {
    cudaEventRecord(e0); kern<V><<<blocks, 256, smem>>>(A, B, K, reps, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * T * T * (double)K * reps * blocks;
  printf("V%d K=%d blocks=%d: %.2f TF/s\n", V, K, blocks, flops / best / 1e9);
}

int main() {
  int K = 1024, blocks = 296;
  double *A, *B, *out;
  CK(cudaMalloc(&A, 64ull * T * K * 8)); CK(cudaMalloc(&B, 64ull * T * K * 8)); CK(cudaMalloc(&out, 64));
  CK(cudaMemset(A, 0, 64ull * T * K * 8)); CK(cudaMemset(B, 0, 64ull * T * K * 8));
  run<0>(A, B, out, K, blocks);
  run<1>(A, B, out, K, blocks);
  run<2>(A, B, out, K, blocks);
  run<3>(A, B, out, K, blocks);
  run<4>(A, B, out, K, blocks);
  run<5>(A, B, out, K, blocks);
  run<3>(A, B, out, 256, blocks);
  run<5>(A, B, out, 256, blocks);
  return 0;
}
