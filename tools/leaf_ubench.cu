
#include <cstdio>
#include <cuda_runtime.h>
constexpr int LDT = 68;
// 1/sqrt(x) and 1/x without the library's out-of-range slow paths (a branch
// there makes the surrounding shuffles warp-collective): MUFU seed + one
// third-order Newton step (~2^-69 relative before rounding), valid for normal
// positive x.  x <= 0 or NaN gives NaN/inf, which the caller flags.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(y * y), x, 1.0);
  return fma(fma(e, 0.375, 0.5), y * e, y);
}
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(fma(e, e, e), y, y);
}

// Warp-level Cholesky + inverse of the 16 x 16 diagonal block at (c0, c0) of St
// (rows/columns >= m are padded with the identity).  Right-looking elimination on
// the symmetric block; the same row operations carried on Z = I give Z = L^{-1}
// (the elimination matrix M with M A = L^T).  Lane l owns column j = l & 15, rows
// i = 8 (l >> 4) + t, t < 8.  Per pivot p (d = current A[p][p]):
//   a[i][j] -= A[i][p] A[p][j] / d   (i, j > p),   z[i][j] -= A[i][p] Z[p][j] / d  (i > p),
//   column p of L = A[:, p] / sqrt(d), row p of Z scaled by 1 / sqrt(d).
// The next pivot d' = A[p+1][p+1] - A[p+1][p]^2 / d is formed by every lane
// from two values shuffled one step early, so the serial chain per pivot is one
// reciprocal and one FMA (no shuffle, no sqrt on it).  Writes L (upper zeroed)
// to St, Z to Wt, the pivots to dv, the first non-positive pivot to *s_bad.
// Must be called by a whole, converged warp.
__device__ __forceinline__ void leaf_chol16(double *St, double *Wt, double *dv, int c0, int m, int *s_bad) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, j = lane & 15, h = lane >> 4;
  double a[8], z[8], dj = 1.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int i = 8 * h + t;
    const bool valid = (c0 + i < m) && (c0 + j < m);
    a[t] = valid ? St[(c0 + i) * LDT + c0 + j] : ((i == j) ? 1.0 : 0.0);
    z[t] = (i == j) ? 1.0 : 0.0;
  }
  double d = __shfl_sync(FULL, a[0], 0);
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    const int tp = p & 7, hp = p >> 3;
    const int t1 = (p + 1) & 7, h1 = (p + 1) >> 3;
    double x = 0.0, y = 1.0;
    if (p < 15) {  // compile-time
      x = __shfl_sync(FULL, a[t1], p + 16 * h1);      // A[p+1][p]
      y = __shfl_sync(FULL, a[t1], p + 1 + 16 * h1);  // A[p+1][p+1]
    }
    const double apj = __shfl_sync(FULL, a[tp], j + 16 * hp);
    const double zpj = __shfl_sync(FULL, z[tp], j + 16 * hp);
    double colp[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) colp[t] = __shfl_sync(FULL, a[t], p + 16 * h);
    const double id = rcp_nr(d);
    const double dn = fma(-(x * x), id, y);
    const double rs = rsqrt_nr(d);
    const double fa = (j > p) ? apj * id : 0.0;
    const double fz = zpj * id;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const bool below = 8 * h + t > p;
      a[t] = below ? fma(-colp[t], fa, a[t]) : a[t];
      z[t] = below ? fma(-colp[t], fz, z[t]) : z[t];
    }
    // branch-free (a divergent branch here turns every shuffle into a collective)
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = 8 * h + t;
      const double sc = (i > p) ? a[t] * rs : ((i == p) ? d * rs : 0.0);
      a[t] = (j == p) ? sc : a[t];
    }
    z[tp] = (h == hp) ? z[tp] * rs : z[tp];
    dj = (j == p) ? d : dj;
    d = dn;
  }
  if (h == (j >> 3) && c0 + j < m) {
    dv[c0 + j] = dj;
    if (!(dj > 0.0)) atomicMin(s_bad, c0 + j);
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int i = 8 * h + t;
    const bool valid = (c0 + i < m) && (c0 + j < m) && i >= j;
    St[(c0 + i) * LDT + c0 + j] = valid ? a[t] : 0.0;
    Wt[(c0 + i) * LDT + c0 + j] = valid ? z[t] : 0.0;
  }
}

__global__ void k(double *out, long long *cyc, int reps) {
  __shared__ double St[16*LDT], Wt[16*LDT], dv[64];
  __shared__ int s_bad;
  for (int i = threadIdx.x; i < 16*LDT; i += blockDim.x) { Wt[i] = 0; }
  for (int i = threadIdx.x; i < 16*LDT; i += blockDim.x) { int r = i / LDT, c = i % LDT; if (c < 64) St[i] = (r==c) ? 20.0 : 0.01*(((r*7+c*3)+(c*7+r*3))%11); }
  s_bad = 1<<30;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    leaf_chol16(St, Wt, dv, 0, 64, &s_bad);
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; out[0] = St[0] + Wt[5*LDT+3]; }
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  for (int nt : {32, 128, 256}) {
    k<<<1, nt>>>(o, c, 10); cudaDeviceSynchronize();
    k<<<1, nt>>>(o, c, 1000); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("leaf16 (%d threads, all warps run it) cycles per call: %lld  (err %s)\n", nt, h, cudaGetErrorString(cudaGetLastError()));
  }
}
