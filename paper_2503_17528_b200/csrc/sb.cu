// sb.cu -- small-block engine: the partitioned selected inversion of PAPER.md
// Sec. 3 (PPOBTAF Alg. 3-4, POBTARSSI Sec. 3.3, PPOBTASI Alg. 5-6) with nested
// solving of the reduced systems (Sec. 4.2), for b <= 64, a <= 16.
//
// Why a second engine.  With b = 64 a block step of Alg. 1 is ~0.5 MFLOP: the
// tile-task executor (exec.cu) pays a dependency hop (global counter publish /
// poll, operand re-staging through L2) between every POTRF, TRSM and SYRK of the
// chain, and the chain is the bound (BASELINE C5).  Here ONE CTA carries a whole
// partition's chain: the running diagonal block, the coupling, the fill-in block
// B_i (Alg. 4) and the arrow rows stay in shared memory from step to step, the
// persistent accumulators (A_ff, A_{n,f}, U_p of Alg. 4 l.9-12) in registers, and
// the partitions of a level run concurrently on all SMs.  Two kernels per level:
//   sb_factor_kernel   PPOBTAF of every partition of the level (2 CTAs / SM, so
//                      one CTA's latency-bound 64 x 64 Cholesky overlaps the
//                      other's DMMA products) writing the boundary blocks straight
//                      into the next level's reduced arrays (order of reading R14,
//                      DESIGN.md); the last level (one partition) is the plain
//                      sequential POBTAF incl. the tip (Alg. 1).
//   sb_inverse_kernel  PPOBTASI of every partition (1 CTA / SM, 224 KB of
//                      operands resident), seeded by the next level's X.
// Block products are warp-level DMMA (mma.sync m8n8k4 f64; tcgen05 has no f64
// kind) on shared-memory tiles whose 64-double rows are XOR-swizzled so that the
// fragment loads of both operand orientations are bank-conflict free.  TRSM is a
// product with W = L_ii^{-1}; W is what the factor pass stores in the
// diagonal slot (the inverse pass needs W, not L_ii).  Padding: blocks of b < 64
// are embedded in 64 x 64 tiles with an identity diagonal, arrow rows a < 16 with
// zeros, so the padded problem has the same factors / inverse on the real part.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "graph.h"
#include "sb.h"

namespace serinv {
namespace sb {
namespace dev {

constexpr int T = 64;
constexpr int NT = 256;

constexpr unsigned FULL = 0xffffffffu;
constexpr int TD = T * T;        // doubles per 64 x 64 tile


enum PartType { P_TOP = 0, P_MID = 1, P_BOT = 2, P_SEQ = 3 };

// element (r, c) of a tile with 64-double rows: bank-conflict-free DMMA fragment
// loads for [row][k] (lanes: r = l/4, c = l%4) and [k][row] (r = l%4, c = l/4)
__device__ __forceinline__ int swz(int r, int c) { return (r << 6) + (c ^ (((r & 3) << 3) | (r & 4))); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// the same with an L2 evict-first policy (streamed operands that must not push other
// kernels' working sets out of L2)
__device__ __forceinline__ void cp_async16_ef(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile(
      "{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, pol;\n}\n" ::"r"(s),
      "l"(gmem)
      : "memory");
}
__device__ __forceinline__ void cp_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

__device__ void record_info(int *info, int v) {
  int old = *(volatile int *)info;
  while (old == 0 || v < old) {
    int prev = atomicCAS(info, old, v);
    if (prev == old) break;
    old = prev;
  }
}

// ---------------------------------------------------------------------------
// Tile movement.  A tile is rows_t x 64 (rows_t = 64 or AR) in swizzled smem.
// ---------------------------------------------------------------------------
// s <- op(g) padded: (r, c) = trans ? g[c*ld + r] : g[r*ld + c] for r < rows, c < cols,
// else (pad && r == c).  Full 64 x 64 untransposed blocks go by cp.async (caller waits).
__device__ void ld_tile(double *s, const double *g, int rows_t, int rows, int cols, int ld, bool trans,
                        bool pad, bool stream = false) {
  const int tid = threadIdx.x;
  if (!trans && rows == T && cols == T && ld == T && rows_t == T) {
#pragma unroll 4
    for (int i = tid; i < TD / 2; i += NT) {
      const int r = i >> 5, c = (i & 31) * 2;
      if (stream)
        cp_async16_ef(s + swz(r, c), g + r * T + c);
      else
        cp_async16(s + swz(r, c), g + r * T + c);
    }
    return;
  }
  if (!trans && cols == T && ld == T && rows <= rows_t && !(pad && rows < rows_t) && !((uintptr_t)g & 15)) {
    // full 64-double rows (e.g. the arrow rows at b = 64): cp.async too, zero pad rows
    for (int i = tid; i < rows_t * (T / 2); i += NT) {
      const int r = i >> 5, c = (i & 31) * 2;
      if (r < rows && stream)
        cp_async16_ef(s + swz(r, c), g + r * T + c);
      else if (r < rows)
        cp_async16(s + swz(r, c), g + r * T + c);
      else
        *(double2 *)(s + swz(r, c)) = make_double2(0.0, 0.0);
    }
    return;
  }
  for (int i = tid; i < rows_t * T; i += NT) {
    int r, c;
    if (trans) {  // consecutive threads read consecutive global addresses
      r = i & 63;
      c = i >> 6;
      if (rows_t < T) {  // r ranges over rows_t
        r = i % rows_t;
        c = i / rows_t;
      }
    } else {
      r = i >> 6;
      c = i & 63;
    }
    double v;
    if (r < rows && c < cols)
      v = trans ? __ldg(g + (int64_t)c * ld + r) : __ldg(g + (int64_t)r * ld + c);
    else
      v = (pad && r == c) ? 1.0 : 0.0;
    s[swz(r, c)] = v;
  }
}

// g <- op(s) (rows x cols of the tile; trans: g[c*ld + r] = s(r, c))
__device__ void st_tile(double *g, const double *s, int rows, int cols, int ld, bool trans) {
  const int tid = threadIdx.x;
  if (!trans && rows == T && cols == T && ld == T) {
    for (int i = tid; i < TD / 2; i += NT) {
      const int r = i >> 5, c = (i & 31) * 2;
      *(double2 *)(g + r * T + c) = *(const double2 *)(s + swz(r, c));
    }
    return;
  }
  for (int i = tid; i < rows * cols; i += NT) {
    if (trans) {
      const int c = i / rows, r = i % rows;  // consecutive threads: consecutive g addresses
      g[(int64_t)c * ld + r] = s[swz(r, c)];
    } else {
      const int r = i / cols, c = i % cols;
      g[(int64_t)r * ld + c] = s[swz(r, c)];
    }
  }
}

// global -> global copy of a rows x cols block (same ld)
__device__ void cp_block(double *dst, const double *src, int64_t count) {
  for (int64_t i = threadIdx.x; i < count; i += NT) dst[i] = __ldg(src + i);
}

// ---------------------------------------------------------------------------
// Warp-level DMMA products on smem tiles.  A warp owns the 8 x 8 output
// fragments (rf[i], cf[j]) (lane l holds (l/4, 2(l%4) + {0,1}) of each):
//   acc[i][j] += sgn * sum_k op(A)[8 rf[i] + .][k] op(B)[k][8 cf[j] + .]
// Layout of 64 x 64 outputs (lay64): warp w = 2 rg + h owns row fragments
// {rg, 7 - rg} and column fragments {0,1,6,7} (h = 0) or {2,3,4,5} (h = 1).  It
// balances the warps for the triangular operands (W = L^{-1}: the k range of
// column fragment c is [8c, 64) or [0, 8c + 8)) and for lower-triangle-only
// products of symmetric results (5 or 4 of the 36 lower fragments per warp), and
// each A row strip is shared by exactly one warp pair (pair barriers).
// Operand k-range modes: A_GE (A[m][k] = 0 for k < m: A = W^T), B_GE (B[k][n] = 0
// for k < n: B = W), B_LE (B[k][n] = 0 for k > n: B = W^T); LOW: only fragments
// with rf >= cf.
// ---------------------------------------------------------------------------
enum { K_FULL = 0, A_GE = 1, B_GE = 2, B_LE = 3 };

template <int MI, int NI>
struct Frags {
  int rf[MI], cf[NI];
};

__device__ __forceinline__ Frags<2, 4> lay64(int w) {
  Frags<2, 4> F;
  const int rg = w >> 1, h = w & 1;
  F.rf[0] = rg;
  F.rf[1] = 7 - rg;
  F.cf[0] = h ? 2 : 0;
  F.cf[1] = h ? 3 : 1;
  F.cf[2] = h ? 4 : 6;
  F.cf[3] = h ? 5 : 7;
  return F;
}
// ARR x 64 outputs (arrow rows, ARR = 8 or 16): ARR = 16: row fragment w & 1, column
// fragments {w/2, 7 - w/2}; ARR = 8: the one row fragment, column fragment w
template <int ARR>
__device__ __forceinline__ Frags<1, ARR / 8> layA(int w) {
  Frags<1, ARR / 8> F;
  if (ARR == 16) {
    F.rf[0] = w & 1;
    F.cf[0] = w >> 1;
    F.cf[ARR / 8 - 1] = 7 - (w >> 1);
  } else {
    F.rf[0] = 0;
    F.cf[0] = w;
  }
  return F;
}
// ARR x ARR outputs (tip-sized): warps 0 .. (ARR/8)^2 - 1
template <int ARR>
__device__ __forceinline__ Frags<1, 1> layU(int w) {
  Frags<1, 1> F;
  F.rf[0] = ARR == 16 ? (w >> 1) & 1 : 0;
  F.cf[0] = ARR == 16 ? w & 1 : 0;
  return F;
}

// column fragments of the two lay64 column sets
__device__ __forceinline__ constexpr int colfrag(int h, int j) { return h ? 2 + j : (j < 2 ? j : j + 4); }

// 64 x 64 products in lay64 for the warp's column set H (compile time): the k loop
// is unrolled, so the triangular k ranges (BM) are compile-time per fragment; LOW
// skips the warp-uniform strictly-upper fragments (rf < cf).  KK = contraction
// length (64, or AR for the arrow contractions).
template <int H, bool TA, bool TB, bool NEG, int BM, bool LOW, int KK>
__device__ __forceinline__ void mma_h(double (&acc)[2][4][2], const double *A, const double *B, const int rf0,
                                      const int rf1) {
  const int l = threadIdx.x & 31, lr = l >> 2, lc = l & 3;
  const int rf[2] = {rf0, rf1};
  bool on[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) on[i][j] = !LOW || rf[i] >= colfrag(H, j);
#pragma unroll
  for (int k = 0; k < KK; k += 4) {
    bool col[4];
    bool any = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = colfrag(H, j);
      col[j] = BM == B_LE ? k < 8 * c + 8 : (BM == B_GE ? k >= 8 * c : true);
      any |= col[j];
    }
    if (!any) continue;
    const int kk = k + lc;
    double af[2], bf[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int m = 8 * rf[i] + lr;
      const double v = TA ? A[swz(kk, m)] : A[swz(m, kk)];
      af[i] = NEG ? -v : v;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      bf[j] = 0.0;
      if (!col[j]) continue;
      const int n = 8 * colfrag(H, j) + lr;
      bf[j] = TB ? B[swz(n, kk)] : B[swz(kk, n)];
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (col[j] && on[i][j]) dmma(acc[i][j], af[i], bf[j]);
  }
}

template <bool TA, bool TB, bool NEG, int BM = K_FULL, bool LOW = false, int KK = T>
__device__ __forceinline__ void mma64(double (&acc)[2][4][2], const double *A, const double *B,
                                      const Frags<2, 4> &F) {
  if (threadIdx.x & 32)
    mma_h<1, TA, TB, NEG, BM, LOW, KK>(acc, A, B, F.rf[0], F.rf[1]);
  else
    mma_h<0, TA, TB, NEG, BM, LOW, KK>(acc, A, B, F.rf[0], F.rf[1]);
}

// small products (arrow / tip outputs) with run-time fragments: warp-level k range only
template <int MI, int NI, bool TA, bool TB, bool NEG, int BM = K_FULL>
__device__ __forceinline__ void mma(double (&acc)[MI][NI][2], const double *A, const double *B,
                                    const Frags<MI, NI> &F, int K) {
  const int l = threadIdx.x & 31, lr = l >> 2, lc = l & 3;
  int klo = K, khi = 0;
#pragma unroll
  for (int j = 0; j < NI; ++j) {
    klo = min(klo, BM == B_GE ? 8 * F.cf[j] : 0);
    khi = max(khi, BM == B_LE ? min(K, 8 * F.cf[j] + 8) : K);
  }
  if (BM == K_FULL && K == T) {  // full products: fully unrolled k loop
    if (K == T) {
#pragma unroll
      for (int k = 0; k < T; k += 4) {
        double af[MI], bf[NI];
        const int kk = k + lc;
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int m = 8 * F.rf[i] + lr;
          const double v = TA ? A[swz(kk, m)] : A[swz(m, kk)];
          af[i] = NEG ? -v : v;
        }
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const int n = 8 * F.cf[j] + lr;
          bf[j] = TB ? B[swz(n, kk)] : B[swz(kk, n)];
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
      return;
    }
  }
#pragma unroll 2
  for (int k = klo; k < khi; k += 4) {
    double af[MI], bf[NI];
    const int kk = k + lc;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int m = 8 * F.rf[i] + lr;
      const double v = TA ? A[swz(kk, m)] : A[swz(m, kk)];
      af[i] = NEG ? -v : v;
    }
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int n = 8 * F.cf[j] + lr;
      bf[j] = TB ? B[swz(n, kk)] : B[swz(kk, n)];
    }
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) dmma(acc[i][j], af[i], bf[j]);
  }
}

template <int MI, int NI>
__device__ __forceinline__ void acc_zero(double (&acc)[MI][NI][2]) {
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// acc <- g (rows x cols block, ld), padded with the identity (pad) or zeros
template <int MI, int NI>
__device__ __forceinline__ void acc_ld(double (&acc)[MI][NI][2], const double *g, int ld, int rows, int cols,
                                       const Frags<MI, NI> &F, bool pad) {
  const int l = threadIdx.x & 31, lr = l >> 2, lc = l & 3;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int m = 8 * F.rf[i] + lr, n = 8 * F.cf[j] + 2 * lc;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = n + e;
        acc[i][j][e] = (m < rows && c < cols) ? __ldg(g + (int64_t)m * ld + c) : ((pad && m == c) ? 1.0 : 0.0);
      }
    }
}

// acc <- s (a swizzled smem tile)
template <int MI, int NI>
__device__ __forceinline__ void acc_ld_smem(double (&acc)[MI][NI][2], const double *s, const Frags<MI, NI> &F) {
  const int l = threadIdx.x & 31, lr = l >> 2, lc = l & 3;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const double2 v = *(const double2 *)(s + swz(8 * F.rf[i] + lr, 8 * F.cf[j] + 2 * lc));
      acc[i][j][0] = v.x;
      acc[i][j][1] = v.y;
    }
}

// s <- sgn * acc; LOW: only fragments rf >= cf, mirrored to (cf, rf) when MIR
template <int MI, int NI, bool LOW = false, bool MIR = false>
__device__ __forceinline__ void acc_st_smem(double *s, const double (&acc)[MI][NI][2], const Frags<MI, NI> &F,
                                            double sgn) {
  const int l = threadIdx.x & 31, lr = l >> 2, lc = l & 3;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      if (LOW && F.rf[i] < F.cf[j]) continue;
      const int m = 8 * F.rf[i] + lr, n = 8 * F.cf[j] + 2 * lc;
      const double v0 = sgn * acc[i][j][0], v1 = sgn * acc[i][j][1];
      *(double2 *)(s + swz(m, n)) = make_double2(v0, v1);
      if (MIR && F.rf[i] != F.cf[j]) {
        s[swz(n, m)] = v0;
        s[swz(n + 1, m)] = v1;
      }
    }
}

// g <- sgn * acc (rows x cols of the block; trans: g[c*ld + r] = value (r, c)); LOW / MIR as above
template <int MI, int NI, bool LOW = false, bool MIR = false, bool CS = false>
__device__ __forceinline__ void acc_st_global(double *g, const double (&acc)[MI][NI][2], int ld, int rows,
                                              int cols, const Frags<MI, NI> &F, bool trans, double sgn) {
  const int l = threadIdx.x & 31, lr = l >> 2, lc = l & 3;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      if (LOW && F.rf[i] < F.cf[j]) continue;
      const int m = 8 * F.rf[i] + lr, n = 8 * F.cf[j] + 2 * lc;
      if (!trans && !MIR && m < rows && n + 1 < cols && !(ld & 1) && !((uintptr_t)g & 15)) {  // 16-byte store
        const double2 v2 = make_double2(sgn * acc[i][j][0], sgn * acc[i][j][1]);
        if (CS)
          __stcs((double2 *)(g + (int64_t)m * ld + n), v2);  // streaming: evict first
        else
          *(double2 *)(g + (int64_t)m * ld + n) = v2;
        continue;
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = n + e;
        if (m >= rows || c >= cols) continue;
        const double v = sgn * acc[i][j][e];
        if (trans || (MIR && F.rf[i] != F.cf[j])) g[(int64_t)c * ld + m] = v;
        if (!trans) g[(int64_t)m * ld + c] = v;
      }
    }
}

// barrier of the warp pair sharing a row strip in lay64 (warps 2rg, 2rg+1)
__device__ __forceinline__ void pair_sync() {
  asm volatile("bar.sync %0, 64;\n" ::"r"(1 + (int)(threadIdx.x >> 6)) : "memory");
}

// 1 / sqrt(x): MUFU approximation + 2 Newton steps (full double precision; NaN for x <= 0)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// ---------------------------------------------------------------------------
// In-place Cholesky + triangular inverse of a 64 x 64 SPD tile (lower triangle
// read): D <- W = L^{-1} (lower, strict upper zero).  ldg[t] = L_tt.
// Right-looking on 8-column panels with look-ahead:
//   warp 0 (the critical chain), round j: factors the 8 x 8 diagonal block (j,j)
//     on ONE thread in registers (8 rsqrt + FMA steps, the product-form inverse
//     W_jj alongside; W_jj replaces the block), publishes it (named barrier,
//     arrive), waits for the workers' round j-1, then computes L_{j+1,j} =
//     A_{j+1,j} W_jj^T and the panel-j update of the next diagonal block itself;
//   warps 1..7 (workers), round j: wait for W_jj; update every other trailing
//     tile (i,k), j < k <= i, computing the panel blocks they need themselves
//     (L_ij = A_ij W_jj^T, written transposed into the free upper block (j,i) --
//     the same values from every warp that computes them -- and read back as
//     fragments); and block row j of W: W_jm = -W_jj sum_{k=m}^{j-1} L_jk W_km
//     (m < j), written over the dead A_jm; then arrive on the round's barrier.
// L itself is never assembled: only W = L^{-1} and the pivots are outputs.
// *s_bad = 2 x the first non-positive pivot index + 1 if that pivot is NaN; 128 if
// none.  Wd: 8 x 64 per-warp scratch; Pscr: 8 x 512 doubles of per-warp scratch.  Called by all NT threads; needs the
// registers of one thread for the leaf (the kernels that call it run 1 CTA / SM).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void nbar_arrive(int id) { asm volatile("bar.arrive %0, 256;\n" ::"r"(id) : "memory"); }
__device__ __forceinline__ void nbar_sync(int id) { asm volatile("bar.sync %0, 256;\n" ::"r"(id) : "memory"); }

// the trailing update of tile (i, k) by panel j (R = 8j): L_ij, L_kj computed in-warp
// (through the warp's private scratch Pw: 8 blocks of 8 x 8, stored transposed with
// row stride 8, conflict-free for both fragment reads), then A_ik -= L_ij L_kj^T; the
// owner of tile (i, j+1) also writes L_ij^T to the shared scratch block (j, i) (the
// upper triangle, free) for block row i of W later.  Up to 4 tiles of one warp in
// flight together.
__device__ __forceinline__ void trail_tiles(double *D, double *Pw, int R, const int (&ti)[4], const int (&tk)[4],
                                            const bool (&on)[4]) {
  const int l = threadIdx.x & 31, lr = l >> 2, lc = l & 3;
  const int j1 = R / 8 + 1;
  double li[4][2], lk[4][2];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    li[u][0] = li[u][1] = lk[u][0] = lk[u][1] = 0.0;
    if (!on[u]) continue;
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4) {
      const double wv = D[swz(R + lr, R + kk + lc)];  // (W_jj^T)[kk][n] = W_jj[n][kk]
      dmma(li[u], D[swz(8 * ti[u] + lr, R + kk + lc)], wv);
      if (tk[u] != ti[u]) dmma(lk[u], D[swz(8 * tk[u] + lr, R + kk + lc)], wv);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (!on[u]) continue;
    double *pi = Pw + 128 * u, *pk = pi + 64;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      pi[(2 * lc + e) * 8 + lr] = li[u][e];
      pk[(2 * lc + e) * 8 + lr] = lk[u][e];
      if (tk[u] == j1) D[swz(R + 2 * lc + e, 8 * ti[u] + lr)] = li[u][e];  // shared copy, one writer
    }
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (!on[u]) continue;
    const int i = ti[u], k = tk[u];
    const double *pi = Pw + 128 * u, *pk = (k != i) ? pi + 64 : pi;
    double2 cv = *(const double2 *)(D + swz(8 * i + lr, 8 * k + 2 * lc));
    double acc[2] = {cv.x, cv.y};
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4) dmma(acc, -pi[(kk + lc) * 8 + lr], pk[(kk + lc) * 8 + lr]);
    *(double2 *)(D + swz(8 * i + lr, 8 * k + 2 * lc)) = make_double2(acc[0], acc[1]);
  }
  __syncwarp();
}

__device__ void chol_inv64(double *D, double *Wd, double *Pscr, double *ldg, int *s_bad,
                           unsigned long long *stamp = nullptr) {
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31, lr = l >> 2, lc = l & 3;
  if (w == 0) {
    int bad = 128;  // 2 * (first failing pivot) + (pivot is NaN): genuine failures sort first (lane 0)
    for (int j = 0; j < 8; ++j) {
      const int R = 8 * j;
      // element (R + i, R + c) of the swizzled tile = (row base)[c ^ (i & 4)]: R = 8j has no bits
      // below 3, so the XOR splits into a per-row base and a compile-time column offset
      if (l == 0) {
        double a[8][8], wv[8][8];  // lower triangles used (indices are compile-time after unrolling)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double *rp = D + (R + i) * T + (R ^ ((i & 3) << 3));
#pragma unroll
          for (int c = 0; c <= i; c += 2) {  // 16-byte loads: positions (c, c+1) ^ (i & 4) stay paired
            const double2 v = *(const double2 *)(rp + (c ^ (i & 4)));
            a[i][c] = v.x;
            a[i][c + 1] = v.y;
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (c > i) a[i][c] = 0.0;
            wv[i][c] = i == c ? 1.0 : 0.0;
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double dkk = a[k][k];
          if (!(dkk > 0.0) && bad == 128) bad = 2 * (R + k) + (dkk != dkk ? 1 : 0);
          const double rs = rsqrt_nr(dkk);
          a[k][k] = dkk * rs;
#pragma unroll
          for (int i = k + 1; i < 8; ++i) a[i][k] *= rs;
#pragma unroll
          for (int i = k + 1; i < 8; ++i)
#pragma unroll
            for (int c = k + 1; c <= i; ++c) a[i][c] = fma(-a[i][k], a[c][k], a[i][c]);
          // W <- E_k^{-1} W: row k scaled by 1/l_kk, rows i > k minus l_ik * (new row k)
#pragma unroll
          for (int c = 0; c <= k; ++c) wv[k][c] *= rs;
#pragma unroll
          for (int i = k + 1; i < 8; ++i)
#pragma unroll
            for (int c = 0; c <= k; ++c) wv[i][c] = fma(-a[i][k], wv[k][c], wv[i][c]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          ldg[R + i] = a[i][i];
          double *rp = D + (R + i) * T + (R ^ ((i & 3) << 3));
#pragma unroll
          for (int c = 0; c < 8; c += 2)
            *(double2 *)(rp + (c ^ (i & 4))) =
                make_double2(c <= i ? wv[i][c] : 0.0, c + 1 <= i ? wv[i][c + 1] : 0.0);
        }
      }
      __syncwarp();
      if (stamp && l == 0) stamp[2 * j] = gtimer();
      nbar_arrive(1 + (j & 1));  // W_jj published
      if (j == 7) {
        nbar_sync(3 + (6 & 1));  // the workers' round 6 (complete every barrier generation)
        break;
      }
      if (j > 0) nbar_sync(3 + ((j - 1) & 1));  // the workers' round j-1 is done
      // look-ahead: the next diagonal block gets its panel-j update from this warp
      const int ti[4] = {j + 1, 0, 0, 0}, tk[4] = {j + 1, 0, 0, 0};
      const bool on[4] = {true, false, false, false};
      trail_tiles(D, Pscr, R, ti, tk, on);
      if (stamp && l == 0) stamp[2 * j + 1] = gtimer();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) bad = min(bad, __shfl_xor_sync(FULL, bad, o));
    if (l == 0) *s_bad = bad;
  } else {
    const int wk = w - 1;
    // this warp's 8 x 8 scratch: columns 8w..8w+7 of Wd
    for (int j = 0; j < 8; ++j) {
      const int R = 8 * j;
      nbar_sync(1 + (j & 1));  // W_jj ready
      // items: trailing tiles (i, k), j < k <= i, except (j+1, j+1); then the blocks
      // (j, m), m < j, of W; round-robin over the 7 workers (<= 4 each)
      const int nb = 7 - j, np = j < 7 ? nb * (nb + 1) / 2 - 1 : 0;
      int ti[4], tk[4];
      bool on[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = wk + 7 * u;
        on[u] = t < np;
        int ii = 0, tt = on[u] ? t + 1 : 1;  // skip tile 0 = (j+1, j+1)
        while (tt > ii) {
          tt -= ii + 1;
          ++ii;
        }
        ti[u] = j + 1 + ii;
        tk[u] = j + 1 + tt;
      }
      if (np > 0) trail_tiles(D, Pscr + 512 * w, R, ti, tk, on);
#pragma unroll 1
      for (int u = 0; u < 4; ++u) {
        const int m = wk + 7 * u - np;
        if (m < 0 || m >= j) continue;
        // T = sum_{k=m}^{j-1} L_jk W_km (L_jk^T in the scratch block (k, j))
        double t2[2] = {0.0, 0.0};
        for (int k = m; k < j; ++k) {
#pragma unroll
          for (int kk = 0; kk < 8; kk += 4)
            dmma(t2, D[swz(8 * k + kk + lc, R + lr)], D[swz(8 * k + kk + lc, 8 * m + lr)]);
        }
        *(double2 *)(Wd + swz(lr, 8 * w + 2 * lc)) = make_double2(t2[0], t2[1]);
        __syncwarp();
        double w2[2] = {0.0, 0.0};
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4) dmma(w2, -D[swz(R + lr, R + kk + lc)], Wd[swz(kk + lc, 8 * w + lr)]);
        *(double2 *)(D + swz(R + lr, 8 * m + 2 * lc)) = make_double2(w2[0], w2[1]);
        __syncwarp();
      }
      if (j < 7) nbar_arrive(3 + (j & 1));  // round j done
    }
  }
  __syncthreads();
  // strict-upper blocks (the panel scratch) -> 0: W is lower triangular
  for (int i = tid; i < TD; i += NT) {
    const int r = i >> 6, c = i & 63;
    if ((c >> 3) > (r >> 3)) D[swz(r, c)] = 0.0;
  }
  __syncthreads();
  if (stamp && tid == 0) stamp[15] = gtimer();
}

// sum_t log(ldg[t]) in a fixed order (warp w of the caller; all lanes get it)
__device__ __forceinline__ double logsum64(const double *ldg) {
  const int l = threadIdx.x & 31;
  double v = log(ldg[l]) + log(ldg[l + 32]);
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// phase timestamps of the first partition of CTA 1 (a middle partition when P >= 3)
#define SB_STAMP(kern, k, ph)                                                                           \
  if (prm.trace && blockIdx.x == (gridDim.x > 1 ? 1 : 0) && p == (int)blockIdx.x && threadIdx.x == 0 && \
      (k) < 128 && prm.lvl < 16)                                                                        \
    prm.trace[(((size_t)prm.lvl * 2 + (kern)) * 128 + (k)) * 8 + (ph)] = gtimer();

struct Chain {
  int type;
  int64_t s, e;  // block range of the partition
  int nn;        // nodes in the chain
  int nel;       // eliminated nodes (0..nel-1)
  int dir;       // +1: node k = block s0 + k;  -1: node k = block e - 1 - k
  int64_t s0;
  __device__ int64_t blk(int k) const { return dir > 0 ? s0 + k : e - 1 - k; }
};

__device__ Chain chain_of(const Level &L, int p) {
  Chain c;
  c.s = L.starts[p];
  c.e = L.starts[p + 1];
  const int cnt = (int)(c.e - c.s);
  c.type = L.P == 1 ? P_SEQ : (p == 0 ? P_TOP : (p == L.P - 1 ? P_BOT : P_MID));
  c.dir = c.type == P_BOT ? -1 : 1;
  c.s0 = c.type == P_MID ? c.s + 1 : c.s;
  c.nn = c.type == P_MID ? cnt - 1 : cnt;
  c.nel = c.type == P_SEQ ? cnt : (c.type == P_MID ? cnt - 2 : cnt - 1);
  return c;
}

// coupling block between node k+1 and node k (rows of node k+1): storage and orientation
__device__ __forceinline__ double *coupling(const Level &L, const Chain &c, int k, int64_t bb, bool *trans) {
  if (c.dir > 0) {
    *trans = false;
    return L.Lo + c.blk(k) * bb;
  }
  *trans = true;  // A_{j-1,j} = A_{j,j-1}^T, stored at Lo[j-1]
  return L.Lo + (c.blk(k) - 1) * bb;
}

// ---------------------------------------------------------------------------
// PPOBTAF (Alg. 3-4; Alg. 1 for the last level) of the partitions of one level.
// ---------------------------------------------------------------------------
template <int ARR>
constexpr int f_smem_doubles() { return 3 * TD + ARR * T + 8 * T + T + 8 + TD + ARR * T + 8 * 512; }

template <int ARR>
__global__ void __launch_bounds__(NT, 1) sb_factor_kernel(Params prm) {
  constexpr int AR = ARR, AD = ARR * T, NA = ARR / 8, NU = NA * NA;
  extern __shared__ __align__(16) double sm[];
  double *D = sm, *X = D + TD, *B = X + TD, *Ar = B + TD, *Wd = Ar + AD, *ldg = Wd + 8 * T;
  double *Dn = ldg + T + 8, *An = Dn + TD;  // the next node's diagonal / arrow blocks (prefetched)
  double *Pscr = An + AD;                   // Cholesky per-warp scratch
  __shared__ int s_bad;
  const Level &L = prm.L;
  const int b = prm.b, a = prm.a, tid = threadIdx.x, w = tid >> 5;
  const int64_t bb = (int64_t)b * b, ab = (int64_t)a * b;
  const Frags<2, 4> F = lay64(w);
  const Frags<1, NA> FA = layA<ARR>(w);
  const Frags<1, 1> FU = layU<ARR>(w);

  for (int p = blockIdx.x; p < L.P; p += gridDim.x) {
    const Chain c = chain_of(L, p);
    const bool mid = c.type == P_MID;
    double lsum = 0.0;
    int firstbad = 0, firstnan = 0;
    // running diagonal / arrow blocks of node 0 (and B_{s+1} = A_{s+1,s}^T, Alg. 4 l.1)
    ld_tile(D, L.D + c.blk(0) * bb, T, b, b, b, false, true);
    ld_tile(Ar, L.Ar + c.blk(0) * ab, AR, a, b, b, false, false);
    if (mid) ld_tile(B, L.Lo + c.s * bb, T, b, b, b, true, false);
    cp_wait_all();
    __syncthreads();
    double Aff[2][4][2], Anf[1][NA][2], Uac[1][1][2];
    acc_zero(Aff);
    acc_zero(Anf);
    acc_zero(Uac);
    for (int k = 0; k < c.nel; ++k) {
      const int64_t bk = c.blk(k);
      const bool nxt = k + 1 < c.nn;
      SB_STAMP(0, k, 0);
      bool tr = false;
      double *cpl = nxt ? coupling(L, c, k, bb, &tr) : nullptr;
      if (nxt) {  // the step's HBM inputs, in flight while the Cholesky runs
        ld_tile(X, cpl, T, b, b, b, tr, false);
        ld_tile(Dn, L.D + c.blk(k + 1) * bb, T, b, b, b, false, true);
        if (a > 0) ld_tile(An, L.Ar + c.blk(k + 1) * ab, AR, a, b, b, false, false);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      unsigned long long *cst = nullptr;  // chol-internal stamps of the traced partition (level slot 8 + lvl)
      if (prm.trace && blockIdx.x == (gridDim.x > 1 ? 1 : 0) && p == (int)blockIdx.x && k < 64 && prm.lvl < 8)
        cst = prm.trace + (((size_t)(8 + prm.lvl) * 2) * 128 + 2 * k) * 8;
      chol_inv64(D, Wd, Pscr, ldg, &s_bad, cst);  // D <- W_k
      SB_STAMP(0, k, 1);
      if (w == 7) {
        const double ls = logsum64(ldg);
        if (tid == NT - 32) lsum += ls;  // one thread keeps the partition's partial (fixed order)
      }
      if (tid == 0 && s_bad < 2 * b && firstbad == 0) {
        firstbad = (int)(L.grow[bk] + (s_bad >> 1) + 1);
        firstnan = s_bad & 1;
      }
      st_tile(L.D + bk * bb, D, b, b, b, false);  // W_k -> diag slot
      cp_wait_all();
      __syncthreads();
      SB_STAMP(0, k, 2);
      // ---- TRSMs (products with W^T; in place, row strips shared by warp pairs only)
      if (nxt) {  // L_{k+1,k} = A_{k+1,k} W^T
        double acc[2][4][2];
        acc_zero(acc);
        mma64<false, true, false, B_LE>(acc, X, D, F);
        pair_sync();
        acc_st_smem(X, acc, F, 1.0);
        acc_st_global(cpl, acc, b, b, b, F, tr, 1.0);
      }
      if (mid) {  // L_{f,k} = B_k W^T (Alg. 4, fill-in TRSM)
        double acc[2][4][2];
        acc_zero(acc);
        mma64<false, true, false, B_LE>(acc, B, D, F);
        pair_sync();
        acc_st_smem(B, acc, F, 1.0);
        acc_st_global(L.Bf + bk * bb, acc, b, b, b, F, false, 1.0);
      }
      if (a > 0) {  // L_{n,k} = A_{n,k} W^T
        double acc[1][NA][2];
        acc_zero(acc);
        mma<1, NA, false, true, false, B_LE>(acc, Ar, D, FA, T);
        __syncthreads();
        acc_st_smem(Ar, acc, FA, 1.0);
        acc_st_global(L.Ar + bk * ab, acc, b, a, b, FA, false, 1.0);
      }
      __syncthreads();
      SB_STAMP(0, k, 3);
      // ---- Schur updates (Alg. 1 l.5-7, Alg. 4 l.9-12); W is dead
      if (nxt) {  // A_{k+1,k+1} - L_{k+1,k} L_{k+1,k}^T -> D
        double acc[2][4][2];
        acc_ld_smem(acc, Dn, F);
        mma64<false, true, true>(acc, X, X, F);
        acc_st_smem(D, acc, F, 1.0);
      }
      if (a > 0) {
        if (w < NU) mma<1, 1, false, true, true>(Uac, Ar, Ar, FU, T);  // U -= Ln Ln^T
        if (mid) mma<1, NA, false, true, true>(Anf, Ar, B, FA, T);       // A_nf -= Ln B^T
      }
      if (mid) mma64<false, true, true>(Aff, B, B, F);  // A_ff -= B B^T
      double accA[1][NA][2];
      if (a > 0 && nxt) {  // A_{n,k+1} - L_{n,k} L_{k+1,k}^T
        acc_ld_smem(accA, An, FA);
        mma<1, NA, false, true, true>(accA, Ar, X, FA, T);
      }
      double accB[2][4][2];
      if (mid && nxt) {  // B_{k+1} = -B_k L_{k+1,k}^T
        acc_zero(accB);
        mma64<false, true, true>(accB, B, X, F);
      }
      __syncthreads();
      if (a > 0 && nxt) acc_st_smem(Ar, accA, FA, 1.0);
      if (mid && nxt) acc_st_smem(B, accB, F, 1.0);
      __syncthreads();
      SB_STAMP(0, k, 4);
    }
    // a NaN pivot (propagated from a failure elsewhere, or NaN input) counts only if there
    // is no genuine one anywhere (merged by the last level)
    if (tid == 0 && firstbad) record_info(firstnan ? prm.info2 : prm.info, firstbad);
    if (tid == NT - 32) L.ldp[p] = lsum;
    const int64_t aa = (int64_t)a * a;
    if (c.type != P_SEQ) {
      // ---- boundary blocks -> the reduced system (reading R9 / R14 order)
      const int ib = c.type == P_TOP ? 0 : (c.type == P_MID ? 2 * p : 2 * p - 1);
      st_tile(L.Dn + ib * bb, D, b, b, b, false);
      if (a > 0) st_tile(L.Arn + ib * ab, Ar, a, b, b, false);
      if (c.type != P_BOT) cp_block(L.Lon + (int64_t)(c.type == P_TOP ? 0 : 2 * p) * bb, L.Lo + (c.e - 1) * bb, bb);
      if (mid) {
        // A_ff + sum(-B B^T), A_{n,f} + sum(-Ln B^T), (L_p, F_p) coupling = B_{e-1}^T
        double acc[2][4][2];
        acc_ld(acc, L.D + c.s * bb, b, b, b, F, false);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[i][j][0] += Aff[i][j][0];
            acc[i][j][1] += Aff[i][j][1];
          }
        acc_st_global(L.Dn + (2 * p - 1) * bb, acc, b, b, b, F, false, 1.0);
        if (a > 0) {
          double acn[1][NA][2];
          acc_ld(acn, L.Ar + c.s * ab, b, a, b, FA, false);
#pragma unroll
          for (int j = 0; j < NA; ++j) {
            acn[0][j][0] += Anf[0][j][0];
            acn[0][j][1] += Anf[0][j][1];
          }
          acc_st_global(L.Arn + (2 * p - 1) * ab, acn, b, a, b, FA, false, 1.0);
        }
        st_tile(L.Lon + (int64_t)(2 * p - 1) * bb, B, b, b, b, true);
      }
      if (a > 0 && w < NU) acc_st_global(L.U + p * aa, Uac, a, a, a, FU, false, 1.0);
    } else if (a > 0) {
      // ---- tip (Alg. 1 l.12): L_nn = chol(A_nn + sum of every level's U), X_nn = W^T W (Alg. 2 l.1)
      __syncthreads();
      ld_tile(D, prm.tip, T, a, a, a, false, true);
      __syncthreads();
      if (w < NU) {
        const int l = tid & 31, mm = 8 * FU.rf[0] + (l >> 2), nn2 = 8 * FU.cf[0] + 2 * (l & 3);
        D[swz(mm, nn2)] += Uac[0][0][0];
        D[swz(mm, nn2 + 1)] += Uac[0][0][1];
      }
      __syncthreads();
      chol_inv64(D, Wd, Pscr, ldg, &s_bad);
      if (w == 7) {
        const double ls = logsum64(ldg);
        if (tid == NT - 32) lsum += ls;
      }
      if (tid == 0 && s_bad < 2 * a)
        record_info((s_bad & 1) ? prm.info2 : prm.info, (int)(prm.tip_row + (s_bad >> 1) + 1));
      if (w < NU) {
        double acc[1][1][2];
        acc_zero(acc);
        mma<1, 1, true, false, false>(acc, D, D, FU, T);
        acc_st_global(prm.tip, acc, a, a, a, FU, false, 1.0);
      }
      if (tid == NT - 32) L.ldp[p] = lsum;
    }
    __syncthreads();
  }
  // ---- last CTA out: tip += sum_p U_p (partition order, reading R8); last level: log det
  __shared__ int s_last;
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(L.done, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (L.P > 1 && a > 0) {
    for (int i = tid; i < a * a; i += NT) {
      double v = prm.tip[i];
      for (int q = 0; q < L.P; ++q) v += *(volatile double *)(L.U + (int64_t)q * a * a + i);
      prm.tip[i] = v;
    }
  }
  if (L.P == 1 && tid == 0) {
    if (*(volatile int *)prm.info == 0) {
      const int i2 = *(volatile int *)prm.info2;
      if (i2) *prm.info = i2;
    }
    double s = 0.0;
    for (int i = 0; i < prm.n_ldp; ++i) s += *(volatile const double *)(prm.ldp_all + i);
    const int inf = *(volatile int *)prm.info;
    *prm.logdet = inf ? __longlong_as_double(0x7ff8000000000000ULL) : 2.0 * s;
  }
}

// ---------------------------------------------------------------------------
// PPOBTASI (Alg. 5-6; Alg. 2 for the last level), W-form:
//   Lc~ = L_{k+1,k} W, Ln~ = L_{n,k} W, Lf~ = L_{f,k} W, Lam = W^T W
//   X_{k+1,k} = -(X_{k+1,k+1} Lc~ + X_{n,k+1}^T Ln~ + Q_{k+1}^T Lf~)
//   Q_k       = -(Q_{k+1} Lc~ + X_ff Lf~ + X_nf^T Ln~)                 (middle)
//   X_{n,k}   = -(X_{n,k+1} Lc~ + X_nn Ln~ + X_nf Lf~)
//   X_kk      = Lam - X_{k+1,k}^T Lc~ - X_{n,k}^T Ln~ - Q_k^T Lf~
// (reading R11: l.7's L_{0,i} is the factor fill-in block; Q_k = X_{f,k}).
// ---------------------------------------------------------------------------
template <int ARR>
constexpr int i_smem_doubles() { return 6 * TD + 4 * ARR * T; }

// ---------------------------------------------------------------------------
// W-form precompute of one level (level 0), run on the SMs the nested levels leave
// idle (a second stream, between the level's factor and inverse kernels): for every
// eliminated node k, in place,
//   W_k -> Lam_k = W_k^T W_k (diag slot),  L_{k+1,k} -> Lc~ = L_{k+1,k} W_k (coupling slot),
//   L_{f,k} -> Lf~ = L_{f,k} W_k (Bf),     L_{n,k} -> Ln~ = L_{n,k} W_k (arrow slot)
// -- the inverse's first products, which need only the factor.  Nothing else
// reads these slots before the level's inverse kernel (the nested levels work on their
// own arrays; the inter-partition couplings are not eliminated nodes).  2 CTAs / SM.
// ---------------------------------------------------------------------------
template <int ARR>
constexpr int p_smem_doubles() { return 2 * (3 * TD + ARR * T); }

// one CTA per SM (its two operand sets fill the SM's shared memory), so the nested
// levels' kernels keep the SMs the caller leaves free.  Items (partition p, node k) are
// claimed one by one from a shared counter (*claim), item it = (p = it % P, k = it / P),
// so several launches of this kernel (started as the nested levels free SMs) share the
// work; the claim of item j + 2 is in flight while item j is computed and item j + 1's
// operands arrive.
template <int ARR>
__global__ void __launch_bounds__(NT, 1) sb_pre_kernel(Params prm, int kmax, int *claim) {
  constexpr int AR = ARR, NA = ARR / 8, SET = 3 * TD + ARR * T;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_next;
  const Level &L = prm.L;
  const int b = prm.b, a = prm.a, w = threadIdx.x >> 5;
  const int64_t bb = (int64_t)b * b, ab = (int64_t)a * b;
  const Frags<2, 4> F = lay64(w);
  const Frags<1, NA> FA = layA<ARR>(w);
  const int nit = L.P * kmax;
  auto node = [&](int it, Chain &c, int &k) {
    c = chain_of(L, it % L.P);
    k = it / L.P;
    return k < c.nel;
  };
  // operands of item it into set s: W_k, L_{k+1,k}, L_{f,k}, L_{n,k}
  auto load = [&](int it, int s) {
    Chain c;
    int k;
    if (node(it, c, k)) {
      const int64_t bk = c.blk(k);
      double *W = sm + s * SET, *Y = W + TD, *Z = Y + TD, *N = Z + TD;
      ld_tile(W, L.D + bk * bb, T, b, b, b, false, true, true);
      if (k + 1 < c.nn) {
        bool tr = false;
        const double *g = coupling(L, c, k, bb, &tr);
        ld_tile(Y, g, T, b, b, b, tr, false, true);
      }
      if (c.type == P_MID) ld_tile(Z, L.Bf + bk * bb, T, b, b, b, false, false, true);
      if (a > 0) ld_tile(N, L.Ar + bk * ab, AR, a, b, b, false, false, true);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if (threadIdx.x == 0) s_next = atomicAdd(claim, 1);
  __syncthreads();
  int cur = s_next;
  __syncthreads();
  if (threadIdx.x == 0) s_next = atomicAdd(claim, 1);
  __syncthreads();
  int nx = s_next;
  if (cur < nit) load(cur, 0);
  for (int j = 0; cur < nit; ++j) {
    if (nx < nit) {
      load(nx, (j + 1) & 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    int nn = 0;
    if (threadIdx.x == 0 && nx < nit) nn = atomicAdd(claim, 1);  // consumed after this item's products
    __syncthreads();
    Chain c;
    int k;
    if (node(cur, c, k)) {
      const int64_t bk = c.blk(k);
      double *W = sm + (j & 1) * SET, *Y = W + TD, *Z = Y + TD, *N = Z + TD;
      double aX[2][4][2];
      acc_zero(aX);
      mma64<true, false, false, B_GE>(aX, W, W, F);  // Lam = W^T W
      acc_st_global<2, 4, false, false, true>(L.D + bk * bb, aX, b, b, b, F, false, 1.0);
      if (k + 1 < c.nn) {  // Lc~ = L_{k+1,k} W
        bool tr = false;
        double *cpl = coupling(L, c, k, bb, &tr);
        acc_zero(aX);
        mma64<false, false, false, B_GE>(aX, Y, W, F);
        acc_st_global<2, 4, false, false, true>(cpl, aX, b, b, b, F, tr, 1.0);
      }
      if (c.type == P_MID) {  // Lf~ = L_{f,k} W
        acc_zero(aX);
        mma64<false, false, false, B_GE>(aX, Z, W, F);
        acc_st_global<2, 4, false, false, true>(L.Bf + bk * bb, aX, b, b, b, F, false, 1.0);
      }
      if (a > 0) {  // Ln~ = L_{n,k} W
        double aN[1][NA][2];
        acc_zero(aN);
        mma<1, NA, false, false, false, B_GE>(aN, N, W, FA, T);
        acc_st_global<1, NA, false, false, true>(L.Ar + bk * ab, aN, b, a, b, FA, false, 1.0);
      }
    }
    if (threadIdx.x == 0) s_next = nx < nit ? nn : nit;
    __syncthreads();  // set j & 1 is reloaded by the next iteration's prefetch; s_next published
    cur = nx;
    nx = s_next;
  }
}

// PRE: the level's Lam, Lc~, Lf~, Ln~ were precomputed in place (sb_pre_kernel)
template <int ARR, bool PRE>
__global__ void __launch_bounds__(NT, 1) sb_inverse_kernel(Params prm) {
  constexpr int AR = ARR, AD = ARR * T, NA = ARR / 8;
  extern __shared__ __align__(16) double sm[];
  double *W = sm, *Lc = W + TD, *Lf = Lc + TD, *Xd = Lf + TD, *Q = Xd + TD, *Xff = Q + TD;
  double *Ln = Xff + TD, *Xn = Ln + AD, *Xnf = Xn + AD, *Xnn = Xnf + AD;
  const Level &L = prm.L;
  const int b = prm.b, a = prm.a, tid = threadIdx.x, w = tid >> 5;
  const int64_t bb = (int64_t)b * b, ab = (int64_t)a * b;
  const Frags<2, 4> F = lay64(w);
  const Frags<1, NA> FA = layA<ARR>(w);

  for (int p = blockIdx.x; p < L.P; p += gridDim.x) {
    const Chain c = chain_of(L, p);
    const bool mid = c.type == P_MID;
    // ---- seeds: the boundary blocks of X from the solved reduced system (reading R10)
    if (a > 0) ld_tile(Xnn, prm.tip, AR, a, a, a, false, true);
    if (c.type != P_SEQ) {
      const int ib = c.type == P_TOP ? 0 : (c.type == P_MID ? 2 * p : 2 * p - 1);
      const int64_t bblk = c.type == P_BOT ? c.s : c.e - 1;  // the boundary block of the chain
      ld_tile(Xd, L.Dn + ib * bb, T, b, b, b, false, true);
      if (a > 0) ld_tile(Xn, L.Arn + ib * ab, AR, a, b, b, false, false);
      cp_block(L.D + bblk * bb, L.Dn + ib * bb, bb);
      if (a > 0) cp_block(L.Ar + bblk * ab, L.Arn + ib * ab, ab);
      if (c.type != P_BOT) cp_block(L.Lo + (c.e - 1) * bb, L.Lon + (int64_t)(c.type == P_TOP ? 0 : 2 * p) * bb, bb);
      if (mid) {
        ld_tile(Xff, L.Dn + (2 * p - 1) * bb, T, b, b, b, false, true);
        if (a > 0) ld_tile(Xnf, L.Arn + (2 * p - 1) * ab, AR, a, b, b, false, false);
        ld_tile(Q, L.Lon + (int64_t)(2 * p - 1) * bb, T, b, b, b, true, false);  // Q_{e-1} = X_{f,l} = X_r(L,F)^T
        cp_block(L.D + c.s * bb, L.Dn + (2 * p - 1) * bb, bb);
        if (a > 0) cp_block(L.Ar + c.s * ab, L.Arn + (2 * p - 1) * ab, ab);
      }
    }
    cp_wait_all();
    __syncthreads();
    // step operands: group 1 = W_k and L_{k+1,k}, group 2 = L_{f,k} and L_{n,k}.  The
    // first step's are loaded here; every later step's are prefetched by the step
    // before, into buffers as soon as its X_kk products are done with them.
    auto load_wc = [&](int k) {
      ld_tile(W, L.D + c.blk(k) * bb, T, b, b, b, false, true);
      if (k + 1 < c.nn) {
        bool t2 = false;
        const double *g = coupling(L, c, k, bb, &t2);
        ld_tile(Lc, g, T, b, b, b, t2, false);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    auto load_fn = [&](int k) {
      if (mid) ld_tile(Lf, L.Bf + c.blk(k) * bb, T, b, b, b, false, false);
      if (a > 0) ld_tile(Ln, L.Ar + c.blk(k) * ab, AR, a, b, b, false, false);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    if (c.nel > 0) {
      load_wc(c.nel - 1);
      load_fn(c.nel - 1);
    }
    for (int k = c.nel - 1; k >= 0; --k) {
      const int64_t bk = c.blk(k);
      const bool nxt = k + 1 < c.nn;
      bool tr = false;
      double *cpl = nxt ? coupling(L, c, k, bb, &tr) : nullptr;
      SB_STAMP(1, k, 0);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      __syncthreads();
      // ---- Lam = W^T W (lower half) while the other operands arrive
      double aX[2][4][2];
      if (PRE) {
        acc_ld_smem(aX, W, F);  // Lam (precomputed)
      } else {
        acc_zero(aX);
        mma64<true, false, false, B_GE>(aX, W, W, F);
      }
      cp_wait_all();
      __syncthreads();
      SB_STAMP(1, k, 1);
      // ---- Lc~, Lf~, Ln~ (W lower)
      if (!PRE) {
        double aL[2][4][2], aF[2][4][2], aN[1][NA][2];
        if (nxt) {
          acc_zero(aL);
          mma64<false, false, false, B_GE>(aL, Lc, W, F);
        }
        if (mid) {
          acc_zero(aF);
          mma64<false, false, false, B_GE>(aF, Lf, W, F);
        }
        if (a > 0) {
          acc_zero(aN);
          mma<1, NA, false, false, false, B_GE>(aN, Ln, W, FA, T);
        }
        __syncthreads();
        if (nxt) acc_st_smem(Lc, aL, F, 1.0);
        if (mid) acc_st_smem(Lf, aF, F, 1.0);
        if (a > 0) acc_st_smem(Ln, aN, FA, 1.0);
      }
      __syncthreads();
      SB_STAMP(1, k, 2);
      // ---- X_{k+1,k}, Q_k, X_{n,k}  (W is dead: its buffer receives X_{k+1,k})
      {
        double aA[2][4][2], aB[2][4][2], aN[1][NA][2];
        if (nxt) {
          acc_zero(aA);
          mma64<false, false, false>(aA, Xd, Lc, F);
          if (a > 0) mma64<true, false, false, K_FULL, false, AR>(aA, Xn, Ln, F);
          if (mid) mma64<true, false, false>(aA, Q, Lf, F);
        }
        if (mid) {
          acc_zero(aB);
          mma64<false, false, false>(aB, Q, Lc, F);
          mma64<false, false, false>(aB, Xff, Lf, F);
          if (a > 0) mma64<true, false, false, K_FULL, false, AR>(aB, Xnf, Ln, F);
        }
        if (a > 0) {
          acc_zero(aN);
          if (nxt) mma<1, NA, false, false, false>(aN, Xn, Lc, FA, T);
          mma<1, NA, false, false, false>(aN, Xnn, Ln, FA, AR);
          if (mid) mma<1, NA, false, false, false>(aN, Xnf, Lf, FA, T);
        }
        __syncthreads();
        if (nxt) {
          acc_st_smem(W, aA, F, -1.0);
          acc_st_global(cpl, aA, b, b, b, F, tr, -1.0);
        }
        if (mid) acc_st_smem(Q, aB, F, -1.0);
        if (a > 0) {
          acc_st_smem(Xn, aN, FA, -1.0);
          acc_st_global(L.Ar + bk * ab, aN, b, a, b, FA, false, -1.0);
        }
      }
      __syncthreads();
      SB_STAMP(1, k, 3);
      // ---- X_kk = Lam - X_{k+1,k}^T Lc~ - X_{n,k}^T Ln~ - Q_k^T Lf~; the next step's
      // W, L_{k,k-1} go into the W / Lc buffers once the first product has read them,
      // its L_{f,k-1}, L_{n,k-1} into Lf / Ln after the last
      if (nxt) mma64<true, false, true>(aX, W, Lc, F);
      __syncthreads();
      if (k > 0) load_wc(k - 1);
      if (a > 0) mma64<true, false, true, K_FULL, false, AR>(aX, Xn, Ln, F);
      if (mid) mma64<true, false, true>(aX, Q, Lf, F);
      acc_st_smem(Xd, aX, F, 1.0);
      __syncthreads();
      if (k > 0) load_fn(k - 1);
      st_tile(L.D + bk * bb, Xd, b, b, b, false);  // coalesced
      SB_STAMP(1, k, 4);
    }
    if (mid) {  // X_{s+1,s} = Q_{s+1}^T (reading R10)
      st_tile(L.Lo + c.s * bb, Q, b, b, b, true);
      __syncthreads();
    }
  }
}

}  // namespace dev

// ---------------------------------------------------------------------------
// Host: plan and launches
// ---------------------------------------------------------------------------
bool make_plan(int64_t n, int64_t b, int64_t a, const std::vector<int> &Ps, Plan &pl) {
  if (n < 1 || b < 1 || b > kMaxB || a < 0 || a > kMaxA) return false;
  pl = Plan();
  pl.n = n;
  pl.b = b;
  pl.a = a;
  pl.Ps = Ps;
  const int nl = (int)Ps.size();
  std::vector<int64_t> grow0(n);
  for (int64_t i = 0; i < n; ++i) grow0[i] = i * b;
  pl.grow.push_back(grow0);
  pl.nlev.push_back(n);
  int64_t m = n;
  for (int l = 0; l < nl; ++l) {
    const int P = Ps[l];
    std::vector<int64_t> st;
    if (P < 2 || !plan_partitions_ends(m, P, 1.0, st)) return false;
    for (int p = 0; p < P; ++p) {  // sizes: ends >= 1, middles >= 2
      const int64_t cnt = st[p + 1] - st[p];
      if (cnt < ((p == 0 || p == P - 1) ? 1 : 2)) return false;
    }
    pl.starts.push_back(st);
    const int64_t nr = 2 * (int64_t)P - 2;
    const std::vector<int64_t> &g = pl.grow.back();
    std::vector<int64_t> gr(nr);
    gr[0] = g[st[1] - 1];
    for (int p = 1; p < P; ++p) {
      gr[2 * p - 1] = g[st[p]];
      if (p < P - 1) gr[2 * p] = g[st[p + 1] - 1];
    }
    pl.grow.push_back(gr);
    pl.nlev.push_back(nr);
    m = nr;
  }
  // workspace: per level l >= 1 arrays D, Lo, Ar; per partitioned level Bf, U, ldp; tables; counters
  int64_t o = 0;
  auto take = [&](int64_t d) {
    const int64_t r = o;
    o += (std::max<int64_t>(d, 1) + 31) / 32 * 32;
    return r;
  };
  const int L = nl + 1;
  pl.off_D.assign(L, -1);
  pl.off_Lo.assign(L, -1);
  pl.off_Ar.assign(L, -1);
  pl.off_Bf.assign(L, -1);
  pl.off_U.assign(L, -1);
  pl.off_ldp.assign(L, -1);
  for (int l = 1; l < L; ++l) {
    const int64_t nr = pl.nlev[l];
    pl.off_D[l] = take(nr * b * b);
    pl.off_Lo[l] = take(std::max<int64_t>(nr - 1, 1) * b * b);
    pl.off_Ar[l] = take(nr * a * b);
  }
  for (int l = 0; l < L; ++l) {
    const int P = l < nl ? Ps[l] : 1;
    if (l < nl) {
      pl.off_Bf[l] = take(pl.nlev[l] * b * b);
      pl.off_U[l] = take((int64_t)P * a * a);
    }
  }
  // all log-det partials contiguous (summed in level order, partition order)
  {
    int64_t tot = 0;
    for (int l = 0; l < L; ++l) tot += l < nl ? Ps[l] : 1;
    const int64_t base = take(tot);
    int64_t q = base;
    for (int l = 0; l < L; ++l) {
      pl.off_ldp[l] = q;
      q += l < nl ? Ps[l] : 1;
    }
  }
  int64_t t = 0;  // offsets into the plan's index table (int64, library-owned device copy)
  pl.off_starts.assign(L, -1);
  pl.off_grow.assign(L, -1);
  for (int l = 0; l < L; ++l) {
    pl.off_starts[l] = t;
    t += l < nl ? Ps[l] + 1 : 2;
    pl.off_grow[l] = t;
    t += pl.nlev[l];
  }
  pl.off_ctr = take(L + 1);  // exit counters per level, then info2
  pl.ws_doubles = o;
  return true;
}

std::vector<int64_t> plan_tables(const Plan &pl) {
  std::vector<int64_t> tab;
  const int nl = (int)pl.Ps.size();
  for (int l = 0; l <= nl; ++l) {
    if (l < nl)
      tab.insert(tab.end(), pl.starts[l].begin(), pl.starts[l].end());
    else {
      tab.push_back(0);
      tab.push_back(pl.nlev[l]);
    }
    tab.insert(tab.end(), pl.grow[l].begin(), pl.grow[l].end());
  }
  return tab;
}

// Level 0: one partition per SM (the chain of ~n/148 blocks is the level's
// critical path).  Deeper levels: short partitions (~6 blocks) until the reduced
// system has <= 12 blocks, then its two ends (P = 2), then the last level solves the
// remaining <= 4 blocks as one chain.
std::vector<int> auto_plan(int64_t n, int64_t b, int sms) {
  (void)b;
  std::vector<int> Ps;
  int64_t m = n;
  const int64_t seq_max = 4;
  bool first = true;
  while (m > seq_max) {
    // level 0: one partition per SM; then ~6-block partitions; a short last system
    // (<= 12 blocks) is split once more into its two fill-in-free ends (measured ~1 %)
    int64_t P = first ? std::min<int64_t>(sms, m / 8) : (m <= 12 ? 2 : m / 6);
    if (P < 2) break;
    std::vector<int64_t> st;
    while (P >= 2 && !plan_partitions_ends(m, (int)P, 1.0, st)) --P;
    if (P < 2) break;
    Ps.push_back((int)P);
    m = 2 * P - 2;
    first = false;
    if (Ps.size() > 12) break;
  }
  return Ps;
}

bool Side::ensure() {
  if (s) return true;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&fork2, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&join2, cudaEventDisableTiming) != cudaSuccess) {
    destroy();
    return false;
  }
  return true;
}

void Side::destroy() {
  if (s) cudaStreamDestroy(s);
  if (s2) cudaStreamDestroy(s2);
  for (cudaEvent_t e : {fork, join, fork2, join2})
    if (e) cudaEventDestroy(e);
  s = s2 = nullptr;
  fork = join = fork2 = join2 = nullptr;
}

int run(const Plan &pl, const int64_t *d_tab, double *diag, double *lower, double *arrow, double *tip, double *ws,
        int *d_info, double *d_logdet, int sms, cudaStream_t st, int *launches, Side *side, unsigned long long *trace) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(dev::sb_pre_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dev::p_smem_doubles<8>() * 8) != cudaSuccess ||
        cudaFuncSetAttribute(dev::sb_pre_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dev::p_smem_doubles<16>() * 8) != cudaSuccess ||
        cudaFuncSetAttribute(dev::sb_inverse_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dev::i_smem_doubles<8>() * 8) != cudaSuccess ||
        cudaFuncSetAttribute(dev::sb_inverse_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dev::i_smem_doubles<16>() * 8) != cudaSuccess)
      return 1;
    if (cudaFuncSetAttribute(dev::sb_factor_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dev::f_smem_doubles<8>() * 8) != cudaSuccess ||
        cudaFuncSetAttribute(dev::sb_factor_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dev::f_smem_doubles<16>() * 8) != cudaSuccess ||
        cudaFuncSetAttribute(dev::sb_inverse_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dev::i_smem_doubles<8>() * 8) != cudaSuccess ||
        cudaFuncSetAttribute(dev::sb_inverse_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dev::i_smem_doubles<16>() * 8) != cudaSuccess)
      return 1;
    attr = true;
  }
  const bool a8 = pl.a <= 8;  // arrow tiles of 8 rows (a <= 8) or 16
  const int nl = (int)pl.Ps.size();
  const int L = nl + 1;
  // exit counters per level, info2, the precompute's claim counter (off_ctr holds L + 1 doubles)
  if (cudaMemsetAsync(ws + pl.off_ctr, 0, (size_t)(L + 2) * sizeof(int), st) != cudaSuccess ||
      cudaMemsetAsync(d_info, 0, sizeof(int), st) != cudaSuccess)
    return 1;
  const int64_t b = pl.b, a = pl.a;
  std::vector<Params> prm(L);
  for (int l = 0; l < L; ++l) {
    Params &q = prm[l];
    Level &v = q.L;
    v.n = pl.nlev[l];
    v.P = l < nl ? pl.Ps[l] : 1;
    v.starts = d_tab + pl.off_starts[l];
    v.grow = d_tab + pl.off_grow[l];
    if (l == 0) {
      v.D = diag;
      v.Lo = lower;
      v.Ar = arrow;
    } else {
      v.D = ws + pl.off_D[l];
      v.Lo = ws + pl.off_Lo[l];
      v.Ar = ws + pl.off_Ar[l];
    }
    v.Bf = l < nl ? ws + pl.off_Bf[l] : nullptr;
    v.U = l < nl ? ws + pl.off_U[l] : nullptr;
    v.ldp = ws + pl.off_ldp[l];
    v.done = (int *)(ws + pl.off_ctr) + l;
    if (l < nl) {
      v.Dn = ws + pl.off_D[l + 1];
      v.Lon = ws + pl.off_Lo[l + 1];
      v.Arn = ws + pl.off_Ar[l + 1];
    } else {
      v.Dn = v.Lon = v.Arn = nullptr;
    }
    q.tip = tip;
    q.b = (int)b;
    q.a = (int)a;
    q.info = d_info;
    q.info2 = (int *)(ws + pl.off_ctr) + L;
    q.lvl = l;
    q.trace = trace;
    q.logdet = d_logdet;
    q.ldp_all = ws + pl.off_ldp[0];
    int64_t tot = 0;
    for (int k = 0; k < L; ++k) tot += k < nl ? pl.Ps[k] : 1;
    q.n_ldp = (int)tot;
    q.tip_row = pl.n * b;
  }
  int nlaunch = 0;
  // level-0 W-form precompute on the SMs the nested levels leave idle (side stream,
  // forked after the level-0 factor kernel, joined before the level-0 inverse kernel)
  int maxp = 1, maxp2 = 1;
  for (int l = 1; l < L; ++l) maxp = std::max(maxp, prm[l].L.P);
  for (int l = 2; l < L; ++l) maxp2 = std::max(maxp2, prm[l].L.P);
  Side *sd = (nl >= 1 && side && side->ensure()) ? side : nullptr;
  const bool pre = sd != nullptr && sms - maxp >= 16;
  bool pre2 = false;
  int *claim = (int *)(ws + pl.off_ctr) + L + 1;
  int kmax = 0;
  if (pre)
    for (int p = 0; p < pl.Ps[0]; ++p) kmax = (int)std::max<int64_t>(kmax, pl.starts[0][p + 1] - pl.starts[0][p]);
  for (int l = 0; l < L; ++l) {
    const int grid = std::max(1, std::min(prm[l].L.P, sms));
    if (a8)
      dev::sb_factor_kernel<8><<<grid, dev::NT, dev::f_smem_doubles<8>() * 8, st>>>(prm[l]);
    else
      dev::sb_factor_kernel<16><<<grid, dev::NT, dev::f_smem_doubles<16>() * 8, st>>>(prm[l]);
    ++nlaunch;
    if (l == 0 && pre) {
      // first share of the SMs the nested levels leave free: all but level 1's
      const int pgrid = sms - prm[1].L.P;
      if (cudaEventRecord(sd->fork, st) != cudaSuccess || cudaStreamWaitEvent(sd->s, sd->fork, 0) != cudaSuccess)
        return 1;
      if (a8)
        dev::sb_pre_kernel<8><<<pgrid, dev::NT, dev::p_smem_doubles<8>() * 8, sd->s>>>(prm[0], kmax, claim);
      else
        dev::sb_pre_kernel<16><<<pgrid, dev::NT, dev::p_smem_doubles<16>() * 8, sd->s>>>(prm[0], kmax, claim);
      ++nlaunch;
      if (cudaEventRecord(sd->join, sd->s) != cudaSuccess) return 1;
    }
    if (l == 1 && pre && L > 2 && prm[1].L.P - maxp2 >= 8) {
      // level 1 done: its SMs (less the deeper levels' widest) join the precompute
      const int pgrid = prm[1].L.P - maxp2;
      if (cudaEventRecord(sd->fork2, st) != cudaSuccess || cudaStreamWaitEvent(sd->s2, sd->fork2, 0) != cudaSuccess)
        return 1;
      if (a8)
        dev::sb_pre_kernel<8><<<pgrid, dev::NT, dev::p_smem_doubles<8>() * 8, sd->s2>>>(prm[0], kmax, claim);
      else
        dev::sb_pre_kernel<16><<<pgrid, dev::NT, dev::p_smem_doubles<16>() * 8, sd->s2>>>(prm[0], kmax, claim);
      ++nlaunch;
      if (cudaEventRecord(sd->join2, sd->s2) != cudaSuccess) return 1;
      pre2 = true;
    }
  }
  for (int l = L - 1; l >= 0; --l) {
    const int grid = std::max(1, std::min(prm[l].L.P, sms));
    const bool pl0 = l == 0 && pre;
    if (pl0 && cudaStreamWaitEvent(st, sd->join, 0) != cudaSuccess) return 1;
    if (pl0 && pre2 && cudaStreamWaitEvent(st, sd->join2, 0) != cudaSuccess) return 1;
    if (a8) {
      if (pl0)
        dev::sb_inverse_kernel<8, true><<<grid, dev::NT, dev::i_smem_doubles<8>() * 8, st>>>(prm[l]);
      else
        dev::sb_inverse_kernel<8, false><<<grid, dev::NT, dev::i_smem_doubles<8>() * 8, st>>>(prm[l]);
    } else {
      if (pl0)
        dev::sb_inverse_kernel<16, true><<<grid, dev::NT, dev::i_smem_doubles<16>() * 8, st>>>(prm[l]);
      else
        dev::sb_inverse_kernel<16, false><<<grid, dev::NT, dev::i_smem_doubles<16>() * 8, st>>>(prm[l]);
    }
    ++nlaunch;
  }
  if (launches) *launches += nlaunch;
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace sb
}  // namespace serinv
