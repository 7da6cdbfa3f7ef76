// exec.cu -- persistent dataflow executor for serinv task graphs on B200 (sm_100a).
//
// One CTA of 256 threads per claim slot; the grid is sized to the number of
// co-resident CTAs (148 SMs x occupancy) so every claimed task can wait on
// earlier tasks without deadlock.  A CTA claims the next task index with one
// atomic, spins (thread 0, ld.acquire.gpu + nanosleep) until the task's input
// counters reach their targets, executes the tile task, then publishes its
// results (__syncthreads + __threadfence + atomicAdd on its signal counters).
// All tile operands are read through L2 (cp.async.cg / ld.global.cg), never
// L1, so data produced by other SMs inside the same launch is never stale.
//
// FP64 arithmetic: tcgen05 has no f64 kind, so the tensor-core path on
// sm_100a is the warp-level DMMA (mma.sync.aligned.m8n8k4.f64 -> SASS
// DMMA.8x8x4, measured 37.1 TFLOP/s chip-wide = the DFMA peak; see
// profiles/fp64_peaks_r01.json).  Tiles are 64 x 64; each of the 8 warps owns a
// 16 x 32 sub-tile (2 x 4 DMMA fragments); operands are staged in shared memory
// by a 3-stage cp.async pipeline over k-chunks of 32, in bank-conflict-free
// padded layouts (row stride = 4 mod 16 doubles).
#include <cuda_runtime.h>
#include <stdint.h>

#include "exec.h"
#include "task.h"

namespace serinv {
namespace dev {

constexpr int NT = 256;
constexpr int KC = 32;
constexpr int STAGES = 3;
constexpr int LD_MK = KC + 4;            // [row][k] layout stride (36 = 4 mod 16)
constexpr int LD_KM = SERINV_TILE + 4;   // [k][row] layout stride (68 = 4 mod 16)
constexpr int OPSZ = SERINV_TILE * LD_MK;  // doubles per operand stage (2304 >= 32*68)
constexpr int LDT = SERINV_TILE + 4;     // full-tile stride in smem (68)
constexpr int SMEM_DOUBLES = STAGES * 2 * OPSZ;  // 13824 doubles = 110592 bytes
static_assert(KC * LD_KM <= OPSZ, "km layout fits the stage");
static_assert(3 * SERINV_TILE * LDT + 6 * SERINV_TILE <= SMEM_DOUBLES, "post/potrf smem fits");

__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

__device__ __forceinline__ double *lptr(const Params &p, const Loc &l) { return p.bufs[l.buf] + l.off; }

__device__ __forceinline__ void phase_mark(const Params &p, int t, int k) {
  if (p.trace && threadIdx.x == 0) p.trace[4 * (size_t)p.ntasks + 8 * (size_t)t + k] = globaltimer();
}


// thread 0 spins until waits [w0, w1) of the task list are satisfied (20 s watchdog)
__device__ void wait_range(const Params &p, int w0, int w1) {
  for (int w = w0; w < w1; ++w) {
    const Wait W = p.waits[w];
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.ctr + W.ctr) : "memory");
    if (v >= W.target) continue;
    int ns = 32;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.ctr + W.ctr) : "memory");
      if (v >= W.target) break;
      __nanosleep(ns);
      ns = min(ns * 2, 256);
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 20000000000ULL) {
        atomicExch(p.info, -1);
        break;
      }
    }
  }
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
// Operand staging.  op(X) is R x K.  km == false: X stored R x K row-major
// (elem (r,k) at base[r*ld + k]) -> smem [r][k] stride LD_MK.  km == true: X
// stored K x R row-major (elem (r,k) at base[k*ld + r]) -> smem [k][r] stride LD_KM.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load_operand(double *s, const double *base, int ld, bool km, int R, int K, int k0,
                                             bool vec) {
  const int tid = threadIdx.x;
  if (vec && R == SERINV_TILE && k0 + KC <= K) {  // full chunk: no bounds predicates
    if (!km) {
#pragma unroll
      for (int it = 0; it < (SERINV_TILE * (KC / 2)) / NT; ++it) {
        const int idx = tid + it * NT, r = idx >> 4, kk = (idx & 15) * 2;
        cp_async16(s + r * LD_MK + kk, base + (int64_t)r * ld + k0 + kk, 16);
      }
    } else {
#pragma unroll
      for (int it = 0; it < (KC * (SERINV_TILE / 2)) / NT; ++it) {
        const int idx = tid + it * NT, kk = idx >> 5, r = (idx & 31) * 2;
        cp_async16(s + kk * LD_KM + r, base + (int64_t)(k0 + kk) * ld + r, 16);
      }
    }
    return;
  }
  if (!km) {
#pragma unroll
    for (int it = 0; it < (SERINV_TILE * (KC / 2)) / NT; ++it) {
      int idx = tid + it * NT;
      int r = idx >> 4, kk = (idx & 15) * 2;
      int kg = k0 + kk;
      int nv = (r < R) ? max(0, min(2, K - kg)) : 0;
      double *dst = s + r * LD_MK + kk;
      const double *src = base + (int64_t)r * ld + kg;
      if (vec) {
        cp_async16(dst, nv ? src : base, nv * 8);
      } else {
        dst[0] = nv > 0 ? __ldcg(src) : 0.0;
        dst[1] = nv > 1 ? __ldcg(src + 1) : 0.0;
      }
    }
  } else {
#pragma unroll
    for (int it = 0; it < (KC * (SERINV_TILE / 2)) / NT; ++it) {
      int idx = tid + it * NT;
      int kk = idx >> 5, r = (idx & 31) * 2;
      int kg = k0 + kk;
      int nv = (kg < K) ? max(0, min(2, R - r)) : 0;
      double *dst = s + kk * LD_KM + r;
      const double *src = base + (int64_t)kg * ld + r;
      if (vec) {
        cp_async16(dst, nv ? src : base, nv * 8);
      } else {
        dst[0] = nv > 0 ? __ldcg(src) : 0.0;
        dst[1] = nv > 1 ? __ldcg(src + 1) : 0.0;
      }
    }
  }
}

// acc += A(16x32 warp slab) * B over `ksteps` k-steps of 4; generic strides:
// A elem (row, k) at As[row*sAr + k*sAk]; B elem (k, col) at Bs[col*sBn + k*sBk].
__device__ __forceinline__ void mma_steps(const double *As, int sAr, int sAk, const double *Bs, int sBn, int sBk,
                                          double (&acc)[2][4][2], int ksteps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = (warp >> 1) * 16 + (lane >> 2);
  const int c0 = (warp & 1) * 32 + (lane >> 2);
  const int kq = lane & 3;
#pragma unroll 4
  for (int ks = 0; ks < ksteps; ++ks) {
    const int kk = ks * 4 + kq;
    double a0 = As[r0 * sAr + kk * sAk];
    double a1 = As[(r0 + 8) * sAr + kk * sAk];
    double b[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(c0 + ni * 8) * sBn + kk * sBk];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      dmma(acc[0][ni], a0, b[ni]);
      dmma(acc[1][ni], a1, b[ni]);
    }
  }
}

// mma_steps on the two staged operand layouts with compile-time strides
// (immediate LDS offsets); a full chunk (KC/4 k-steps) is fully unrolled.
template <bool AKM, bool BKM>
__device__ __forceinline__ void mma_chunk(const double *As, const double *Bs, double (&acc)[2][4][2], int ksteps) {
  constexpr int sAr = AKM ? 1 : LD_MK, sAk = AKM ? LD_KM : 1;
  constexpr int sBn = BKM ? 1 : LD_MK, sBk = BKM ? LD_KM : 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kq = lane & 3;
  const double *Ap = As + ((warp >> 1) * 16 + (lane >> 2)) * sAr + kq * sAk;
  const double *Bp = Bs + ((warp & 1) * 32 + (lane >> 2)) * sBn + kq * sBk;
  auto step = [&](int ks) {
    const double a0 = Ap[ks * 4 * sAk], a1 = Ap[8 * sAr + ks * 4 * sAk];
    double b[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bp[ni * 8 * sBn + ks * 4 * sBk];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      dmma(acc[0][ni], a0, b[ni]);
      dmma(acc[1][ni], a1, b[ni]);
    }
  };
  if (ksteps == KC / 4) {
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) step(ks);
  } else {
    for (int ks = 0; ks < ksteps; ++ks) step(ks);
  }
}

__device__ __forceinline__ void mma_chunk_lay(bool akm, bool bkm, const double *As, const double *Bs,
                                              double (&acc)[2][4][2], int ksteps) {
  if (akm) {
    if (bkm) mma_chunk<true, true>(As, Bs, acc, ksteps);
    else mma_chunk<true, false>(As, Bs, acc, ksteps);
  } else {
    if (bkm) mma_chunk<false, true>(As, Bs, acc, ksteps);
    else mma_chunk<false, false>(As, Bs, acc, ksteps);
  }
}

// Main loop over one or two segment lists sharing ONE cp.async pipeline:
//   acc  = sum_{s in [s0, s0+ns)}  op(A_s) op(B_s)   (output m  x n)
//   acc2 = sum_{s in [s0b, s0b+nsb)} op(A_s) op(B_s)  (output mb x n)   [if acc2 != nullptr]
// full 64 x 64 tile (row-major, ld, 16-byte aligned) -> smem [64][LDT] via cp.async
__device__ __forceinline__ void tile_async(double *s, const double *g, int ld) {
#pragma unroll
  for (int it = 0; it < (SERINV_TILE * SERINV_TILE / 2) / NT; ++it) {
    const int idx = threadIdx.x + it * NT, r = idx >> 5, c2 = (idx & 31) * 2;
    cp_async16(s + r * LDT + c2, g + (int64_t)r * ld + c2, 16);
  }
}

// pf0 / pf1 (optional, full aligned 64 x 64 tiles): staged with cp.async into the
// pipeline stages freed after the last k-chunk is issued -- pf0 lands in stage
// nchunks % STAGES, pf1 in (nchunks + 1) % STAGES (complete when this returns).
template <bool DUAL>
__device__ __forceinline__ void gemm_mainloop2(const Params &p, int s0, int ns, int m, int s0b, int nsb, int mb,
                                               int n, double *smem, double (&acc)[2][4][2],
                                               double (&acc2)[2][4][2], const double *pf0 = nullptr, int ld0 = 0,
                                               const double *pf1 = nullptr, int ld1 = 0) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (DUAL) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc2[i][j][0] = acc2[i][j][1] = 0.0;
  } else {
    nsb = 0;
  }
  if (ns + nsb == 0) return;
  const Seg *segsA = p.segs + s0;
  const Seg *segsB = p.segs + s0b;
  int nchA = 0, nchB = 0;
  for (int s = 0; s < ns; ++s) nchA += (segsA[s].k + KC - 1) / KC;
  for (int s = 0; s < nsb; ++s) nchB += (segsB[s].k + KC - 1) / KC;
  const int nchunks = nchA + nchB;
  // Segment descriptors are copied into registers at segment switches only:
  // the cp.async asm carries a memory clobber, so reading them through a
  // reference would re-load them from global memory on every chunk.
  struct Cur {
    const double *a, *b;
    int lda, ldb, k, R;
    bool akm, bkm, va, vb;
  };
  auto fetch = [&](int idx, bool inB) {
    const Seg S = inB ? segsB[idx] : segsA[idx];
    Cur c;
    c.a = lptr(p, S.A);
    c.b = lptr(p, S.B);
    c.lda = S.A.ld;
    c.ldb = S.B.ld;
    c.k = S.k;
    c.R = inB ? mb : m;
    c.akm = S.ta != 0;
    c.bkm = S.tb == 0;
    c.va = ((S.A.off | S.A.ld) & 1) == 0;
    c.vb = ((S.B.off | S.B.ld) & 1) == 0;
    return c;
  };
  // load-side cursor (list A, then list B)
  int ls = 0, lk = 0, lj = 0;
  Cur L = fetch(0, nchA == 0);
  auto issue = [&](int stage) {
    ++lj;
    double *As = smem + stage * 2 * OPSZ;
    load_operand(As, L.a, L.lda, L.akm, L.R, L.k, lk, L.va);
    load_operand(As + OPSZ, L.b, L.ldb, L.bkm, n, L.k, lk, L.vb);
    lk += KC;
    if (lk >= L.k && lj < nchunks) {
      lk = 0;
      ++ls;
      if (lj == nchA) ls = 0;  // switch to list B
      L = fetch(ls, lj >= nchA);
    }
  };
  // compute-side cursor
  int cs = 0, ck = 0;
  Cur C = L;
  // issue slot `slot` (>= nchunks): the prefetch tiles
  auto issue_extra = [&](int slot) {
    double *st = smem + (slot % STAGES) * 2 * OPSZ;
    if (slot == nchunks && pf0) tile_async(st, pf0, ld0);
    if (slot == nchunks + 1 && pf1) tile_async(st, pf1, ld1);
  };
#pragma unroll
  for (int j = 0; j < STAGES - 1; ++j) {
    if (j < nchunks) issue(j);
    else issue_extra(j);
    cp_commit();
  }
  for (int j = 0; j < nchunks; ++j) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    if (j + STAGES - 1 < nchunks) issue((j + STAGES - 1) % STAGES);
    else issue_extra(j + STAGES - 1);
    cp_commit();
    const bool inB = j >= nchA;
    const double *As = smem + (j % STAGES) * 2 * OPSZ;
    const double *Bs = As + OPSZ;
    int kleft = C.k - ck;
    int ksteps = kleft >= KC ? KC / 4 : (kleft + 3) / 4;
    if (DUAL && inB)
      mma_chunk_lay(C.akm, C.bkm, As, Bs, acc2, ksteps);
    else
      mma_chunk_lay(C.akm, C.bkm, As, Bs, acc, ksteps);
    ck += KC;
    if (ck >= C.k && j + 1 < nchunks) {
      ck = 0;
      ++cs;
      if (j + 1 == nchA) cs = 0;
      C = fetch(cs, j + 1 >= nchA);
    }
  }
  cp_wait<0>();
  __syncthreads();
}

// Single-stage main loop (stage buffers at `stage`, 2 * OPSZ doubles): used
// where the rest of shared memory holds live data (the late tile of a chain task).
__device__ void gemm_onestage(const Params &p, int s0, int ns, int m, int n, double *stage, double (&acc)[2][4][2]) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const Seg *segs = p.segs + s0;
  double *As = stage, *Bs = stage + OPSZ;
  for (int s = 0; s < ns; ++s) {
    const Seg &S = segs[s];
    const bool vecA = ((S.A.off | S.A.ld) & 1) == 0, vecB = ((S.B.off | S.B.ld) & 1) == 0;
    const bool akm = S.ta != 0, bkm = S.tb == 0;
    for (int k0 = 0; k0 < S.k; k0 += KC) {
      load_operand(As, lptr(p, S.A), S.A.ld, akm, m, S.k, k0, vecA);
      load_operand(Bs, lptr(p, S.B), S.B.ld, bkm, n, S.k, k0, vecB);
      cp_commit();
      cp_wait<0>();
      __syncthreads();
      const int kleft = S.k - k0;
      const int ksteps = kleft >= KC ? KC / 4 : (kleft + 3) / 4;
      mma_steps(As, akm ? 1 : LD_MK, akm ? LD_KM : 1, Bs, bkm ? 1 : LD_MK, bkm ? LD_KM : 1, acc, ksteps);
      __syncthreads();
    }
  }
}

__device__ __forceinline__ void gemm_mainloop(const Params &p, int s0, int ns, int m, int n, double *smem,
                                              double (&acc)[2][4][2]) {
  gemm_mainloop2<false>(p, s0, ns, m, 0, 0, 0, n, smem, acc, acc);
}

// Fragment element coordinates of acc[mi][ni][h].
__device__ __forceinline__ void frag_rc(int mi, int ni, int h, int &r, int &c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  r = (warp >> 1) * 16 + mi * 8 + (lane >> 2);
  c = (warp & 1) * 32 + ni * 8 + 2 * (lane & 3) + h;
}

// acc = alpha * acc + beta * C0   (C0: m x n at loc)
__device__ __forceinline__ void apply_c0(const Params &p, double alpha, double beta, const Loc &loc, int m, int n,
                                         double (&acc)[2][4][2]) {
  const double *c0 = (beta != 0.0) ? lptr(p, loc) : nullptr;
  if (c0 && m == SERINV_TILE && n == SERINV_TILE && ((loc.off | loc.ld) & 1) == 0) {
    // full tile: 16-byte loads, four in flight per fragment row
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      double2 cv[4];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        int r, cc;
        frag_rc(mi, ni, 0, r, cc);
        cv[ni] = __ldcg(reinterpret_cast<const double2 *>(c0 + (int64_t)r * loc.ld + cc));
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        acc[mi][ni][0] = fma(alpha, acc[mi][ni][0], beta * cv[ni].x);
        acc[mi][ni][1] = fma(alpha, acc[mi][ni][1], beta * cv[ni].y);
      }
    }
    return;
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int r, cc;
        frag_rc(mi, ni, h, r, cc);
        double v = alpha * acc[mi][ni][h];
        if (c0 && r < m && cc < n) v += beta * __ldcg(c0 + (int64_t)r * loc.ld + cc);
        acc[mi][ni][h] = v;
      }
}

__device__ __forceinline__ void acc_to_smem(double *St, const double (&acc)[2][4][2]) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int r, c;
        frag_rc(mi, ni, h, r, c);
        St[r * LDT + c] = acc[mi][ni][h];
      }
}

// load an m x n tile (row-major, ld) into smem [64][LDT], zero padded
__device__ __forceinline__ void tile_to_smem(double *St, const double *g, int ld, int m, int n) {
  if (m == SERINV_TILE && n == SERINV_TILE && (((uintptr_t)g | (uintptr_t)ld) & 1) == 0 &&
      ((uintptr_t)g & 15) == 0) {
    // full aligned tile: all 16-byte loads in flight together (cp.async), one wait
#pragma unroll
    for (int it = 0; it < (SERINV_TILE * SERINV_TILE / 2) / NT; ++it) {
      const int idx = threadIdx.x + it * NT, r = idx >> 5, c2 = (idx & 31) * 2;
      unsigned s = (unsigned)__cvta_generic_to_shared(St + r * LDT + c2);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g + (int64_t)r * ld + c2) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    return;
  }
  for (int idx = threadIdx.x; idx < SERINV_TILE * SERINV_TILE; idx += NT) {
    int r = idx >> 6, c = idx & 63;
    St[r * LDT + c] = (r < m && c < n) ? __ldcg(g + (int64_t)r * ld + c) : 0.0;
  }
}

// acc(16 x 32 warp slab of a 64 x 64 result) += A B over K = 64 from two [64][LDT]
// smem tiles, compile-time strides, fully unrolled: A(r,k) = As[r][k];
// B(k,c) = Bs[c][k] (BT) or Bs[k][c]
template <bool BT>
__device__ __forceinline__ void mma_smem64(const double *As, const double *Bs, double (&acc)[2][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kq = lane & 3;
  const double *Ap = As + ((warp >> 1) * 16 + (lane >> 2)) * LDT + kq;
  const double *Bp = BT ? Bs + ((warp & 1) * 32 + (lane >> 2)) * LDT + kq : Bs + kq * LDT + (warp & 1) * 32 + (lane >> 2);
#pragma unroll
  for (int ks = 0; ks < SERINV_TILE / 4; ++ks) {
    const double a0 = Ap[ks * 4], a1 = Ap[8 * LDT + ks * 4];
    double b[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = BT ? Bp[ni * 8 * LDT + ks * 4] : Bp[ks * 4 * LDT + ni * 8];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      dmma(acc[0][ni], a0, b[ni]);
      dmma(acc[1][ni], a1, b[ni]);
    }
  }
}

// smem [64][LDT] tile -> global (m x n at g, row stride ld); 16-byte stores when full and aligned
__device__ __forceinline__ void smem_to_global(double *g, int64_t ld, const double *S, int m, int n) {
  if (m == SERINV_TILE && n == SERINV_TILE && (((uintptr_t)g & 15) | (ld & 1)) == 0) {
#pragma unroll 4
    for (int idx = threadIdx.x; idx < SERINV_TILE * SERINV_TILE / 2; idx += NT) {
      const int i = idx >> 5, k2 = (idx & 31) * 2;
      *reinterpret_cast<double2 *>(g + (int64_t)i * ld + k2) = make_double2(S[i * LDT + k2], S[i * LDT + k2 + 1]);
    }
    return;
  }
  for (int idx = threadIdx.x; idx < SERINV_TILE * SERINV_TILE; idx += NT) {
    const int i = idx >> 6, k = idx & 63;
    if (i < m && k < n) g[(int64_t)i * ld + k] = S[i * LDT + k];
  }
}

__device__ void store_tile(const Params &p, const Loc &loc, int m, int n, const double (&acc)[2][4][2]) {
  double *o = lptr(p, loc);
  const bool vec = ((loc.off | loc.ld) & 1) == 0;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      int r, c;
      frag_rc(mi, ni, 0, r, c);
      if (r >= m) continue;
      double *dst = o + (int64_t)r * loc.ld + c;
      if (vec && c + 1 < n) {
        *reinterpret_cast<double2 *>(dst) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      } else {
        if (c < n) dst[0] = acc[mi][ni][0];
        if (c + 1 < n) dst[1] = acc[mi][ni][1];
      }
    }
}

__device__ void store_acc(const Params &p, const Task &T, const double (&acc)[2][4][2]) {
  double *o = lptr(p, T.out);
  const bool vec = ((T.out.off | T.out.ld) & 1) == 0;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      int r, c;
      frag_rc(mi, ni, 0, r, c);
      if (r >= T.m) continue;
      double *dst = o + (int64_t)r * T.out.ld + c;
      if (vec && c + 1 < T.n) {
        *reinterpret_cast<double2 *>(dst) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      } else {
        if (c < T.n) dst[0] = acc[mi][ni][0];
        if (c + 1 < T.n) dst[1] = acc[mi][ni][1];
      }
    }
  if (T.flags & (TF_MIRROR | TF_ZERO_MIRROR)) {
    double *o2 = lptr(p, T.out2);
    const bool zero = (T.flags & TF_ZERO_MIRROR) != 0;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int r, c;
          frag_rc(mi, ni, h, r, c);
          if (r < T.m && c < T.n) o2[(int64_t)c * T.out2.ld + r] = zero ? 0.0 : acc[mi][ni][h];
        }
  }
}

// ---------------------------------------------------------------------------
// Wide GEMM tasks: m <= 128 output rows (two row tiles) x n <= 64 columns.
// Same task semantics as run_gemm (segments, alpha/beta C0, TF_POST, TF_MIRROR)
// for the bulk updates whose row tiles share their operand lists (the
// Takahashi tile products, the L W precompute): the A panel feeds 128 rows per
// B panel, so each staged byte carries 1.33x the DMMA work of a 64 x 64 tile
// (L2 -> SMEM traffic per flop -25 %), and the per-task overhead is amortised
// over twice the flops.  8 warps of 32 x 32 (4 x 4 DMMA fragments), a 2-stage
// cp.async pipeline over k-chunks of 32 in the same 110.6 KB of shared memory.
// ---------------------------------------------------------------------------
constexpr int WROWS = 2 * SERINV_TILE;          // 128
constexpr int LDW_KM = WROWS + 4;               // [k][row] stride for 128 rows (132 = 4 mod 16)
constexpr int WA_SZ = WROWS * LD_MK;            // 4608 doubles >= 32 * 132
constexpr int WSTAGE = WA_SZ + OPSZ;            // A (128 rows) + B (64 rows)
static_assert(2 * WSTAGE <= SMEM_DOUBLES, "wide stages fit");
static_assert(KC * LDW_KM <= WA_SZ, "wide km layout fits");
static_assert((WROWS + SERINV_TILE) * LDT <= SMEM_DOUBLES, "wide post-multiply fits");

// op(X) is R x K (R <= ROWS); layouts as in load_operand, km stride ROWS + 4
template <int ROWS>
__device__ __forceinline__ void load_operand_w(double *s, const double *base, int ld, bool km, int R, int K, int k0,
                                               bool vec) {
  constexpr int LDK = ROWS + 4;
  const int tid = threadIdx.x;
  if (!km) {
#pragma unroll
    for (int it = 0; it < (ROWS * (KC / 2)) / NT; ++it) {
      const int idx = tid + it * NT, r = idx >> 4, kk = (idx & 15) * 2;
      const int kg = k0 + kk;
      const int nv = (r < R) ? max(0, min(2, K - kg)) : 0;
      double *dst = s + r * LD_MK + kk;
      const double *src = base + (int64_t)r * ld + kg;
      if (vec) {
        cp_async16(dst, nv ? src : base, nv * 8);
      } else {
        dst[0] = nv > 0 ? __ldcg(src) : 0.0;
        dst[1] = nv > 1 ? __ldcg(src + 1) : 0.0;
      }
    }
  } else {
#pragma unroll
    for (int it = 0; it < (KC * (ROWS / 2)) / NT; ++it) {
      const int idx = tid + it * NT, kk = idx / (ROWS / 2), r = (idx % (ROWS / 2)) * 2;
      const int kg = k0 + kk;
      const int nv = (kg < K) ? max(0, min(2, R - r)) : 0;
      double *dst = s + kk * LDK + r;
      const double *src = base + (int64_t)kg * ld + r;
      if (vec) {
        cp_async16(dst, nv ? src : base, nv * 8);
      } else {
        dst[0] = nv > 0 ? __ldcg(src) : 0.0;
        dst[1] = nv > 1 ? __ldcg(src + 1) : 0.0;
      }
    }
  }
}

// acc(32 x 32 warp tile of a 128 x 64 output) += A * B over `ksteps` k-steps of 4;
// A elem (row, k) at As[row*sAr + k*sAk]; B elem (k, col) at Bs[col*sBn + k*sBk].
template <int sAr, int sAk, int sBn, int sBk>
__device__ __forceinline__ void wide_steps(const double *As, const double *Bs, double (&acc)[4][4][2], int ksteps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kq = lane & 3;
  const double *Ap = As + ((warp >> 1) * 32 + (lane >> 2)) * sAr + kq * sAk;
  const double *Bp = Bs + ((warp & 1) * 32 + (lane >> 2)) * sBn + kq * sBk;
  auto step = [&](int ks) {
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = Ap[mi * 8 * sAr + ks * 4 * sAk];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bp[ni * 8 * sBn + ks * 4 * sBk];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
  };
  if (ksteps == KC / 4) {
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) step(ks);
  } else {
    for (int ks = 0; ks < ksteps; ++ks) step(ks);
  }
}

__device__ __forceinline__ void wide_chunk(bool akm, bool bkm, const double *As, const double *Bs,
                                           double (&acc)[4][4][2], int ksteps) {
  if (akm) {
    if (bkm) wide_steps<1, LDW_KM, 1, LD_KM>(As, Bs, acc, ksteps);
    else wide_steps<1, LDW_KM, LD_MK, 1>(As, Bs, acc, ksteps);
  } else {
    if (bkm) wide_steps<LD_MK, 1, 1, LD_KM>(As, Bs, acc, ksteps);
    else wide_steps<LD_MK, 1, LD_MK, 1>(As, Bs, acc, ksteps);
  }
}

__device__ __forceinline__ void wide_rc(int mi, int ni, int h, int &r, int &c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  r = (warp >> 1) * 32 + mi * 8 + (lane >> 2);
  c = (warp & 1) * 32 + ni * 8 + 2 * (lane & 3) + h;
}

__device__ void run_gemm_wide(const Params &p, const Task &T, double *smem) {
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int m = T.m, n = T.n;
  const Seg *segs = p.segs + T.seg0;
  int nch = 0;
  for (int s = 0; s < T.nseg; ++s) nch += (segs[s].k + KC - 1) / KC;
  struct Cur {
    const double *a, *b;
    int lda, ldb, k;
    bool akm, bkm, va, vb;
  };
  auto fetch = [&](int idx) {
    const Seg S = segs[idx];
    Cur c;
    c.a = lptr(p, S.A);
    c.b = lptr(p, S.B);
    c.lda = S.A.ld;
    c.ldb = S.B.ld;
    c.k = S.k;
    c.akm = S.ta != 0;
    c.bkm = S.tb == 0;
    c.va = ((S.A.off | S.A.ld) & 1) == 0;
    c.vb = ((S.B.off | S.B.ld) & 1) == 0;
    return c;
  };
  if (nch > 0) {
    int ls = 0, lk = 0, lj = 0;
    Cur L = fetch(0);
    auto issue = [&](int stage) {
      ++lj;
      double *As = smem + stage * WSTAGE;
      load_operand_w<WROWS>(As, L.a, L.lda, L.akm, m, L.k, lk, L.va);
      load_operand_w<SERINV_TILE>(As + WA_SZ, L.b, L.ldb, L.bkm, n, L.k, lk, L.vb);
      lk += KC;
      if (lk >= L.k && lj < nch) {
        lk = 0;
        L = fetch(++ls);
      }
    };
    int cs = 0, ck = 0;
    Cur C = L;
    issue(0);
    cp_commit();
    for (int j = 0; j < nch; ++j) {
      cp_wait<0>();
      __syncthreads();
      if (j + 1 < nch) issue((j + 1) & 1);
      cp_commit();
      const double *As = smem + (j & 1) * WSTAGE;
      const int kleft = C.k - ck;
      const int ksteps = kleft >= KC ? KC / 4 : (kleft + 3) / 4;
      wide_chunk(C.akm, C.bkm, As, As + WA_SZ, acc, ksteps);
      ck += KC;
      if (ck >= C.k && j + 1 < nch) {
        ck = 0;
        C = fetch(++cs);
      }
    }
    cp_wait<0>();
    __syncthreads();
  }
  // acc = alpha * acc + beta * C0
  if (T.beta != 0.0 && m == WROWS && n == SERINV_TILE && ((T.c0.off | T.c0.ld) & 1) == 0) {
    const double *c0 = lptr(p, T.c0);  // full tile: 16-byte loads, four in flight per row group
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      double2 cv[4];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        int r, cc;
        wide_rc(mi, ni, 0, r, cc);
        cv[ni] = __ldcg(reinterpret_cast<const double2 *>(c0 + (int64_t)r * T.c0.ld + cc));
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        acc[mi][ni][0] = fma(T.alpha, acc[mi][ni][0], T.beta * cv[ni].x);
        acc[mi][ni][1] = fma(T.alpha, acc[mi][ni][1], T.beta * cv[ni].y);
      }
    }
  } else {
    const double *c0 = (T.beta != 0.0) ? lptr(p, T.c0) : nullptr;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int r, cc;
          wide_rc(mi, ni, h, r, cc);
          double v = T.alpha * acc[mi][ni][h];
          if (c0 && r < m && cc < n) v += T.beta * __ldcg(c0 + (int64_t)r * T.c0.ld + cc);
          acc[mi][ni][h] = v;
        }
  }
  if (T.flags & TF_POST) {  // out = S op(R), S = the 128 x n result, R n x n
    double *St = smem;
    double *Rt = smem + WROWS * LDT;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int r, cc;
          wide_rc(mi, ni, h, r, cc);
          St[r * LDT + cc] = acc[mi][ni][h];
          acc[mi][ni][h] = 0.0;
        }
    tile_to_smem(Rt, lptr(p, T.r), T.r.ld, n, n);
    __syncthreads();
    if (T.flags & TF_POST_T)
      wide_steps<LDT, 1, LDT, 1>(St, Rt, acc, (n + 3) / 4);
    else
      wide_steps<LDT, 1, 1, LDT>(St, Rt, acc, (n + 3) / 4);
    __syncthreads();
  }
  double *o = lptr(p, T.out);
  const bool vec = ((T.out.off | T.out.ld) & 1) == 0;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      int r, cc;
      wide_rc(mi, ni, 0, r, cc);
      if (r >= m) continue;
      double *dst = o + (int64_t)r * T.out.ld + cc;
      if (vec && cc + 1 < n) {
        *reinterpret_cast<double2 *>(dst) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      } else {
        if (cc < n) dst[0] = acc[mi][ni][0];
        if (cc + 1 < n) dst[1] = acc[mi][ni][1];
      }
    }
  if (T.flags & TF_MIRROR) {
    double *o2 = lptr(p, T.out2);
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int r, cc;
          wide_rc(mi, ni, h, r, cc);
          if (r < m && cc < n) o2[(int64_t)cc * T.out2.ld + r] = acc[mi][ni][h];
        }
  }
}

// ---------------------------------------------------------------------------
// Tile tasks
// ---------------------------------------------------------------------------
__device__ void run_gemm(const Params &p, const Task &T, double *smem, int tsk) {
  double acc[2][4][2];
  // C0 and the post-multiply tile ride in the pipeline's freed stages when the
  // task has k-chunks and the tiles are full and 16-byte aligned (the post tile
  // only if it is not a late input)
  int nch = 0;
  for (int s = 0; s < T.nseg; ++s) nch += (p.segs[T.seg0 + s].k + KC - 1) / KC;
  const bool full = T.m == SERINV_TILE && T.n == SERINV_TILE && nch > 0;
  const bool pfc = full && T.beta != 0.0 && ((T.c0.off | T.c0.ld) & 1) == 0;
  const bool pfr = full && (T.flags & TF_POST) && T.nlate == 0 && ((T.r.off | T.r.ld) & 1) == 0;
  const double *pc = pfc ? lptr(p, T.c0) : nullptr;
  const double *pr = pfr ? lptr(p, T.r) : nullptr;
  // stage assignment: pf0 -> nch % 3, pf1 -> (nch + 1) % 3; with only R, R takes pf0's slot
  gemm_mainloop2<false>(p, T.seg0, T.nseg, T.m, 0, 0, 0, T.n, smem, acc, acc, pfc ? pc : pr,
                        pfc ? T.c0.ld : T.r.ld, pfc ? pr : nullptr, T.r.ld);
  phase_mark(p, tsk, 5);
  double *Cs = smem + (nch % STAGES) * 2 * OPSZ;
  double *Rs = pfc ? smem + ((nch + 1) % STAGES) * 2 * OPSZ : Cs;
  if (pfc) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int r, cc;
          frag_rc(mi, ni, h, r, cc);
          acc[mi][ni][h] = fma(T.alpha, acc[mi][ni][h], T.beta * Cs[r * LDT + cc]);
        }
  } else {
    apply_c0(p, T.alpha, T.beta, T.c0, T.m, T.n, acc);
  }
  if (T.nlate > 0) {  // late inputs (the post-multiply tile, the SYRK target's updates)
    if (threadIdx.x == 0) wait_range(p, T.wait0 + T.nwait - T.nlate, T.wait0 + T.nwait);
    __syncthreads();
  }
  if (T.flags & TF_POST) {
    // S (this result) goes to the stage after the prefetched ones; R from its stage
    // carried chain: W is the previous task's (the POTRF's) Wt; smem[0..) stays free
    // for the SYRK target that the next POTRF consumes
    const bool carry = (T.flags & TF_CARRY) != 0;
    double *St = carry ? smem + 2 * SERINV_TILE * LDT : (pfr ? smem + ((nch + 2) % STAGES) * 2 * OPSZ : smem);
    double *Rt = carry ? smem + SERINV_TILE * LDT : (pfr ? Rs : smem + SERINV_TILE * LDT);
    if (!pfr && pfc && !carry) __syncthreads();  // C0 (read above) may overlap St / Rt
    acc_to_smem(St, acc);
    if (!pfr && !carry) tile_to_smem(Rt, lptr(p, T.r), T.r.ld, T.n, T.n);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const bool rt = (T.flags & TF_POST_T) != 0;
    // out = S * op(R): B(k, j) = R[j][k] (POST_T) or R[k][j]
    if (T.n == SERINV_TILE) {
      if (rt) mma_smem64<true>(St, Rt, acc);
      else mma_smem64<false>(St, Rt, acc);
    } else {
      mma_steps(St, LDT, 1, Rt, rt ? LDT : 1, rt ? 1 : LDT, acc, (T.n + 3) / 4);
    }
    __syncthreads();
  }
  phase_mark(p, tsk, 6);
  store_acc(p, T, acc);
  phase_mark(p, tsk, 7);
  if (T.flags & TF_SYRK3) {
    // the next diagonal tile of the chain: out3 -= L L^T (L = this result, m x n);
    // stage the target tile into smem with cp.async while the SYRK runs
    const bool carry = (T.flags & TF_CARRY) != 0;
    double *Lt = carry ? smem + 2 * SERINV_TILE * LDT : smem;
    double *Ct = carry ? smem : smem + SERINV_TILE * LDT;
    {
      const double *g = lptr(p, T.out3);
      const bool vec = ((T.out3.off | T.out3.ld) & 1) == 0;
      for (int idx = threadIdx.x; idx < SERINV_TILE * (SERINV_TILE / 2); idx += NT) {
        const int r = idx >> 5, c = (idx & 31) * 2;
        const int nv = (r < T.m) ? max(0, min(2, T.m - c)) : 0;
        const double *src = g + (int64_t)r * T.out3.ld + c;
        if (vec) {
          cp_async16(Ct + r * LDT + c, nv ? src : g, nv * 8);
        } else {
          Ct[r * LDT + c] = nv > 0 ? __ldcg(src) : 0.0;
          Ct[r * LDT + c + 1] = nv > 1 ? __ldcg(src + 1) : 0.0;
        }
      }
      cp_commit();
    }
    acc_to_smem(Lt, acc);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (T.n == SERINV_TILE) {
      // only the lower triangle of L L^T is used downstream: the warp whose slab is
      // strictly upper (rows 0-15, columns 32-63) skips its products
      if (!((threadIdx.x >> 5) == 1)) mma_smem64<true>(Lt, Lt, acc);
    } else {
      mma_steps(Lt, LDT, 1, Lt, LDT, 1, acc, (T.n + 3) / 4);
    }
    cp_wait<0>();
    __syncthreads();
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int r, c;
          frag_rc(mi, ni, h, r, c);
          acc[mi][ni][h] = Ct[r * LDT + c] - acc[mi][ni][h];
        }
    store_tile(p, T.out3, T.m, T.m, acc);
    if (carry) {  // the updated diagonal tile stays in smem[0..) for the next POTRF (same CTA)
      __syncthreads();
      acc_to_smem(Ct, acc);
    }
    __syncthreads();
  }
}


// select row[kk] for runtime kk without dynamic register indexing
__device__ __forceinline__ double sel4(const double (&row)[4], int kk) {
  double x = row[0];
  x = (kk == 1) ? row[1] : x;
  x = (kk == 2) ? row[2] : x;
  x = (kk == 3) ? row[3] : x;
  return x;
}
__device__ __forceinline__ void set4(double (&row)[4], int kk, double x) {
  row[0] = (kk == 0) ? x : row[0];
  row[1] = (kk == 1) ? x : row[1];
  row[2] = (kk == 2) ? x : row[2];
  row[3] = (kk == 3) ? x : row[3];
}

// 16x16 (x K) warp product on smem operands: acc(16 x 16, 2 x 2 m8n8 fragments) +=
// A[r][k] * B[k][c],  A at As (row stride lda), B at Bs (row stride ldb).
__device__ __forceinline__ void warp_mma16(const double *As, int lda, const double *Bs, int ldb, int K,
                                           double (&acc)[2][2][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  for (int k0 = 0; k0 < K; k0 += 4) {
    double a0 = As[g * lda + k0 + q], a1 = As[(g + 8) * lda + k0 + q];
    double b0 = Bs[(k0 + q) * ldb + g], b1 = Bs[(k0 + q) * ldb + g + 8];
    dmma(acc[0][0], a0, b0);
    dmma(acc[0][1], a0, b1);
    dmma(acc[1][0], a1, b0);
    dmma(acc[1][1], a1, b1);
  }
}

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
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int i = 8 * h + t;
    const bool valid = (c0 + i < m) && (c0 + j < m) && i >= j;
    St[(c0 + i) * LDT + c0 + j] = valid ? a[t] : 0.0;
    Wt[(c0 + i) * LDT + c0 + j] = valid ? z[t] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// 8 x 8 block helpers (one warp).  A block is addressed by its top-left element
// in a [64][LDT] smem tile.  Accumulator layout (DMMA m8n8): lane (g = lane >> 2,
// q = lane & 3) holds row g, columns 2q, 2q + 1.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void blk_load(const double *B, double (&v)[2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  v[0] = B[g * LDT + 2 * q];
  v[1] = B[g * LDT + 2 * q + 1];
}
__device__ __forceinline__ void blk_store(double *B, const double (&v)[2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  B[g * LDT + 2 * q] = v[0];
  B[g * LDT + 2 * q + 1] = v[1];
}
// acc += X Y^T
__device__ __forceinline__ void blk_mma_nt(double (&acc)[2], const double *X, const double *Y) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  dmma(acc, X[g * LDT + q], Y[g * LDT + q]);
  dmma(acc, X[g * LDT + 4 + q], Y[g * LDT + 4 + q]);
}
// acc += X Y
__device__ __forceinline__ void blk_mma_nn(double (&acc)[2], const double *X, const double *Y) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  dmma(acc, X[g * LDT + q], Y[q * LDT + g]);
  dmma(acc, X[g * LDT + 4 + q], Y[(4 + q) * LDT + g]);
}

// acc -= X Y^T with acc holding C on entry: the DMMA accumulates onto C directly
// (negated A operand), so no FP64 ALU op waits on the tensor-pipe result
__device__ __forceinline__ void blk_mma_nt_sub(double (&acc)[2], const double *X, const double *Y) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  dmma(acc, -X[g * LDT + q], Y[g * LDT + q]);
  dmma(acc, -X[g * LDT + 4 + q], Y[g * LDT + 4 + q]);
}

// Cholesky + inverse of one 8 x 8 block (one converged warp, registers +
// shuffles), the block given in accumulator layout (a0, a1 = A[g][2q], A[g][2q+1]):
// Ab <- L (strict upper zeroed), Zb <- Z = L^{-1}, dv8[j] <- pivot j.
// Right-looking elimination with the row operations mirrored on Z = I (see
// leaf_chol16 for the algebra: M A = L^T, Z = D^{-1/2} M = L^{-1}).  The column
// scaling by 1/sqrt(d_p) (L) and the row scaling of Z are postponed to the end
// (the updates only read the unscaled current column), and the next pivot
// d' = A[p+1][p+1] - A[p+1][p]^2 / d is formed from two values shuffled before
// pivot p's update, so the serial chain per pivot is one FMA and one reciprocal.
__device__ __forceinline__ void leaf_chol8r(double a0, double a1, double *Ab, double *Zb, double *dv8) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  double z0 = (g == 2 * q) ? 1.0 : 0.0, z1 = (g == 2 * q + 1) ? 1.0 : 0.0;
  double dmine = 1.0;
  double d = __shfl_sync(FULL, a0, 0);
  double id = rcp_nr(d);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int sq = p >> 1;
    const double ap = (p & 1) ? a1 : a0;
    double x = 0.0, y = 1.0;
    if (p < 7) {  // compile-time
      const int p1 = p + 1;
      x = __shfl_sync(FULL, ap, 4 * p1 + sq);                               // A[p+1][p]
      y = __shfl_sync(FULL, (p1 & 1) ? a1 : a0, 4 * p1 + (p1 >> 1));        // A[p+1][p+1]
    }
    const double ai = __shfl_sync(FULL, ap, 4 * g + sq);        // A[g][p]
    const double aj0 = __shfl_sync(FULL, ap, 8 * q + sq);       // A[2q][p]
    const double aj1 = __shfl_sync(FULL, ap, 8 * q + 4 + sq);   // A[2q+1][p]
    const double zp0 = __shfl_sync(FULL, z0, 4 * p + q);        // Z[p][2q]
    const double zp1 = __shfl_sync(FULL, z1, 4 * p + q);        // Z[p][2q+1]
    const double dn = fma(-(x * x), id, y);
    const double idn = rcp_nr(dn);
    const double f = ai * id;
    const bool below = g > p;
    a0 = (below && 2 * q > p) ? fma(-f, aj0, a0) : a0;
    a1 = (below && 2 * q + 1 > p) ? fma(-f, aj1, a1) : a1;
    z0 = below ? fma(-f, zp0, z0) : z0;
    z1 = below ? fma(-f, zp1, z1) : z1;
    dmine = (lane == p) ? d : dmine;
    d = dn;
    id = idn;
  }
  // postponed scaling: L[g][j] = A[g][j] / sqrt(d_j) (g > j), sqrt(d_j) on the
  // diagonal, 0 above; Z[g][:] /= sqrt(d_g)
  const double dj0 = __shfl_sync(FULL, dmine, 2 * q), dj1 = __shfl_sync(FULL, dmine, 2 * q + 1);
  const double dg = __shfl_sync(FULL, dmine, g);
  const double r0 = rsqrt_nr(dj0), r1 = rsqrt_nr(dj1), rg = rsqrt_nr(dg);
  a0 = (g > 2 * q) ? a0 * r0 : ((g == 2 * q) ? dj0 * r0 : 0.0);
  a1 = (g > 2 * q + 1) ? a1 * r1 : ((g == 2 * q + 1) ? dj1 * r1 : 0.0);
  Ab[g * LDT + 2 * q] = a0;
  Ab[g * LDT + 2 * q + 1] = a1;
  Zb[g * LDT + 2 * q] = z0 * rg;
  Zb[g * LDT + 2 * q + 1] = z1 * rg;
  if (lane < 8) dv8[lane] = dmine;
}
__device__ __forceinline__ void leaf_chol8(double *Ab, double *Zb, double *dv8) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  leaf_chol8r(Ab[g * LDT + 2 * q], Ab[g * LDT + 2 * q + 1], Ab, Zb, dv8);
}

// the 36 blocks (i, j), j <= i < 8, of an 8 x 8-block lower triangle, column-major: (i << 4) | j
__constant__ unsigned char c_lower8[36] = {
    0x00, 0x10, 0x20, 0x30, 0x40, 0x50, 0x60, 0x70, 0x11, 0x21, 0x31, 0x41, 0x51, 0x61, 0x71, 0x22, 0x32, 0x42,
    0x52, 0x62, 0x72, 0x33, 0x43, 0x53, 0x63, 0x73, 0x44, 0x54, 0x64, 0x74, 0x55, 0x65, 0x75, 0x66, 0x76, 0x77};

// Cholesky L and inverse W = L^{-1} of the 64 x 64 tile St (rows / columns >= m
// padded with the identity) on 8 x 8 blocks, software-pipelined across warps so
// the serial chain is just the 8 leaves.  Step k (k = 0..7), after a CTA barrier:
//   warp 0 (critical): L(k,k-1) = A(k,k-1) Z_{k-1}^T (published to the workers
//     through a named barrier), A(k,k) -= L(k,k-1) L(k,k-1)^T, leaf_chol8(k);
//   warps 1-7: the panel L(i,k-1) = A(i,k-1) Z_{k-1}^T (i > k), then the
//     trailing update A(i,j) -= L(i,k-1) L(j,k-1)^T (k <= j <= i, (i,j) != (k,k))
//     and block row k-1 of W: W(k-1,j) = -Z_{k-1} sum_{l=j}^{k-2} L(k-1,l) W(l,j).
// The last block row of W follows the final step.  Writes L (strict upper
// zeroed) to St, W to Wt (must be zero on entry), pivots to dv[0..63].
__device__ void chol8_pipelined(double *St, double *Wt, double *S2, double *dv, int m) {
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
    if (__all_sync(0xffffffffu, warp == 0)) {
      double *Akk = blk(St, k, k);
      if (k > 0) {
        double l[2] = {0.0, 0.0};
        blk_mma_nt(l, blk(St, k, k - 1), blk(Wt, k - 1, k - 1));
        __syncwarp();  // in-place: every lane's operand reads before any lane's store
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
        __syncwarp();  // in-place: every lane's operand reads before any lane's store
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

// Diagonal-tile task: optional fused pre-update (GEMM), Cholesky (factor) of the
// 64 x 64 tile, its inverse W = L^{-1}, log-det partial, info, and the fused TRSM
// of the sub-diagonal tile (next link of the critical chain).
//
// Cholesky: left-looking over 16-column blocks, the 16 x 16 diagonal blocks
// factored and inverted by one warp in registers (leaf_chol16), the rows below
// by DMMA with the leaf's inverse.
// Inverse: blocked on 16 x 16 blocks: the 4 diagonal blocks come from the leaves
// (TRTRI-only tasks: right-looking substitution in 4 warps), then the off-diagonal
// blocks level by level
// W_ij = -W_ii (sum_k L_ik W_kj) with DMMA (one warp per block).
__device__ void run_potrf_trtri(const Params &p, const Task &T, double *smem, bool factor, int tsk) {
  const int tid = threadIdx.x, r = tid & 15, c = tid >> 4;
  const int lane = tid & 31, warp = tid >> 5;
  const int m = T.m;
  double *St = smem;                      // [64][LDT] L
  double *Wt = St + SERINV_TILE * LDT;    // [64][LDT] W
  double *S2 = Wt + SERINV_TILE * LDT;    // [64][LDT] TRSM2 staging / scratch
  double *lb = S2 + SERINV_TILE * LDT;    // [4][64] published pivot columns
  double *rsv = lb + 4 * SERINV_TILE;     // [64] 1 / L_jj
  double *dv = rsv + SERINV_TILE;         // [64] pivots
  __shared__ int s_bad, s_nan;  // first genuine / NaN-pivot failure in the tile
  const bool trsm2 = factor && (T.flags & TF_TRSM2);
  double acc2[2][4][2];
  if (factor && (T.flags & TF_CARRY)) {
    // carried chain: the previous task on this CTA (the chain TRSM+SYRK) left the
    // fully updated tile in St
  } else if (factor) {
    double acc1[2][4][2];
    // both fused updates (diagonal tile, sub-diagonal tile) through one pipeline
    if (trsm2)
      gemm_mainloop2<true>(p, T.seg0, T.nseg1, T.m, T.seg0 + T.nseg1, T.nseg2 - T.nseg1, T.m3, T.n, smem, acc1, acc2);
    else
      gemm_mainloop2<false>(p, T.seg0, T.nseg1, T.m, 0, 0, 0, T.n, smem, acc1, acc1);
    apply_c0(p, T.alpha, T.beta, T.c0, T.m, T.n, acc1);
    if (trsm2) apply_c0(p, (T.nseg2 > T.nseg1) ? T.alpha : 0.0, T.beta3, T.out3, T.m3, m, acc2);
    __syncthreads();
    acc_to_smem(St, acc1);
  } else {
    tile_to_smem(St, lptr(p, T.c0), T.c0.ld, m, m);
  }
  for (int idx = tid; idx < SERINV_TILE * LDT; idx += NT) Wt[idx] = 0.0;
  if (tid < SERINV_TILE) rsv[tid] = 0.0;
  if (tid == 0) s_bad = s_nan = 1 << 30;
  __syncthreads();
  phase_mark(p, tsk, 0);
  const bool chol8 = factor && (T.flags & TF_CHOL8);
  if (chol8) {
    chol8_pipelined(St, Wt, S2, dv, m);
  } else if (factor) {
    // Left-looking over 16-column blocks.  Per block: (1) DMMA update of the
    // block columns from the finished columns to the left, (2) one warp factors
    // and inverts the 16 x 16 diagonal block in registers (leaf_chol16, no CTA
    // barrier per pivot), (3) the rows below: L = A W_kk^T by DMMA.
    for (int cb = 0; cb * 16 < m; ++cb) {
      const int c0 = 16 * cb;
      const int nrow = m - c0;  // rows c0..m-1
      // (1) left-looking block update: A[c0:, c0:c0+16] -= L[c0:, :c0] L[c0:c0+16, :c0]^T
      if (cb > 0) {
        const int nrg = (nrow + 7) / 8;  // 8-row groups
        for (int f = warp; f < nrg * 2; f += 8) {
          const int r8 = c0 + 8 * (f >> 1), n8 = c0 + 8 * (f & 1);
          const int g = lane >> 2, q = lane & 3;
          double acc[2] = {0.0, 0.0};
          for (int k0 = 0; k0 < c0; k0 += 4) {
            const double av = St[(r8 + g) * LDT + k0 + q];
            const double bv = St[(n8 + g) * LDT + k0 + q];
            dmma(acc, av, bv);
          }
          St[(r8 + g) * LDT + n8 + 2 * q] -= acc[0];
          St[(r8 + g) * LDT + n8 + 2 * q + 1] -= acc[1];
        }
        __syncthreads();
      }
      // (2) diagonal block (warp 0); the other warps zero the strict upper part above it
      if (__all_sync(0xffffffffu, warp == 0)) {  // vote: the compiler sees a converged warp
        leaf_chol16(St, Wt, dv, c0, m, &s_bad);
      } else {
        for (int idx = tid - 32; idx < c0 * 16; idx += NT - 32) St[(idx >> 4) * LDT + c0 + (idx & 15)] = 0.0;
      }
      __syncthreads();
      // (3) panel below the diagonal block
      const int r0 = c0 + 16;
      if (r0 < m) {
        const int ngr = (m - r0 + 7) / 8;
        if (warp < ngr) {
          const int r8 = r0 + 8 * warp, g = lane >> 2, q = lane & 3;
          double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
          for (int k0 = 0; k0 < 16; k0 += 4) {
            const double av = St[(r8 + g) * LDT + c0 + k0 + q];
            const double b0 = Wt[(c0 + g) * LDT + c0 + k0 + q];
            const double b1 = Wt[(c0 + 8 + g) * LDT + c0 + k0 + q];
            dmma(acc[0], av, b0);
            dmma(acc[1], av, b1);
          }
          __syncwarp();
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            St[(r8 + g) * LDT + c0 + 8 * ni + 2 * q] = acc[ni][0];
            St[(r8 + g) * LDT + c0 + 8 * ni + 2 * q + 1] = acc[ni][1];
          }
        }
        __syncthreads();
      }
    }
  } else {
    // TRTRI-only: L given; zero its upper part, 1 / L_jj
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int i = r + 16 * ii, k = c + 16 * kk;
        if (k > i) St[i * LDT + k] = 0.0;
      }
    if (tid < m) {
      const double d = St[tid * LDT + tid];
      rsv[tid] = 1.0 / d;
      if (!(d != 0.0) || !isfinite(d)) atomicMin(isnan(d) ? &s_nan : &s_bad, tid);
    }
  }
  __syncthreads();
  if (factor && tid < m) {  // pivots (before the square root) of either factorisation path
    const double d = dv[tid];
    if (!(d > 0.0)) atomicMin(isnan(d) ? &s_nan : &s_bad, tid);
  }
  __syncthreads();
  phase_mark(p, tsk, 1);
  // ---- inverse, diagonal 16 x 16 blocks (TRTRI-only; the factor path's leaves produced
  // them): warp w < 4 inverts block w (lanes 0..15 = columns)
  if (!factor && warp < 4 && 16 * warp < m && lane < 16) {
    const int base = 16 * warp, cc = lane;
    double w[16], a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double x = (k >= cc) ? (((k == cc) ? 1.0 : 0.0) - a[k]) * rsv[base + k] : 0.0;
      w[k] = x;
#pragma unroll
      for (int i = k + 1; i < 16; ++i) a[i] = fma(St[(base + i) * LDT + base + k], x, a[i]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) Wt[(base + i) * LDT + base + cc] = w[i];
  }
  __syncthreads();
  // ---- off-diagonal blocks, level d = i - j
  for (int d = 1; d < (chol8 ? 1 : 4); ++d) {  // chol8: W is complete
    const int bj = warp, bi = warp + d;
    if (bi < 4 && 16 * bi < m) {
      double acc[2][2][2] = {};
      for (int k = bj; k < bi; ++k)
        warp_mma16(St + (16 * bi) * LDT + 16 * k, LDT, Wt + (16 * k) * LDT + 16 * bj, LDT, 16, acc);
      double *sc = S2 + warp * 16 * 17;  // per-warp 16 x 16 scratch (stride 17)
      const int g = lane >> 2, q = lane & 3;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) sc[(g + 8 * mi) * 17 + 8 * ni + 2 * q + h] = acc[mi][ni][h];
      __syncwarp();
      double acc2b[2][2][2] = {};
      warp_mma16(Wt + (16 * bi) * LDT + 16 * bi, LDT, sc, 17, 16, acc2b);
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            Wt[(16 * bi + g + 8 * mi) * LDT + 16 * bj + 8 * ni + 2 * q + h] = -acc2b[mi][ni][h];
    }
    __syncthreads();
  }
  phase_mark(p, tsk, 2);
  if (tid == 0 && s_bad < (1 << 30)) record_info(p.info, T.aux1 + s_bad + 1);
  if (tid == 0 && s_nan < (1 << 30)) record_info(p.info2, T.aux1 + s_nan + 1);
  const bool early = factor && (T.flags & TF_EARLY_SIG) && (T.flags & TF_W_OUT);
  if (early) {
    // W = L^{-1} is what the chain's next TRSM waits for: store it and publish the
    // task's own counter now; the log-det partial and L follow (their readers wait
    // on the factor-done counter, signalled at the end)
    smem_to_global(lptr(p, T.out2), T.out2.ld, Wt, m, m);
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(p.ctr + p.sigs[T.sig0 + ((T.flags & TF_CHAINSTEP) ? 1 : 0)], 1);
    }
  }
  const bool chainstep = factor && (T.flags & TF_CHAINSTEP) && early;
  if (chainstep) {
    // fused chain step: E's and the next tile's earlier updates (bulk tasks) are the
    // late inputs; W stays in Wt, E W^T and the next tile are formed in smem
    if (tid == 0) wait_range(p, T.wait0 + T.nwait - T.nlate, T.wait0 + T.nwait);
    __syncthreads();
    tile_to_smem(S2, lptr(p, T.out3), T.out3.ld, T.m3, m);
    __syncthreads();
    double acc[2][4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
    mma_smem64<true>(S2, Wt, acc);  // L(K+1,K) = E W^T
    store_tile(p, T.out3, T.m3, m, acc);
    if (T.zmask & 1) {  // strict-upper tile (c, c+1) of the diagonal block
      double *z = lptr(p, T.out) + SERINV_TILE;
      for (int idx = tid; idx < m * T.m3; idx += NT) {
        const int rr = idx / T.m3, cc = idx - rr * T.m3;
        z[(int64_t)rr * T.out.ld + cc] = 0.0;
      }
    }
    __syncthreads();
    if (tid == 0) {  // publish the sub-diagonal tile (sigs[1]) for the bulk updates
      __threadfence();
      atomicAdd(p.ctr + p.sigs[T.sig0 + 2], 1);
    }
    smem_to_global(lptr(p, T.out), T.out.ld, St, m, m);  // L(K,K); St is reused below
    acc_to_smem(S2, acc);
    __syncthreads();
    tile_to_smem(St, lptr(p, T.out4), T.out4.ld, T.m4, T.m4);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
    if (warp != 1) mma_smem64<true>(S2, S2, acc);  // lower triangle of L L^T (warp 1's slab is upper)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int rr, cc;
          frag_rc(mi, ni, h, rr, cc);
          acc[mi][ni][h] = St[rr * LDT + cc] - acc[mi][ni][h];
        }
    store_tile(p, T.out4, T.m4, T.m4, acc);
    __syncthreads();
    acc_to_smem(St, acc);  // carried into the next POTRF on this CTA
  }
  if (factor) {
    // log det partial: sum_j 0.5 log d_j, fixed-order tree over 64 values
    double *lg = lb;
    if (tid < 64) lg[tid] = (tid < m) ? 0.5 * log(dv[tid]) : 0.0;
    __syncthreads();
    for (int h = 32; h > 0; h >>= 1) {
      if (tid < h) lg[tid] += lg[tid + h];
      __syncthreads();
    }
    if (tid == 0 && T.aux0 >= 0) *lptr(p, T.r) = lg[0];
  }
  // ---- TRSM of the sub-diagonal tile: L2 = S2 * W^T (the update was applied up front)
  if (trsm2) {
    acc_to_smem(S2, acc2);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc2[i][jj][0] = acc2[i][jj][1] = 0.0;
    mma_steps(S2, LDT, 1, Wt, LDT, 1, acc2, (m + 3) / 4);
    store_tile(p, T.out3, T.m3, m, acc2);
    if (T.zmask & 1) {  // strict-upper tile (c, c+1) of the diagonal block
      double *z = lptr(p, T.out) + SERINV_TILE;
      for (int idx = tid; idx < m * T.m3; idx += NT) {
        const int rr = idx / T.m3, cc = idx - rr * T.m3;
        z[(int64_t)rr * T.out.ld + cc] = 0.0;
      }
    }
    if (T.flags & TF_TRSM3) {
      // second sub-diagonal tile: its inputs were produced by bulk tasks while this
      // task factorised the diagonal tile -- await them now
      if (tid == 0) wait_range(p, T.wait0 + T.nwait - T.nlate, T.wait0 + T.nwait);
      __syncthreads();
      double *stage = smem + 2 * SERINV_TILE * LDT;  // St (L) and Wt (W) stay live
      gemm_onestage(p, T.seg0 + T.nseg2, T.nseg - T.nseg2, T.m4, m, stage, acc2);
      apply_c0(p, (T.nseg > T.nseg2) ? T.alpha : 0.0, T.beta4, T.out4, T.m4, m, acc2);
      acc_to_smem(S2, acc2);
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc2[i][jj][0] = acc2[i][jj][1] = 0.0;
      mma_steps(S2, LDT, 1, Wt, LDT, 1, acc2, (m + 3) / 4);
      store_tile(p, T.out4, T.m4, m, acc2);
      if (T.zmask & 2) {  // strict-upper tile (c, c+2)
        double *z = lptr(p, T.out) + 2 * SERINV_TILE;
        for (int idx = tid; idx < m * T.m4; idx += NT) {
          const int rr = idx / T.m4, cc = idx - rr * T.m4;
          z[(int64_t)rr * T.out.ld + cc] = 0.0;
        }
      }
    }
  }
  phase_mark(p, tsk, 3);
  // ---- store L (factor) and W
  {
    const bool wout = (!factor || (T.flags & TF_W_OUT)) && !early;
    const Loc &wl = factor ? T.out2 : T.out;
    if (factor && !chainstep) smem_to_global(lptr(p, T.out), T.out.ld, St, m, m);
    if (wout) smem_to_global(lptr(p, wl), wl.ld, Wt, m, m);
  }
  phase_mark(p, tsk, 4);
}

__device__ void run_reduce(const Params &p, const Task &T) {
  // out = beta * C0 + alpha * sum_{j < cnt} P_j, fixed order j = 0..cnt-1; element pairs
  const double *src = lptr(p, T.r);
  const double *c0 = T.beta != 0.0 ? lptr(p, T.c0) : nullptr;
  double *o = lptr(p, T.out);
  const int n2 = (T.n + 1) >> 1;
  for (int idx = threadIdx.x; idx < T.m * n2; idx += NT) {
    const int r = idx / n2, c = 2 * (idx - r * n2);
    const bool two = c + 1 < T.n;
    double s0 = 0.0, s1 = 0.0;
    const double *sp = src + (int64_t)r * T.r.ld + c;
#pragma unroll 4
    for (int j = 0; j < T.aux0; ++j) {
      const double *q = sp + T.aux2 * j;
      s0 += __ldcg(q);
      if (two) s1 += __ldcg(q + 1);
    }
    double v0 = T.alpha * s0, v1 = T.alpha * s1;
    if (c0) {
      v0 += T.beta * __ldcg(c0 + (int64_t)r * T.c0.ld + c);
      if (two) v1 += T.beta * __ldcg(c0 + (int64_t)r * T.c0.ld + c + 1);
    }
    double *op = o + (int64_t)r * T.out.ld + c;
    op[0] = v0;
    if (two) op[1] = v1;
    if (T.flags & TF_MIRROR) {
      double *o2 = lptr(p, T.out2);
      o2[(int64_t)c * T.out2.ld + r] = v0;
      if (two) o2[(int64_t)(c + 1) * T.out2.ld + r] = v1;
    }
  }
}

__device__ void run_copy(const Params &p, const Task &T) {
  const double *c0 = lptr(p, T.c0);
  double *o = lptr(p, T.out);
  const bool tr = (T.flags & TF_TRANS_C0) != 0;
  for (int idx = threadIdx.x; idx < T.m * T.n; idx += NT) {
    int r = idx / T.n, c = idx - r * T.n;
    double v = tr ? __ldcg(c0 + (int64_t)c * T.c0.ld + r) : __ldcg(c0 + (int64_t)r * T.c0.ld + c);
    o[(int64_t)r * T.out.ld + c] = T.alpha * v;
  }
}

__device__ void run_logdet(const Params &p, const Task &T, double *smem) {
  // *out = 2 * sum slots (fixed per-thread strides + fixed tree) + sum extras (rank order)
  const double *slots = lptr(p, T.r);
  double s = 0.0;
  for (int j = threadIdx.x; j < T.aux0; j += NT) s += __ldcg(slots + j);
  smem[threadIdx.x] = s;
  __syncthreads();
  for (int w = NT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) smem[threadIdx.x] += smem[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double v = 2.0 * smem[0];
    if (T.aux1 > 0) {
      const double *ex = lptr(p, T.c0);
      for (int j = 0; j < T.aux1; ++j) v += __ldcg(ex + T.aux2 * j);
    }
    const int inf = *(volatile int *)p.info | *(volatile int *)p.info2;
    *lptr(p, T.out) = inf ? __longlong_as_double(0x7ff8000000000000ULL) : v;
  }
}

}  // namespace dev

extern "C" __global__ void __launch_bounds__(dev::NT, 2) serinv_exec_kernel(dev::Params p) {
  using namespace dev;
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_task, s_q;
  // ---- roles: the first nq-1 CTAs to arrive serve the critical queues and get
  // their SM to themselves (co-resident siblings on those SMs exit); the rest
  // serve the bulk queue.  All CTAs are co-resident, so the barrier is safe.
  if (threadIdx.x == 0) {
    int32_t *role = p.qclaim + p.nq;
    const int rank = atomicAdd(role, 1);
    const int me = (int)smid();
    role[2 + rank] = me;
    __threadfence();
    atomicAdd(role + 1, 1);
    const unsigned long long t0 = globaltimer();
    while (ld_acquire(role + 1) < (int)gridDim.x) {
      __nanosleep(64);
      if (globaltimer() - t0 > 20000000000ULL) {  // watchdog (grid not co-resident)
        atomicExch(p.info, -1);
        break;
      }
    }
    // The first ncrit DISTINCT SMs in arrival order become critical SMs; on each,
    // the earliest-arrived CTA serves one critical queue and the others exit, so
    // every critical chain owns a whole SM.
    int q = 0;
    const int ncrit = p.ncrit;
    int found = 0, last_crit_rank = -1;
    for (int r = 0; r < (int)gridDim.x && found < ncrit; ++r) {
      const int sr = ld_acquire(role + 2 + r);
      bool seen = false;
      for (int r2 = 0; r2 < r; ++r2)
        if (ld_acquire(role + 2 + r2) == sr) {
          seen = true;
          break;
        }
      if (seen) continue;
      ++found;  // sr is critical SM number `found`
      last_crit_rank = r;
      if (sr == me) q = (r == rank) ? found : -1;
    }
    // the urgent queue: the first nurgent CTAs (arrival order) not on a critical SM
    if (q == 0 && p.nurgent > 0 && p.nq > ncrit + 1) {
      int cnt = 0;
      for (int r = 0; r < rank; ++r) {
        const int sr = ld_acquire(role + 2 + r);
        bool crit = false;
        for (int r2 = 0; r2 <= last_crit_rank; ++r2)
          if (ld_acquire(role + 2 + r2) == sr) {
            crit = true;
            break;
          }
        if (!crit) ++cnt;
      }
      if (cnt < p.nurgent) q = ncrit + 1;
    }
    s_q = q;
  }
  __syncthreads();
  const int q0 = s_q;  // read before thread 0 reuses s_q for the claims
  __syncthreads();
  if (q0 >= 0) {
    unsigned long long t_claim = 0, t_start = 0;
    for (;;) {
      if (threadIdx.x == 0) {
        int q = s_q, t = -1;
        for (;;) {
          const int idx = atomicAdd(p.qclaim + q, 1);
          if (idx < p.qoff[q + 1] - p.qoff[q]) {
            t = p.qlist[p.qoff[q] + idx];
            break;
          }
          if (q == 0) break;
          q = 0;  // critical queue drained: help with the bulk queue
        }
        s_q = q;
        s_task = t;
      }
      __syncthreads();
      const int t = s_task;
      if (t < 0) break;
      const Task T = p.tasks[t];
      if (p.trace && threadIdx.x == 0) t_claim = globaltimer();
      if (threadIdx.x == 0) {
        for (int w = 0; w < T.nwait - T.nlate; ++w) {
          const Wait W = p.waits[T.wait0 + w];
          if (ld_acquire(p.ctr + W.ctr) >= W.target) continue;
          int ns = 32;
          const unsigned long long t0 = globaltimer();
          while (ld_acquire(p.ctr + W.ctr) < W.target) {
            __nanosleep(ns);
            ns = min(ns * 2, 256);
            if (globaltimer() - t0 > 20000000000ULL) {  // 20 s watchdog: never hang the GPU
              atomicExch(p.info, -1);
              break;
            }
          }
        }
      }
      if (p.trace && threadIdx.x == 0) t_start = globaltimer();
      __syncthreads();
      switch (T.type) {
        case TK_GEMM:
          if (T.m > SERINV_TILE) run_gemm_wide(p, T, smem);
          else run_gemm(p, T, smem, t);
          break;
        case TK_POTRF: run_potrf_trtri(p, T, smem, true, t); break;
        case TK_TRTRI: run_potrf_trtri(p, T, smem, false, t); break;
        case TK_REDUCE: run_reduce(p, T); break;
        case TK_COPY: run_copy(p, T); break;
        case TK_LOGDET: run_logdet(p, T, smem); break;
        default: break;
      }
      // publish: barrier (CTA-scope ordering of every thread's stores) then one
      // gpu-scope fence by the signalling thread (cumulative) and the increments.
      // The last warp publishes while thread 0 already claims the next task.
      __syncthreads();
      if (threadIdx.x == NT - 32) {
        __threadfence();
        const bool ew = T.type == TK_POTRF && (T.flags & TF_EARLY_SIG) && (T.flags & TF_W_OUT);
        const bool cs = ew && (T.flags & TF_CHAINSTEP);
        // early-published signals: sigs[0] (W), or sigs[1] (W) and sigs[2] (sub-diagonal tile) of a chain step
        for (int s = (ew && !cs) ? 1 : 0; s < T.nsig; ++s)
          if (!(cs && (s == 1 || s == 2))) atomicAdd(p.ctr + p.sigs[T.sig0 + s], 1);
        if (p.trace) {
          unsigned long long *rec = p.trace + 4 * (size_t)t;
          rec[2] = globaltimer();
          rec[3] = (unsigned long long)(unsigned)T.type | ((unsigned long long)smid() << 16) |
                   ((unsigned long long)(unsigned)T.m << 32) | ((unsigned long long)(unsigned)T.flags << 48);
        }
      }
      if (threadIdx.x == 0 && p.trace) {
        unsigned long long *rec = p.trace + 4 * (size_t)t;
        rec[0] = t_claim;
        rec[1] = t_start;
      }
    }
  }
  // the last CTA out merges the NaN-pivot failures into *info (only if there was
  // no genuine failure): every other CTA's records are ordered before its
  // fence + increment of the exit counter
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.done, 1) == (int)gridDim.x - 1) {
      __threadfence();
      const int i2 = *(volatile int *)p.info2;
      if (i2 != 0) atomicCAS(p.info, 0, i2);
    }
  }
}


int exec_smem_bytes() { return dev::SMEM_DOUBLES * 8; }

}  // namespace serinv
