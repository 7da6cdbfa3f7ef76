// task.h -- task-graph records shared by the host graph builder (graph.cpp) and
// the persistent sm_100a executor (exec.cu).
//
// The whole BTA factorisation / selected inversion (Alg. 1-6) is lowered
// to a DAG of TILE tasks (tile edge TILE = 64 doubles).  Every task writes one
// output tile (<= 64 x 64) and is one of:
//   TK_GEMM    out = (alpha * sum_s op(A_s) op(B_s) + beta * C0) [* op(R)]
//              -- Schur updates (Alg. 1 l.5-7, Alg. 4 l.7-12), TRSM as
//              GEMM with the inverted diagonal tile, the POBTASI
//              products (Alg. 2 l.7-12, Alg. 6), triangular inverses.
//   TK_POTRF   L = chol(alpha * sum_s ... + beta * C0) of a diagonal tile, plus
//              W = L^{-1} (so later TRSMs are GEMMs), log-diag partial, info.
//   TK_TRTRI   W = L^{-1} of a stored lower-triangular tile.
//   TK_REDUCE  out = beta * C0 + alpha * sum_j P_j  (fixed order j = 0..cnt-1).
//   TK_COPY    out = alpha * op(C0)   (op = transpose if TF_TRANS_C0).
//   TK_LOGDET  *logdet = 2 * sum_j slot_j (fixed tree order), NaN if info != 0.
// Dependencies are counters: a task waits until counter[c] >= target for each
// of its waits, and after its stores increments each counter in its signal
// list.  Task records are emitted in a topological order (graph.cpp), so a
// task only ever waits on tasks claimed before it -- the persistent grid
// cannot deadlock as long as all its CTAs are co-resident.
#pragma once
#include <stdint.h>

#define SERINV_TILE 64

enum TaskKind : int16_t {
  TK_NOP = 0,
  TK_GEMM = 1,
  TK_POTRF = 2,
  TK_TRTRI = 3,
  TK_REDUCE = 4,
  TK_COPY = 5,
  TK_LOGDET = 6,
};

enum TaskFlags : uint16_t {
  TF_MIRROR = 1,      // also store the transpose of the result at out2
  TF_POST = 2,        // right-multiply the result by op(R) (R is n x n)
  TF_POST_T = 4,      // op(R) = R^T (else R)
  TF_ZERO_MIRROR = 8, // store zeros at out2 (transposed footprint): strict-upper tiles of L
  TF_TRANS_C0 = 16,   // TK_COPY: out = alpha * C0^T
  TF_W_OUT = 32,      // TK_POTRF: store W = L^{-1} at out2
  TF_TRSM2 = 64,      // TK_POTRF: fused TRSM of the sub-diagonal tile (out3)
  TF_TRSM3 = 128,     // TK_POTRF: fused TRSM of the second sub-diagonal tile (out4)
  TF_SYRK3 = 256,     // TK_GEMM (+TF_POST): then out3 (m x m) -= L L^T with L the result
  TF_CHOL8 = 512,     // TK_POTRF: warp-pipelined 8 x 8-block Cholesky + inverse (chol8_pipelined)
  TF_EARLY_SIG = 1024,  // TK_POTRF (+TF_W_OUT, no TF_TRSM2): own counter signalled once W is stored
  TF_CARRY = 2048,    // carried chain (same CTA, consecutive tasks): TK_POTRF reads its tile from smem St;
                      // TK_GEMM (+TF_POST|TF_SYRK3) reads W from smem Wt and leaves the SYRK result in St
  TF_CHAINSTEP = 4096,  // TK_POTRF: then E W^T for the sub-diagonal tile out3 (sigs[1] after its store) and
                        // the next diagonal tile out4 -= (E W^T)(E W^T)^T, left in St (carry); late inputs
};

// Buffer ids (kernel argument `bufs[]`, offsets in doubles).
enum BufId : int32_t {
  BUF_DIAG = 0,
  BUF_LOWER = 1,
  BUF_ARROW = 2,
  BUF_TIP = 3,
  BUF_WS = 4,     // workspace (doubles)
  BUF_EXT0 = 5,   // extra user buffers (exchange send / recv)
  BUF_EXT1 = 6,
  BUF_LOGDET = 7, // double* scalar
  BUF_COUNT = 8
};

struct Loc {
  int32_t buf;
  int32_t ld;
  int64_t off;
};

struct Seg {
  Loc A, B;
  int32_t k;
  int8_t ta, tb;  // 0: op(X) = X, 1: op(X) = X^T
  int8_t pad0, pad1;
};

struct Wait {
  int32_t ctr, target;
};

struct Task {
  int16_t type;
  uint16_t flags;
  int16_t m, n;         // output tile dims (<= SERINV_TILE)
  int32_t seg0, nseg;
  int32_t wait0, nwait;
  int32_t sig0, nsig;
  Loc out, c0, r, out2;
  double alpha, beta;
  int32_t aux0, aux1;   // POTRF: aux0 = logdet slot (-1 none), aux1 = global row base (info)
  int64_t aux2;         // REDUCE: stride between partials (doubles); count in aux0
  // TK_POTRF with TF_TRSM2: also L2 = (beta3 * C3 - sum_{s >= nseg1} ...) W^T for the
  // sub-diagonal tile at out3 (m3 rows), i.e. the next link of the critical chain.
  Loc out3;
  double beta3;
  int32_t m3, nseg1;
  // TK_POTRF with TF_TRSM3: the second sub-diagonal tile at out4 (m4 rows),
  // update segments [nseg2, nseg); its inputs are awaited LATE: waits
  // [nwait - nlate, nwait) are checked only after the diagonal tile is done.
  // zmask bit0 / bit1: zero the strict-upper mirror tile at out + 64 / out + 128.
  Loc out4;
  double beta4;
  int32_t m4, nseg2;
  int32_t nlate, zmask;
};

static_assert(sizeof(Loc) == 16, "Loc layout");
static_assert(sizeof(Seg) == 40, "Seg layout");
static_assert(sizeof(Task) == 200, "Task layout");
