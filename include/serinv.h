/*
 * serinv.h -- C-ABI of libserinv.so: FP64 block Cholesky (POBTAF) and selected
 * inversion (POBTASI) of SPD block-tridiagonal-with-arrowhead (BTA) matrices on
 * NVIDIA B200 (sm_100a), plus the partitioned variants PPOBTAF / PPOBTASI.
 *
 * Method: Serinv, arXiv 2503.17528.  Citations "P:n" are PAPER.md lines.
 *
 * ---------------------------------------------------------------------------
 * Matrix layout (Sec. 2.1, Table 2).  A BTA matrix of order
 * N = n*b + a has n diagonal blocks A_{i,i} (b x b), n-1 lower blocks A_{i+1,i}
 * (b x b), n arrow blocks A_{n,i} (a x b) and the tip A_{n,n} (a x a).  a = 0 is
 * the BT special case; then arrow/tip may be NULL.
 *
 * All blocks are FP64, ROW-MAJOR, stored contiguously per kind in DEVICE memory
 * that the caller owns (typically torch tensors):
 *     diag  [n][b][b]     A_{i,i}   -> L_{i,i} (strict upper set to 0) -> X_{i,i} (full symmetric)
 *     lower [n-1][b][b]   A_{i+1,i} -> L_{i+1,i}                      -> X_{i+1,i}
 *     arrow [n][a][b]     A_{n,i}   -> L_{n,i}                        -> X_{n,i}
 *     tip   [a][a]        A_{n,n}   -> L_{n,n} (strict upper set to 0) -> X_{n,n} (full symmetric)
 * Only the lower triangles of diag/tip are read on input.  Base pointers must be
 * 16-byte aligned (cudaMalloc / torch allocations are).
 *
 * Results (the plain definitions the method reaches):
 *   serinv_pobtaf : L = the Cholesky factor of A restricted to the BTA pattern
 *                   (fill-in stays in the pattern), and log det A = 2 sum log diag L.
 *   serinv_pobtasi: X = A^{-1} restricted to the BTA pattern ("true inverse blocks
 *                   with the exact same coordinates as the non-zero blocks of A").
 *
 * Ownership: the caller allocates every buffer, including the workspace whose
 * size the *_ws queries return.  The library allocates only its cached task
 * graphs (one per problem shape, on first use; see serinv_prepare).
 *
 * Errors: the host return value (int) is synchronous and reports argument /
 * launch problems:  SERINV_OK, -k = argument k invalid, SERINV_ERR_* below.
 * Numerical status is stream-ordered in *d_info (device int):
 *     0      success
 *     k > 0  (pobtaf) the 1-based global row of the first non-positive pivot
 *            (LAPACK dpotrf semantics): block (k-1)/b, or the tip if k > n*b.
 *            Outputs are then undefined and *d_logdet is NaN.
 *     k > 0  (pobtasi) zero / non-finite diagonal entry of L at global row k.
 *     -1     internal watchdog fired (a dependency never completed within 20 s);
 *            outputs undefined.  Indicates a library bug, never a property of A.
 * No host synchronisation happens inside any call (all work is enqueued on
 * `stream`, a cudaStream_t passed as void*).
 */
#ifndef SERINV_H
#define SERINV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SERINV_OK 0
#define SERINV_ERR_CUDA 1001     /* a CUDA runtime call failed                  */
#define SERINV_ERR_WS 1002       /* workspace too small / misaligned            */
#define SERINV_ERR_NCCL 1003     /* NCCL call failed (distributed entry points) */
#define SERINV_ERR_HANDLE 1004   /* NULL / destroyed handle                      */
#define SERINV_ERR_SHAPE 1005    /* unsupported shape (e.g. n < 1, b < 1)        */
#define SERINV_ERR_ALIGN 1006    /* a base pointer is not 16-byte aligned        */
#define SERINV_ERR_PLAN 1007     /* infeasible partition plan (too few blocks)   */

/* A BTA matrix on the device (see layout above). */
typedef struct {
  int64_t n, b, a;
  double *diag;   /* [n][b][b]   */
  double *lower;  /* [n-1][b][b] */
  double *arrow;  /* [n][a][b]   (NULL allowed if a == 0) */
  double *tip;    /* [a][a]      (NULL allowed if a == 0) */
} serinv_bta_t;

typedef struct serinv_ctx *serinv_handle_t;

/* Version string of the library ("serinv-b200 <ver> sm_100a"). */
const char *serinv_version(void);
/* Human-readable text for a status code. */
const char *serinv_status_string(int status);

/* Create / destroy a handle bound to CUDA device `cuda_device`.  One handle per
 * host thread; the handle caches task graphs keyed by problem shape. */
int serinv_create(serinv_handle_t *h, int cuda_device);
int serinv_destroy(serinv_handle_t h);

/* Workspace sizes in bytes (device memory, 256-byte aligned by the caller). */
int serinv_pobtaf_ws(int64_t n, int64_t b, int64_t a, size_t *bytes);
int serinv_pobtasi_ws(int64_t n, int64_t b, int64_t a, size_t *bytes);
/* serinv_selinv needs max(pobtaf_ws, pobtasi_ws) == serinv_selinv_ws. */
int serinv_selinv_ws(int64_t n, int64_t b, int64_t a, size_t *bytes);

/* Build and upload the task graph for shape (n, b, a) ahead of time
 * (kind: 0 = pobtaf, 1 = pobtasi, 2 = selinv).  Optional: the compute entry
 * points build it on first use. */
int serinv_prepare(serinv_handle_t h, int kind, int64_t n, int64_t b, int64_t a);

/*
 * POBTAF (Alg. 1): in-place block Cholesky  A -> L.
 *   A        device BTA (overwritten by L; strict upper of diag/tip zeroed)
 *   d_ws     device workspace of >= serinv_pobtaf_ws bytes
 *   d_info   device int (written; see above)
 *   d_logdet device double: log det A = 2 sum log diag(L) (NaN if info != 0);
 *            may be NULL.
 */
int serinv_pobtaf(serinv_handle_t h, const serinv_bta_t *A, void *d_ws, size_t ws_bytes,
                  int *d_info, double *d_logdet, void *stream);

/*
 * POBTASI (Alg. 2): in-place selected inversion  L -> X.
 * L must be the output of serinv_pobtaf (any workspace); the inverse of each
 * L_{i,i} is formed once and the TRSMs become GEMMs.
 */
int serinv_pobtasi(serinv_handle_t h, const serinv_bta_t *L, void *d_ws, size_t ws_bytes,
                   int *d_info, void *stream);

/*
 * POBTAF followed by POBTASI as ONE task graph (A -> X, plus log det): the
 * L_{i,i}^{-1} precompute of the inversion overlaps the factorisation chain.
 * Same result as serinv_pobtaf + serinv_pobtasi.
 */
int serinv_selinv(serinv_handle_t h, const serinv_bta_t *A, void *d_ws, size_t ws_bytes,
                  int *d_info, double *d_logdet, void *stream);

/*
 * serinv_selinv with HOST buffers and streaming IO: A_host (pinned host memory,
 * same layout) is copied into the device buffers A_dev in chunks of blocks on an
 * internal copy stream while the factorisation runs (each chunk bumps an arrival
 * counter the task graph waits on, via cuStreamWriteValue32); the selected
 * inverse is copied back to X_host (pinned; may equal A_host) node by node as
 * soon as the backward pass finalises it (cuStreamWaitValue32 on the node's
 * counter).  A_dev is overwritten by X.  `stream` is joined with both copy
 * streams before the call's work completes on it.  Workspace: serinv_selinv_ws.
 */
int serinv_selinv_host(serinv_handle_t h, const serinv_bta_t *A_host, const serinv_bta_t *X_host,
                       const serinv_bta_t *A_dev, void *d_ws, size_t ws_bytes, int *d_info, double *d_logdet,
                       void *stream);

/* ------------------------------------------------------------------------- */
/* Partitioned method (Sec. 3, Alg. 3-6).                 */
/* ------------------------------------------------------------------------- */

/*
 * Partition plan (Sec. 3.1, Sec. 4.3; reading R6 in
 * DESIGN.md): P contiguous ranges of the n diagonal blocks, rank 0 the top
 * partition.  top = floor(r*n/(r+P-1)) clamped to [1, n-2(P-1)], the rest split
 * evenly over ranks 1..P-1 with the remainder going to the earliest ones.
 *   starts: host array of P+1 int64; rank p owns blocks [starts[p], starts[p+1]).
 * Returns SERINV_ERR_PLAN if n < 2P-1.
 */
int serinv_plan(int64_t n, int P, double r, int64_t *starts);

/* Partition plan for the twisted scheme (reading R14: the last partition
 * is eliminated bottom-up, so the first and the last partition are fill-in free):
 * both ends get r times a middle partition's blocks, middles split the rest evenly
 * (each >= 2), the remainder to the earliest; P = 2 gives equal halves, r = 1 the
 * same partition as serinv_plan.  starts: host int64[P + 1], caller-owned.
 * Returns 0, -3 (r not positive/finite), -4 (NULL), SERINV_ERR_PLAN (infeasible). */
int serinv_plan_ends(int64_t n, int P, double r, int64_t *starts);

/*
 * In-process partitioned selected inversion on ONE device: PPOBTAF (Alg. 3-4)
 * over P partitions, POBTARSSI on the reduced system of 2P-1 blocks (Sec. 3.3),
 * PPOBTASI (Alg. 5-6), executed as one task graph whose partitions run
 * concurrently on disjoint SMs.  Equivalent to serinv_selinv (same X and log
 * det up to rounding).  Breaks the length-n dependency chain into
 * chains of length ~n/P.  A is overwritten by X.  P = 1 is
 * serinv_selinv.
 */
int serinv_pselinv_ws(int64_t n, int64_t b, int64_t a, int P, double r, size_t *bytes);
int serinv_pselinv(serinv_handle_t h, const serinv_bta_t *A, int P, double r, void *d_ws,
                   size_t ws_bytes, int *d_info, double *d_logdet, void *stream);

/*
 * Nested solving (Sec. 4.2 "nested solving"; SURVEY 8(f)
 * f1/f3) on ONE device: Ps[0] partitions of A; the reduced system A_r (2 Ps[0]-1
 * blocks) is itself solved by the partitioned algorithm with Ps[1] partitions,
 * and so on for nlev <= SERINV_MAX_LEVELS levels; the last reduced system is
 * solved as one chain.  Every level must be feasible (serinv_plan with ratio r;
 * levels >= 1 need Ps[k] >= 2 and 2 Ps[k-1] - 1 >= 2 Ps[k] - 1).  Same result
 * as serinv_selinv (X in place, log det) up to rounding.  Errors as
 * serinv_pselinv; SERINV_ERR_PLAN for an infeasible level.
 *
 * serinv_auto_partitions: the library's default plan for n blocks of size b on
 * one B200 (partitions of ~64 blocks for b <= 128, ~32 for b <= 512, nested
 * until the last reduced system has <= 48 / 16 blocks; {1} = sequential for
 * large b, where the chains are throughput-bound).  Writes min(levels, cap)
 * entries of Ps and returns the number of levels (>= 1).
 */
#define SERINV_MAX_LEVELS 4
int serinv_auto_partitions(int64_t n, int64_t b, int *Ps, int cap);
int serinv_pselinv_nested_ws(int64_t n, int64_t b, int64_t a, int nlev, const int *Ps, double r,
                             size_t *bytes);
int serinv_pselinv_nested(serinv_handle_t h, const serinv_bta_t *A, int nlev, const int *Ps, double r,
                          void *d_ws, size_t ws_bytes, int *d_info, double *d_logdet, void *stream);

/*
 * Distributed partitioned method, one process per GPU (rank p of P owns the
 * blocks [starts[p], starts[p+1]) of serinv_plan).  The caller passes its LOCAL
 * blocks:
 *     diag  [count][b][b], arrow [count][a][b],
 *     lower [count][b][b]  where lower[count-1] is the coupling A_{e,e-1} to the
 *                          next rank (P:378 assigns A_{i+1,i} to column i's
 *                          partition); the last rank passes count-1 lower blocks.
 *     tip   replicated: every rank passes the same A_{n,n} and receives X_{n,n}.
 * part = {P, rank, n_global, start, count}.
 *
 *   serinv_ppobtaf   PARTIAL_POBTAF (rank 0) or PERMUTED_POBTAF (rank > 0) on
 *                    the local blocks (no communication), then packs this rank's
 *                    boundary blocks + U_p + partial log det into d_sendbuf
 *                    (serinv_exchange_bytes bytes).
 *   (caller)         all-gather of the P send buffers into d_recvbuf (rank
 *                    order) -- NCCL via torch.distributed in the Python binding.
 *   serinv_ppobtasi  assembles the reduced system A_r from d_recvbuf in a fixed
 *                    rank order (bit-identical on every rank), runs POBTARSSI
 *                    redundantly, then PARTIAL_/PERMUTED_POBTASI on the local
 *                    blocks.  Writes X in place and the global log det.
 * d_ws must be passed unchanged from serinv_ppobtaf to serinv_ppobtasi (it keeps
 * the fill-in factor blocks B_i, Alg. 6 l.3/l.11).
 */
typedef struct {
  int P, rank;
  int64_t n_global, start, count;
} serinv_part_t;

int serinv_exchange_bytes(int64_t b, int64_t a, size_t *bytes);
int serinv_ppobtaf_ws(const serinv_part_t *part, int64_t b, int64_t a, size_t *bytes);
int serinv_ppobtaf(serinv_handle_t h, const serinv_part_t *part, const serinv_bta_t *A_local,
                   void *d_ws, size_t ws_bytes, void *d_sendbuf, int *d_info, void *stream);
int serinv_ppobtasi(serinv_handle_t h, const serinv_part_t *part, const serinv_bta_t *L_local,
                    void *d_ws, size_t ws_bytes, const void *d_recvbuf, int *d_info,
                    double *d_logdet, void *stream);

/*
 * Hierarchical variant: intra-GPU partitioning of each rank's blocks (SURVEY
 * §8(f) f1 applied per rank; nested solving of the reduced system, PAPER.md
 * Sec. 4.2).  Rank p splits its blocks [start, start+count) into Q
 * consecutive sub-partitions (even sizes, remainder to the earliest; each needs
 * >= 2 blocks, count >= 2Q), so the whole matrix has P*Q partitions, rank p
 * owning partitions [pQ, (p+1)Q).  Q must be the same on every rank.
 *   serinv_ppobtaf_q   factors the Q sub-partitions (one launch) and packs Q
 *                      exchange records (Q * serinv_exchange_bytes bytes in
 *                      d_sendbuf; the rank's partial log det in the first).
 *   (caller)           all-gather of the P send buffers (rank order) into
 *                      d_recvbuf: P * Q records in global partition order.
 *   serinv_ppobtasi_q  assembles the reduced system (2PQ-2 blocks with the
 *                      twisted last partition, reading R14), solves it
 *                      redundantly -- by the nested partitioned algorithm when
 *                      long (serinv_auto_partitions), else as one chain --
 *                      then the backward pass of the Q sub-partitions.
 * Q = 1 is exactly serinv_ppobtaf / serinv_ppobtasi.  Errors as above, plus
 * SERINV_ERR_PLAN if Q < 1 or count < 2Q (Q > 1).  d_ws from
 * serinv_ppobtaf_q_ws(part, Q, ...), passed unchanged between the two calls.
 * serinv_dist_auto_q: the library's default Q for a rank of `count` blocks of
 * size b (the first level of serinv_auto_partitions(count, b)); >= 1, or a
 * negative status.
 */
int serinv_ppobtaf_q_ws(const serinv_part_t *part, int Q, int64_t b, int64_t a, size_t *bytes);
int serinv_ppobtaf_q(serinv_handle_t h, const serinv_part_t *part, int Q, const serinv_bta_t *A_local,
                     void *d_ws, size_t ws_bytes, void *d_sendbuf, int *d_info, void *stream);
int serinv_ppobtasi_q(serinv_handle_t h, const serinv_part_t *part, int Q, const serinv_bta_t *L_local,
                      void *d_ws, size_t ws_bytes, const void *d_recvbuf, int *d_info,
                      double *d_logdet, void *stream);
int serinv_dist_auto_q(int64_t count, int64_t b);

/* ------------------------------------------------------------------------- */
/* Introspection (tests / bench).                                            */
/* ------------------------------------------------------------------------- */

/* Statistics of the cached graph for (kind, n, b, a[, P]): number of tasks,
 * executed FP64 flops (model), persistent grid size.  kind as serinv_prepare,
 * 3 = pselinv (P given), 4 = ppobtaf, 5 = ppobtasi. */
typedef struct {
  int64_t tasks;
  int64_t counters;
  double flops;
  int grid;
  int tile;
} serinv_graph_stats_t;
int serinv_graph_stats(serinv_handle_t h, int kind, int64_t n, int64_t b, int64_t a, int P,
                       double r, serinv_graph_stats_t *out);
/* the same for the nested partitioned graph of serinv_pselinv_nested */
/* Diagnostic (tools/): the claimed task list of the cached graph for (kind, n, b, a, P, r).
 * rec: ntasks x 10 int32 {type, flags, m, n, wait0, nwait, nlate, sig0, nsig, claim queue};
 * waits / sigs: counter ids (sizes returned in *nw / *ns; pass NULL arrays to query).
 * Host pointers, caller-owned.  Returns 0 or a negative argument / SERINV_ERR_* code. */
int serinv_graph_dump(serinv_handle_t h, int kind, int64_t n, int64_t b, int64_t a, int P, double r,
                      int32_t *rec, int32_t *waits, int64_t *nw, int32_t *sigs, int64_t *ns);
int serinv_graph_stats_nested(serinv_handle_t h, int64_t n, int64_t b, int64_t a, int nlev, const int *Ps,
                              double r, serinv_graph_stats_t *out);

/* Tracing: while d_trace != NULL, every launch whose graph has at most
 * bytes/96 tasks records 4 x uint64 per task (in emission order):
 * {claim time, start time (inputs ready), end time, meta}, times from the GPU
 * global timer (ns); meta = type | smid << 16 | m << 32 | flags << 48; followed
 * by 8 x uint64 per task of phase timestamps (POTRF / TRTRI tasks). 
 * Pass NULL to disable. */
int serinv_set_trace(serinv_handle_t h, void *d_trace, size_t bytes);

/* Diagnostic: `ntasks` independent 64 x 64 tile GEMMs (K = k, in nseg segments)
 * through the persistent executor; measures the tile engine's throughput.
 * d_ws needs >= 8 * (2 * 64 * 64 * k + 64^3) bytes. */
int serinv_bench_gemm(serinv_handle_t h, int ntasks, int k, int nseg, void *d_ws, size_t ws_bytes, void *stream);

/* Number of kernel launches enqueued by the last compute call of this handle. */
int serinv_last_launches(serinv_handle_t h, int *launches);

#ifdef __cplusplus
}
#endif
#endif /* SERINV_H */
