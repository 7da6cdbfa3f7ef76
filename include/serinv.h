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

/* Create / destroy a handle bound to CUDA device `cuda_device`.  The handle caches
 * task graphs keyed by problem shape (and SERINV_OPT).  Calls through one handle
 * execute on the device in call order, whatever streams they use (each call waits
 * for the previous one's work; the enqueue is serialised across host threads), so
 * a handle may be shared, at the price of that serialisation. */
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
 * Partition plan the partitioned solvers (serinv_pselinv, serinv_pselinv_nested)
 * actually use: serinv_plan_ends with the twisted last partition (the default,
 * reading R14), serinv_plan when SERINV_OPT=twist_last=0 selects the paper's
 * scheme.  Same arguments and errors as serinv_plan.
 */
int serinv_pselinv_plan(int64_t n, int P, double r, int64_t *starts);

/*
 * Small-block engine (b <= 64, a <= 16): the same partitioned method with nested
 * solving (Sec. 3, Alg. 3-6; Sec. 4.2) executed by two kernels
 * per nesting level in which one CTA carries a whole partition's chain with its
 * blocks resident in shared memory.  Ps[0..nlev-1]: partitions
 * per level (each >= 2; level k+1 works on the 2 Ps[k] - 2 block reduced system of
 * level k, twisted last partition, reading R14); the last reduced system is
 * solved as one chain (Alg. 1 + Alg. 2).  nlev = 0: the whole matrix as one chain;
 * nlev < 0: the library's plan (serinv_sb_auto_plan; Ps ignored).  A -> X in
 * place, log det in *d_logdet, *d_info as serinv_selinv (dpotrf row semantics).
 * Errors: SERINV_ERR_SHAPE (b > 64, a > 16, n < 1), SERINV_ERR_PLAN (a level has a
 * middle partition of < 2 blocks or an end partition of < 1), SERINV_ERR_WS.
 * The library caches the plan's index tables per shape in the handle.
 *   serinv_sb_auto_plan  writes min(levels, cap) entries, returns the level count
 *                        (>= 0) or a negative status.
 */
int serinv_sb_auto_plan(int64_t n, int64_t b, int64_t a, int *Ps, int cap);
int serinv_sb_ws(int64_t n, int64_t b, int64_t a, int nlev, const int *Ps, size_t *bytes);
int serinv_sb_selinv(serinv_handle_t h, const serinv_bta_t *A, int nlev, const int *Ps, void *d_ws,
                     size_t ws_bytes, int *d_info, double *d_logdet, void *stream);

/* ------------------------------------------------------------------------- */
/* Distributed method, one process per GPU (Sec. 3, Alg. 3-6; the    */
/* paper's exchange is NCCL).                                      */
/* ------------------------------------------------------------------------- */

/*
 * Communicator.  An NCCL communicator owned by the library; it carries the one
 * exchange step of the method (an all-gather of the per-partition records, which
 * replaces the paper's Reduce + Gather + Scatter).  NCCL is loaded at run
 * time (libnccl.so.2; the copy already mapped into the process is reused), so the
 * library itself does not depend on it.
 *   serinv_nccl_unique_id  on ONE rank: writes SERINV_NCCL_ID_BYTES bytes that the
 *                          caller broadcasts to every rank (e.g. torch.distributed).
 *   serinv_comm_init       collective over the P ranks (ncclCommInitRank) on CUDA
 *                          device `cuda_device`; id may be NULL only for P == 1 (no
 *                          NCCL: the all-gather of one rank is a device copy).
 *   serinv_comm_destroy    collective; frees the communicator.
 * Errors: SERINV_ERR_NCCL (NCCL missing or an NCCL call failed), -k argument k.
 */
#define SERINV_NCCL_ID_BYTES 128
typedef struct serinv_comm *serinv_comm_t;
int serinv_nccl_unique_id(unsigned char *id);
int serinv_comm_init(serinv_comm_t *comm, const unsigned char *id, int P, int rank, int cuda_device);
int serinv_comm_destroy(serinv_comm_t comm);

/*
 * Rank p of P owns the global blocks [start, start+count) (e.g. of serinv_plan /
 * serinv_plan_ends) and passes its LOCAL blocks:
 *     diag  [count][b][b], arrow [count][a][b],
 *     lower [count][b][b]  where lower[count-1] is the coupling A_{e,e-1} to the
 *                          next rank (P:378 assigns A_{i+1,i} to column i's
 *                          partition); the last rank passes count-1 lower blocks.
 *     tip   replicated: every rank passes the same A_{n,n} and receives X_{n,n}.
 * part = {P, rank, n_global, start, count}.  Each rank splits its blocks into Q
 * consecutive sub-partitions (intra-GPU partitioning; even sizes,
 * remainder to the earliest, each >= 2 blocks when Q > 1): the matrix has P*Q
 * partitions.  Q = 1 is the paper's one partition per process; Q must be the
 * same on every rank (serinv_dist_auto_q is the library's default).
 *
 *   serinv_ppobtaf   PARTIAL_POBTAF (partition 0) / PERMUTED_POBTAF (middle
 *                    partitions, Alg. 4 fill-in chain) / the twisted last partition
 *                    (reading R14) on the local blocks -- no communication -- then
 *                    packs the Q exchange records (boundary blocks, couplings, U_p,
 *                    the partial log det, this rank's info and the partition
 *                    bounds) and all-gathers the P*Q records over `comm` (one
 *                    ncclAllGather on `stream`).
 *   serinv_ppobtasi  assembles the reduced system A_r (2PQ-2 blocks; 2PQ-1 with
 *                    twist_last=0) from the gathered records in partition order --
 *                    bit-identical on every rank --, solves it redundantly
 *                    (POBTARSSI; nested partitioned solve when long, Sec. 4.2), then
 *                    PARTIAL_/PERMUTED_POBTASI on the local blocks: X in place,
 *                    X_{n,n} in tip, the global log det in *d_logdet.
 * d_ws: serinv_ppobtaf_ws(part, Q, ...) bytes, passed UNCHANGED from serinv_ppobtaf
 * to serinv_ppobtasi (it holds the fill-in factor blocks B_i, Alg. 6 l.3/l.11, and
 * the gathered records).  comm must have P == part->P and rank == part->rank.
 * Status: *d_info after serinv_ppobtasi is the SAME on every rank: the smallest
 * 1-based global row of a non-positive pivot any rank's PPOBTAF met; else the
 * reduced system's; else 0 (-1: watchdog).  The global log det is NaN when it is
 * non-zero.  The log det is only known after the reduced solve, so it is an
 * output of serinv_ppobtasi (SURVEY 8(b)'s sketch had it on ppobtaf).
 */
typedef struct {
  int P, rank;
  int64_t n_global, start, count;
} serinv_part_t;

int serinv_ppobtaf_ws(const serinv_part_t *part, int Q, int64_t b, int64_t a, size_t *bytes);
int serinv_ppobtaf(serinv_handle_t h, serinv_comm_t comm, const serinv_part_t *part, int Q,
                   const serinv_bta_t *A_local, void *d_ws, size_t ws_bytes, int *d_info, void *stream);
int serinv_ppobtasi(serinv_handle_t h, serinv_comm_t comm, const serinv_part_t *part, int Q,
                    const serinv_bta_t *L_local, void *d_ws, size_t ws_bytes, int *d_info, double *d_logdet,
                    void *stream);

/*
 * The same two phases with the exchange left to the caller (any transport):
 *   serinv_ppobtaf_q   factors and packs the Q records into d_sendbuf
 *                      (Q * serinv_exchange_bytes bytes);
 *   (caller)           all-gather of the P send buffers, rank order, into
 *                      d_recvbuf (P * Q records);
 *   serinv_ppobtasi_q  as serinv_ppobtasi, reading d_recvbuf.
 * d_ws: serinv_ppobtaf_q_ws bytes, passed unchanged between the two calls.
 * serinv_dist_auto_q: the library's default Q for a rank of `count` blocks of size
 * b (>= 1), or a negative status.  Errors as above, plus SERINV_ERR_PLAN if
 * Q < 1 or count < 2Q (Q > 1).
 */
int serinv_exchange_bytes(int64_t b, int64_t a, size_t *bytes);
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
