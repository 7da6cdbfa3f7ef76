// graph.h -- host-side task-graph builder and scheduler (C++17, no CUDA).
//
// The block algorithms of PAPER.md (Alg. 1 POBTAF, Alg. 2 POBTASI, Alg. 3-6
// PPOBTAF / PPOBTASI, Sec. 3.3 POBTARSSI) are lowered to a DAG of 64 x 64 tile
// tasks (task.h).  The lowering is exact block algebra: a block Cholesky at
// block size b equals the tiled Cholesky at tile size 64 on the same pattern,
// and the Takahashi recurrence of Alg. 2 / Alg. 6 is evaluated with the
// inverted diagonal blocks W_X = L_XX^{-1} ("invert L_ii once", P:567-569,
// P:649):  X_{Y,X} = -sum_Z X_{Y,Z} (L_{Z,X} W_X),
//          X_{X,X} = W_X^T W_X - sum_Y X_{Y,X}^T (L_{Y,X} W_X).
// The scheduler orders tasks by a list-scheduling simulation with critical-
// path (bottom-level) priority so the persistent executor claims the
// latency-critical POTRF/TRSM chain first and fills the idle SMs with the
// bulk updates and the inversion precompute.
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "task.h"

namespace serinv {

constexpr int TILE = SERINV_TILE;

// Finalised graph: flat arrays ready for upload.
struct Graph {
  std::vector<Task> tasks;
  std::vector<Seg> segs;
  std::vector<Wait> waits;
  std::vector<int32_t> sigs;
  int32_t nctr = 0;
  double flops = 0.0;        // executed FP64 flops (model)
  int grid = 0;              // worker count the schedule was simulated for
  int64_t ws_doubles = 0;    // workspace doubles used (excluding counters)
  int64_t nslots = 0;        // logdet slots
  double sim_ns = 0.0;       // simulated makespan of the schedule (ns)
  // claim queues: queue 0 = bulk, queues 1..nq-1 = critical chains (one CTA each,
  // alone on its SM).  qlist holds task indices, queue q = qlist[qoff[q] .. qoff[q+1]).
  std::vector<int32_t> qlist, qoff;
  // streaming IO (kind 6): blocks-arrived counter written by the H2D stream, and per
  // node (fin[k].target = #producers) the counter of its final-X tasks, in the order
  // the nodes finish (tip first, then blocks n-1 .. 0)
  int32_t arr_ctr = -1;
  std::vector<Wait> fin;
  std::vector<int32_t> fin_blk;   // block of fin[k] (-1: the tip)
  // twisted streaming IO: arr_ctr counts top units (blocks 0, 1, ..., m) and
  // arr_ctr2 bottom units (blocks n-1, n-2, ..., m+1; unit j holds diag[j],
  // arrow[j] and lower[j-1]); twist_m = m (-1: one-sided, units in block order)
  int32_t arr_ctr2 = -1;
  int64_t twist_m = -1;
  int ncrit = 0;     // queues 1..ncrit: one CTA each, alone on its SM
  int nurgent = 0;   // queue ncrit+1 (if any): served by nurgent CTAs (near-critical tasks)
  std::string error;         // non-empty if building failed
};

// A storage place for a block: base Loc (top-left) of a rows x cols block.
struct BlkRef {
  Loc base{};
  int rows = 0, cols = 0;
  bool zero_init = false;    // starts as fill-in zero (beta = 0 on first write)
  bool valid = false;
};

// Generic description of one elimination problem (one partition, the whole
// matrix, or a reduced system) on top of which factor / inverse tasks are built.
struct Problem {
  // nodes in elimination order
  std::vector<int> size;          // node size (b or a)
  std::vector<char> elim;         // factorised here
  std::vector<int64_t> rowbase;   // global row of the node's first row (info)
  std::vector<std::vector<int>> rows;     // rows[X]: nodes Y > X with blk(Y,X) nonzero (elim X)
  std::map<std::pair<int, int>, BlkRef> blk;   // (Y, X), Y >= X
  std::vector<char> accum;        // targets in this node's column receive whole-node update groups
  // workspace placements (filled by the builder)
  std::vector<Loc> W;             // W_X = L_XX^{-1}
  std::vector<Loc> Lam;           // Lambda_X = W_X^T W_X
  std::map<std::pair<int, int>, Loc> Lchk;     // Lchk(Z,X) = L_{Z,X} W_X
  std::vector<int64_t> slot;      // logdet slot base per node (-1: none)
  int queue = 0;                  // claim queue of this problem's POTRF chain (0 = bulk)
  int queue2 = 0;                 // claim queue of the chain's sub-diagonal TRSMs (split chain)
  // per-node overrides of (queue, queue2) (empty: every node uses queue / queue2);
  // a twisted problem runs two independent chains, each on its own critical CTAs
  std::vector<int> nqueue, nqueue2;
  int q1(int X) const { return nqueue.empty() ? queue : nqueue[X]; }
  int q2(int X) const { return nqueue2.empty() ? queue2 : nqueue2[X]; }
};

struct BuildOptions {
  int grid = 296;          // persistent CTAs (for the simulated schedule)
  int update_group = 4;    // tile columns per chained update task (regular targets)
  bool schedule = true;
  bool critical_queues = true;  // dedicated CTAs for the POTRF chains
  bool fuse_trsm = false;       // fuse the sub-diagonal TRSM into each POTRF task
  bool fuse_trsm3 = false;      // ... and the second sub-diagonal TRSM (late inputs)
  bool split_chain = true;      // POTRF chain on one critical CTA, its TRSMs on a second one
  bool chain_syrk = true;       // the sub-diagonal TRSM also applies its SYRK to the next diagonal tile
  int urgent_ctas = 0;          // CTAs serving the near-critical queue (0: no urgent queue)
  int si_split = 320;           // K per partial GEMM of the Takahashi tile tasks (0 = no split)
  bool rts1_chain = false;      // the second sub-diagonal TRSM also on the chain's TRSM queue
  int max_crit = 16;            // partitioned solves: exclusive-SM chains only if 2P <= max_crit
  int twist_min_n = 4;          // selinv: two-sided (twisted) elimination if n >= twist_min_n (0: never)
  bool twist_last = true;       // partitioned solves: the last partition eliminates bottom-up (no fill-in)
  bool chol8 = true;
  bool early_sig = true;
  bool carry_chain = true;      // chain TRSM+SYRK on the POTRF's CTA, operands carried in shared memory
  int carry_min_b = 2048;       // ... for nodes of at least this size
  bool chain_step = false;      // POTRF + sub-diagonal TRSM + next-tile SYRK as ONE carried task (all sizes;
                                // measured slower: E's last update becomes a bulk round trip on the chain)        // POTRF publishes W before its log-det partial and L (TF_EARLY_SIG)            // POTRF tasks: 8 x 8-block warp-pipelined Cholesky (else 16 x 16 leaves)
  int wide_min_wave = 512;      // 128 x 64 tasks for inversion waves of >= this many tiles (0: never)
  int twist_max_b = 1024;       // ... and b <= twist_max_b (larger blocks: the one-sided chain hides under the work)
  bool twist_reduced = true;    // reduced systems (>= 4 blocks) solved in the twisted order (two chains)
  int dist_len = 0;             // distributed reduced system: nested partitions of ~dist_len blocks (0: measured default)
  double cost_gemm_fixed = 2500.0;  // scheduler cost model: GEMM task fixed ns
  double cost_potrf = 19000.0;      // ... POTRF tile task ns
  double cost_gflops = 85.0;        // ... bulk GEMM GFLOP/s per CTA
  bool cost_set = false;            // cost model set through SERINV_OPT (else per block size, build_sequential)
  int split_last = 0;           // carried chain: the newest N updates of the tiles it awaits as single-column tasks (measured: no gain at C3)
  // overrides from the environment (SERINV_OPT="key=value,..."), for tuning runs
  void apply_env();
};

// Sequential problems (whole matrix).  kind: 0 = pobtaf, 1 = pobtasi, 2 = selinv,
// 6 = selinv with streaming host IO (external arrival counter + per-node final counters).
Graph build_sequential(int kind, int64_t n, int64_t b, int64_t a, const BuildOptions &opt);

// Workspace bytes for the sequential kinds (doubles region + counters).
int64_t sequential_ws_bytes(int kind, int64_t n, int64_t b, int64_t a, const BuildOptions &opt = BuildOptions());

// In-process partitioned pipeline on one device (PPOBTAF -> POBTARSSI -> PPOBTASI).
Graph build_pselinv(int64_t n, int64_t b, int64_t a, int P, double r, const BuildOptions &opt);
int64_t pselinv_ws_bytes(int64_t n, int64_t b, int64_t a, int P, double r);
// nested partitioned solve: Ps[0] partitions of the matrix, Ps[1] of its reduced
// system, ... (the last reduced system is solved as one chain)
Graph build_pselinv(int64_t n, int64_t b, int64_t a, const std::vector<int> &Ps, double r, const BuildOptions &opt);
int64_t pselinv_ws_bytes(int64_t n, int64_t b, int64_t a, const std::vector<int> &Ps, double r);
// default one-device nesting plan for n blocks of size b ({1} = sequential)
std::vector<int> auto_partitions(int64_t n, int64_t b);

// Distributed per-rank graphs.  phase 0 = ppobtaf (+ pack into EXT0 send buffer),
// phase 1 = ppobtasi (assemble from EXT1 recv buffer, POBTARSSI, backward).
// Q = sub-partitions per rank (intra-GPU partitioning of the rank's blocks).
Graph build_distributed(int phase, int P, int rank, int64_t n_global, int64_t start,
                        int64_t count, int64_t b, int64_t a, const BuildOptions &opt, int Q = 1);
int64_t distributed_ws_bytes(int P, int rank, int64_t n_global, int64_t start, int64_t count,
                             int64_t b, int64_t a, int Q = 1);
int64_t exchange_doubles(int64_t b, int64_t a);
// offset of the record's meta tail (dist_meta.h: log det partial, info, s, e)
int64_t exchange_meta_offset(int64_t b, int64_t a);

// Diagnostic: independent tile GEMMs (engine throughput).
Graph build_gemm_bench(int ntasks, int k, int nseg, const BuildOptions &opt);

// Blocks of the reduced system of P partitions: 2P-1 (paper), 2P-2 with the
// twisted last partition (reading R14).
int reduced_size(int P, bool twisted_last);

// Partition plan (reading R6).  Returns false if infeasible.
bool plan_partitions(int64_t n, int P, double r, std::vector<int64_t> &starts);
// Twisted-scheme plan (reading R14): first and last partition r x a middle one.
bool plan_partitions_ends(int64_t n, int P, double r, std::vector<int64_t> &starts);
// The plan the partitioned solvers actually use: plan_partitions_ends with the
// twisted last partition (default), else the paper's plan_partitions.
bool plan_partitions_for(int64_t n, int P, double r, bool twist_last, std::vector<int64_t> &starts);

// Bytes reserved at the end of the workspace for counters (+1 claim counter).
int64_t counter_bytes(int32_t nctr);

}  // namespace serinv
