// sb.h -- the small-block engine (sb.cu): the partitioned method of PAPER.md
// Sec. 3 (PPOBTAF -> POBTARSSI -> PPOBTASI, Alg. 3-6) with nested solving
// (Sec. 4.2) for blocks of b <= 64 and arrowheads of a <= 16, run as
// two kernels per nesting level in which ONE CTA carries a whole partition's
// dependent chain with its working blocks resident in shared memory.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace serinv {
namespace sb {

constexpr int kMaxB = 64;
constexpr int kMaxA = 16;

// One nesting level: the BTA matrix it works on (level 0 = the user's arrays,
// deeper levels = the reduced systems in workspace) and its partition plan.
struct Level {
  int64_t n = 0;            // blocks
  int P = 1;                // partitions (1: the last level, solved as one chain with the tip)
  const int64_t *starts;    // device [P + 1]
  const int64_t *grow;      // device [n]: 0-based global row of node i's first row (info)
  double *D, *Lo, *Ar;      // the level's blocks (b x b, b x b, a x b; row-major, contiguous)
  double *Bf;               // fill-in factor blocks L_{f,i} of middle partitions, by block index
  double *U;                // [P][a][a] tip updates of the partitions
  double *ldp;              // [P] log-det partials
  double *Dn, *Lon, *Arn;   // the next level's blocks (the reduced system, P >= 2)
  int *done;                // CTA exit counter (zeroed per call)
};

struct Params {
  Level L;
  double *tip;              // a x a, in place: A_nn (+ sum of U over the levels) -> X_nn
  int b, a;
  int *info;                // dpotrf-style 1-based global row of the first non-positive pivot
  int *info2;               // the same for NaN pivots (merged into info only if it stays 0)
  int lvl;                  // level index (trace)
  unsigned long long *trace;  // optional phase timestamps of CTA 0 (tools/sb_trace.py)
  double *logdet;           // written by the last level's factor kernel
  const double *ldp_all;    // every level's partials (fixed summation order)
  int n_ldp;
  int64_t tip_row;          // 0-based global row of the tip's first row
};

// Host-side plan of all levels for (n, b, a) and the level partition counts Ps
// (Ps.size() levels of partitioned elimination, then the last reduced system as
// one chain).  Workspace layout in doubles; device arrays filled by setup().
struct Plan {
  int64_t n, b, a;
  std::vector<int> Ps;
  std::vector<std::vector<int64_t>> starts;  // per partitioned level
  std::vector<std::vector<int64_t>> grow;    // per level (incl. the last)
  std::vector<int64_t> nlev;                 // blocks per level (incl. the last)
  // workspace offsets (doubles)
  std::vector<int64_t> off_D, off_Lo, off_Ar, off_Bf, off_U, off_ldp;  // workspace (doubles)
  std::vector<int64_t> off_starts, off_grow;                          // index table (int64)
  int64_t off_ctr = 0;   // int counters (as doubles) [levels]
  int64_t ws_doubles = 0;
};

// Build the plan; false if a level is infeasible (partitions of < 2 blocks in the middle,
// < 1 at the ends) or b / a unsupported.
// Side streams of the level-0 precompute (sb_pre_kernel) and their fork / join events;
// owned by the caller's handle (one call at a time per handle), created on first use.
struct Side {
  cudaStream_t s = nullptr, s2 = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, fork2 = nullptr, join2 = nullptr;
  bool ensure();   // create on the current device; false on a CUDA error
  void destroy();
};

bool make_plan(int64_t n, int64_t b, int64_t a, const std::vector<int> &Ps, Plan &pl);
// Default nesting for one B200 (148 SMs).
std::vector<int> auto_plan(int64_t n, int64_t b, int sms);
// Host image of the plan's index tables (starts / grow), copied once into the workspace.
std::vector<int64_t> plan_tables(const Plan &pl);
// Enqueue the whole solve on `st`: memset of counters + info, factor kernels level
// 0..L, inverse kernels level L..0.  d_tab: device copy of plan_tables(pl).
int run(const Plan &pl, const int64_t *d_tab, double *diag, double *lower, double *arrow, double *tip, double *ws,
        int *d_info, double *d_logdet, int sms, cudaStream_t st, int *launches, Side *side,
        unsigned long long *trace = nullptr);
// trace layout: [level < 16][kernel 0 factor / 1 inverse][step < 128][8 phase stamps] (u64 ns)
constexpr int kTraceWords = 16 * 2 * 128 * 8;

}  // namespace sb
}  // namespace serinv
