// exec.h -- launch interface of the persistent executor (exec.cu).
#pragma once
#include <stdint.h>

#include "task.h"

namespace serinv {
namespace dev {
struct Params {
  const Task *tasks;
  const Seg *segs;
  const Wait *waits;
  const int32_t *sigs;
  int32_t *ctr;          // dependency counters (zeroed before each launch)
  int32_t *qclaim;       // [nq] claim counters, then [2 + grid] role table (zeroed before each launch)
  const int32_t *qlist;  // task indices per queue
  const int32_t *qoff;   // [nq + 1]
  int nq;                // queue 0 = bulk, 1..ncrit = critical chains, ncrit+1 = urgent (if nq > ncrit+1)
  int ncrit;             // critical queues (one CTA each, exclusive SM)
  int nurgent;           // CTAs serving the urgent queue
  int ntasks;
  double *bufs[BUF_COUNT];
  int *info;             // first genuine failure (finite pivot <= 0 / zero diagonal), dpotrf row
  int *info2;            // failures with a NaN pivot (propagated, or NaN input): merged by the last CTA out
  int *done;             // CTAs that finished (zeroed before each launch)
  unsigned long long *trace;  // optional: 4 x u64 per task {claim, start, end, meta}
};
}  // namespace dev
int exec_smem_bytes();
}  // namespace serinv

extern "C" __global__ void serinv_exec_kernel(serinv::dev::Params p);
