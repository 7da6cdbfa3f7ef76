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
  int32_t *ctr;    // dependency counters (zeroed before each launch)
  int32_t *claim;  // next-task claim counter (zeroed before each launch)
  int ntasks;
  double *bufs[BUF_COUNT];
  int *info;
};
}  // namespace dev
int exec_smem_bytes();
}  // namespace serinv

extern "C" __global__ void serinv_exec_kernel(serinv::dev::Params p);
