// comm.h -- the library's NCCL communicator (serinv_comm_t, include/serinv.h).
// NCCL is resolved at run time (dlopen of libnccl.so.2, reusing the copy the
// process already loaded, e.g. torch's), so libserinv.so loads without NCCL and
// only the distributed entry points that take a communicator need it.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/serinv.h"

namespace serinv {
// all-gather of `count` doubles per rank (rank order) on `stream`; SERINV_OK or SERINV_ERR_NCCL
int comm_allgather_f64(serinv_comm_t c, const double *send, double *recv, size_t count, cudaStream_t stream);
int comm_size(serinv_comm_t c);
int comm_rank(serinv_comm_t c);
int comm_device(serinv_comm_t c);
}  // namespace serinv
