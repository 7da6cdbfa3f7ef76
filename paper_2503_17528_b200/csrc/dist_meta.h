// dist_meta.h -- metadata carried in the exchange records of the distributed path
// (PPOBTAF -> all-gather -> PPOBTASI, Alg. 3 l.8 P:413, Sec. 3.3), shared by
// the library's small device kernels (serinv.cu) and the host interpreter test tool.
//
// Record tail (doubles, after the blocks and U_p; XRec::ld() in graph.cpp):
//   ld()      the partition's partial log det (NaN if its factorisation failed)
//   ld() + 1  info of the rank's PPOBTAF (dpotrf semantics: 1-based global row, 0 ok, -1 watchdog)
//   ld() + 2  first global block s of the partition
//   ld() + 3  end e of the partition (exclusive)
// With them every rank derives the SAME status after the exchange: the smallest
// positive row any rank's PPOBTAF reported, else the reduced system's (whose rows
// of other ranks' partitions are labelled kEncRow + node * b at graph build time,
// because a rank does not know the other ranks' sub-partition starts, and decoded
// here from the records), else this rank's backward pass.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define SERINV_HD __host__ __device__
#else
#define SERINV_HD
#endif

namespace serinv {

constexpr int32_t kEncRow = 1 << 30;  // encoded reduced-system row base (unknown partition start)
constexpr int kMetaDoubles = 4;       // ld, info, s, e

// start of sub-partition q of a rank owning [start, start+count) split into Q
// (even sizes, remainder to the earliest; graph.cpp split_rank)
SERINV_HD inline int64_t meta_sub_start(int64_t start, int64_t count, int Q, int q) {
  const int64_t base = count / Q, rem = count % Q;
  return start + q * base + (q < rem ? q : rem);
}

// after PPOBTAF: info, s, e into each of the rank's Q records
SERINV_HD inline void meta_write(double *send, int Q, int64_t recsz, int64_t ld, int info, int64_t start,
                                 int64_t count, int q) {
  double *r = send + q * recsz + ld;
  r[1] = (double)info;
  r[2] = (double)meta_sub_start(start, count, Q, q);
  r[3] = (double)meta_sub_start(start, count, Q, q + 1);
}

// before PPOBTASI: the status all ranks' PPOBTAF reported (watchdog first, then the smallest row)
SERINV_HD inline int meta_combine_info(const double *recv, int nrec, int64_t recsz, int64_t ld) {
  int best = 0;
  for (int k = 0; k < nrec; ++k) {
    const int v = (int)recv[k * recsz + ld + 1];
    if (v < 0) return v;
    if (v > 0 && (best == 0 || v < best)) best = v;
  }
  return best;
}

// after PPOBTASI: the final status -- the records' status if any rank's PPOBTAF failed
// (what the reduced solve then reports is a consequence), else the decoded own status
SERINV_HD inline int meta_final_info(int info, const double *recv, int nrec, int64_t recsz, int64_t ld, int64_t b);

// after PPOBTASI: decode an encoded reduced-system row (node k of A_r: 0 = last block
// of partition 0, 2p-1 = first block of partition p, 2p = last block of partition p)
SERINV_HD inline int meta_decode_info(int info, const double *recv, int64_t recsz, int64_t ld, int64_t b) {
  if (info < kEncRow) return info;
  const int64_t e = (int64_t)info - kEncRow - 1, k = e / b, piv = e % b;
  int64_t blk;
  if (k == 0) {
    blk = (int64_t)recv[ld + 3] - 1;
  } else {
    const int64_t p = (k + 1) / 2;
    blk = (k & 1) ? (int64_t)recv[p * recsz + ld + 2] : (int64_t)recv[p * recsz + ld + 3] - 1;
  }
  return (int)(blk * b + piv + 1);
}

SERINV_HD inline int meta_final_info(int info, const double *recv, int nrec, int64_t recsz, int64_t ld, int64_t b) {
  const int comb = meta_combine_info(recv, nrec, recsz, ld);
  return comb ? comb : meta_decode_info(info, recv, recsz, ld, b);
}

}  // namespace serinv
