// serinv.cu -- C-ABI of libserinv.so (include/serinv.h).
//
// Each compute entry point: validate arguments, fetch (or build + upload) the
// cached task graph for the problem shape, reset its dependency counters, and
// launch ONE persistent executor kernel (exec.cu) on the caller's stream.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/serinv.h"
#include "comm.h"
#include "dist_meta.h"
#include "graph.h"
#include "task.h"

#include "exec.h"
#include "sb.h"

using namespace serinv;

namespace {

struct DevGraph {
  Graph g;                 // host copy (stats); task arrays freed after upload
  void *blob = nullptr;    // tasks | segs | waits | sigs | qlist | qoff
  int32_t *ctr = nullptr;  // nctr counters, nq queue claims, 2 + grid role table
  const Task *d_tasks = nullptr;
  const Seg *d_segs = nullptr;
  const Wait *d_waits = nullptr;
  const int32_t *d_sigs = nullptr;
  const int32_t *d_qlist = nullptr;
  const int32_t *d_qoff = nullptr;
  int nq = 1;
  int ncrit = 0, nurgent = 0;
  int64_t nctr_alloc = 0;
  int64_t ntasks = 0, nwaits = 0, nsigs = 0;
  ~DevGraph() {
    if (blob) cudaFree(blob);
    if (ctr) cudaFree(ctr);
  }
};

typedef std::tuple<int, int64_t, int64_t, int64_t, int, int64_t, int, int64_t, int64_t> GKey;
// graphs and workspace layouts depend on the build options (SERINV_OPT): part of every cache key
typedef std::pair<GKey, std::string> CKey;
inline std::string opt_string() {
  const char *e = getenv("SERINV_OPT");
  return e ? std::string(e) : std::string();
}

}  // namespace

namespace {
// a cached small-block engine plan and its device index table (serinv_sb_*)
struct SbEntry {
  sb::Plan pl;
  int64_t *d_tab = nullptr;
  ~SbEntry() {
    if (d_tab) cudaFree(d_tab);
  }
};
}  // namespace

struct serinv_ctx {
  std::map<std::vector<int64_t>, std::unique_ptr<SbEntry>> sb_cache;
  int device = 0;
  int sms = 0;
  int grid = 0;
  int smem = 0;
  int last_launches = 0;
  double *dummy = nullptr;  // logdet sink when the caller passes NULL
  int *dummy_info = nullptr;
  unsigned long long *trace = nullptr;  // optional per-task trace buffer (device)
  size_t trace_cap = 0;                 // records
  cudaStream_t s_in = nullptr, s_out = nullptr;  // streaming host IO copy streams
  sb::Side sb_side;                               // small-block engine's precompute side streams
  cudaEvent_t ev_start = nullptr, ev_in = nullptr, ev_out = nullptr;
  std::map<CKey, std::unique_ptr<DevGraph>> cache;
  std::mutex mu;
  // A handle's calls execute in call order, whatever streams they are enqueued on:
  // every call waits for the previous call's device work (ev_last) and the whole
  // enqueue sequence is one critical section.  The cached graphs' dependency
  // counters are reset by each call, so two calls must never overlap on the device.
  std::recursive_mutex call_mu;
  cudaEvent_t ev_last = nullptr;
  int depth = 0;
};

namespace {

inline bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

// One API call's critical section (see serinv_ctx::call_mu); nests.
struct CallGuard {
  serinv_handle_t h;
  cudaStream_t st;
  std::unique_lock<std::recursive_mutex> lk;
  CallGuard(serinv_handle_t h_, cudaStream_t st_) : h(h_), st(st_), lk(h_->call_mu) {
    if (h->depth++ == 0) {
      h->last_launches = 0;
      cudaStreamWaitEvent(st, h->ev_last, 0);
    }
  }
  ~CallGuard() {
    if (--h->depth == 0) cudaEventRecord(h->ev_last, st);
  }
};

int upload(DevGraph &dg, int grid) {
  Graph &g = dg.g;
  size_t bt = g.tasks.size() * sizeof(Task), bs = g.segs.size() * sizeof(Seg);
  size_t bw = g.waits.size() * sizeof(Wait), bg = g.sigs.size() * sizeof(int32_t);
  size_t bq = g.qlist.size() * sizeof(int32_t), bo = g.qoff.size() * sizeof(int32_t);
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  size_t total = up(bt) + up(bs) + up(bw) + up(bg) + up(bq) + up(bo) + 256;
  if (cudaMalloc(&dg.blob, total) != cudaSuccess) return SERINV_ERR_CUDA;
  char *base = (char *)dg.blob;
  size_t o = 0;
  auto put = [&](const void *src, size_t n) {
    char *dst = base + o;
    if (n) cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
    o += up(n);
    return (const void *)dst;
  };
  dg.d_tasks = (const Task *)put(g.tasks.data(), bt);
  dg.d_segs = (const Seg *)put(g.segs.data(), bs);
  dg.d_waits = (const Wait *)put(g.waits.data(), bw);
  dg.d_sigs = (const int32_t *)put(g.sigs.data(), bg);
  dg.d_qlist = (const int32_t *)put(g.qlist.data(), bq);
  dg.d_qoff = (const int32_t *)put(g.qoff.data(), bo);
  dg.nq = (int)g.qoff.size() - 1;
  dg.ncrit = g.ncrit;
  dg.nurgent = g.nurgent;
  dg.nctr_alloc = (int64_t)g.nctr + dg.nq + 2 + grid + 2;  // + done, info2 (exec.h)
  if (cudaMalloc(&dg.ctr, (size_t)dg.nctr_alloc * sizeof(int32_t)) != cudaSuccess) return SERINV_ERR_CUDA;
  dg.ntasks = (int64_t)g.tasks.size();
  dg.nwaits = (int64_t)g.waits.size();
  dg.nsigs = (int64_t)g.sigs.size();
  if (cudaGetLastError() != cudaSuccess) return SERINV_ERR_CUDA;
  // keep stats, drop the big host arrays
  std::vector<Task>().swap(g.tasks);
  std::vector<Seg>().swap(g.segs);
  std::vector<Wait>().swap(g.waits);
  std::vector<int32_t>().swap(g.sigs);
  std::vector<int32_t>().swap(g.qlist);
  return SERINV_OK;
}

int get_graph_impl(serinv_handle_t h, const GKey &key, DevGraph **out);
int get_graph(serinv_handle_t h, const GKey &key, DevGraph **out) {
  try {
    return get_graph_impl(h, key, out);
  } catch (const std::exception &e) {
    fprintf(stderr, "serinv: graph build failed: %s\n", e.what());
    return SERINV_ERR_SHAPE;
  }
}
int get_graph_impl(serinv_handle_t h, const GKey &key, DevGraph **out) {
  std::lock_guard<std::mutex> lk(h->mu);
  const CKey ckey(key, opt_string());
  auto it = h->cache.find(ckey);
  if (it != h->cache.end()) {
    *out = it->second.get();
    return SERINV_OK;
  }
  int kind = std::get<0>(key);
  int64_t n = std::get<1>(key), b = std::get<2>(key), a = std::get<3>(key);
  BuildOptions opt;
  opt.grid = h->grid;
  opt.apply_env();
  std::unique_ptr<DevGraph> dg(new DevGraph());
  if (kind == 9) {
    dg->g = build_gemm_bench((int)n, (int)b, (int)std::max<int64_t>(1, a), opt);
  } else if (kind <= 2 || kind == 6) {
    dg->g = build_sequential(kind, n, b, a, opt);
  } else if (kind == 3) {
    int P = std::get<4>(key);
    double r;
    int64_t rb = std::get<5>(key);
    memcpy(&r, &rb, 8);
    std::vector<int> Ps{P};
    int64_t more = std::get<7>(key);  // nested levels 1.. (16 bits each)
    for (int l = 1; l < (int)std::get<8>(key); ++l) Ps.push_back((int)((more >> (16 * (l - 1))) & 0xffff));
    dg->g = build_pselinv(n, b, a, Ps, r, opt);
  } else {
    int P = std::get<4>(key);
    int rank = std::get<6>(key);
    int64_t start = std::get<7>(key), count = std::get<8>(key);
    if (kind != 4 && kind != 5) return SERINV_ERR_SHAPE;
    int Q = (int)std::max<int64_t>(1, std::get<5>(key));
    dg->g = build_distributed(kind - 4, P, rank, n, start, count, b, a, opt, Q);
  }
  if (!dg->g.error.empty()) {
    fprintf(stderr, "serinv: graph build failed: %s\n", dg->g.error.c_str());
    return SERINV_ERR_SHAPE;
  }
  int rc = upload(*dg, h->grid);
  if (rc) return rc;
  *out = dg.get();
  h->cache[ckey] = std::move(dg);
  return SERINV_OK;
}

// reset: clear the graph's counters (and *d_info unless keep_info) before the kernel
int launch(serinv_handle_t h, DevGraph &dg, double *bufs[BUF_COUNT], int *d_info, cudaStream_t st,
           bool reset = true, bool keep_info = false) {
  CallGuard guard(h, st);
  if (reset) {
    if (cudaMemsetAsync(dg.ctr, 0, (size_t)dg.nctr_alloc * sizeof(int32_t), st) != cudaSuccess)
      return SERINV_ERR_CUDA;
    if (!keep_info && cudaMemsetAsync(d_info, 0, sizeof(int), st) != cudaSuccess) return SERINV_ERR_CUDA;
  }
  dev::Params p;
  p.tasks = dg.d_tasks;
  p.segs = dg.d_segs;
  p.waits = dg.d_waits;
  p.sigs = dg.d_sigs;
  p.ctr = dg.ctr;
  p.qclaim = dg.ctr + dg.g.nctr;
  p.qlist = dg.d_qlist;
  p.qoff = dg.d_qoff;
  p.nq = dg.nq;
  p.ncrit = dg.ncrit;
  p.nurgent = dg.nurgent;
  p.ntasks = (int)dg.ntasks;
  for (int i = 0; i < BUF_COUNT; ++i) p.bufs[i] = bufs[i];
  p.info = d_info;
  p.info2 = dg.ctr + dg.nctr_alloc - 1;
  p.done = dg.ctr + dg.nctr_alloc - 2;
  p.trace = (h->trace && (size_t)dg.ntasks <= h->trace_cap) ? h->trace : nullptr;
  serinv_exec_kernel<<<h->grid, 256, h->smem, st>>>(p);
  h->last_launches += 1;
  return cudaGetLastError() == cudaSuccess ? SERINV_OK : SERINV_ERR_CUDA;
}

int check_bta(const serinv_bta_t *A) {
  if (!A) return -2;
  if (A->n < 1 || A->b < 1 || A->a < 0) return SERINV_ERR_SHAPE;
  if (A->b > 64 * 4000 || A->a > 64 * 4000 || A->n >= (1 << 19)) return SERINV_ERR_SHAPE;
  if (!A->diag) return -2;
  if (A->n > 1 && !A->lower) return -2;
  if (A->a > 0 && (!A->arrow || !A->tip)) return -2;
  if (!aligned16(A->diag) || (A->lower && !aligned16(A->lower)) || (A->arrow && !aligned16(A->arrow)) ||
      (A->tip && !aligned16(A->tip)))
    return SERINV_ERR_ALIGN;
  return SERINV_OK;
}

int run_seq(serinv_handle_t h, int kind, const serinv_bta_t *A, void *ws, size_t ws_bytes, int *d_info,
            double *d_logdet, void *stream) {
  if (!h) return SERINV_ERR_HANDLE;
  int rc = check_bta(A);
  if (rc) return rc;
  if (!d_info) return -5;
  if (!ws || !aligned16(ws)) return SERINV_ERR_WS;
  if (cudaSetDevice(h->device) != cudaSuccess) return SERINV_ERR_CUDA;
  DevGraph *dg = nullptr;
  rc = get_graph(h, GKey(kind, A->n, A->b, A->a, 1, 0, 0, 0, 0), &dg);
  if (rc) return rc;
  if ((int64_t)ws_bytes < dg->g.ws_doubles * 8) return SERINV_ERR_WS;
  double *bufs[BUF_COUNT] = {A->diag, A->lower, A->arrow, A->tip, (double *)ws, nullptr, nullptr,
                             d_logdet ? d_logdet : h->dummy};
  return launch(h, *dg, bufs, d_info, (cudaStream_t)stream);
}

}  // namespace

extern "C" {

const char *serinv_version(void) { return "serinv-b200 0.1.0 sm_100a"; }

const char *serinv_status_string(int s) {
  switch (s) {
    case SERINV_OK: return "ok";
    case SERINV_ERR_CUDA: return "CUDA error";
    case SERINV_ERR_WS: return "workspace too small or misaligned";
    case SERINV_ERR_NCCL: return "NCCL error";
    case SERINV_ERR_HANDLE: return "invalid handle";
    case SERINV_ERR_SHAPE: return "unsupported shape";
    case SERINV_ERR_ALIGN: return "base pointer not 16-byte aligned";
    case SERINV_ERR_PLAN: return "infeasible partition plan";
    default: return s < 0 ? "invalid argument" : "unknown status";
  }
}

int serinv_create(serinv_handle_t *h, int cuda_device) {
  if (!h) return -1;
  *h = nullptr;
  if (cudaSetDevice(cuda_device) != cudaSuccess) return SERINV_ERR_CUDA;
  std::unique_ptr<serinv_ctx> c(new serinv_ctx());
  c->device = cuda_device;
  if (cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, cuda_device) != cudaSuccess)
    return SERINV_ERR_CUDA;
  c->smem = exec_smem_bytes();
  if (cudaFuncSetAttribute(serinv_exec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem) !=
      cudaSuccess)
    return SERINV_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, serinv_exec_kernel, 256, c->smem) != cudaSuccess ||
      per_sm < 1)
    return SERINV_ERR_CUDA;
  c->grid = c->sms * per_sm;
  if (cudaMalloc(&c->dummy, 256) != cudaSuccess) return SERINV_ERR_CUDA;
  c->dummy_info = (int *)(c->dummy + 16);
  if (cudaEventCreateWithFlags(&c->ev_last, cudaEventDisableTiming) != cudaSuccess) return SERINV_ERR_CUDA;
  *h = c.release();
  return SERINV_OK;
}

int serinv_destroy(serinv_handle_t h) {
  if (!h) return SERINV_ERR_HANDLE;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  h->cache.clear();
  h->sb_cache.clear();
  if (h->dummy) cudaFree(h->dummy);
  h->sb_side.destroy();
  if (h->s_in) cudaStreamDestroy(h->s_in);
  if (h->s_out) cudaStreamDestroy(h->s_out);
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_out) cudaEventDestroy(h->ev_out);
  if (h->ev_last) cudaEventDestroy(h->ev_last);
  delete h;
  return SERINV_OK;
}

static BuildOptions env_opt() {
  BuildOptions o;
  o.apply_env();
  return o;
}

int serinv_pobtaf_ws(int64_t n, int64_t b, int64_t a, size_t *bytes) {
  if (!bytes) return -4;
  if (n < 1 || b < 1 || a < 0) return SERINV_ERR_SHAPE;
  *bytes = (size_t)sequential_ws_bytes(0, n, b, a, env_opt());
  return SERINV_OK;
}
int serinv_pobtasi_ws(int64_t n, int64_t b, int64_t a, size_t *bytes) {
  if (!bytes) return -4;
  if (n < 1 || b < 1 || a < 0) return SERINV_ERR_SHAPE;
  *bytes = (size_t)sequential_ws_bytes(1, n, b, a, env_opt());
  return SERINV_OK;
}
int serinv_selinv_ws(int64_t n, int64_t b, int64_t a, size_t *bytes) {
  if (!bytes) return -4;
  if (n < 1 || b < 1 || a < 0) return SERINV_ERR_SHAPE;
  *bytes = (size_t)sequential_ws_bytes(2, n, b, a, env_opt());
  return SERINV_OK;
}

int serinv_prepare(serinv_handle_t h, int kind, int64_t n, int64_t b, int64_t a) {
  if (!h) return SERINV_ERR_HANDLE;
  if (kind < 0 || kind > 2) return -2;
  if (n < 1 || b < 1 || a < 0) return SERINV_ERR_SHAPE;
  cudaSetDevice(h->device);
  DevGraph *dg;
  return get_graph(h, GKey(kind, n, b, a, 1, 0, 0, 0, 0), &dg);
}

int serinv_pobtaf(serinv_handle_t h, const serinv_bta_t *A, void *d_ws, size_t ws_bytes, int *d_info,
                  double *d_logdet, void *stream) {
  return run_seq(h, 0, A, d_ws, ws_bytes, d_info, d_logdet, stream);
}

int serinv_pobtasi(serinv_handle_t h, const serinv_bta_t *L, void *d_ws, size_t ws_bytes, int *d_info,
                   void *stream) {
  return run_seq(h, 1, L, d_ws, ws_bytes, d_info, nullptr, stream);
}

int serinv_selinv(serinv_handle_t h, const serinv_bta_t *A, void *d_ws, size_t ws_bytes, int *d_info,
                  double *d_logdet, void *stream) {
  return run_seq(h, 2, A, d_ws, ws_bytes, d_info, d_logdet, stream);
}

int serinv_plan(int64_t n, int P, double r, int64_t *starts) {
  if (!starts) return -4;
  if (!(r > 0.0) || !std::isfinite(r)) return -3;
  std::vector<int64_t> s;
  if (!plan_partitions(n, P, r, s)) return SERINV_ERR_PLAN;
  for (size_t i = 0; i < s.size(); ++i) starts[i] = s[i];
  return SERINV_OK;
}

int serinv_pselinv_plan(int64_t n, int P, double r, int64_t *starts) {
  if (!starts) return -4;
  if (!(r > 0.0) || !std::isfinite(r)) return -3;
  std::vector<int64_t> s;
  if (!plan_partitions_for(n, P, r, env_opt().twist_last, s)) return SERINV_ERR_PLAN;
  for (size_t i = 0; i < s.size(); ++i) starts[i] = s[i];
  return SERINV_OK;
}

int serinv_plan_ends(int64_t n, int P, double r, int64_t *starts) {
  if (!starts) return -4;
  if (!(r > 0.0) || !std::isfinite(r)) return -3;
  std::vector<int64_t> s;
  if (!plan_partitions_ends(n, P, r, s)) return SERINV_ERR_PLAN;
  for (size_t i = 0; i < s.size(); ++i) starts[i] = s[i];
  return SERINV_OK;
}

// workspace queries of the partitioned graphs build the graph: memoise them
static std::mutex g_ws_mu;
static std::map<CKey, int64_t> g_ws_cache;

int serinv_pselinv_ws(int64_t n, int64_t b, int64_t a, int P, double r, size_t *bytes) {
  if (!bytes) return -6;
  if (n < 1 || b < 1 || a < 0) return SERINV_ERR_SHAPE;
  std::vector<int64_t> s;
  if (!(r > 0.0) || !std::isfinite(r) || !plan_partitions_for(n, P, r, env_opt().twist_last, s))
    return SERINV_ERR_PLAN;
  int64_t rb;
  memcpy(&rb, &r, 8);
  auto key = std::make_tuple(3, n, b, a, P, rb, 0, (int64_t)0, (int64_t)0);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  const CKey ckey(key, opt_string());
  auto it = g_ws_cache.find(ckey);
  int64_t v = it != g_ws_cache.end() ? it->second : (g_ws_cache[ckey] = pselinv_ws_bytes(n, b, a, P, r));
  if (v < 0) return SERINV_ERR_SHAPE;
  *bytes = (size_t)v;
  return SERINV_OK;
}

int serinv_pselinv(serinv_handle_t h, const serinv_bta_t *A, int P, double r, void *d_ws, size_t ws_bytes,
                   int *d_info, double *d_logdet, void *stream) {
  if (!h) return SERINV_ERR_HANDLE;
  int rc = check_bta(A);
  if (rc) return rc;
  if (!d_info) return -7;
  if (!d_ws || !aligned16(d_ws)) return SERINV_ERR_WS;
  std::vector<int64_t> s;
  if (!(r > 0.0) || !std::isfinite(r) || !plan_partitions_for(A->n, P, r, env_opt().twist_last, s))
    return SERINV_ERR_PLAN;
  if (P == 1) return run_seq(h, 2, A, d_ws, ws_bytes, d_info, d_logdet, stream);
  if (cudaSetDevice(h->device) != cudaSuccess) return SERINV_ERR_CUDA;
  int64_t rb;
  memcpy(&rb, &r, 8);
  DevGraph *dg = nullptr;
  rc = get_graph(h, GKey(3, A->n, A->b, A->a, P, rb, 0, 0, 0), &dg);
  if (rc) return rc;
  if ((int64_t)ws_bytes < dg->g.ws_doubles * 8) return SERINV_ERR_WS;
  double *bufs[BUF_COUNT] = {A->diag, A->lower, A->arrow, A->tip, (double *)d_ws, nullptr, nullptr,
                             d_logdet ? d_logdet : h->dummy};
  return launch(h, *dg, bufs, d_info, (cudaStream_t)stream);
}

// nested plan -> (feasible, key fields)
static int nested_key(int64_t n, int nlev, const int *Ps, double r, int64_t *more) {
  if (nlev < 1 || nlev > SERINV_MAX_LEVELS || !Ps) return SERINV_ERR_PLAN;
  int64_t m = n;
  *more = 0;
  BuildOptions opt;
  opt.apply_env();
  for (int l = 0; l < nlev; ++l) {
    std::vector<int64_t> s;
    if (Ps[l] < 1 || Ps[l] > 0xffff || (l > 0 && Ps[l] < 2) || !plan_partitions_for(m, Ps[l], r, opt.twist_last, s))
      return SERINV_ERR_PLAN;
    if (l > 0) *more |= (int64_t)Ps[l] << (16 * (l - 1));
    m = reduced_size(Ps[l], opt.twist_last);
  }
  if (nlev > 1 && Ps[0] < 2) return SERINV_ERR_PLAN;
  return SERINV_OK;
}

int serinv_auto_partitions(int64_t n, int64_t b, int *Ps, int cap) {
  if (n < 1 || b < 1 || !Ps || cap < 1) return SERINV_ERR_SHAPE;
  std::vector<int> v = auto_partitions(n, b);
  if ((int)v.size() > SERINV_MAX_LEVELS) v.resize(SERINV_MAX_LEVELS);
  for (int i = 0; i < (int)v.size() && i < cap; ++i) Ps[i] = v[i];
  return (int)v.size();
}

int serinv_pselinv_nested_ws(int64_t n, int64_t b, int64_t a, int nlev, const int *Ps, double r, size_t *bytes) {
  if (!bytes) return -7;
  if (n < 1 || b < 1 || a < 0) return SERINV_ERR_SHAPE;
  int64_t more;
  int rc = nested_key(n, nlev, Ps, r, &more);
  if (rc) return rc;
  if (nlev == 1) return serinv_pselinv_ws(n, b, a, Ps[0], r, bytes);
  int64_t rb;
  memcpy(&rb, &r, 8);
  auto key = std::make_tuple(3, n, b, a, Ps[0], rb, 0, more, (int64_t)nlev);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  const CKey ckey(key, opt_string());
  auto it = g_ws_cache.find(ckey);
  int64_t v = it != g_ws_cache.end()
                  ? it->second
                  : (g_ws_cache[ckey] = pselinv_ws_bytes(n, b, a, std::vector<int>(Ps, Ps + nlev), r));
  if (v < 0) return SERINV_ERR_SHAPE;
  *bytes = (size_t)v;
  return SERINV_OK;
}

int serinv_pselinv_nested(serinv_handle_t h, const serinv_bta_t *A, int nlev, const int *Ps, double r, void *d_ws,
                          size_t ws_bytes, int *d_info, double *d_logdet, void *stream) {
  if (!h) return SERINV_ERR_HANDLE;
  int rc = check_bta(A);
  if (rc) return rc;
  if (!d_info) return -8;
  if (!d_ws || !aligned16(d_ws)) return SERINV_ERR_WS;
  int64_t more;
  rc = nested_key(A->n, nlev, Ps, r, &more);
  if (rc) return rc;
  if (nlev == 1) return serinv_pselinv(h, A, Ps[0], r, d_ws, ws_bytes, d_info, d_logdet, stream);
  if (cudaSetDevice(h->device) != cudaSuccess) return SERINV_ERR_CUDA;
  int64_t rb;
  memcpy(&rb, &r, 8);
  DevGraph *dg = nullptr;
  rc = get_graph(h, GKey(3, A->n, A->b, A->a, Ps[0], rb, 0, more, nlev), &dg);
  if (rc) return rc;
  if ((int64_t)ws_bytes < dg->g.ws_doubles * 8) return SERINV_ERR_WS;
  double *bufs[BUF_COUNT] = {A->diag, A->lower, A->arrow, A->tip, (double *)d_ws, nullptr, nullptr,
                             d_logdet ? d_logdet : h->dummy};
  return launch(h, *dg, bufs, d_info, (cudaStream_t)stream);
}

int serinv_exchange_bytes(int64_t b, int64_t a, size_t *bytes) {
  if (!bytes) return -3;
  if (b < 1 || a < 0) return SERINV_ERR_SHAPE;
  *bytes = (size_t)exchange_doubles(b, a) * 8;
  return SERINV_OK;
}

static int check_part(const serinv_part_t *pt, int Q = 1) {
  if (!pt) return -1;
  if (Q < 1 || Q > 65536) return SERINV_ERR_PLAN;
  if (pt->P < 1 || pt->rank < 0 || pt->rank >= pt->P || pt->count < 1 || pt->start < 0 ||
      pt->start + pt->count > pt->n_global)
    return SERINV_ERR_PLAN;
  if (pt->P > 1 && pt->rank > 0 && pt->count < 2) return SERINV_ERR_PLAN;
  if (Q > 1 && pt->count < 2 * (int64_t)Q) return SERINV_ERR_PLAN;
  return SERINV_OK;
}

int serinv_ppobtaf_q_ws(const serinv_part_t *part, int Q, int64_t b, int64_t a, size_t *bytes) {
  int rc = check_part(part, Q);
  if (rc) return rc;
  if (!bytes) return -5;
  if (b < 1 || a < 0) return SERINV_ERR_SHAPE;
  auto key = std::make_tuple(4, part->n_global, b, a, part->P, (int64_t)Q, part->rank, part->start, part->count);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  const CKey ckey(key, opt_string());
  auto it = g_ws_cache.find(ckey);
  int64_t v = it != g_ws_cache.end()
                  ? it->second
                  : (g_ws_cache[ckey] = distributed_ws_bytes(part->P, part->rank, part->n_global, part->start,
                                                            part->count, b, a, Q));
  if (v < 0) return SERINV_ERR_SHAPE;
  *bytes = (size_t)v;
  return SERINV_OK;
}

int serinv_dist_auto_q(int64_t count, int64_t b) {
  if (count < 1 || b < 1) return SERINV_ERR_SHAPE;
  std::vector<int> v = auto_partitions(count, b);
  int Q = v.empty() ? 1 : v[0];
  // chain-bound blocks (b <= 1024, where the single-device selinv twists): two
  // chains per rank (measured with tools/scaling_sim.py, C2 at P = 4 / 8:
  // E_weak 40.6 / 38.5 % at Q = 1 -> 46.9 / 44.8 % at Q = 2); b = 2048 (C3) is
  // FP64-bound and keeps Q = 1
  if (Q == 1 && b <= 1024 && count >= 64) Q = 2;
  while (Q > 1 && count < 2 * (int64_t)Q) --Q;
  return Q;
}

}  // extern "C"

namespace {
// Status handling of the distributed path (dist_meta.h): PPOBTAF's info and the
// partition's [s, e) go into the rank's records before the exchange; PPOBTASI
// starts from the smallest row any rank reported and decodes reduced-system rows
// of other ranks' partitions afterwards -- every rank ends with the same status.
__global__ void dist_meta_kernel(double *send, int Q, int64_t recsz, int64_t mo, const int *info, int64_t start,
                                 int64_t count) {
  const int v = *(volatile const int *)info;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Q; q += gridDim.x * blockDim.x)
    meta_write(send, Q, recsz, mo, v, start, count, q);
}
__global__ void dist_combine_kernel(const double *recv, int nrec, int64_t recsz, int64_t mo, int *info) {
  if (threadIdx.x == 0) *info = meta_combine_info(recv, nrec, recsz, mo);
}
__global__ void dist_final_kernel(const double *recv, int nrec, int64_t recsz, int64_t mo, int64_t b, int *info) {
  if (threadIdx.x == 0) *info = meta_final_info(*info, recv, nrec, recsz, mo, b);
}
}  // namespace

static int run_dist(serinv_handle_t h, int phase, const serinv_part_t *part, int Q, const serinv_bta_t *A,
                    void *d_ws, size_t ws_bytes, void *ext0, const void *ext1, int *d_info, double *d_logdet,
                    void *stream) {
  if (!h) return SERINV_ERR_HANDLE;
  int rc = check_part(part, Q);
  if (rc) return rc;
  if (!A || !A->diag || A->b < 1 || A->a < 0) return -3;
  if (A->n != part->count) return -3;
  if (A->a > 0 && (!A->arrow || !A->tip)) return -3;
  if (part->count > 1 && !A->lower) return -3;
  if (!d_ws || !aligned16(d_ws)) return SERINV_ERR_WS;
  if (!d_info) return -8;
  if (cudaSetDevice(h->device) != cudaSuccess) return SERINV_ERR_CUDA;
  DevGraph *dg = nullptr;
  rc = get_graph(h, GKey(4 + phase, part->n_global, A->b, A->a, part->P, (int64_t)Q, part->rank, part->start,
                        part->count),
                 &dg);
  if (rc) return rc;
  if ((int64_t)ws_bytes < dg->g.ws_doubles * 8) return SERINV_ERR_WS;
  double *bufs[BUF_COUNT] = {A->diag, A->lower, A->arrow, A->tip, (double *)d_ws, (double *)ext0,
                             (double *)ext1, d_logdet ? d_logdet : h->dummy};
  cudaStream_t st = (cudaStream_t)stream;
  CallGuard guard(h, st);
  const int64_t recsz = exchange_doubles(A->b, A->a), mo = exchange_meta_offset(A->b, A->a);
  if (phase == 0) {
    rc = launch(h, *dg, bufs, d_info, st);
    if (rc) return rc;
    dist_meta_kernel<<<(Q + 127) / 128, 128, 0, st>>>((double *)ext0, Q, recsz, mo, d_info, part->start,
                                                      part->count);
    h->last_launches += 1;
    return cudaGetLastError() == cudaSuccess ? SERINV_OK : SERINV_ERR_CUDA;
  }
  dist_combine_kernel<<<1, 32, 0, st>>>((const double *)ext1, part->P * Q, recsz, mo, d_info);
  rc = launch(h, *dg, bufs, d_info, st, true, /*keep_info=*/true);
  if (rc) return rc;
  dist_final_kernel<<<1, 32, 0, st>>>((const double *)ext1, part->P * Q, recsz, mo, A->b, d_info);
  h->last_launches += 2;
  return cudaGetLastError() == cudaSuccess ? SERINV_OK : SERINV_ERR_CUDA;
}

// comm entry points: workspace = graph workspace | send records | recv records
static int64_t up256(int64_t x) { return (x + 255) / 256 * 256; }

extern "C" {

int serinv_ppobtaf_q(serinv_handle_t h, const serinv_part_t *part, int Q, const serinv_bta_t *A_local, void *d_ws,
                     size_t ws_bytes, void *d_sendbuf, int *d_info, void *stream) {
  if (!d_sendbuf) return -7;
  return run_dist(h, 0, part, Q, A_local, d_ws, ws_bytes, d_sendbuf, nullptr, d_info, nullptr, stream);
}

int serinv_ppobtasi_q(serinv_handle_t h, const serinv_part_t *part, int Q, const serinv_bta_t *L_local, void *d_ws,
                      size_t ws_bytes, const void *d_recvbuf, int *d_info, double *d_logdet, void *stream) {
  if (!d_recvbuf) return -7;
  return run_dist(h, 1, part, Q, L_local, d_ws, ws_bytes, nullptr, d_recvbuf, d_info, d_logdet, stream);
}

int serinv_ppobtaf_ws(const serinv_part_t *part, int Q, int64_t b, int64_t a, size_t *bytes) {
  if (!bytes) return -5;
  size_t g = 0;
  int rc = serinv_ppobtaf_q_ws(part, Q, b, a, &g);
  if (rc) return rc;
  const int64_t rec = exchange_doubles(b, a) * 8;
  *bytes = (size_t)(up256((int64_t)g) + up256((int64_t)Q * rec) + up256((int64_t)part->P * Q * rec));
  return SERINV_OK;
}

static int comm_split_ws(serinv_comm_t comm, const serinv_part_t *part, int Q, const serinv_bta_t *A, void *d_ws,
                         size_t ws_bytes, size_t *gbytes, double **send, double **recv) {
  if (!comm) return -2;
  if (!part || !A) return -3;
  if (comm_size(comm) != part->P || comm_rank(comm) != part->rank) return -3;
  size_t total = 0;
  int rc = serinv_ppobtaf_ws(part, Q, A->b, A->a, &total);
  if (rc) return rc;
  if (!d_ws || ws_bytes < total) return SERINV_ERR_WS;
  size_t g = 0;
  serinv_ppobtaf_q_ws(part, Q, A->b, A->a, &g);
  const int64_t rec = exchange_doubles(A->b, A->a) * 8;
  *gbytes = (size_t)up256((int64_t)g);
  *send = (double *)((char *)d_ws + *gbytes);
  *recv = (double *)((char *)*send + up256((int64_t)Q * rec));
  return SERINV_OK;
}

int serinv_ppobtaf(serinv_handle_t h, serinv_comm_t comm, const serinv_part_t *part, int Q,
                   const serinv_bta_t *A_local, void *d_ws, size_t ws_bytes, int *d_info, void *stream) {
  if (!h) return SERINV_ERR_HANDLE;
  size_t g = 0;
  double *send = nullptr, *recv = nullptr;
  int rc = comm_split_ws(comm, part, Q, A_local, d_ws, ws_bytes, &g, &send, &recv);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  CallGuard guard(h, st);
  rc = run_dist(h, 0, part, Q, A_local, d_ws, g, send, nullptr, d_info, nullptr, stream);
  if (rc) return rc;
  return comm_allgather_f64(comm, send, recv, (size_t)Q * exchange_doubles(A_local->b, A_local->a), st);
}

int serinv_ppobtasi(serinv_handle_t h, serinv_comm_t comm, const serinv_part_t *part, int Q,
                    const serinv_bta_t *L_local, void *d_ws, size_t ws_bytes, int *d_info, double *d_logdet,
                    void *stream) {
  if (!h) return SERINV_ERR_HANDLE;
  size_t g = 0;
  double *send = nullptr, *recv = nullptr;
  int rc = comm_split_ws(comm, part, Q, L_local, d_ws, ws_bytes, &g, &send, &recv);
  if (rc) return rc;
  return run_dist(h, 1, part, Q, L_local, d_ws, g, nullptr, recv, d_info, d_logdet, stream);
}

int serinv_graph_stats(serinv_handle_t h, int kind, int64_t n, int64_t b, int64_t a, int P, double r,
                       serinv_graph_stats_t *out) {
  if (!h) return SERINV_ERR_HANDLE;
  if (!out) return -8;
  if (kind < 0 || kind > 3) return -2;
  int64_t rb = 0;
  if (kind == 3) memcpy(&rb, &r, 8);
  cudaSetDevice(h->device);
  DevGraph *dg = nullptr;
  int rc = get_graph(h, GKey(kind, n, b, a, kind == 3 ? P : 1, rb, 0, 0, 0), &dg);
  if (rc) return rc;
  out->tasks = dg->ntasks;
  out->counters = dg->g.nctr;
  out->flops = dg->g.flops;
  out->grid = h->grid;
  out->tile = SERINV_TILE;
  return SERINV_OK;
}

// Diagnostic: the claimed task list of a cached sequential / partitioned graph.
// rec (ntasks x 10 int32): type, flags, m, n, wait0, nwait, nlate, sig0, nsig, queue;
// waits (nwaits int32 counter ids), sigs (nsigs int32).  Sizes via *nw, *ns.
int serinv_graph_dump(serinv_handle_t h, int kind, int64_t n, int64_t b, int64_t a, int P, double r, int32_t *rec,
                      int32_t *waits, int64_t *nw, int32_t *sigs, int64_t *ns) {
  if (!h) return SERINV_ERR_HANDLE;
  if (kind < 0 || kind > 3) return -2;
  int64_t rb = 0;
  if (kind == 3) memcpy(&rb, &r, 8);
  cudaSetDevice(h->device);
  DevGraph *dg = nullptr;
  int rc = get_graph(h, GKey(kind, n, b, a, kind == 3 ? P : 1, rb, 0, 0, 0), &dg);
  if (rc) return rc;
  // the host arrays were dropped after upload: read the device copies back
  const Graph &g = dg->g;
  if (nw) *nw = dg->nwaits;
  if (ns) *ns = dg->nsigs;
  if (rec) {
    std::vector<Task> tasks(dg->ntasks);
    std::vector<int32_t> ql(dg->ntasks);
    cudaMemcpy(tasks.data(), dg->d_tasks, tasks.size() * sizeof(Task), cudaMemcpyDeviceToHost);
    cudaMemcpy(ql.data(), dg->d_qlist, ql.size() * sizeof(int32_t), cudaMemcpyDeviceToHost);
    std::vector<int32_t> q(tasks.size(), 0);
    for (size_t qq = 0; qq + 1 < g.qoff.size(); ++qq)
      for (int32_t k = g.qoff[qq]; k < g.qoff[qq + 1]; ++k) q[ql[k]] = (int32_t)qq;
    for (size_t t = 0; t < tasks.size(); ++t) {
      const Task &T = tasks[t];
      int32_t *o = rec + 10 * t;
      o[0] = T.type; o[1] = T.flags; o[2] = T.m; o[3] = T.n; o[4] = T.wait0; o[5] = T.nwait;
      o[6] = T.nlate; o[7] = T.sig0; o[8] = T.nsig; o[9] = q[t];
    }
  }
  if (waits) {
    std::vector<Wait> w(dg->nwaits);
    cudaMemcpy(w.data(), dg->d_waits, w.size() * sizeof(Wait), cudaMemcpyDeviceToHost);
    for (size_t k = 0; k < w.size(); ++k) waits[k] = w[k].ctr;
  }
  if (sigs) cudaMemcpy(sigs, dg->d_sigs, dg->nsigs * sizeof(int32_t), cudaMemcpyDeviceToHost);
  return SERINV_OK;
}

int serinv_graph_stats_nested(serinv_handle_t h, int64_t n, int64_t b, int64_t a, int nlev, const int *Ps, double r,
                              serinv_graph_stats_t *out) {
  if (!h) return SERINV_ERR_HANDLE;
  if (!out) return -8;
  int64_t more;
  int rc = nested_key(n, nlev, Ps, r, &more);
  if (rc) return rc;
  int64_t rb = 0;
  memcpy(&rb, &r, 8);
  cudaSetDevice(h->device);
  DevGraph *dg = nullptr;
  rc = get_graph(h, nlev == 1 ? GKey(3, n, b, a, Ps[0], rb, 0, 0, 0) : GKey(3, n, b, a, Ps[0], rb, 0, more, nlev),
                 &dg);
  if (rc) return rc;
  out->tasks = dg->ntasks;
  out->counters = dg->g.nctr;
  out->flops = dg->g.flops;
  out->grid = h->grid;
  out->tile = SERINV_TILE;
  return SERINV_OK;
}

// Driver stream memory operations, resolved through the runtime (no link-time
// dependency on libcuda, so the library also loads on machines without a GPU).
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_writeValue32 p_writeValue32 = nullptr;
static PFN_waitValue32 p_waitValue32 = nullptr;
static bool load_stream_memops() {
  if (p_writeValue32 && p_waitValue32) return true;
  void *f1 = nullptr, *f2 = nullptr;
  cudaDriverEntryPointQueryResult q1, q2;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f1, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPoint("cuStreamWaitValue32", &f2, cudaEnableDefault, &q2) != cudaSuccess || !f1 || !f2)
    return false;
  p_writeValue32 = (PFN_writeValue32)f1;
  p_waitValue32 = (PFN_waitValue32)f2;
  return true;
}

// Streaming host IO: H2D of the input blocks and D2H of the selected inverse
// overlap the factorisation / inversion.  The H2D stream copies chunks of blocks
// in order and bumps the graph's arrival counter (cuStreamWriteValue32); the
// D2H stream waits on each node's final-X counter (cuStreamWaitValue32) and
// copies the node's blocks back while the kernel works on earlier blocks.
// Streaming host IO for the twisted selinv graph: units stream in from both ends
// (top units 0..m on the arrival counter arr_ctr, bottom units n-1..m+1 on
// arr_ctr2; bottom unit j carries lower[j-1]) and each node's outputs stream out
// as soon as its final-X counter completes (the graph's fin list, in completion
// order: tip, m, then both chains outwards), in contiguous per-side chunks.
static int selinv_host_twisted(serinv_handle_t h, DevGraph &dg, const serinv_bta_t *A_host, const serinv_bta_t *X_host,
                               const serinv_bta_t *A_dev, void *d_ws, int *d_info, double *d_logdet, cudaStream_t st,
                               int64_t chunk) {
  const int64_t n = A_dev->n, b = A_dev->b, a = A_dev->a, m = dg.g.twist_m;
  const size_t bb = (size_t)b * b, ab = (size_t)a * b;
  auto cp = [&](double *dst, const double *src, size_t doubles, cudaMemcpyKind k, cudaStream_t s) {
    return doubles ? cudaMemcpyAsync(dst, src, doubles * 8, k, s) == cudaSuccess : true;
  };
  // blocks [j0, j1) of one side with their lower blocks (top: lower[j], bottom: lower[j-1])
  auto unit_range = [&](const serinv_bta_t *dst, const serinv_bta_t *src, int64_t j0, int64_t j1, bool top,
                        cudaMemcpyKind k, cudaStream_t s) {
    if (j1 <= j0) return true;
    bool ok = cp(dst->diag + j0 * bb, src->diag + j0 * bb, (j1 - j0) * bb, k, s);
    if (a > 0) ok = ok && cp(dst->arrow + j0 * ab, src->arrow + j0 * ab, (j1 - j0) * ab, k, s);
    const int64_t l0 = top ? j0 : j0 - 1, l1 = top ? std::min(j1, m) : j1 - 1;
    if (l1 > l0) ok = ok && cp(dst->lower + l0 * bb, src->lower + l0 * bb, (l1 - l0) * bb, k, s);
    return ok;
  };
  CUdeviceptr arr = (CUdeviceptr)(dg.ctr + dg.g.arr_ctr), arr2 = (CUdeviceptr)(dg.ctr + dg.g.arr_ctr2);
  const int64_t nbot = n - 1 - m;
  for (int64_t t = 0, s = 0; t <= m || s < nbot;) {
    if (t <= m) {
      const int64_t t1 = std::min(m + 1, t + chunk);
      if (!unit_range(A_dev, A_host, t, t1, true, cudaMemcpyHostToDevice, h->s_in) ||
          p_writeValue32((CUstream)h->s_in, arr, (cuuint32_t)t1, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
        return SERINV_ERR_CUDA;
      t = t1;
    }
    if (s < nbot) {
      const int64_t s1 = std::min(nbot, s + chunk);
      if (!unit_range(A_dev, A_host, n - s1, n - s, false, cudaMemcpyHostToDevice, h->s_in) ||
          p_writeValue32((CUstream)h->s_in, arr2, (cuuint32_t)s1, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
        return SERINV_ERR_CUDA;
      s = s1;
    }
  }
  double *bufs[BUF_COUNT] = {A_dev->diag, A_dev->lower, A_dev->arrow, A_dev->tip, (double *)d_ws, nullptr, nullptr,
                             d_logdet ? d_logdet : h->dummy};
  int rc = launch(h, dg, bufs, d_info, st, false);
  if (rc) return rc;
  // D2H in completion order; per side a pending contiguous range, flushed per chunk
  int64_t tlo = -1, thi = -1, blo = -1, bhi = -1;  // top [tlo, thi), bottom [blo, bhi)
  auto flush_top = [&]() {
    bool ok = unit_range(X_host, A_dev, tlo, thi, true, cudaMemcpyDeviceToHost, h->s_out);
    tlo = thi = -1;
    return ok;
  };
  auto flush_bot = [&]() {
    bool ok = unit_range(X_host, A_dev, blo, bhi, false, cudaMemcpyDeviceToHost, h->s_out);
    blo = bhi = -1;
    return ok;
  };
  for (size_t k = 0; k < dg.g.fin.size(); ++k) {
    const Wait &w = dg.g.fin[k];
    if (p_waitValue32((CUstream)h->s_out, (CUdeviceptr)(dg.ctr + w.ctr), (cuuint32_t)w.target,
                      CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return SERINV_ERR_CUDA;
    const int64_t i = dg.g.fin_blk[k];
    if (i < 0) {
      if (!cp(X_host->tip, A_dev->tip, (size_t)a * a, cudaMemcpyDeviceToHost, h->s_out)) return SERINV_ERR_CUDA;
    } else if (i <= m) {  // top side finishes m, m-1, ..., 0
      if (tlo < 0) tlo = thi = i + 1;
      tlo = i;
      if (thi - tlo >= chunk && !flush_top()) return SERINV_ERR_CUDA;
    } else {  // bottom side finishes m+1, m+2, ..., n-1
      if (blo < 0) blo = bhi = i;
      bhi = i + 1;
      if (bhi - blo >= chunk && !flush_bot()) return SERINV_ERR_CUDA;
    }
  }
  if ((tlo >= 0 && !flush_top()) || (blo >= 0 && !flush_bot())) return SERINV_ERR_CUDA;
  if (cudaEventRecord(h->ev_in, h->s_in) != cudaSuccess || cudaEventRecord(h->ev_out, h->s_out) != cudaSuccess ||
      cudaStreamWaitEvent(st, h->ev_in, 0) != cudaSuccess || cudaStreamWaitEvent(st, h->ev_out, 0) != cudaSuccess)
    return SERINV_ERR_CUDA;
  return SERINV_OK;
}

int serinv_selinv_host(serinv_handle_t h, const serinv_bta_t *A_host, const serinv_bta_t *X_host,
                       const serinv_bta_t *A_dev, void *d_ws, size_t ws_bytes, int *d_info, double *d_logdet,
                       void *stream) {
  if (!h) return SERINV_ERR_HANDLE;
  int rc = check_bta(A_dev);
  if (rc) return rc;
  if (!A_host || !X_host) return -2;
  if (A_host->n != A_dev->n || A_host->b != A_dev->b || A_host->a != A_dev->a || X_host->n != A_dev->n ||
      X_host->b != A_dev->b || X_host->a != A_dev->a)
    return -2;
  if (!A_host->diag || !X_host->diag || (A_dev->n > 1 && (!A_host->lower || !X_host->lower)) ||
      (A_dev->a > 0 && (!A_host->arrow || !A_host->tip || !X_host->arrow || !X_host->tip)))
    return -2;
  if (!d_info) return -7;
  if (!d_ws || !aligned16(d_ws)) return SERINV_ERR_WS;
  if (cudaSetDevice(h->device) != cudaSuccess) return SERINV_ERR_CUDA;
  if (!load_stream_memops()) return SERINV_ERR_CUDA;
  DevGraph *dg = nullptr;
  const int64_t n = A_dev->n, b = A_dev->b, a = A_dev->a;
  rc = get_graph(h, GKey(6, n, b, a, 1, 0, 0, 0, 0), &dg);
  if (rc) return rc;
  if ((int64_t)ws_bytes < dg->g.ws_doubles * 8) return SERINV_ERR_WS;
  if (!h->s_in) {
    if (cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming) != cudaSuccess)
      return SERINV_ERR_CUDA;
  }
  cudaStream_t st = (cudaStream_t)stream;
  CallGuard guard(h, st);
  if (cudaMemsetAsync(dg->ctr, 0, (size_t)dg->nctr_alloc * sizeof(int32_t), st) != cudaSuccess ||
      cudaMemsetAsync(d_info, 0, sizeof(int), st) != cudaSuccess || cudaEventRecord(h->ev_start, st) != cudaSuccess)
    return SERINV_ERR_CUDA;
  if (cudaStreamWaitEvent(h->s_in, h->ev_start, 0) != cudaSuccess ||
      cudaStreamWaitEvent(h->s_out, h->ev_start, 0) != cudaSuccess)
    return SERINV_ERR_CUDA;
  const size_t bb = (size_t)b * b * 8, ab = (size_t)a * b * 8;
  // chunks of ~8 MB of blocks
  const int64_t per_block = (int64_t)(2 * bb + ab);
  const int64_t chunk = std::max<int64_t>(1, (8ll << 20) / std::max<int64_t>(per_block, 1));
  // ---- H2D (in order), arrival counter = number of blocks present
  auto h2d = [&](void *dst, const void *src, size_t bytes) {
    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->s_in) : cudaSuccess;
  };
  auto d2h = [&](void *dst, const void *src, size_t bytes) {
    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->s_out) : cudaSuccess;
  };
  CUdeviceptr arr = (CUdeviceptr)(dg->ctr + dg->g.arr_ctr);
  if (a > 0 && h2d(A_dev->tip, A_host->tip, (size_t)a * a * 8) != cudaSuccess) return SERINV_ERR_CUDA;
  if (dg->g.twist_m >= 0) return selinv_host_twisted(h, *dg, A_host, X_host, A_dev, d_ws, d_info, d_logdet, st, chunk);
  for (int64_t i0 = 0; i0 < n; i0 += chunk) {
    const int64_t i1 = std::min(n, i0 + chunk);
    if (h2d(A_dev->diag + i0 * b * b, A_host->diag + i0 * b * b, (size_t)(i1 - i0) * bb) != cudaSuccess)
      return SERINV_ERR_CUDA;
    const int64_t l1 = std::min(i1, n - 1);
    if (l1 > i0 && h2d(A_dev->lower + i0 * b * b, A_host->lower + i0 * b * b, (size_t)(l1 - i0) * bb) != cudaSuccess)
      return SERINV_ERR_CUDA;
    if (a > 0 && h2d(A_dev->arrow + i0 * a * b, A_host->arrow + i0 * a * b, (size_t)(i1 - i0) * ab) != cudaSuccess)
      return SERINV_ERR_CUDA;
    if (p_writeValue32((CUstream)h->s_in, arr, (cuuint32_t)i1, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      return SERINV_ERR_CUDA;
  }
  // ---- the kernel (counters already reset on `st`)
  double *bufs[BUF_COUNT] = {A_dev->diag, A_dev->lower, A_dev->arrow, A_dev->tip, (double *)d_ws, nullptr, nullptr,
                             d_logdet ? d_logdet : h->dummy};
  rc = launch(h, *dg, bufs, d_info, st, false);
  if (rc) return rc;
  // ---- D2H as nodes finish: fin[] = [tip (if a > 0), block n-1, ..., block 0]
  auto waitv = [&](const Wait &w) {
    return p_waitValue32((CUstream)h->s_out, (CUdeviceptr)(dg->ctr + w.ctr), (cuuint32_t)w.target,
                               CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS;
  };
  size_t k = 0;
  if (a > 0) {
    if (!waitv(dg->g.fin[k++])) return SERINV_ERR_CUDA;
    if (d2h(X_host->tip, A_dev->tip, (size_t)a * a * 8) != cudaSuccess) return SERINV_ERR_CUDA;
  }
  for (int64_t i1 = n; i1 > 0; i1 -= chunk) {
    const int64_t i0 = std::max<int64_t>(0, i1 - chunk);
    for (int64_t i = i1 - 1; i >= i0; --i)
      if (!waitv(dg->g.fin[k++])) return SERINV_ERR_CUDA;
    if (d2h(X_host->diag + i0 * b * b, A_dev->diag + i0 * b * b, (size_t)(i1 - i0) * bb) != cudaSuccess)
      return SERINV_ERR_CUDA;
    const int64_t l1 = std::min(i1, n - 1);
    if (l1 > i0 && d2h(X_host->lower + i0 * b * b, A_dev->lower + i0 * b * b, (size_t)(l1 - i0) * bb) != cudaSuccess)
      return SERINV_ERR_CUDA;
    if (a > 0 && d2h(X_host->arrow + i0 * a * b, A_dev->arrow + i0 * a * b, (size_t)(i1 - i0) * ab) != cudaSuccess)
      return SERINV_ERR_CUDA;
  }
  if (cudaEventRecord(h->ev_in, h->s_in) != cudaSuccess || cudaEventRecord(h->ev_out, h->s_out) != cudaSuccess ||
      cudaStreamWaitEvent(st, h->ev_in, 0) != cudaSuccess || cudaStreamWaitEvent(st, h->ev_out, 0) != cudaSuccess)
    return SERINV_ERR_CUDA;
  return SERINV_OK;
}

int serinv_bench_gemm(serinv_handle_t h, int ntasks, int k, int nseg, void *d_ws, size_t ws_bytes, void *stream) {
  if (!h) return SERINV_ERR_HANDLE;
  if (ntasks < 1 || k < 1 || nseg < 1 || k % nseg) return -2;
  if (!d_ws || !aligned16(d_ws)) return SERINV_ERR_WS;
  if (cudaSetDevice(h->device) != cudaSuccess) return SERINV_ERR_CUDA;
  DevGraph *dg = nullptr;
  int rc = get_graph(h, GKey(9, ntasks, k, nseg, 1, 0, 0, 0, 0), &dg);
  if (rc) return rc;
  if ((int64_t)ws_bytes < dg->g.ws_doubles * 8) return SERINV_ERR_WS;
  double *bufs[BUF_COUNT] = {nullptr, nullptr, nullptr, nullptr, (double *)d_ws, nullptr, nullptr, h->dummy};
  return launch(h, *dg, bufs, h->dummy_info, (cudaStream_t)stream);
}

int serinv_set_trace(serinv_handle_t h, void *d_trace, size_t bytes) {
  if (!h) return SERINV_ERR_HANDLE;
  if (d_trace && ((uintptr_t)d_trace & 7)) return SERINV_ERR_ALIGN;
  h->trace = (unsigned long long *)d_trace;
  h->trace_cap = d_trace ? bytes / 96 : 0;  // 4 + 8 u64 per task
  return SERINV_OK;
}

// ---------------------------------------------------------------------------
// small-block engine (sb.cu)
// ---------------------------------------------------------------------------
static int sb_levels(int64_t n, int64_t b, int64_t a, int nlev, const int *Ps, std::vector<int> &v) {
  if (n < 1 || b < 1 || a < 0) return SERINV_ERR_SHAPE;
  if (b > sb::kMaxB || a > sb::kMaxA) return SERINV_ERR_SHAPE;
  if (nlev < 0) {
    v = sb::auto_plan(n, b, 148);  // B200: 148 SMs (fixed, so the ws query needs no device)
  } else {
    if (nlev > 0 && !Ps) return -5;
    v.assign(Ps, Ps + nlev);
  }
  return SERINV_OK;
}

int serinv_sb_auto_plan(int64_t n, int64_t b, int64_t a, int *Ps, int cap) {
  if (!Ps || cap < 0) return -4;
  std::vector<int> v;
  int rc = sb_levels(n, b, a, -1, nullptr, v);
  if (rc) return -rc;
  for (int i = 0; i < (int)v.size() && i < cap; ++i) Ps[i] = v[i];
  return (int)v.size();
}

int serinv_sb_ws(int64_t n, int64_t b, int64_t a, int nlev, const int *Ps, size_t *bytes) {
  if (!bytes) return -6;
  std::vector<int> v;
  int rc = sb_levels(n, b, a, nlev, Ps, v);
  if (rc) return rc;
  sb::Plan pl;
  if (!sb::make_plan(n, b, a, v, pl)) return SERINV_ERR_PLAN;
  *bytes = (size_t)pl.ws_doubles * 8;
  return SERINV_OK;
}

int serinv_sb_selinv(serinv_handle_t h, const serinv_bta_t *A, int nlev, const int *Ps, void *d_ws, size_t ws_bytes,
                     int *d_info, double *d_logdet, void *stream) {
  if (!h) return SERINV_ERR_HANDLE;
  int rc = check_bta(A);
  if (rc) return rc;
  if (!d_info) return -8;
  if (!d_ws || !aligned16(d_ws)) return SERINV_ERR_WS;
  if (cudaSetDevice(h->device) != cudaSuccess) return SERINV_ERR_CUDA;
  std::vector<int> v;
  rc = sb_levels(A->n, A->b, A->a, nlev, Ps, v);
  if (rc) return rc;
  std::vector<int64_t> key{A->n, A->b, A->a};
  key.insert(key.end(), v.begin(), v.end());
  SbEntry *e = nullptr;
  {
    std::lock_guard<std::mutex> lk(h->mu);
    auto it = h->sb_cache.find(key);
    if (it == h->sb_cache.end()) {
      std::unique_ptr<SbEntry> ne(new SbEntry);
      if (!sb::make_plan(A->n, A->b, A->a, v, ne->pl)) return SERINV_ERR_PLAN;
      const std::vector<int64_t> tab = sb::plan_tables(ne->pl);
      if (cudaMalloc(&ne->d_tab, tab.size() * sizeof(int64_t)) != cudaSuccess ||
          cudaMemcpy(ne->d_tab, tab.data(), tab.size() * sizeof(int64_t), cudaMemcpyHostToDevice) != cudaSuccess)
        return SERINV_ERR_CUDA;
      it = h->sb_cache.emplace(key, std::move(ne)).first;
    }
    e = it->second.get();
  }
  if ((int64_t)ws_bytes < e->pl.ws_doubles * 8) return SERINV_ERR_WS;
  cudaStream_t st = (cudaStream_t)stream;
  CallGuard guard(h, st);
  int nl = 0;
  if (sb::run(e->pl, e->d_tab, A->diag, A->lower, A->arrow, A->tip, (double *)d_ws, d_info,
              d_logdet ? d_logdet : h->dummy, h->sms, st, &nl, &h->sb_side,
              (h->trace && h->trace_cap * 96 >= (size_t)sb::kTraceWords * 8) ? h->trace : nullptr))
    return SERINV_ERR_CUDA;
  h->last_launches += nl;
  return SERINV_OK;
}

int serinv_last_launches(serinv_handle_t h, int *launches) {
  if (!h || !launches) return SERINV_ERR_HANDLE;
  *launches = h->last_launches;
  return SERINV_OK;
}

}  // extern "C"
