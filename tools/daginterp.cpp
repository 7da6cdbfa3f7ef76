// daginterp.cpp -- TEST TOOL: executes a serinv task graph on the host, task by
// task in emission order, with plain loops.  Used only by tests/test_graph_host.py
// to validate the graph builder (dependencies, locations, task semantics) on a
// machine without a GPU.  It is not linked into libserinv.so and is never on
// the product path.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>

#include "../paper_2503_17528_b200/csrc/graph.h"
#include "../paper_2503_17528_b200/csrc/dist_meta.h"

using namespace serinv;

namespace {

struct Ctx {
  double *bufs[BUF_COUNT];
  std::vector<int32_t> ctr;
  int info = 0;   // first genuine failure (finite pivot <= 0, zero / infinite diagonal)
  int info2 = 0;  // failures with a NaN pivot (propagated from an earlier failure or NaN input)
};
inline void rec_info(int &slot, int v) {
  if (!slot || v < slot) slot = v;
}

inline double *ptr(Ctx &c, const Loc &l) { return c.bufs[l.buf] + l.off; }
inline double get(Ctx &c, const Loc &l, int r, int k) { return ptr(c, l)[(int64_t)r * l.ld + k]; }
// op(X)[i][j]
inline double opget(Ctx &c, const Loc &l, int trans, int i, int j) {
  return trans ? get(c, l, j, i) : get(c, l, i, j);
}

int run_tasks(const Graph &g, Ctx &c);
// as the device launch: NaN-pivot failures count only when there is no genuine one
int run(const Graph &g, Ctx &c) {
  c.info2 = 0;
  const int rc = run_tasks(g, c);
  if (!c.info) c.info = c.info2;
  return rc;
}

int run_tasks(const Graph &g, Ctx &c) {
  c.ctr.assign(g.nctr, 0);
  if (g.arr_ctr >= 0) c.ctr[g.arr_ctr] = 1 << 30;  // streaming IO: every block has arrived
  if (g.arr_ctr2 >= 0) c.ctr[g.arr_ctr2] = 1 << 30;
  std::vector<double> acc(2 * SERINV_TILE * SERINV_TILE), tmp(2 * SERINV_TILE * SERINV_TILE);  // wide GEMM: m <= 128
  for (size_t t = 0; t < g.tasks.size(); ++t) {
    const Task &T = g.tasks[t];
    for (int w = 0; w < T.nwait; ++w) {
      const Wait &W = g.waits[T.wait0 + w];
      if (c.ctr[W.ctr] < W.target) {
        fprintf(stderr, "task %zu (type %d): wait on counter %d not satisfied (%d < %d)\n", t, T.type, W.ctr,
                c.ctr[W.ctr], W.target);
        return -1;
      }
    }
    const int m = T.m, n = T.n;
    if (m > SERINV_TILE && (T.type != TK_GEMM || m > 2 * SERINV_TILE || n > SERINV_TILE || T.nlate ||
                            (T.flags & (TF_SYRK3 | TF_ZERO_MIRROR)))) {
      fprintf(stderr, "task %zu: unsupported wide task (type %d, %d x %d, flags %d)\n", t, T.type, m, n, T.flags);
      return -4;
    }
    if (getenv("DAG_DUMP"))
      fprintf(stderr, "t%zu type %d m %d n %d out(%d,%lld) c0(%d,%lld) nseg %d nseg1 %d alpha %g beta %g flags %d out3(%d,%lld) m3 %d beta3 %g\n", t, T.type, m, n,
              T.out.buf, (long long)T.out.off, T.c0.buf, (long long)T.c0.off, T.nseg, T.nseg1, T.alpha, T.beta, T.flags,
              T.out3.buf, (long long)T.out3.off, T.m3, T.beta3);
    auto A_ = [&](int i, int j) -> double & { return acc[i * SERINV_TILE + j]; };
    if (T.type == TK_GEMM || T.type == TK_POTRF) {
      int ns = (T.type == TK_POTRF) ? T.nseg1 : T.nseg;
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
          double s = 0;
          for (int si = 0; si < ns; ++si) {
            const Seg &S = g.segs[T.seg0 + si];
            for (int k = 0; k < S.k; ++k) s += opget(c, S.A, S.ta, i, k) * opget(c, S.B, S.tb, k, j);
          }
          double v = T.alpha * s;
          if (T.beta != 0.0) v += T.beta * get(c, T.c0, i, j);
          A_(i, j) = v;
        }
    }
    if (T.type == TK_GEMM) {
      if (T.flags & TF_POST) {
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < n; ++j) {
            double s = 0;
            for (int k = 0; k < n; ++k) s += A_(i, k) * opget(c, T.r, (T.flags & TF_POST_T) ? 1 : 0, k, j);
            tmp[i * SERINV_TILE + j] = s;
          }
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < n; ++j) A_(i, j) = tmp[i * SERINV_TILE + j];
      }
      double *o = ptr(c, T.out);
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) o[(int64_t)i * T.out.ld + j] = A_(i, j);
      if (T.flags & TF_SYRK3) {
        double *o3 = ptr(c, T.out3);
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < m; ++j) {
            double s = 0;
            for (int k = 0; k < n; ++k) s += A_(i, k) * A_(j, k);
            o3[(int64_t)i * T.out3.ld + j] -= s;
          }
      }
      if (T.flags & TF_MIRROR) {
        double *o2 = ptr(c, T.out2);
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < n; ++j) o2[(int64_t)j * T.out2.ld + i] = A_(i, j);
      }
      if (T.flags & TF_ZERO_MIRROR) {
        double *o2 = ptr(c, T.out2);
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < n; ++j) o2[(int64_t)j * T.out2.ld + i] = 0.0;
      }
    } else if (T.type == TK_POTRF || T.type == TK_TRTRI) {
      if (T.type == TK_TRTRI) {
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < m; ++j) A_(i, j) = j <= i ? get(c, T.c0, i, j) : 0.0;
      } else {
        // Cholesky (lower) of acc
        double ls = 0;
        for (int j = 0; j < m; ++j) {
          double d = A_(j, j);
          for (int k = 0; k < j; ++k) d -= A_(j, k) * A_(j, k);
          if (!(d > 0.0)) {
            rec_info(std::isnan(d) ? c.info2 : c.info, T.aux1 + j + 1);
            d = NAN;
          }
          d = std::sqrt(d);
          A_(j, j) = d;
          for (int i = j + 1; i < m; ++i) {
            double s = A_(i, j);
            for (int k = 0; k < j; ++k) s -= A_(i, k) * A_(j, k);
            A_(i, j) = s / d;
          }
          ls += std::log(d);
        }
        for (int i = 0; i < m; ++i)
          for (int j = i + 1; j < m; ++j) A_(i, j) = 0.0;
        if (T.r.buf >= 0 && T.aux0 >= 0) *ptr(c, T.r) = ls;
        double *o = ptr(c, T.out);
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < m; ++j) o[(int64_t)i * T.out.ld + j] = A_(i, j);
      }
      // W = L^{-1}
      std::vector<double> W(m * m, 0.0);
      for (int j = 0; j < m; ++j) {
        W[j * m + j] = 1.0 / A_(j, j);
        for (int i = j + 1; i < m; ++i) {
          double s = 0;
          for (int k = j; k < i; ++k) s += A_(i, k) * W[k * m + j];
          W[i * m + j] = -s / A_(i, i);
        }
      }
      Loc wl = (T.type == TK_TRTRI) ? T.out : T.out2;
      if (T.type == TK_TRTRI || (T.flags & TF_W_OUT)) {
        double *o = ptr(c, wl);
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < m; ++j) o[(int64_t)i * wl.ld + j] = W[i * m + j];
      }
      if (T.type == TK_TRTRI) {
        for (int j = 0; j < m; ++j)
          if (!(A_(j, j) != 0.0) || !std::isfinite(A_(j, j)))
            rec_info(std::isnan(A_(j, j)) ? c.info2 : c.info, T.aux1 + j + 1);
      }
      auto trsm_tile = [&](int s0, int s1, const Loc &out, int mm, double beta) {
        // (beta * C + alpha * sum_{s0 <= s < s1} ...) * W^T  at out (mm x m)
        double alpha = (s1 > s0) ? T.alpha : 0.0;
        std::vector<double> S2(mm * m);
        for (int i = 0; i < mm; ++i)
          for (int j = 0; j < m; ++j) {
            double s = 0;
            for (int si = s0; si < s1; ++si) {
              const Seg &S = g.segs[T.seg0 + si];
              for (int k = 0; k < S.k; ++k) s += opget(c, S.A, S.ta, i, k) * opget(c, S.B, S.tb, k, j);
            }
            double v = alpha * s;
            if (beta != 0.0) v += beta * get(c, out, i, j);
            S2[i * m + j] = v;
          }
        double *o3 = ptr(c, out);
        for (int i = 0; i < mm; ++i)
          for (int j = 0; j < m; ++j) {
            double s = 0;
            for (int k = 0; k < m; ++k) s += S2[i * m + k] * W[j * m + k];
            o3[(int64_t)i * out.ld + j] = s;
          }
      };
      if (T.type == TK_POTRF && (T.flags & TF_TRSM2)) {
        trsm_tile(T.nseg1, T.nseg2, T.out3, T.m3, T.beta3);
        if (T.zmask & 1) {
          double *z = ptr(c, T.out) + SERINV_TILE;
          for (int i = 0; i < m; ++i)
            for (int j = 0; j < T.m3; ++j) z[(int64_t)i * T.out.ld + j] = 0.0;
        }
      }
      if (T.type == TK_POTRF && (T.flags & TF_CHAINSTEP)) {
        // E <- E W^T (no update segments: E's updates were bulk tasks), zero the mirror
        // tile, then the next diagonal tile out4 -= E E^T
        trsm_tile(0, 0, T.out3, T.m3, 1.0);
        if (T.zmask & 1) {
          double *z = ptr(c, T.out) + SERINV_TILE;
          for (int i = 0; i < m; ++i)
            for (int j = 0; j < T.m3; ++j) z[(int64_t)i * T.out.ld + j] = 0.0;
        }
        double *o4 = ptr(c, T.out4);
        for (int i = 0; i < T.m4; ++i)
          for (int j = 0; j < T.m4; ++j) {
            double s = 0;
            for (int k = 0; k < m; ++k) s += get(c, T.out3, i, k) * get(c, T.out3, j, k);
            o4[(int64_t)i * T.out4.ld + j] -= s;
          }
      }
      if (T.type == TK_POTRF && (T.flags & TF_TRSM3)) {
        trsm_tile(T.nseg2, T.nseg, T.out4, T.m4, T.beta4);
        if (T.zmask & 2) {
          double *z = ptr(c, T.out) + 2 * SERINV_TILE;
          for (int i = 0; i < m; ++i)
            for (int j = 0; j < T.m4; ++j) z[(int64_t)i * T.out.ld + j] = 0.0;
        }
      }
    } else if (T.type == TK_REDUCE) {
      double *o = ptr(c, T.out);
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
          double s = 0;
          for (int p = 0; p < T.aux0; ++p) s += ptr(c, T.r)[T.aux2 * p + (int64_t)i * T.r.ld + j];
          double v = T.alpha * s;
          if (T.beta != 0.0) v += T.beta * get(c, T.c0, i, j);
          o[(int64_t)i * T.out.ld + j] = v;
          if (T.flags & TF_MIRROR) ptr(c, T.out2)[(int64_t)j * T.out2.ld + i] = v;
        }
    } else if (T.type == TK_COPY) {
      double *o = ptr(c, T.out);
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j)
          o[(int64_t)i * T.out.ld + j] = T.alpha * ((T.flags & TF_TRANS_C0) ? get(c, T.c0, j, i) : get(c, T.c0, i, j));
    } else if (T.type == TK_LOGDET) {
      double s = 0;
      for (int i = 0; i < T.aux0; ++i) s += ptr(c, T.r)[i];
      double v = 2.0 * s;
      for (int j = 0; j < T.aux1; ++j) v += ptr(c, T.c0)[T.aux2 * j];
      *ptr(c, T.out) = (c.info || c.info2) ? NAN : v;
    }
    for (int s = 0; s < T.nsig; ++s) c.ctr[g.sigs[T.sig0 + s]]++;
  }
  return 0;
}

}  // namespace

extern "C" {

// kind: 0 pobtaf, 1 pobtasi, 2 selinv.  Returns 0 on success; *info as serinv.
int dag_run_sequential(int kind, int64_t n, int64_t b, int64_t a, double *diag, double *lower, double *arrow,
                       double *tip, double *logdet, int *info, int grid, int update_group, int64_t *ntasks,
                       int si_split) {
  BuildOptions opt;
  opt.grid = grid;
  opt.update_group = update_group;
  if (si_split >= 0) opt.si_split = si_split;
  opt.apply_env();  // SERINV_OPT (e.g. twist_min_n=0: one-sided chain)
  Graph g = build_sequential(kind, n, b, a, opt);
  if (!g.error.empty()) {
    fprintf(stderr, "graph error: %s\n", g.error.c_str());
    return -2;
  }
  std::vector<double> ws(g.ws_doubles + 64, 0.0);
  double ld = 0;
  Ctx c;
  memset(c.bufs, 0, sizeof(c.bufs));
  c.bufs[BUF_DIAG] = diag;
  c.bufs[BUF_LOWER] = lower;
  c.bufs[BUF_ARROW] = arrow;
  c.bufs[BUF_TIP] = tip;
  c.bufs[BUF_WS] = ws.data();
  c.bufs[BUF_LOGDET] = &ld;
  int rc = run(g, c);
  *info = c.info;
  if (logdet) *logdet = ld;
  if (ntasks) *ntasks = (int64_t)g.tasks.size();
  // streaming IO: every final-X counter reached its target
  if (rc == 0)
    for (const Wait &w : g.fin)
      if (c.ctr[w.ctr] != w.target) return -5;
  return rc;
}

int dag_run_pselinv_nested(int64_t n, int64_t b, int64_t a, int nlev, const int *Ps, double r, double *diag,
                           double *lower, double *arrow, double *tip, double *logdet, int *info, int grid,
                           int64_t *ntasks) {
  BuildOptions opt;
  opt.grid = grid;
  opt.apply_env();
  Graph g = build_pselinv(n, b, a, std::vector<int>(Ps, Ps + nlev), r, opt);
  if (!g.error.empty()) {
    fprintf(stderr, "graph error: %s\n", g.error.c_str());
    return -2;
  }
  std::vector<double> ws(g.ws_doubles + 64, 0.0);
  double ld = 0;
  Ctx c;
  memset(c.bufs, 0, sizeof(c.bufs));
  c.bufs[BUF_DIAG] = diag;
  c.bufs[BUF_LOWER] = lower;
  c.bufs[BUF_ARROW] = arrow;
  c.bufs[BUF_TIP] = tip;
  c.bufs[BUF_WS] = ws.data();
  c.bufs[BUF_LOGDET] = &ld;
  int rc = run(g, c);
  *info = c.info;
  if (logdet) *logdet = ld;
  if (ntasks) *ntasks = (int64_t)g.tasks.size();
  return rc;
}

int dag_run_pselinv(int64_t n, int64_t b, int64_t a, int P, double r, double *diag, double *lower, double *arrow,
                    double *tip, double *logdet, int *info, int grid, int64_t *ntasks) {
  return dag_run_pselinv_nested(n, b, a, 1, &P, r, diag, lower, arrow, tip, logdet, info, grid, ntasks);
}

int dag_auto_partitions(int64_t n, int64_t b, int *Ps, int cap) {
  std::vector<int> v = auto_partitions(n, b);
  for (int i = 0; i < (int)v.size() && i < cap; ++i) Ps[i] = v[i];
  return (int)v.size();
}

// Simulate P ranks of the distributed path on the host.  Global arrays in, X out
// (in place); each rank works on copies of its local blocks.
// Q = sub-partitions per rank (serinv_ppobtaf_q / serinv_ppobtasi_q).
int dag_run_distributed_q(int64_t n, int64_t b, int64_t a, int P, int Q, double r, double *diag, double *lower,
                          double *arrow, double *tip, double *logdet, int *info) {
  std::vector<int64_t> st;
  if (!plan_partitions(n, P, r, st)) return -3;
  int64_t rec = exchange_doubles(b, a), mo = exchange_meta_offset(b, a);
  std::vector<double> records(rec * P * Q, 0.0);
  struct Rank {
    std::vector<double> D, L, A, T, ws;
    int64_t cnt;
    Ctx c;
  };
  std::vector<Rank> R(P);
  BuildOptions opt;
  opt.grid = 8;
  opt.apply_env();
  for (int p = 0; p < P; ++p) {
    Rank &k = R[p];
    int64_t s = st[p], e = st[p + 1], cnt = e - s;
    k.cnt = cnt;
    k.D.assign(diag + s * b * b, diag + e * b * b);
    int64_t nl = (p < P - 1) ? cnt : cnt - 1;
    k.L.assign(std::max<int64_t>(nl, 1) * b * b, 0.0);
    if (nl > 0) std::copy(lower + s * b * b, lower + (s + nl) * b * b, k.L.begin());
    k.A.assign(std::max<int64_t>(cnt * a * b, 1), 0.0);
    if (a) std::copy(arrow + s * a * b, arrow + e * a * b, k.A.begin());
    k.T.assign(std::max<int64_t>(a * a, 1), 0.0);
    if (a) std::copy(tip, tip + a * a, k.T.begin());
    Graph g0 = build_distributed(0, P, p, n, s, cnt, b, a, opt, Q);
    Graph g1 = build_distributed(1, P, p, n, s, cnt, b, a, opt, Q);
    if (!g0.error.empty() || !g1.error.empty()) {
      fprintf(stderr, "graph error: %s %s\n", g0.error.c_str(), g1.error.c_str());
      return -2;
    }
    k.ws.assign(std::max(g0.ws_doubles, g1.ws_doubles) + 64, 0.0);
    memset(k.c.bufs, 0, sizeof(k.c.bufs));
    k.c.bufs[BUF_DIAG] = k.D.data();
    k.c.bufs[BUF_LOWER] = k.L.data();
    k.c.bufs[BUF_ARROW] = k.A.data();
    k.c.bufs[BUF_TIP] = k.T.data();
    k.c.bufs[BUF_WS] = k.ws.data();
    k.c.bufs[BUF_EXT0] = records.data() + p * Q * rec;
    if (run(g0, k.c)) return -1;
    for (int q = 0; q < Q; ++q) meta_write(records.data() + p * Q * rec, Q, rec, mo, k.c.info, s, cnt, q);
  }
  double ld = 0;
  *info = 0;
  for (int p = 0; p < P; ++p) {
    Rank &k = R[p];
    Graph g1 = build_distributed(1, P, p, n, st[p], k.cnt, b, a, opt, Q);
    double ldp = 0;
    k.c.bufs[BUF_EXT0] = nullptr;
    k.c.bufs[BUF_EXT1] = records.data();
    k.c.bufs[BUF_LOGDET] = &ldp;
    const int comb = meta_combine_info(records.data(), P * Q, rec, mo);  // as serinv_ppobtasi
    k.c.info = comb;
    if (run(g1, k.c)) return -1;
    k.c.info = comb ? comb : meta_decode_info(k.c.info, records.data(), rec, mo, b);
    if (p == 0) *info = k.c.info;
    else if (k.c.info != *info) {
      fprintf(stderr, "rank info mismatch: %d vs %d\n", k.c.info, *info);
      return -4;
    }
    if (p == 0) ld = ldp;
    else if (!(ldp == ld) && !(std::isnan(ld) && std::isnan(ldp))) fprintf(stderr, "rank logdet mismatch\n");
    int64_t s = st[p], e = st[p + 1], cnt = k.cnt;
    std::copy(k.D.begin(), k.D.begin() + cnt * b * b, diag + s * b * b);
    int64_t nl = (p < P - 1) ? cnt : cnt - 1;
    if (nl > 0) std::copy(k.L.begin(), k.L.begin() + nl * b * b, lower + s * b * b);
    if (a) std::copy(k.A.begin(), k.A.begin() + cnt * a * b, arrow + s * a * b);
    if (a && p == 0) std::copy(k.T.begin(), k.T.begin() + a * a, tip);
  }
  *logdet = ld;
  return 0;
}

int dag_run_distributed(int64_t n, int64_t b, int64_t a, int P, double r, double *diag, double *lower, double *arrow,
                        double *tip, double *logdet, int *info) {
  return dag_run_distributed_q(n, b, a, P, 1, r, diag, lower, arrow, tip, logdet, info);
}

// One distributed phase on caller buffers (used by the gloo multi-process test).
int64_t dag_dist_ws_doubles_q(int P, int Q, int rank, int64_t n, int64_t start, int64_t count, int64_t b,
                              int64_t a) {
  return distributed_ws_bytes(P, rank, n, start, count, b, a, Q) / 8;
}
int64_t dag_dist_ws_doubles(int P, int rank, int64_t n, int64_t start, int64_t count, int64_t b, int64_t a) {
  return dag_dist_ws_doubles_q(P, 1, rank, n, start, count, b, a);
}
int64_t dag_exchange_doubles(int64_t b, int64_t a) { return exchange_doubles(b, a); }
int dag_run_dist_phase_q(int phase, int P, int Q, int rank, int64_t n, int64_t start, int64_t count, int64_t b,
                         int64_t a, double *diag, double *lower, double *arrow, double *tip, double *ws, double *ext0,
                         double *ext1, double *logdet, int *info) {
  BuildOptions opt;
  opt.grid = 8;
  Graph g = build_distributed(phase, P, rank, n, start, count, b, a, opt, Q);
  if (!g.error.empty()) return -2;
  Ctx c;
  memset(c.bufs, 0, sizeof(c.bufs));
  double ld = 0;
  c.bufs[BUF_DIAG] = diag;
  c.bufs[BUF_LOWER] = lower;
  c.bufs[BUF_ARROW] = arrow;
  c.bufs[BUF_TIP] = tip;
  c.bufs[BUF_WS] = ws;
  c.bufs[BUF_EXT0] = ext0;
  c.bufs[BUF_EXT1] = ext1;
  c.bufs[BUF_LOGDET] = &ld;
  // the status handling of serinv_ppobtaf / serinv_ppobtasi (dist_meta.h)
  const int64_t rec = exchange_doubles(b, a), mo = exchange_meta_offset(b, a);
  const int comb = phase == 1 ? meta_combine_info(ext1, P * Q, rec, mo) : 0;
  c.info = comb;
  int rc = run(g, c);
  if (phase == 0)
    for (int q = 0; q < Q; ++q) meta_write(ext0, Q, rec, mo, c.info, start, count, q);
  else
    c.info = comb ? comb : meta_decode_info(c.info, ext1, rec, mo, b);
  *info = c.info;
  if (logdet) *logdet = ld;
  return rc;
}

int dag_run_dist_phase(int phase, int P, int rank, int64_t n, int64_t start, int64_t count, int64_t b, int64_t a,
                       double *diag, double *lower, double *arrow, double *tip, double *ws, double *ext0,
                       double *ext1, double *logdet, int *info) {
  return dag_run_dist_phase_q(phase, P, 1, rank, n, start, count, b, a, diag, lower, arrow, tip, ws, ext0, ext1,
                              logdet, info);
}

int dag_stats_sequential(int kind, int64_t n, int64_t b, int64_t a, int grid, int64_t *ntasks, double *flops,
                         int64_t *nctr) {
  BuildOptions opt;
  opt.grid = grid;
  Graph g = build_sequential(kind, n, b, a, opt);
  if (!g.error.empty()) return -2;
  *ntasks = (int64_t)g.tasks.size();
  *flops = g.flops;
  *nctr = g.nctr;
  return 0;
}
}
