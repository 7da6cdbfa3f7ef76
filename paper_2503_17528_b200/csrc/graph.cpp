// graph.cpp -- lowering of PAPER.md Alg. 1-6 to a tile-task DAG + scheduler.
// See graph.h for the overview and task.h for the task semantics.
#include "graph.h"

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstring>
#include <functional>
#include <queue>
#include <unordered_map>

namespace serinv {

namespace {

inline int ntiles(int64_t s) { return (int)((s + TILE - 1) / TILE); }
inline int tdim(int64_t s, int t) { return (int)std::min<int64_t>(TILE, s - (int64_t)t * TILE); }

inline Loc at(const Loc &base, int64_t r, int64_t c) {
  Loc l = base;
  l.off += r * (int64_t)base.ld + c;
  return l;
}
inline Loc tileloc(const Loc &base, int q, int c) { return at(base, (int64_t)q * TILE, (int64_t)c * TILE); }

// ---------------------------------------------------------------------------
// Raw graph under construction (tasks in creation order = a topological order).
// ---------------------------------------------------------------------------
struct RawTask {
  Task t{};
  std::vector<Seg> segs;
  std::vector<int32_t> waits;   // counters (target = #producers, fixed at finalize)
  std::vector<int32_t> sigs;    // counters signalled (own counter first)
  double cost = 0.0;            // ns (scheduler model)
  double flops = 0.0;
};

struct Raw {
  std::vector<RawTask> tasks;
  int32_t nctr = 0;
  int32_t new_ctr() { return nctr++; }
  // returns task id; the task's own completion counter == its id counter
  int add(RawTask &&rt) {
    int id = (int)tasks.size();
    int32_t own = new_ctr();
    rt.sigs.insert(rt.sigs.begin(), own);
    own_ctr.push_back(own);
    tasks.push_back(std::move(rt));
    return id;
  }
  int32_t ctr_of(int task) const { return own_ctr[task]; }
  std::vector<int32_t> own_ctr;
};

double gemm_flops(int m, int n, const std::vector<Seg> &segs) {
  double k = 0;
  for (auto &s : segs) k += s.k;
  return 2.0 * m * n * k;
}

// Scheduler cost model (ns): one CTA of a 2-CTA/SM persistent grid.
double task_cost(const RawTask &rt) {
  const double ns_per_flop = 1.0 / 110.0;  // ~110 GFLOP/s per CTA
  switch (rt.t.type) {
    case TK_POTRF: return 5000.0 + rt.flops * ns_per_flop;
    case TK_TRTRI: return 2500.0;
    case TK_GEMM: return 900.0 + rt.flops * ns_per_flop;
    default: return 700.0;
  }
}

// ---------------------------------------------------------------------------
// Builder over a Problem.
// ---------------------------------------------------------------------------
struct Builder {
  Raw raw;
  Problem &P;
  BuildOptions opt;
  int64_t ws_top = 0;           // next free workspace double
  int64_t slot_top = 0;         // next logdet slot (in the slot region)
  int64_t slot_region = -1;     // WS offset of the slot region

  // L tile producers: key (Y, q, X, c) -> task
  std::unordered_map<uint64_t, int> Lprod;
  // per target tile chain state
  struct TileState {
    std::vector<std::pair<int, int>> pending;  // columns (X, c) not yet applied
    int last = -1;                             // last task that wrote the tile
    bool written = false;
  };
  std::unordered_map<uint64_t, TileState> tstate;
  // group counters
  std::map<int, int32_t> factordone;   // node -> counter (all final L tiles of column-node X)
  std::map<int, int32_t> predone;      // node -> counter (precompute of node X done)
  std::map<std::tuple<int, int, int, int>, int32_t> xr, xc;  // (Y,X,tile, kind) final-X row/col
  std::map<std::tuple<int, int>, int32_t> wcol;               // (X, c) W column complete
  std::map<std::tuple<int, int, int>, int32_t> lcol;          // (Z, X, c) Lchk column complete
  std::map<int, int> wdiag_task;       // (X*4096 + c) -> task producing W(c,c)

  Builder(Problem &p, const BuildOptions &o) : P(p), opt(o) {}

  // key of tile (row node Y, row tile q) x (column node X, column tile c)
  static uint64_t key4(int Y, int q, int X, int c) {
    return ((uint64_t)(uint32_t)Y << 44) | ((uint64_t)(uint32_t)q << 32) | ((uint64_t)(uint32_t)X << 12) |
           (uint64_t)(uint32_t)c;
  }
  static void unkey4(uint64_t k, int &Y, int &q, int &X, int &c) {
    Y = (int)(k >> 44);
    q = (int)((k >> 32) & 0xFFF);
    X = (int)((k >> 12) & 0xFFFFF);
    c = (int)(k & 0xFFF);
  }

  int64_t alloc(int64_t doubles) {
    int64_t off = ws_top;
    ws_top += (doubles + 31) / 32 * 32;  // 256-byte granules
    return off;
  }

  int32_t group_ctr(std::map<int, int32_t> &m, int k) {
    auto it = m.find(k);
    if (it != m.end()) return it->second;
    int32_t c = raw.new_ctr();
    m[k] = c;
    return c;
  }
  template <class K>
  int32_t gctr(std::map<K, int32_t> &m, const K &k) {
    auto it = m.find(k);
    if (it != m.end()) return it->second;
    int32_t c = raw.new_ctr();
    m[k] = c;
    return c;
  }

  const BlkRef &B(int Y, int X) const {
    auto it = P.blk.find({Y, X});
    if (it == P.blk.end() || !it->second.valid) {
      static BlkRef bad;
      fprintf(stderr, "serinv graph: missing block (%d,%d)\n", Y, X);
      return bad;
    }
    return it->second;
  }
  bool has(int Y, int X) const {
    auto it = P.blk.find({Y, X});
    return it != P.blk.end() && it->second.valid;
  }

  // ------------------------------------------------------------------ helpers
  static Seg seg(Loc A, int ta, Loc Bm, int tb, int k) {
    Seg s{};
    s.A = A;
    s.B = Bm;
    s.k = k;
    s.ta = (int8_t)ta;
    s.tb = (int8_t)tb;
    return s;
  }

  int emit(RawTask &&rt) {
    if (rt.t.type == TK_GEMM) rt.flops = gemm_flops(rt.t.m, rt.t.n, rt.segs) +
                                        ((rt.t.flags & TF_POST) ? 2.0 * rt.t.m * rt.t.n * rt.t.n : 0.0);
    if (rt.t.type == TK_POTRF)
      rt.flops = gemm_flops(rt.t.m, rt.t.n, rt.segs) + 2.0 * rt.t.m * rt.t.m * rt.t.m / 3.0;
    if (rt.t.type == TK_TRTRI) rt.flops = rt.t.m * (double)rt.t.m * rt.t.m / 3.0;
    rt.cost = task_cost(rt);
    // dedupe waits
    std::sort(rt.waits.begin(), rt.waits.end());
    rt.waits.erase(std::unique(rt.waits.begin(), rt.waits.end()), rt.waits.end());
    return raw.add(std::move(rt));
  }

  // ===================================================================
  // Factorisation (Alg. 1 / Alg. 4, tile-level right-looking)
  // ===================================================================
  struct RT {
    int Y, q, h;
    Loc loc;  // L(Y q, X c) tile
  };

  // column row-tiles of tile column (X, c)
  std::vector<RT> column_rows(int X, int c) {
    std::vector<RT> v;
    const BlkRef &d = B(X, X);
    int nt = ntiles(P.size[X]);
    for (int r = c + 1; r < nt; ++r) v.push_back({X, r, tdim(P.size[X], r), tileloc(d.base, r, c)});
    for (int Y : P.rows[X]) {
      const BlkRef &bb = B(Y, X);
      int nq = ntiles(P.size[Y]);
      for (int q = 0; q < nq; ++q) v.push_back({Y, q, tdim(P.size[Y], q), tileloc(bb.base, q, c)});
    }
    return v;
  }

  // target tile storage for update pair (Yi qi) >= (Yj qj) from column node X
  BlkRef target_blk(int Yi, int Yj, int X, bool &ok) {
    ok = true;
    if (Yj == X) return B(Yi, X);
    if (!has(Yi, Yj)) {
      ok = false;
      return BlkRef{};
    }
    return B(Yi, Yj);
  }

  uint64_t tkey(int Yi, int Yj, int qi, int qj) { return key4(Yi, qi, Yj, qj); }

  // Flush pending columns of a target tile into one chained update task.
  // cols: list of (X, c) columns; all L tiles of rows (Yi qi) and (Yj qj) at those
  // columns are final.  The group may span two nodes -> two segments.
  int update_task(int Yi, int qi, int Yj, int qj, const BlkRef &tb, TileState &st,
                  const std::vector<std::pair<int, int>> &cols) {
    RawTask rt;
    rt.t.type = TK_GEMM;
    int m = tdim(P.size[Yi], qi), n = tdim(P.size[Yj], qj);
    rt.t.m = (int16_t)m;
    rt.t.n = (int16_t)n;
    rt.t.out = tileloc(tb.base, qi, qj);
    rt.t.alpha = -1.0;
    bool first = !st.written;
    rt.t.beta = (first && tb.zero_init) ? 0.0 : 1.0;
    rt.t.c0 = rt.t.out;
    add_update_segs(rt, Yi, qi, Yj, qj, cols);
    if (st.last >= 0) rt.waits.push_back(raw.ctr_of(st.last));
    int id = emit(std::move(rt));
    st.last = id;
    st.written = true;
    return id;
  }

  void add_update_segs(RawTask &rt, int Yi, int qi, int Yj, int qj, const std::vector<std::pair<int, int>> &cols) {
    size_t s = 0;
    while (s < cols.size()) {
      int X = cols[s].first, c0 = cols[s].second;
      size_t e = s + 1;
      while (e < cols.size() && cols[e].first == X && cols[e].second == cols[e - 1].second + 1) ++e;
      int c1 = cols[e - 1].second;
      // L(Yi qi, X c0..c1) and L(Yj qj, X c0..c1) are contiguous row strips
      const BlkRef &bi = (Yi == X) ? B(X, X) : B(Yi, X);
      const BlkRef &bj = (Yj == X) ? B(X, X) : B(Yj, X);
      int k = (int)(std::min<int64_t>((int64_t)(c1 + 1) * TILE, P.size[X]) - (int64_t)c0 * TILE);
      rt.segs.push_back(seg(tileloc(bi.base, qi, c0), 0, tileloc(bj.base, qj, c0), 1, k));
      for (size_t u = s; u < e; ++u) {
        int c = cols[u].second;
        rt.waits.push_back(raw.ctr_of(Lprod.at(key4(Yi, qi, X, c))));
        rt.waits.push_back(raw.ctr_of(Lprod.at(key4(Yj, qj, X, c))));
      }
      s = e;
    }
  }

  void flush(int Yi, int qi, int Yj, int qj, const BlkRef &tb, TileState &st, size_t keep_last) {
    // flush all pending columns except the last `keep_last`, in groups
    size_t upto = st.pending.size() - std::min(keep_last, st.pending.size());
    size_t s = 0;
    while (s < upto) {
      int G = opt.update_group;
      bool whole_node = P.accum[Yj];
      std::vector<std::pair<int, int>> g;
      int X0 = st.pending[s].first;
      size_t e = s;
      while (e < upto && st.pending[e].first == X0 && (whole_node || (int)g.size() < G)) {
        g.push_back(st.pending[e]);
        ++e;
      }
      update_task(Yi, qi, Yj, qj, tb, st, g);
      s = e;
    }
    st.pending.erase(st.pending.begin(), st.pending.begin() + upto);
  }

  // logdet slot for a diagonal tile
  int64_t next_slot() { return slot_top++; }

  void factor_node(int X, bool fuse_w) {
    int nt = ntiles(P.size[X]);
    const BlkRef &d = B(X, X);
    int32_t fd = group_ctr(factordone, X);
    for (int c = 0; c < nt; ++c) {
      int w = tdim(P.size[X], c);
      // ---- POTRF of the diagonal tile (X c, X c)
      {
        uint64_t k = tkey(X, X, c, c);
        TileState &st = tstate[k];
        flush(X, c, X, c, d, st, 1);
        RawTask rt;
        rt.t.type = TK_POTRF;
        rt.t.m = rt.t.n = (int16_t)w;
        rt.t.out = tileloc(d.base, c, c);
        rt.t.c0 = rt.t.out;
        rt.t.alpha = -1.0;
        rt.t.beta = 1.0;
        if (!st.pending.empty()) add_update_segs(rt, X, c, X, c, st.pending);
        if (st.last >= 0) rt.waits.push_back(raw.ctr_of(st.last));
        rt.t.flags = TF_W_OUT;
        rt.t.out2 = tileloc(P.W[X], c, c);
        rt.t.aux0 = (int32_t)(P.slot[X] + c);
        rt.t.r = Loc{BUF_WS, 0, slot_region + P.slot[X] + c};
        rt.t.aux1 = (int32_t)(P.rowbase[X] + (int64_t)c * TILE);
        rt.sigs.push_back(fd);
        int id = emit(std::move(rt));
        st.pending.clear();
        st.last = id;
        Lprod[key4(X, c, X, c)] = id;
        wdiag_task[X * 4096 + c] = id;
      }
      // ---- TRSM of every row tile below: L = (A - last update) W(c,c)^T
      std::vector<RT> rts = column_rows(X, c);
      for (auto &r : rts) {
        const BlkRef &tb = (r.Y == X) ? d : B(r.Y, X);
        uint64_t k = tkey(r.Y, X, r.q, c);
        TileState &st = tstate[k];
        flush(r.Y, r.q, X, c, tb, st, 1);
        RawTask rt;
        rt.t.type = TK_GEMM;
        rt.t.m = (int16_t)r.h;
        rt.t.n = (int16_t)w;
        rt.t.out = r.loc;
        rt.t.c0 = r.loc;
        rt.t.alpha = -1.0;
        rt.t.beta = (!st.written && tb.zero_init) ? 0.0 : 1.0;
        if (!st.pending.empty()) {
          add_update_segs(rt, r.Y, r.q, X, c, st.pending);
        } else {
          rt.t.alpha = 0.0;  // no update: out = C0 * W^T
        }
        if (st.last >= 0) rt.waits.push_back(raw.ctr_of(st.last));
        rt.waits.push_back(raw.ctr_of(Lprod.at(key4(X, c, X, c))));
        rt.t.flags = TF_POST | TF_POST_T;
        rt.t.r = tileloc(P.W[X], c, c);
        if (r.Y == X) {  // strict-upper tile (c, r.q) of the diagonal block: zero it
          rt.t.flags |= TF_ZERO_MIRROR;
          rt.t.out2 = tileloc(d.base, c, r.q);
        }
        rt.sigs.push_back(fd);
        int id = emit(std::move(rt));
        st.pending.clear();
        st.last = id;
        st.written = true;
        Lprod[key4(r.Y, r.q, X, c)] = id;
      }
      // ---- register this column's contributions to every later target tile
      // pairs (i >= j) of the row tiles; j must be a later column than (X, c)
      for (size_t j = 0; j < rts.size(); ++j) {
        for (size_t i = j; i < rts.size(); ++i) {
          const RT &ri = rts[i], &rj = rts[j];
          bool ok;
          BlkRef tb = target_blk(ri.Y, rj.Y, X, ok);
          if (!ok) continue;
          if (ri.Y == rj.Y && ri.q < rj.q) continue;
          uint64_t k = tkey(ri.Y, rj.Y, ri.q, rj.q);
          tstate[k].pending.push_back({X, c});
        }
      }
      (void)fuse_w;
    }
  }

  // Flush all pending updates onto non-eliminated (boundary) targets.
  void flush_boundary() {
    // deterministic order: iterate sorted keys
    std::vector<uint64_t> keys;
    for (auto &kv : tstate)
      if (!kv.second.pending.empty()) keys.push_back(kv.first);
    std::sort(keys.begin(), keys.end());
    for (uint64_t k : keys) {
      int Yi, qi, Yj, qj;
      unkey4(k, Yi, qi, Yj, qj);
      TileState &st = tstate[k];
      flush(Yi, qi, Yj, qj, B(Yi, Yj), st, 0);
    }
  }

  // ===================================================================
  // Selected inversion (Alg. 2 / Alg. 6 with L^{-1} precompute)
  // ===================================================================
  // W_X = L_XX^{-1}: diagonal tiles from POTRF (fused) or TRTRI, then
  // W(r,c) = -(sum_{k=c+1..r} W(r,k) L(k,c)) W(c,c)   (from W L = I).
  void precompute_node(int X, bool have_wdiag) {
    int nt = ntiles(P.size[X]);
    const BlkRef &d = B(X, X);
    // in a pobtasi-only graph L is an input: no factor-done counter to wait on
    int32_t fd = have_wdiag ? group_ctr(factordone, X) : -1;
    int32_t pre = group_ctr(predone, X);
    std::vector<std::vector<int>> Wt(nt, std::vector<int>(nt, -1));
    for (int c = 0; c < nt; ++c) {
      int w = tdim(P.size[X], c);
      if (have_wdiag) {
        Wt[c][c] = wdiag_task.at(X * 4096 + c);
      } else {
        RawTask rt;
        rt.t.type = TK_TRTRI;
        rt.t.m = rt.t.n = (int16_t)w;
        rt.t.c0 = tileloc(d.base, c, c);
        rt.t.out = tileloc(P.W[X], c, c);
        rt.t.aux1 = (int32_t)(P.rowbase[X] + (int64_t)c * TILE);
        if (fd >= 0) rt.waits.push_back(fd);
        rt.sigs.push_back(pre);
        Wt[c][c] = emit(std::move(rt));
      }
    }
    for (int r = 1; r < nt; ++r) {
      for (int c = r - 1; c >= 0; --c) {
        RawTask rt;
        rt.t.type = TK_GEMM;
        rt.t.m = (int16_t)tdim(P.size[X], r);
        rt.t.n = (int16_t)tdim(P.size[X], c);
        rt.t.out = tileloc(P.W[X], r, c);
        rt.t.alpha = -1.0;
        rt.t.beta = 0.0;
        int k = (int)(std::min<int64_t>((int64_t)(r + 1) * TILE, P.size[X]) - (int64_t)(c + 1) * TILE);
        rt.segs.push_back(seg(tileloc(P.W[X], r, c + 1), 0, tileloc(d.base, c + 1, c), 0, k));
        rt.t.flags = TF_POST;  // * W(c,c)
        rt.t.r = tileloc(P.W[X], c, c);
        for (int kk = c + 1; kk <= r; ++kk) rt.waits.push_back(raw.ctr_of(Wt[r][kk]));
        rt.waits.push_back(raw.ctr_of(Wt[c][c]));
        if (fd >= 0) rt.waits.push_back(fd);
        rt.sigs.push_back(pre);
        Wt[r][c] = emit(std::move(rt));
      }
    }
    auto wcol_wait = [&](RawTask &rt, int c) {
      for (int r = c; r < nt; ++r) rt.waits.push_back(raw.ctr_of(Wt[r][c]));
    };
    // Lchk(Z, X)(q, c) = sum_{k >= c} L_{Z,X}(q, k) W(k, c)
    for (int Z : P.rows[X]) {
      const BlkRef &bz = B(Z, X);
      Loc lc = P.Lchk.at({Z, X});
      int nq = ntiles(P.size[Z]);
      for (int c = 0; c < nt; ++c) {
        int32_t lcc = gctr(lcol, std::make_tuple(Z, X, c));
        for (int q = 0; q < nq; ++q) {
          RawTask rt;
          rt.t.type = TK_GEMM;
          rt.t.m = (int16_t)tdim(P.size[Z], q);
          rt.t.n = (int16_t)tdim(P.size[X], c);
          rt.t.out = tileloc(lc, q, c);
          rt.t.alpha = 1.0;
          rt.t.beta = 0.0;
          int k = (int)(P.size[X] - (int64_t)c * TILE);
          rt.segs.push_back(seg(tileloc(bz.base, q, c), 0, tileloc(P.W[X], c, c), 0, k));
          wcol_wait(rt, c);
          if (fd >= 0) rt.waits.push_back(fd);
          rt.sigs.push_back(pre);
          rt.sigs.push_back(lcc);
          emit(std::move(rt));
        }
      }
    }
    // Lambda_X(r, c) = sum_{k >= r} W(k,r)^T W(k,c), r >= c
    for (int r = 0; r < nt; ++r) {
      for (int c = 0; c <= r; ++c) {
        RawTask rt;
        rt.t.type = TK_GEMM;
        rt.t.m = (int16_t)tdim(P.size[X], r);
        rt.t.n = (int16_t)tdim(P.size[X], c);
        rt.t.out = tileloc(P.Lam[X], r, c);
        rt.t.alpha = 1.0;
        rt.t.beta = 0.0;
        int k = (int)(P.size[X] - (int64_t)r * TILE);
        rt.segs.push_back(seg(tileloc(P.W[X], r, r), 1, tileloc(P.W[X], r, c), 0, k));
        wcol_wait(rt, r);
        wcol_wait(rt, c);
        rt.sigs.push_back(pre);
        lam_task[std::make_tuple(X, r, c)] = emit(std::move(rt));
      }
    }
  }
  std::map<std::tuple<int, int, int>, int> lam_task;

  // counters for final-X rows / columns of storage block (Y, X)
  int32_t XR(int Y, int X, int q) { return gctr(xr, std::make_tuple(Y, X, q, 0)); }
  int32_t XC(int Y, int X, int c) { return gctr(xc, std::make_tuple(Y, X, c, 0)); }

  // Register external producers of final X blocks (e.g. copies of X_r): a task
  // that writes the whole block (Y, X) signals all its row/col counters.
  void signal_whole_block(RawTask &rt, int Y, int X) {
    int nr = ntiles(P.size[Y]), nc = ntiles(P.size[X]);
    for (int q = 0; q < nr; ++q) rt.sigs.push_back(XR(Y, X, q));
    for (int c = 0; c < nc; ++c) rt.sigs.push_back(XC(Y, X, c));
  }

  // Read X_{Y,Z} row tile q (Y, Z in rows[X] U diag): location + transpose + waits
  // X_{Y,Z}: if Y >= Z stored at blk(Y,Z) (row tile q, op N); else at blk(Z,Y)^T
  // (column tile q, op T).
  void xrow(RawTask &rt, int Y, int Z, int q, Loc &loc, int &trans, int &k) {
    if (Y >= Z) {
      loc = tileloc(B(Y, Z).base, q, 0);
      trans = 0;
      rt.waits.push_back(XR(Y, Z, q));
    } else {
      loc = tileloc(B(Z, Y).base, 0, q);
      trans = 1;
      rt.waits.push_back(XC(Z, Y, q));
    }
    k = P.size[Z];
  }

  // Takahashi step for node X (all Y in rows[X] already hold final X values).
  void invert_node(int X) {
    int nt = ntiles(P.size[X]);
    int32_t pre = group_ctr(predone, X);
    const auto &R = P.rows[X];
    // X_{Y,X}(q, c) = - sum_Z X_{Y,Z}(q, :) Lchk(Z,X)(:, c)
    for (int Y : R) {
      const BlkRef &by = B(Y, X);
      int nq = ntiles(P.size[Y]);
      for (int q = 0; q < nq; ++q) {
        for (int c = 0; c < nt; ++c) {
          RawTask rt;
          rt.t.type = TK_GEMM;
          rt.t.m = (int16_t)tdim(P.size[Y], q);
          rt.t.n = (int16_t)tdim(P.size[X], c);
          rt.t.out = tileloc(by.base, q, c);
          rt.t.alpha = -1.0;
          rt.t.beta = 0.0;
          for (int Z : R) {
            Loc a;
            int tr, k;
            xrow(rt, Y, Z, q, a, tr, k);
            rt.segs.push_back(seg(a, tr, tileloc(P.Lchk.at({Z, X}), 0, c), 0, k));
            rt.waits.push_back(gctr(lcol, std::make_tuple(Z, X, c)));
          }
          rt.waits.push_back(pre);  // WAR: L_{Y,X} consumed by the precompute
          rt.sigs.push_back(XR(Y, X, q));
          rt.sigs.push_back(XC(Y, X, c));
          emit(std::move(rt));
        }
      }
    }
    // X_{X,X}(r, c) = Lambda(r,c) - sum_Y X_{Y,X}(:, r)^T Lchk(Y,X)(:, c), r >= c, mirrored
    const BlkRef &d = B(X, X);
    for (int r = 0; r < nt; ++r) {
      for (int c = 0; c <= r; ++c) {
        RawTask rt;
        rt.t.type = TK_GEMM;
        rt.t.m = (int16_t)tdim(P.size[X], r);
        rt.t.n = (int16_t)tdim(P.size[X], c);
        rt.t.out = tileloc(d.base, r, c);
        rt.t.c0 = tileloc(P.Lam[X], r, c);
        rt.t.alpha = -1.0;
        rt.t.beta = 1.0;
        for (int Y : R) {
          rt.segs.push_back(seg(tileloc(B(Y, X).base, 0, r), 1, tileloc(P.Lchk.at({Y, X}), 0, c), 0, P.size[Y]));
          rt.waits.push_back(XC(Y, X, r));
          rt.waits.push_back(gctr(lcol, std::make_tuple(Y, X, c)));
        }
        if (R.empty()) rt.t.alpha = 0.0;
        rt.waits.push_back(raw.ctr_of(lam_task.at(std::make_tuple(X, r, c))));
        rt.waits.push_back(pre);
        if (r != c) {
          rt.t.flags = TF_MIRROR;
          rt.t.out2 = tileloc(d.base, c, r);
        }
        rt.sigs.push_back(XR(X, X, r));
        rt.sigs.push_back(XC(X, X, c));
        if (r != c) {
          rt.sigs.push_back(XR(X, X, c));
          rt.sigs.push_back(XC(X, X, r));
        }
        emit(std::move(rt));
      }
    }
  }

  // LOGDET over slots [0, nslots) of the slot region
  void logdet_task(int64_t nslots) {
    RawTask rt;
    rt.t.type = TK_LOGDET;
    rt.t.r = Loc{BUF_WS, 0, slot_region};
    rt.t.aux0 = (int32_t)nslots;
    rt.t.out = Loc{BUF_LOGDET, 0, 0};
    // waits on every POTRF (all factordone counters)
    for (auto &kv : factordone) rt.waits.push_back(kv.second);
    emit(std::move(rt));
  }

  // ------------------------------------------------------------------ finalize
  Graph finalize() {
    Graph g;
    const int N = (int)raw.tasks.size();
    const int C = raw.nctr;
    // Bipartite DAG: task -> counters it signals -> tasks waiting on them.
    std::vector<int32_t> nprod(C, 0), nwaiter(C, 0);
    for (auto &t : raw.tasks) {
      for (int32_t s : t.sigs) nprod[s]++;
      for (int32_t w : t.waits) nwaiter[w]++;
    }
    // CSR of waiters per counter
    std::vector<int64_t> wptr(C + 1, 0);
    for (int c = 0; c < C; ++c) wptr[c + 1] = wptr[c] + nwaiter[c];
    std::vector<int32_t> wlist(wptr[C]);
    {
      std::vector<int64_t> fill(wptr.begin(), wptr.end() - 1);
      for (int i = 0; i < N; ++i)
        for (int32_t w : raw.tasks[i].waits) wlist[fill[w]++] = i;
    }
    for (int i = 0; i < N; ++i)
      for (int32_t w : raw.tasks[i].waits)
        if (nprod[w] == 0) {
          g.error = "counter with no producer";
          return g;
        }
    // topological order of tasks (Kahn over the bipartite graph, creation order ties)
    std::vector<int32_t> tdeg(N), cdeg(nprod);
    for (int i = 0; i < N; ++i) tdeg[i] = (int32_t)raw.tasks[i].waits.size();
    std::vector<int> topo;
    topo.reserve(N);
    {
      std::priority_queue<int, std::vector<int>, std::greater<int>> q;
      for (int i = 0; i < N; ++i)
        if (!tdeg[i]) q.push(i);
      while (!q.empty()) {
        int t = q.top();
        q.pop();
        topo.push_back(t);
        for (int32_t s : raw.tasks[t].sigs)
          if (--cdeg[s] == 0)
            for (int64_t k = wptr[s]; k < wptr[s + 1]; ++k)
              if (--tdeg[wlist[k]] == 0) q.push(wlist[k]);
      }
      if ((int)topo.size() != N) {
        g.error = "dependency cycle";
        return g;
      }
    }
    // bottom levels: bl(task) = cost + max over signalled counters of max waiter bl
    std::vector<double> bl(N, 0.0), cbl(C, 0.0);
    for (int k = N - 1; k >= 0; --k) {
      int t = topo[k];
      double m = 0;
      for (int32_t s : raw.tasks[t].sigs) m = std::max(m, cbl[s]);
      bl[t] = raw.tasks[t].cost + m;
      for (int32_t w : raw.tasks[t].waits) cbl[w] = std::max(cbl[w], bl[t]);
    }
    // list scheduling simulation
    std::vector<int> order;
    order.reserve(N);
    if (opt.schedule) {
      auto cmp = [&](int x, int y) {
        if (bl[x] != bl[y]) return bl[x] < bl[y];
        return x > y;
      };
      std::priority_queue<int, std::vector<int>, decltype(cmp)> ready(cmp);
      typedef std::pair<double, int> Ev;
      std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> ev;
      for (int i = 0; i < N; ++i) tdeg[i] = (int32_t)raw.tasks[i].waits.size();
      cdeg = nprod;
      for (int i = 0; i < N; ++i)
        if (!tdeg[i]) ready.push(i);
      int free_w = std::max(1, opt.grid);
      double now = 0;
      while ((int)order.size() < N) {
        while (free_w > 0 && !ready.empty()) {
          int t = ready.top();
          ready.pop();
          order.push_back(t);
          ev.push({now + raw.tasks[t].cost, t});
          --free_w;
        }
        if (ev.empty()) break;
        Ev e = ev.top();
        ev.pop();
        now = e.first;
        ++free_w;
        for (int32_t s : raw.tasks[e.second].sigs)
          if (--cdeg[s] == 0)
            for (int64_t k = wptr[s]; k < wptr[s + 1]; ++k)
              if (--tdeg[wlist[k]] == 0) ready.push(wlist[k]);
      }
      if ((int)order.size() != N) {
        g.error = "schedule incomplete";
        return g;
      }
      g.sim_ns = now;
    } else {
      order = topo;
    }
    // emit flat arrays
    g.tasks.reserve(N);
    for (int t : order) {
      RawTask &rt = raw.tasks[t];
      Task task = rt.t;
      task.seg0 = (int32_t)g.segs.size();
      task.nseg = (int32_t)rt.segs.size();
      for (auto &s : rt.segs) g.segs.push_back(s);
      task.wait0 = (int32_t)g.waits.size();
      task.nwait = (int32_t)rt.waits.size();
      for (int32_t w : rt.waits) g.waits.push_back(Wait{w, nprod[w]});
      task.sig0 = (int32_t)g.sigs.size();
      task.nsig = (int32_t)rt.sigs.size();
      for (int32_t s : rt.sigs) g.sigs.push_back(s);
      g.tasks.push_back(task);
      g.flops += rt.flops;
    }
    g.nctr = raw.nctr;
    g.grid = opt.grid;
    g.ws_doubles = ws_top;
    g.nslots = slot_top;
    return g;
  }
};

// ---------------------------------------------------------------------------
// Sequential problem: nodes 0..n-1 (blocks) and n (the arrow tip, if a > 0).
// ---------------------------------------------------------------------------
struct SeqLayout {
  int64_t n, b, a;
  int64_t W, Wtip, Lchk, Lnchk, Lam, Lamtip, slots, total;
};

SeqLayout seq_layout(int kind, int64_t n, int64_t b, int64_t a) {
  SeqLayout L{};
  L.n = n;
  L.b = b;
  L.a = a;
  int64_t top = 0;
  auto take = [&](int64_t d) {
    int64_t o = top;
    top += (d + 31) / 32 * 32;
    return o;
  };
  L.W = take(n * b * b);
  L.Wtip = take(a * a);
  bool inv = kind != 0;
  L.Lchk = inv ? take(std::max<int64_t>(n - 1, 0) * b * b) : -1;
  L.Lnchk = inv ? take(n * a * b) : -1;
  L.Lam = inv ? take(n * b * b) : -1;
  L.Lamtip = inv ? take(a * a) : -1;
  L.slots = take(n * ntiles(b) + ntiles(a) + 1);
  L.total = top;
  return L;
}

void seq_problem(Problem &P, const SeqLayout &L) {
  int64_t n = L.n, b = L.b, a = L.a;
  int nn = (int)n + (a > 0 ? 1 : 0);
  int A = (int)n;  // arrow node id
  P.size.assign(nn, (int)b);
  if (a > 0) P.size[A] = (int)a;
  P.elim.assign(nn, 1);
  P.accum.assign(nn, 0);
  if (a > 0) P.accum[A] = 1;
  P.rowbase.resize(nn);
  for (int i = 0; i < nn; ++i) P.rowbase[i] = (int64_t)i * b;
  P.rows.assign(nn, {});
  P.W.resize(nn);
  P.Lam.resize(nn);
  P.slot.resize(nn);
  for (int i = 0; i < (int)n; ++i) {
    BlkRef d;
    d.base = Loc{BUF_DIAG, (int32_t)b, (int64_t)i * b * b};
    d.rows = d.cols = (int)b;
    d.valid = true;
    P.blk[{i, i}] = d;
    if (i + 1 < (int)n) {
      BlkRef l;
      l.base = Loc{BUF_LOWER, (int32_t)b, (int64_t)i * b * b};
      l.rows = l.cols = (int)b;
      l.valid = true;
      P.blk[{i + 1, i}] = l;
      P.rows[i].push_back(i + 1);
    }
    if (a > 0) {
      BlkRef ar;
      ar.base = Loc{BUF_ARROW, (int32_t)b, (int64_t)i * a * b};
      ar.rows = (int)a;
      ar.cols = (int)b;
      ar.valid = true;
      P.blk[{A, i}] = ar;
      P.rows[i].push_back(A);
    }
    P.W[i] = Loc{BUF_WS, (int32_t)b, L.W + (int64_t)i * b * b};
    P.Lam[i] = Loc{BUF_WS, (int32_t)b, L.Lam >= 0 ? L.Lam + (int64_t)i * b * b : 0};
    if (L.Lchk >= 0 && i + 1 < (int)n) P.Lchk[{i + 1, i}] = Loc{BUF_WS, (int32_t)b, L.Lchk + (int64_t)i * b * b};
    if (L.Lnchk >= 0 && a > 0) P.Lchk[{A, i}] = Loc{BUF_WS, (int32_t)b, L.Lnchk + (int64_t)i * a * b};
    P.slot[i] = (int64_t)i * ntiles(b);
  }
  if (a > 0) {
    BlkRef t;
    t.base = Loc{BUF_TIP, (int32_t)a, 0};
    t.rows = t.cols = (int)a;
    t.valid = true;
    P.blk[{A, A}] = t;
    P.W[A] = Loc{BUF_WS, (int32_t)a, L.Wtip};
    P.Lam[A] = Loc{BUF_WS, (int32_t)a, L.Lamtip >= 0 ? L.Lamtip : 0};
    P.slot[A] = n * ntiles(b);
  }
}

}  // namespace

int64_t sequential_ws_bytes(int kind, int64_t n, int64_t b, int64_t a) {
  return seq_layout(kind, n, b, a).total * 8;
}

Graph build_sequential(int kind, int64_t n, int64_t b, int64_t a, const BuildOptions &opt) {
  SeqLayout L = seq_layout(kind, n, b, a);
  Problem P;
  seq_problem(P, L);
  Builder bld(P, opt);
  bld.ws_top = L.total;
  bld.slot_region = L.slots;
  int nn = (int)P.size.size();
  bool fact = kind != 1, inv = kind != 0;
  if (fact) {
    for (int X = 0; X < nn; ++X) bld.factor_node(X, true);
    bld.slot_top = n * ntiles(b) + ntiles(a);
    bld.logdet_task(bld.slot_top);
  }
  if (inv) {
    for (int X = 0; X < nn; ++X) bld.precompute_node(X, fact);
    for (int X = nn - 1; X >= 0; --X) bld.invert_node(X);
  }
  Graph g = bld.finalize();
  g.ws_doubles = L.total;
  return g;
}

bool plan_partitions(int64_t n, int P, double r, std::vector<int64_t> &starts) {
  starts.clear();
  if (P < 1 || n < 1) return false;
  if (P == 1) {
    starts = {0, n};
    return true;
  }
  if (n < 2 * (int64_t)P - 1) return false;
  int64_t top = (int64_t)std::floor(r * (double)n / (r + (double)(P - 1)));
  top = std::max<int64_t>(1, std::min<int64_t>(top, n - 2 * (int64_t)(P - 1)));
  int64_t rest = n - top, base = rest / (P - 1), rem = rest % (P - 1);
  starts.push_back(0);
  starts.push_back(top);
  int64_t s = top;
  for (int p = 1; p < P; ++p) {
    s += base + ((p - 1) < rem ? 1 : 0);
    starts.push_back(s);
  }
  return s == n;
}

}  // namespace serinv

namespace serinv {
Graph build_pselinv(int64_t, int64_t, int64_t, int, double, const BuildOptions &) {
  Graph g;
  g.error = "pselinv not built yet";
  return g;
}
int64_t pselinv_ws_bytes(int64_t, int64_t, int64_t, int, double) { return 0; }
Graph build_distributed(int, int, int, int64_t, int64_t, int64_t, int64_t, int64_t, const BuildOptions &) {
  Graph g;
  g.error = "distributed not built yet";
  return g;
}
int64_t distributed_ws_bytes(int, int, int64_t, int64_t, int64_t, int64_t, int64_t) { return 0; }
int64_t exchange_doubles(int64_t, int64_t) { return 0; }
}  // namespace serinv
