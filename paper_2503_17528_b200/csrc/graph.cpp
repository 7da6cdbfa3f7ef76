// graph.cpp -- lowering of PAPER.md Alg. 1-6 to a tile-task DAG + scheduler.
// See graph.h for the overview and task.h for the task semantics.
//
// Structure
//   Ctx      the graph under construction (tasks, counters, workspace bump
//            allocator, logdet slots, location-keyed "final X" counters) and
//            the scheduler (finalize).
//   Problem  one elimination problem: nodes (blocks) in elimination order and
//            the storage of every structurally non-zero block (Y, X).
//   Builder  lowers one Problem: factor_node (tile right-looking Cholesky,
//            Alg. 1 / Alg. 4 lines 3-12), precompute_node (W = L^{-1},
//            L W, W^T W: "invert L_ii once"), invert_node
//            (Takahashi step, Alg. 2 lines 7-12 / Alg. 6 lines 2-12).
//   build_*  assemble the problems of POBTAF / POBTASI / selinv (sequential),
//            the in-process partitioned pipeline (Alg. 3-6 + Sec. 3.3) and the
//            per-rank distributed graphs.
#include "graph.h"
#include "dist_meta.h"

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <memory>
#include <queue>
#include <unordered_map>

namespace serinv {

int reduced_size(int P, bool tw);

namespace {

constexpr int URGENT_QUEUE = 1 << 20;  // placeholder id, renumbered to ncrit + 1 in finalize

inline int ntiles(int64_t s) { return (int)((s + TILE - 1) / TILE); }
inline int tdim(int64_t s, int t) { return (int)std::min<int64_t>(TILE, s - (int64_t)t * TILE); }

inline Loc at(const Loc &base, int64_t r, int64_t c) {
  Loc l = base;
  l.off += r * (int64_t)base.ld + c;
  return l;
}
inline Loc tileloc(const Loc &base, int q, int c) { return at(base, (int64_t)q * TILE, (int64_t)c * TILE); }
inline Loc wsloc(int64_t off, int64_t ld) { return Loc{BUF_WS, (int32_t)ld, off}; }

// ---------------------------------------------------------------------------
// Graph under construction.
// ---------------------------------------------------------------------------
struct RawTask {
  Task t{};
  std::vector<Seg> segs;
  std::vector<int32_t> waits;  // counters (target = #producers, fixed at finalize)
  std::vector<int32_t> late;   // waits checked late (TF_TRSM3 inputs)
  std::vector<Wait> ext;       // waits on EXTERNAL counters (stream-written), explicit targets
  std::vector<int32_t> sigs;   // counters signalled (own counter first)
  double cost = 0.0;           // ns (scheduler model)
  double flops = 0.0;
  int queue = 0;               // claim queue (0 = bulk)
};

double gemm_flops(int m, int n, const std::vector<Seg> &segs) {
  double k = 0;
  for (auto &s : segs) k += s.k;
  return 2.0 * m * n * k;
}

// Scheduler cost model (ns) for one CTA of a 2-CTA/SM persistent grid.
// Calibrated on B200 task traces (tools/trace.py): bulk GEMM ~85 GFLOP/s per CTA with
// two CTAs per SM, POTRF tile task ~21 us, REDUCE ~10 us.
double task_cost(const RawTask &rt, const BuildOptions &o) {
  const double ns_per_flop = 1.0 / o.cost_gflops;
  switch (rt.t.type) {
    case TK_POTRF: return o.cost_potrf + rt.flops * ns_per_flop * 0.5;
    case TK_TRTRI: return 6000.0;
    case TK_GEMM: return o.cost_gemm_fixed + rt.flops * ns_per_flop;
    case TK_REDUCE: return 6000.0;
    default: return 2000.0;
  }
}

Seg mkseg(Loc A, int ta, Loc Bm, int tb, int k) {
  Seg s{};
  s.A = A;
  s.B = Bm;
  s.k = k;
  s.ta = (int8_t)ta;
  s.tb = (int8_t)tb;
  return s;
}

struct Ctx {
  BuildOptions opt;
  std::vector<RawTask> tasks;
  std::vector<int32_t> own;
  int32_t nctr = 0;
  int64_t ws_top = 0;
  int64_t slot_region = 0, slot_cap = 0, slot_count = 0;
  std::map<std::tuple<int32_t, int64_t, int, int>, int32_t> xrc;  // final-X row/col tile counters by location
  std::vector<int32_t> potrf_ctrs;                                  // every factor-done counter (LOGDET waits)
  std::vector<Wait> ext_default;     // external waits added to every task emitted while set
  std::vector<std::pair<int32_t, int>> fin;  // streaming IO: per node, counter of its final-X tasks + block (-1 tip)
  int32_t arr_ctr = -1;                      // streaming IO: blocks-arrived counter (external)
  int32_t arr_ctr2 = -1;                     // twisted streaming IO: bottom units arrived
  int64_t twist_m = -1;
  std::map<int32_t, double> ext_ns;          // scheduler model: ns per unit of an external counter
  std::vector<char> is_ext;          // counter written by a stream (no producer task)

  int32_t new_ctr() { return nctr++; }
  int32_t new_ext_ctr() {
    int32_t c = nctr++;
    if ((int)is_ext.size() < nctr) is_ext.resize(nctr, 0);
    is_ext[c] = 1;
    return c;
  }
  int64_t alloc(int64_t doubles) {
    int64_t o = ws_top;
    ws_top += (std::max<int64_t>(doubles, 1) + 31) / 32 * 32;
    return o;
  }
  int64_t slots(int64_t k) {
    int64_t s = slot_count;
    slot_count += k;
    if (slot_count > slot_cap) fprintf(stderr, "serinv graph: slot overflow\n");
    return s;
  }
  int32_t ctr_of(int task) const { return own[task]; }
  int32_t XRC(const Loc &base, int tile, int rc) {
    auto k = std::make_tuple(base.buf, base.off, tile, rc);
    auto it = xrc.find(k);
    if (it != xrc.end()) return it->second;
    int32_t c = new_ctr();
    xrc[k] = c;
    return c;
  }
  int emit(RawTask &&rt) {
    if (rt.t.type == TK_GEMM)
      rt.flops = gemm_flops(rt.t.m, rt.t.n, rt.segs) + ((rt.t.flags & TF_POST) ? 2.0 * rt.t.m * rt.t.n * rt.t.n : 0.0) +
                 ((rt.t.flags & TF_SYRK3) ? 2.0 * rt.t.m * rt.t.m * rt.t.n : 0.0);
    if (rt.t.type == TK_POTRF)
      rt.flops = 2.0 * rt.t.m * rt.t.n * [&] { double k = 0; for (auto &sg : rt.segs) k += sg.k; return k; }() +
                 2.0 * rt.t.m * rt.t.m * rt.t.m / 3.0 + ((rt.t.flags & TF_TRSM2) ? 2.0 * rt.t.m3 * rt.t.m * rt.t.m : 0.0) +
                 ((rt.t.flags & TF_TRSM3) ? 2.0 * rt.t.m4 * rt.t.m * rt.t.m : 0.0);
    if (rt.t.type == TK_TRTRI) rt.flops = rt.t.m * (double)rt.t.m * rt.t.m / 3.0;
    rt.cost = task_cost(rt, opt);
    std::sort(rt.waits.begin(), rt.waits.end());
    rt.waits.erase(std::unique(rt.waits.begin(), rt.waits.end()), rt.waits.end());
    std::sort(rt.late.begin(), rt.late.end());
    rt.late.erase(std::unique(rt.late.begin(), rt.late.end()), rt.late.end());
    {
      std::vector<int32_t> lt;
      for (int32_t w : rt.late)
        if (!std::binary_search(rt.waits.begin(), rt.waits.end(), w)) lt.push_back(w);
      rt.late.swap(lt);
    }
    for (const Wait &w : ext_default) rt.ext.push_back(w);
    int id = (int)tasks.size();
    int32_t o = new_ctr();
    rt.sigs.insert(rt.sigs.begin(), o);
    own.push_back(o);
    tasks.push_back(std::move(rt));
    return id;
  }

  // ---- data-movement tasks ---------------------------------------------
  // out (rows x cols, row-major) = op(src), tiles of 64 x 64; src is cols x rows if trans
  void copy_block(Loc out, Loc src, int rows, int cols, bool trans, const std::vector<int32_t> &waits,
                  const std::vector<int32_t> &sigs_all, std::function<void(RawTask &, int, int)> tile_sigs = nullptr) {
    for (int q = 0; q < ntiles(rows); ++q)
      for (int c = 0; c < ntiles(cols); ++c) {
        RawTask rt;
        rt.t.type = TK_COPY;
        rt.t.m = (int16_t)tdim(rows, q);
        rt.t.n = (int16_t)tdim(cols, c);
        rt.t.out = tileloc(out, q, c);
        rt.t.c0 = trans ? tileloc(src, c, q) : tileloc(src, q, c);
        rt.t.alpha = 1.0;
        if (trans) rt.t.flags = TF_TRANS_C0;
        rt.waits = waits;
        rt.sigs = sigs_all;
        if (tile_sigs) tile_sigs(rt, q, c);
        emit(std::move(rt));
      }
  }
  void sig_xblock(RawTask &rt, const Loc &base, int q, int c) {
    rt.sigs.push_back(XRC(base, q, 0));
    rt.sigs.push_back(XRC(base, c, 1));
  }
  // out = beta * C0 + alpha * sum_{j<cnt} P_j (P_j at src + j*stride), tiled
  void reduce_block(Loc out, Loc c0, double beta, Loc src, int64_t stride, int cnt, double alpha, int rows, int cols,
                    const std::vector<int32_t> &waits, const std::vector<int32_t> &sigs) {
    for (int q = 0; q < ntiles(rows); ++q)
      for (int c = 0; c < ntiles(cols); ++c) {
        RawTask rt;
        rt.t.type = TK_REDUCE;
        rt.t.m = (int16_t)tdim(rows, q);
        rt.t.n = (int16_t)tdim(cols, c);
        rt.t.out = tileloc(out, q, c);
        rt.t.c0 = tileloc(c0, q, c);
        rt.t.beta = beta;
        rt.t.r = tileloc(src, q, c);
        rt.t.aux2 = stride;
        rt.t.aux0 = cnt;
        rt.t.alpha = alpha;
        rt.waits = waits;
        rt.sigs = sigs;
        emit(std::move(rt));
      }
  }
  // *out = 2 * sum slots[slot0 .. slot0+ns) + sum_{j<ne} extra[j*stride]  (fixed order; NaN if info)
  int logdet(Loc out, int64_t slot0, int64_t ns, Loc extra, int ne, int64_t stride, const std::vector<int32_t> &waits) {
    RawTask rt;
    rt.t.type = TK_LOGDET;
    rt.t.r = wsloc(slot_region + slot0, 0);
    rt.t.aux0 = (int32_t)ns;
    rt.t.c0 = extra;
    rt.t.aux1 = ne;
    rt.t.aux2 = stride;
    rt.t.out = out;
    rt.waits = waits;
    for (int32_t c : potrf_ctrs) rt.waits.push_back(c);
    return emit(std::move(rt));
  }

  Graph finalize();
};

// ---------------------------------------------------------------------------
// Lowering of one elimination problem.
// ---------------------------------------------------------------------------
struct Builder {
  Ctx &cx;
  Problem &P;
  std::unordered_map<uint64_t, int> Lprod;  // L tile producers
  std::unordered_map<uint64_t, int32_t> Lctr;  // L tiles published on a counter other than their producer's own
  int32_t lwait(uint64_t key) {
    auto it = Lctr.find(key);
    return it != Lctr.end() ? it->second : cx.ctr_of(Lprod.at(key));
  }
  struct TileState {
    std::vector<std::pair<int, int>> pending;  // columns (X, c) not yet applied
    int last = -1;
    bool written = false;
  };
  std::unordered_map<uint64_t, TileState> tstate;
  std::map<int, int32_t> factordone, predone;
  std::map<std::tuple<int, int, int>, int32_t> lcol;
  std::map<int64_t, int> wdiag_task;
  std::map<std::tuple<int, int, int>, int> lam_task;
  std::vector<int32_t> input_waits;  // extra waits for tasks reading the problem's inputs
  int flush_queue = 0;               // claim queue of update tasks being flushed
  int concurrency = 1;               // independent chains whose inversion waves overlap (twisted: 2)
  std::map<int, int> last_chain_ts;  // carried chain: last chain TRSM+SYRK task per claim queue
  // wide (128-row) tasks for a wave of `tiles` independent 64 x 64 output tiles
  bool use_wide(int tiles) const {
    return cx.opt.wide_min_wave > 0 && tiles * std::max(1, concurrency) >= cx.opt.wide_min_wave;
  }

  Builder(Ctx &c, Problem &p) : cx(c), P(p) {}

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
  int32_t gctr(std::map<int, int32_t> &m, int k) {
    auto it = m.find(k);
    if (it != m.end()) return it->second;
    int32_t c = cx.new_ctr();
    m[k] = c;
    return c;
  }
  int32_t lcol_ctr(int Z, int X, int c) {
    auto k = std::make_tuple(Z, X, c);
    auto it = lcol.find(k);
    if (it != lcol.end()) return it->second;
    int32_t v = cx.new_ctr();
    lcol[k] = v;
    return v;
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
  int32_t XR(int Y, int X, int q) { return cx.XRC(B(Y, X).base, q, 0); }
  int32_t XC(int Y, int X, int c) { return cx.XRC(B(Y, X).base, c, 1); }

  // workspace for W, Lambda, Lchk of every eliminated node; logdet slots
  void allocate(bool inverse) {
    int nn = (int)P.size.size();
    P.W.assign(nn, Loc{});
    P.Lam.assign(nn, Loc{});
    P.slot.assign(nn, -1);
    for (int X = 0; X < nn; ++X) {
      if (!P.elim[X]) continue;
      int64_t s = P.size[X];
      P.W[X] = wsloc(cx.alloc(s * s), s);
      P.slot[X] = cx.slots(ntiles(s));
      if (inverse) {
        P.Lam[X] = wsloc(cx.alloc(s * s), s);
        for (int Z : P.rows[X]) P.Lchk[{Z, X}] = wsloc(cx.alloc((int64_t)P.size[Z] * s), s);
      }
    }
    if (inverse) allocate_split();
  }

  // =================================================================== factor
  struct RT {
    int Y, q, h;
    Loc loc;
  };
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
  uint64_t tkey(int Yi, int Yj, int qi, int qj) { return key4(Yi, qi, Yj, qj); }

  void add_update_segs(RawTask &rt, int Yi, int qi, int Yj, int qj, const std::vector<std::pair<int, int>> &cols) {
    size_t s = 0;
    while (s < cols.size()) {
      int X = cols[s].first, c0 = cols[s].second;
      size_t e = s + 1;
      while (e < cols.size() && cols[e].first == X && cols[e].second == cols[e - 1].second + 1) ++e;
      int c1 = cols[e - 1].second;
      const BlkRef &bi = (Yi == X) ? B(X, X) : B(Yi, X);
      const BlkRef &bj = (Yj == X) ? B(X, X) : B(Yj, X);
      int k = (int)(std::min<int64_t>((int64_t)(c1 + 1) * TILE, P.size[X]) - (int64_t)c0 * TILE);
      rt.segs.push_back(mkseg(tileloc(bi.base, qi, c0), 0, tileloc(bj.base, qj, c0), 1, k));
      for (size_t u = s; u < e; ++u) {
        int c = cols[u].second;
        rt.waits.push_back(lwait(key4(Yi, qi, X, c)));
        rt.waits.push_back(lwait(key4(Yj, qj, X, c)));
      }
      s = e;
    }
  }

  void update_task(int Yi, int qi, int Yj, int qj, const BlkRef &tb, TileState &st,
                   const std::vector<std::pair<int, int>> &cols) {
    RawTask rt;
    rt.t.type = TK_GEMM;
    rt.t.m = (int16_t)tdim(P.size[Yi], qi);
    rt.t.n = (int16_t)tdim(P.size[Yj], qj);
    rt.t.out = tileloc(tb.base, qi, qj);
    rt.t.c0 = rt.t.out;
    rt.t.alpha = -1.0;
    rt.t.beta = (!st.written && tb.zero_init) ? 0.0 : 1.0;
    add_update_segs(rt, Yi, qi, Yj, qj, cols);
    if (st.last >= 0) rt.waits.push_back(cx.ctr_of(st.last));
    for (int32_t w : input_waits) rt.waits.push_back(w);
    rt.queue = flush_queue;
    st.last = cx.emit(std::move(rt));
    st.written = true;
  }

  // pending updates of a tile -> update tasks of up to update_group columns, except the
  // last keep_last (fused by the caller).  split_last: the newest opt.split_last flushed
  // columns are tasks of their own -- for tiles a carried chain task awaits: a grouped
  // task starts only when its newest column is ready and then runs G x longer, on the
  // chain (measured at C3: a 4-column update, 26 us, bound every chain step).
  void flush(int Yi, int qi, int Yj, int qj, const BlkRef &tb, TileState &st, size_t keep_last,
             bool split_last = false) {
    size_t upto = st.pending.size() - std::min(keep_last, st.pending.size());
    size_t s = 0;
    const int G = cx.opt.update_group;
    const bool whole = P.accum[Yj] != 0;
    const size_t ns = (size_t)std::max(0, cx.opt.split_last);  // newest columns as single tasks
    const size_t cut = (split_last && !whole) ? upto - std::min(ns, upto) : upto;
    while (s < upto) {
      std::vector<std::pair<int, int>> g;
      int X0 = st.pending[s].first;
      size_t e = s;
      const size_t lim = s < cut ? cut : upto;
      const int gmax = s < cut ? G : 1;
      while (e < lim && st.pending[e].first == X0 && (whole || (int)g.size() < gmax)) g.push_back(st.pending[e++]);
      update_task(Yi, qi, Yj, qj, tb, st, g);
      s = e;
    }
    st.pending.erase(st.pending.begin(), st.pending.begin() + upto);
  }

  void factor_node(int X) {
    int nt = ntiles(P.size[X]);
    const BlkRef &d = B(X, X);
    int32_t fd = gctr(factordone, X);
    cx.potrf_ctrs.push_back(fd);
    for (int c = 0; c < nt; ++c) {
      int w = tdim(P.size[X], c);
      std::vector<RT> rts = column_rows(X, c);
      size_t first_trsm = 0;
      // carried chain only for large blocks: there the FP64 work hides the serialised
      // TRSM+SYRK and the freed SM helps (C3 954 -> 937 ms); for b <= 1024 the split
      // chain's overlap wins (C2 57.1 vs 58.2 ms)
      const bool carry = cx.opt.carry_chain && cx.opt.critical_queues && cx.opt.split_chain && cx.opt.chain_syrk &&
                         !cx.opt.fuse_trsm && P.q1(X) > 0 && (P.size[X] >= cx.opt.carry_min_b || cx.opt.chain_step);
      uint64_t step_dk = ~0ull;  // next diagonal tile updated inside a fused chain step
      {  // POTRF of the diagonal tile with the last update fused in (+ the sub-diagonal TRSM)
        TileState &st = tstate[tkey(X, X, c, c)];
        // carried chain: the tile's last writer is the chain TRSM+SYRK that ran just
        // before on this claim queue (same CTA), which left the tile in shared memory
        const bool carry_in = carry && st.pending.empty() && st.last >= 0 && last_chain_ts.count(P.q1(X)) &&
                              last_chain_ts[P.q1(X)] == st.last;
        flush(X, c, X, c, d, st, 1);
        RawTask rt;
        rt.t.type = TK_POTRF;
        rt.t.m = rt.t.n = (int16_t)w;
        rt.t.out = tileloc(d.base, c, c);
        rt.t.c0 = rt.t.out;
        rt.t.alpha = -1.0;
        rt.t.beta = 1.0;
        if (!st.pending.empty()) add_update_segs(rt, X, c, X, c, st.pending);
        rt.t.nseg1 = (int32_t)rt.segs.size();
        if (st.last >= 0) rt.waits.push_back(cx.ctr_of(st.last));
        for (int32_t iw : input_waits) rt.waits.push_back(iw);
        rt.t.flags = TF_W_OUT | (cx.opt.chol8 ? TF_CHOL8 : 0) | (carry_in ? TF_CARRY : 0);
        rt.t.out2 = tileloc(P.W[X], c, c);
        rt.t.aux0 = (int32_t)(P.slot[X] + c);
        rt.t.r = wsloc(cx.slot_region + P.slot[X] + c, 0);
        rt.t.aux1 = (int32_t)(P.rowbase[X] + (int64_t)c * TILE);
        rt.sigs.push_back(fd);
        TileState *st0 = nullptr;
        if (cx.opt.fuse_trsm && !rts.empty()) {
          const RT &r0 = rts[0];
          const BlkRef &tb0 = (r0.Y == X) ? d : B(r0.Y, X);
          st0 = &tstate[tkey(r0.Y, X, r0.q, c)];
          flush(r0.Y, r0.q, X, c, tb0, *st0, 1);
          if (!st0->pending.empty()) add_update_segs(rt, r0.Y, r0.q, X, c, st0->pending);
          if (st0->last >= 0) rt.waits.push_back(cx.ctr_of(st0->last));
          rt.t.flags |= TF_TRSM2;
          rt.t.out3 = r0.loc;
          rt.t.m3 = r0.h;
          rt.t.beta3 = (!st0->written && tb0.zero_init) ? 0.0 : 1.0;
          if (r0.Y == X) rt.t.zmask |= 1;  // zero tile (c, c+1) = out + TILE columns
          first_trsm = 1;
        }
        rt.t.nseg2 = (int32_t)rt.segs.size();
        // fused carried chain step (TF_CHAINSTEP): this task also computes the first
        // sub-diagonal tile E W^T and applies its SYRK to the next diagonal tile,
        // keeping W, E and the updated next tile in shared memory (same CTA); E's and
        // the next tile's earlier updates are bulk tasks, awaited late
        TileState *stE = nullptr, *stD = nullptr;
        int32_t step_sctr = -1;
        if (carry && cx.opt.chain_step && first_trsm == 0 && !rts.empty() && rts[0].h == TILE && w == TILE &&
            has(rts[0].Y, rts[0].Y)) {
          const RT &r0 = rts[0];
          const BlkRef &tbE = (r0.Y == X) ? d : B(r0.Y, X);
          const BlkRef &bd = B(r0.Y, r0.Y);
          const uint64_t dk = tkey(r0.Y, r0.Y, r0.q, r0.q);
          if (!(bd.zero_init && !tstate[dk].written) && !(tbE.zero_init && !tstate[tkey(r0.Y, X, r0.q, c)].written)) {
            stE = &tstate[tkey(r0.Y, X, r0.q, c)];
            flush(r0.Y, r0.q, X, c, tbE, *stE, 0);
            stD = &tstate[dk];
            flush(r0.Y, r0.q, r0.Y, r0.q, bd, *stD, 0);
            if (stE->last >= 0) rt.late.push_back(cx.ctr_of(stE->last));
            if (stD->last >= 0) rt.late.push_back(cx.ctr_of(stD->last));
            rt.t.flags |= TF_CHAINSTEP;
            rt.t.out3 = r0.loc;
            rt.t.m3 = r0.h;
            rt.t.out4 = tileloc(bd.base, r0.q, r0.q);
            rt.t.m4 = r0.h;
            if (r0.Y == X) rt.t.zmask |= 1;  // zero tile (c, c+1) = out + TILE columns
            step_dk = dk;
            first_trsm = 1;  // rts[0] is done here
          }
        }
        TileState *st1 = nullptr;
        if (first_trsm == 1 && cx.opt.fuse_trsm3 && rts.size() >= 2) {
          // the second sub-diagonal tile: its own inputs (a bulk TRSM of the previous
          // column, earlier updates) are awaited late, after the POTRF
          const RT &r1 = rts[1];
          const BlkRef &tb1 = (r1.Y == X) ? d : B(r1.Y, X);
          st1 = &tstate[tkey(r1.Y, X, r1.q, c)];
          flush(r1.Y, r1.q, X, c, tb1, *st1, 1);
          RawTask tmp;
          if (!st1->pending.empty()) add_update_segs(tmp, r1.Y, r1.q, X, c, st1->pending);
          for (auto &sg : tmp.segs) rt.segs.push_back(sg);
          rt.late = tmp.waits;
          if (st1->last >= 0) rt.late.push_back(cx.ctr_of(st1->last));
          rt.t.flags |= TF_TRSM3;
          rt.t.out4 = r1.loc;
          rt.t.m4 = r1.h;
          rt.t.beta4 = (!st1->written && tb1.zero_init) ? 0.0 : 1.0;
          if (r1.Y == X) rt.t.zmask |= 2;  // zero tile (c, c+2)
          first_trsm = 2;
        }
        rt.queue = cx.opt.critical_queues ? P.q1(X) : 0;
        // the own counter (first signal) only guards W = L^{-1}: readers of the
        // factor tile and the log-det slot wait on the factor-done counter fd, and
        // readers of a fused TRSM's tile on its own counter (published at the end)
        int32_t sctr = -1, wctr = -1;
        const bool is_step = (rt.t.flags & TF_CHAINSTEP) != 0;
        if (is_step) {
          // chain step: sigs[0] (own) at the end -- it guards the next diagonal tile --
          // sigs[1] = W (early), sigs[2] = the sub-diagonal tile (mid-task)
          rt.t.flags |= TF_EARLY_SIG;
          wctr = cx.new_ctr();
          sctr = cx.new_ctr();
          rt.sigs.insert(rt.sigs.begin(), sctr);
          rt.sigs.insert(rt.sigs.begin(), wctr);
        } else if (!(rt.t.flags & TF_TRSM3) && cx.opt.early_sig) {
          rt.t.flags |= TF_EARLY_SIG;
          if (rt.t.flags & TF_TRSM2) {
            sctr = cx.new_ctr();
            rt.sigs.push_back(sctr);
          }
        }
        step_sctr = sctr;
        int id = cx.emit(std::move(rt));  // emit puts the own counter first: [own, wctr, sctr, ...]
        if (sctr >= 0) Lctr[key4(rts[0].Y, rts[0].q, X, c)] = sctr;
        if (wctr >= 0) Lctr[key4(X, c, X, c)] = wctr;
        if (is_step) {
          last_chain_ts[P.q1(X)] = id;
          stE->pending.clear();
          stE->last = id;
          stE->written = true;
          Lprod[key4(rts[0].Y, rts[0].q, X, c)] = id;
          stD->pending.clear();
          stD->last = id;
          stD->written = true;
        }
        (void)step_sctr;
        st.pending.clear();
        st.last = id;
        st.written = true;
        Lprod[key4(X, c, X, c)] = id;
        wdiag_task[(int64_t)X * 4096 + c] = id;
        if (st0) {
          st0->pending.clear();
          st0->last = id;
          st0->written = true;
          Lprod[key4(rts[0].Y, rts[0].q, X, c)] = id;
        }
        if (st1) {
          st1->pending.clear();
          st1->last = id;
          st1->written = true;
          Lprod[key4(rts[1].Y, rts[1].q, X, c)] = id;
        }
      }
      uint64_t fused_diag = step_dk;  // next diagonal tile whose column-(X,c) update is fused (step or chain TRSM)
      for (size_t ri = first_trsm; ri < rts.size(); ++ri) {  // TRSM = (A - last update) W(c,c)^T
        const RT &r = rts[ri];
        const BlkRef &tb = (r.Y == X) ? d : B(r.Y, X);
        TileState &st = tstate[tkey(r.Y, X, r.q, c)];
        // updates feeding the chain's next two tiles are near-critical: urgent queue
        const bool near = cx.opt.critical_queues && cx.opt.split_chain && cx.opt.urgent_ctas > 0 && ri < 2;
        flush_queue = near ? URGENT_QUEUE : 0;
        // carried chain TRSM+SYRK: runs on the POTRF's CTA right after it (W in shared
        // memory), so all of its tile's earlier updates are flushed to bulk tasks
        bool chain_carry = false;
        if (carry && ri == 0 && first_trsm == 0 && has(r.Y, r.Y)) {
          const BlkRef &bd = B(r.Y, r.Y);
          const TileState &sd0 = tstate[tkey(r.Y, r.Y, r.q, r.q)];
          chain_carry = !(bd.zero_init && !sd0.written) && r.h == TILE && w == TILE;
        }
        flush(r.Y, r.q, X, c, tb, st, chain_carry ? 0 : 1, chain_carry && cx.opt.split_last > 0);
        RawTask rt;
        rt.t.type = TK_GEMM;
        rt.t.m = (int16_t)r.h;
        rt.t.n = (int16_t)w;
        rt.t.out = r.loc;
        rt.t.c0 = r.loc;
        rt.t.alpha = -1.0;
        rt.t.beta = (!st.written && tb.zero_init) ? 0.0 : 1.0;
        if (!st.pending.empty())
          add_update_segs(rt, r.Y, r.q, X, c, st.pending);
        else
          rt.t.alpha = 0.0;
        if (st.last >= 0) rt.waits.push_back(cx.ctr_of(st.last));
        for (int32_t iw : input_waits) rt.waits.push_back(iw);
        TileState *sdp = nullptr;
        uint64_t dk = tkey(r.Y, r.Y, r.q, r.q);
        if (cx.opt.split_chain && cx.opt.chain_syrk && ri == 0 && first_trsm == 0 && has(r.Y, r.Y)) {
          const BlkRef &bd = B(r.Y, r.Y);
          TileState &sd = tstate[dk];
          if (!(bd.zero_init && !sd.written)) {
            // the chain: L(K+1,K) = E W_K^T, then the next diagonal tile -= L L^T here,
            // so the next POTRF starts from a fully updated tile.  The update of E runs
            // while POTRF(K) is still busy: W_K and the diagonal tile's earlier updates
            // are awaited late.
            flush(r.Y, r.q, r.Y, r.q, bd, sd, 0, chain_carry && cx.opt.split_last > 0);
            flush_queue = 0;
            rt.t.flags = TF_SYRK3;
            rt.t.out3 = tileloc(bd.base, r.q, r.q);
            rt.t.m3 = r.h;
            rt.late.push_back(lwait(key4(X, c, X, c)));
            if (sd.last >= 0) rt.late.push_back(cx.ctr_of(sd.last));
            sdp = &sd;
            fused_diag = dk;
          }
        }
        if (!sdp) rt.waits.push_back(lwait(key4(X, c, X, c)));  // W(c,c)
        rt.t.flags |= TF_POST | TF_POST_T;
        rt.t.r = tileloc(P.W[X], c, c);
        if (r.Y == X) {
          rt.t.flags |= TF_ZERO_MIRROR;
          rt.t.out2 = tileloc(d.base, c, r.q);
        }
        rt.sigs.push_back(fd);
        // the sub-diagonal TRSMs feed the next POTRF: critical queues too
        flush_queue = 0;
        if (chain_carry && sdp) rt.t.flags |= TF_CARRY;
        if (cx.opt.critical_queues) {
          if (chain_carry && sdp) rt.queue = P.q1(X);
          else if (cx.opt.split_chain && first_trsm == 0 && ri == 0) rt.queue = P.q2(X);
          else if (cx.opt.split_chain && first_trsm == 0 && ri == 1 && cx.opt.rts1_chain) rt.queue = P.q2(X);
          else if (cx.opt.split_chain && first_trsm == 0 && ri == 1 && cx.opt.urgent_ctas > 0) rt.queue = URGENT_QUEUE;
          else if (ri == first_trsm && first_trsm == 1 && cx.opt.fuse_trsm) rt.queue = P.q1(X);
        }
        const bool is_carry = (rt.t.flags & TF_CARRY) != 0;
        const int rq = rt.queue;
        int id = cx.emit(std::move(rt));
        if (is_carry) last_chain_ts[rq] = id;
        st.pending.clear();
        st.last = id;
        st.written = true;
        Lprod[key4(r.Y, r.q, X, c)] = id;
        if (sdp) {
          sdp->pending.clear();
          sdp->last = id;
          sdp->written = true;
        }
      }
      for (size_t j = 0; j < rts.size(); ++j)
        for (size_t i = j; i < rts.size(); ++i) {
          const RT &ri = rts[i], &rj = rts[j];
          if (ri.Y == rj.Y && ri.q < rj.q) continue;
          if (rj.Y != X && ri.Y != rj.Y && !has(ri.Y, rj.Y)) continue;
          const uint64_t k = tkey(ri.Y, rj.Y, ri.q, rj.q);
          if (k == fused_diag) continue;  // applied by the fused SYRK of the chain TRSM
          tstate[k].pending.push_back({X, c});
        }
    }
  }

  // all pending updates of non-eliminated (boundary) targets become tasks;
  // their last writers are appended to `done`
  void flush_boundary(std::vector<int32_t> &done) {
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
    for (uint64_t k : keys) done.push_back(cx.ctr_of(tstate[k].last));
  }

  // ========================================================= inverse precompute
  void precompute_node(int X, bool have_wdiag) {
    int nt = ntiles(P.size[X]);
    const BlkRef &d = B(X, X);
    int32_t fd = have_wdiag ? gctr(factordone, X) : -1;
    int32_t pre = gctr(predone, X);
    std::vector<std::vector<int>> Wt(nt, std::vector<int>(nt, -1));
    for (int c = 0; c < nt; ++c) {
      if (have_wdiag) {
        Wt[c][c] = wdiag_task.at((int64_t)X * 4096 + c);
      } else {
        RawTask rt;
        rt.t.type = TK_TRTRI;
        rt.t.m = rt.t.n = (int16_t)tdim(P.size[X], c);
        rt.t.c0 = tileloc(d.base, c, c);
        rt.t.out = tileloc(P.W[X], c, c);
        rt.t.aux1 = (int32_t)(P.rowbase[X] + (int64_t)c * TILE);
        for (int32_t iw : input_waits) rt.waits.push_back(iw);
        rt.sigs.push_back(pre);
        Wt[c][c] = cx.emit(std::move(rt));
      }
    }
    // W(r,c) = -(sum_{k=c+1..r} W(r,k) L(k,c)) W(c,c)     (from W L = I)
    for (int r = 1; r < nt; ++r)
      for (int c = r - 1; c >= 0; --c) {
        RawTask rt;
        rt.t.type = TK_GEMM;
        rt.t.m = (int16_t)tdim(P.size[X], r);
        rt.t.n = (int16_t)tdim(P.size[X], c);
        rt.t.out = tileloc(P.W[X], r, c);
        rt.t.alpha = -1.0;
        rt.t.beta = 0.0;
        int k = (int)(std::min<int64_t>((int64_t)(r + 1) * TILE, P.size[X]) - (int64_t)(c + 1) * TILE);
        rt.segs.push_back(mkseg(tileloc(P.W[X], r, c + 1), 0, tileloc(d.base, c + 1, c), 0, k));
        rt.t.flags = TF_POST;
        rt.t.r = tileloc(P.W[X], c, c);
        for (int kk = c + 1; kk <= r; ++kk) rt.waits.push_back(cx.ctr_of(Wt[r][kk]));
        rt.waits.push_back(cx.ctr_of(Wt[c][c]));
        if (fd >= 0) rt.waits.push_back(fd);
        for (int32_t iw : input_waits) rt.waits.push_back(iw);
        rt.sigs.push_back(pre);
        Wt[r][c] = cx.emit(std::move(rt));
      }
    auto wcol_wait = [&](RawTask &rt, int c) {
      for (int r = c; r < nt; ++r) rt.waits.push_back(cx.ctr_of(Wt[r][c]));
    };
    // Lchk(Z,X)(q,c) = sum_{k >= c} L_{Z,X}(q,k) W(k,c)
    for (int Z : P.rows[X]) {
      const BlkRef &bz = B(Z, X);
      Loc lc = P.Lchk.at({Z, X});
      const int nqz = ntiles(P.size[Z]);
      const bool wide = use_wide(nqz * nt);
      for (int c = 0; c < nt; ++c) {
        int32_t lcc = lcol_ctr(Z, X, c);
        for (int q = 0; q < nqz; q += (wide && q + 1 < nqz) ? 2 : 1) {
          const bool two = wide && q + 1 < nqz;
          RawTask rt;
          rt.t.type = TK_GEMM;
          rt.t.m = (int16_t)(tdim(P.size[Z], q) + (two ? tdim(P.size[Z], q + 1) : 0));
          rt.t.n = (int16_t)tdim(P.size[X], c);
          rt.t.out = tileloc(lc, q, c);
          rt.t.alpha = 1.0;
          rt.t.beta = 0.0;
          rt.segs.push_back(mkseg(tileloc(bz.base, q, c), 0, tileloc(P.W[X], c, c), 0,
                                  (int)(P.size[X] - (int64_t)c * TILE)));
          wcol_wait(rt, c);
          if (fd >= 0) rt.waits.push_back(fd);
          for (int32_t iw : input_waits) rt.waits.push_back(iw);
          rt.sigs.push_back(pre);
          rt.sigs.push_back(lcc);
          cx.emit(std::move(rt));
        }
      }
    }
    // Lambda(r,c) = sum_{k >= r} W(k,r)^T W(k,c),  r >= c
    for (int r = 0; r < nt; ++r)
      for (int c = 0; c <= r; ++c) {
        RawTask rt;
        rt.t.type = TK_GEMM;
        rt.t.m = (int16_t)tdim(P.size[X], r);
        rt.t.n = (int16_t)tdim(P.size[X], c);
        rt.t.out = tileloc(P.Lam[X], r, c);
        rt.t.alpha = 1.0;
        rt.t.beta = 0.0;
        rt.segs.push_back(
            mkseg(tileloc(P.W[X], r, r), 1, tileloc(P.W[X], r, c), 0, (int)(P.size[X] - (int64_t)r * TILE)));
        wcol_wait(rt, r);
        wcol_wait(rt, c);
        rt.sigs.push_back(pre);
        lam_task[std::make_tuple(X, r, c)] = cx.emit(std::move(rt));
      }
  }

  // ---- split-K of the Takahashi tile tasks (better packing of the inversion waves)
  int64_t split_base = -1;      // ring of partial tiles: 2 slots x tiles x pieces x TILE^2
  int split_tiles = 0, split_pieces = 0, split_step = 0;
  std::vector<int> last_reduce;  // per (slot, tile): REDUCE that last read the partials

  void allocate_split() {
    if (cx.opt.si_split <= 0) return;
    int nn = (int)P.size.size();
    for (int X = 0; X < nn; ++X) {
      if (!P.elim[X] || P.rows[X].empty()) continue;
      int nt = ntiles(P.size[X]), tiles = nt * (nt + 1) / 2;
      int64_t K = 0;
      for (int Y : P.rows[X]) {
        tiles += ntiles(P.size[Y]) * nt;
        K += P.size[Y];
      }
      split_tiles = std::max(split_tiles, tiles);
      split_pieces = std::max(split_pieces, (int)((K + cx.opt.si_split - 1) / cx.opt.si_split));
    }
    if (split_pieces < 2) return;
    split_base = cx.alloc((int64_t)2 * split_tiles * split_pieces * TILE * TILE);
    last_reduce.assign((size_t)2 * split_tiles, -1);
  }

  static std::vector<Seg> slice(const std::vector<Seg> &segs, int k0, int k1) {
    std::vector<Seg> out;
    int off = 0;
    for (const Seg &sg : segs) {
      int a = std::max(k0, off), b = std::min(k1, off + sg.k);
      if (a < b) {
        Seg t = sg;
        int lo = a - off;
        t.k = b - a;
        t.A.off += sg.ta ? (int64_t)lo * sg.A.ld : lo;
        t.B.off += sg.tb ? lo : (int64_t)lo * sg.B.ld;
        out.push_back(t);
      }
      off += sg.k;
    }
    return out;
  }

  // emit a Takahashi tile task, split along K into partial GEMMs + a fixed-order REDUCE.
  // wave = number of tile tasks of this dependency wave: split only as much as needed
  // to give every CTA of the grid ~2 tasks (big waves are not split at all).
  void emit_split(RawTask &&rt, int tile, int wave) {
    int K = 0;
    for (auto &sg : rt.segs) K += sg.k;
    const int KS = cx.opt.si_split;
    wave *= std::max(1, concurrency);  // independent chains inverted side by side
    const int want = (2 * std::max(1, cx.opt.grid) + wave - 1) / std::max(1, wave);
    int pieces = std::min({split_pieces, (K + KS - 1) / std::max(1, KS), want});
    if (split_base < 0 || KS <= 0 || pieces < 2 || tile >= split_tiles) {
      cx.emit(std::move(rt));
      return;
    }
    int per = (K + pieces - 1) / pieces;
    const int slot = split_step & 1;
    const int64_t tbase = split_base + (((int64_t)slot * split_tiles + tile) * split_pieces) * TILE * TILE;
    int &lr = last_reduce[(size_t)slot * split_tiles + tile];
    std::vector<int32_t> own;
    for (int j = 0; j < pieces; ++j) {
      RawTask pt;
      pt.t.type = TK_GEMM;
      pt.t.m = rt.t.m;
      pt.t.n = rt.t.n;
      pt.t.out = Loc{BUF_WS, TILE, tbase + (int64_t)j * TILE * TILE};
      pt.t.alpha = 1.0;
      pt.t.beta = 0.0;
      pt.segs = slice(rt.segs, j * per, std::min(K, (j + 1) * per));
      pt.waits = rt.waits;
      if (lr >= 0) pt.waits.push_back(cx.ctr_of(lr));  // WAR on the partial slot
      own.push_back(cx.ctr_of(cx.emit(std::move(pt))));
    }
    RawTask red;
    red.t.type = TK_REDUCE;
    red.t.m = rt.t.m;
    red.t.n = rt.t.n;
    red.t.out = rt.t.out;
    red.t.c0 = rt.t.c0;
    red.t.beta = rt.t.beta;
    red.t.alpha = rt.t.alpha;
    red.t.r = Loc{BUF_WS, TILE, tbase};
    red.t.aux2 = (int64_t)TILE * TILE;
    red.t.aux0 = pieces;
    red.t.flags = rt.t.flags & TF_MIRROR;
    red.t.out2 = rt.t.out2;
    red.waits = rt.waits;
    for (int32_t o : own) red.waits.push_back(o);
    red.sigs = rt.sigs;
    lr = cx.emit(std::move(red));
  }

  // X_{Y,Z} row tile q: Y >= Z at blk(Y,Z) (row tile, op N), else blk(Z,Y)^T (col tile, op T)
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

  // ================================================================ Takahashi
  int32_t fin_ctr = -1;  // streaming IO: counter signalled by every final-X task of the node

  void invert_node(int X) {
    int nt = ntiles(P.size[X]);
    int32_t pre = gctr(predone, X);
    const auto &R = P.rows[X];
    int tile = 0;
    int wave1 = 0;
    for (int Y : R) wave1 += ntiles(P.size[Y]) * nt;
    const int wave2 = nt * (nt + 1) / 2;
    const bool wide = use_wide(wave1);
    for (int Y : R) {  // X_{Y,X}(q,c) = -sum_Z X_{Y,Z}(q,:) Lchk(Z,X)(:,c)
      const BlkRef &by = B(Y, X);
      const int nq = ntiles(P.size[Y]);
      for (int q = 0; q < nq; q += (wide && q + 1 < nq) ? 2 : 1) {
        const bool two = wide && q + 1 < nq;  // rows q, q+1 in one wide task
        for (int c = 0; c < nt; ++c) {
          RawTask rt;
          rt.t.type = TK_GEMM;
          rt.t.m = (int16_t)(tdim(P.size[Y], q) + (two ? tdim(P.size[Y], q + 1) : 0));
          rt.t.n = (int16_t)tdim(P.size[X], c);
          rt.t.out = tileloc(by.base, q, c);
          rt.t.alpha = -1.0;
          rt.t.beta = 0.0;
          for (int Z : R) {
            Loc a, a2;
            int tr, k;
            xrow(rt, Y, Z, q, a, tr, k);
            if (two) xrow(rt, Y, Z, q + 1, a2, tr, k);
            rt.segs.push_back(mkseg(a, tr, tileloc(P.Lchk.at({Z, X}), 0, c), 0, k));
            rt.waits.push_back(lcol_ctr(Z, X, c));
          }
          rt.waits.push_back(pre);  // WAR: L_{Y,X} consumed by the precompute
          rt.sigs.push_back(XR(Y, X, q));
          if (two) rt.sigs.push_back(XR(Y, X, q + 1));
          rt.sigs.push_back(XC(Y, X, c));
          if (fin_ctr >= 0) rt.sigs.push_back(fin_ctr);
          if (two) {
            cx.emit(std::move(rt));
            tile += 2;
          } else {
            emit_split(std::move(rt), tile++, wave1);
          }
        }
      }
    }
    // X_{X,X}(r,c) = Lambda(r,c) - sum_Y X_{Y,X}(:,r)^T Lchk(Y,X)(:,c), r >= c, mirrored
    const BlkRef &d = B(X, X);
    const bool wide2 = use_wide(wave2);
    // X_XX tiles (r, c), r >= c; with wide tasks the off-diagonal rows of column c
    // go in pairs (r, r+1), r > c (each mirrored), the diagonal tile alone
    for (int c = 0; c < nt; ++c)
      for (int r = c; r < nt;) {
        const bool two = wide2 && r > c && r + 1 < nt;
        RawTask rt;
        rt.t.type = TK_GEMM;
        rt.t.m = (int16_t)(tdim(P.size[X], r) + (two ? tdim(P.size[X], r + 1) : 0));
        rt.t.n = (int16_t)tdim(P.size[X], c);
        rt.t.out = tileloc(d.base, r, c);
        rt.t.c0 = tileloc(P.Lam[X], r, c);
        rt.t.alpha = R.empty() ? 0.0 : -1.0;
        rt.t.beta = 1.0;
        for (int Y : R) {
          rt.segs.push_back(mkseg(tileloc(B(Y, X).base, 0, r), 1, tileloc(P.Lchk.at({Y, X}), 0, c), 0, P.size[Y]));
          rt.waits.push_back(XC(Y, X, r));
          if (two) rt.waits.push_back(XC(Y, X, r + 1));
          rt.waits.push_back(lcol_ctr(Y, X, c));
        }
        rt.waits.push_back(cx.ctr_of(lam_task.at(std::make_tuple(X, r, c))));
        if (two) rt.waits.push_back(cx.ctr_of(lam_task.at(std::make_tuple(X, r + 1, c))));
        rt.waits.push_back(pre);
        if (r != c) {
          rt.t.flags = TF_MIRROR;
          rt.t.out2 = tileloc(d.base, c, r);
        }
        for (int rr = r; rr <= r + (two ? 1 : 0); ++rr) {
          rt.sigs.push_back(XR(X, X, rr));
          if (rr != c) rt.sigs.push_back(XC(X, X, rr));
        }
        rt.sigs.push_back(XC(X, X, c));
        if (r != c) rt.sigs.push_back(XR(X, X, c));
        if (fin_ctr >= 0) rt.sigs.push_back(fin_ctr);
        if (two) {
          cx.emit(std::move(rt));
          tile += 2;
          r += 2;
        } else {
          emit_split(std::move(rt), tile++, wave2);
          r += 1;
        }
      }
    ++split_step;
  }
};

// ---------------------------------------------------------------------------
// Scheduler: bipartite DAG (tasks -> counters -> tasks), bottom-level
// priorities, list-scheduling simulation on opt.grid workers.
// ---------------------------------------------------------------------------
Graph Ctx::finalize() {
  Graph g;
  const int N = (int)tasks.size();
  const int C = nctr;
  std::vector<int32_t> nprod(C, 0), nwaiter(C, 0);
  for (auto &t : tasks) {
    for (int32_t w : t.late) t.waits.push_back(w);  // the scheduler sees early + late waits
    for (int32_t s : t.sigs) nprod[s]++;
    for (int32_t w : t.waits) nwaiter[w]++;
  }
  std::vector<int64_t> wptr(C + 1, 0);
  for (int c = 0; c < C; ++c) wptr[c + 1] = wptr[c] + nwaiter[c];
  std::vector<int32_t> wlist(wptr[C]);
  {
    std::vector<int64_t> fill(wptr.begin(), wptr.end() - 1);
    for (int i = 0; i < N; ++i)
      for (int32_t w : tasks[i].waits) wlist[fill[w]++] = i;
  }
  for (int i = 0; i < N; ++i)
    for (int32_t w : tasks[i].waits)
      if (nprod[w] == 0) {
        g.error = "counter with no producer";
        return g;
      }
  (void)is_ext;
  std::vector<int32_t> tdeg(N), cdeg(nprod);
  for (int i = 0; i < N; ++i) tdeg[i] = (int32_t)tasks[i].waits.size();
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
      for (int32_t s : tasks[t].sigs)
        if (--cdeg[s] == 0)
          for (int64_t k = wptr[s]; k < wptr[s + 1]; ++k)
            if (--tdeg[wlist[k]] == 0) q.push(wlist[k]);
    }
    if ((int)topo.size() != N) {
      g.error = "dependency cycle";
      return g;
    }
  }
  std::vector<double> bl(N, 0.0), cbl(C, 0.0);
  for (int k = N - 1; k >= 0; --k) {
    int t = topo[k];
    double m = 0;
    for (int32_t s : tasks[t].sigs) m = std::max(m, cbl[s]);
    bl[t] = tasks[t].cost + m;
    for (int32_t w : tasks[t].waits) cbl[w] = std::max(cbl[w], bl[t]);
  }
  std::vector<int> order;
  order.reserve(N);
  if (opt.schedule) {
    auto cmp = [&](int x, int y) {
      if (bl[x] != bl[y]) return bl[x] < bl[y];
      return x > y;
    };
    std::priority_queue<int, std::vector<int>, decltype(cmp)> ready(cmp);
    typedef std::pair<double, int> Ev;
    std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> ev, rel;
    // streaming IO: a task waiting on an external (stream-written) counter is not
    // released before its input units can have arrived (target x ns per unit)
    std::vector<double> release(N, 0.0);
    if (!ext_ns.empty())
      for (int i = 0; i < N; ++i)
        for (const Wait &w : tasks[i].ext) {
          auto it = ext_ns.find(w.ctr);
          if (it != ext_ns.end()) release[i] = std::max(release[i], w.target * it->second);
        }
    double now = 0;
    auto make_ready = [&](int t) {
      if (release[t] > now) rel.push({release[t], t});
      else ready.push(t);
    };
    for (int i = 0; i < N; ++i) tdeg[i] = (int32_t)tasks[i].waits.size();
    cdeg = nprod;
    for (int i = 0; i < N; ++i)
      if (!tdeg[i]) make_ready(i);
    int free_w = std::max(1, opt.grid);
    while ((int)order.size() < N) {
      while (free_w > 0 && !ready.empty()) {
        int t = ready.top();
        ready.pop();
        order.push_back(t);
        ev.push({now + tasks[t].cost, t});
        --free_w;
      }
      if (ev.empty() && rel.empty()) break;
      if (!rel.empty() && (ev.empty() || rel.top().first <= ev.top().first)) {
        now = std::max(now, rel.top().first);
        ready.push(rel.top().second);
        rel.pop();
        continue;
      }
      Ev e = ev.top();
      ev.pop();
      now = e.first;
      ++free_w;
      for (int32_t s : tasks[e.second].sigs)
        if (--cdeg[s] == 0)
          for (int64_t k = wptr[s]; k < wptr[s + 1]; ++k)
            if (--tdeg[wlist[k]] == 0) make_ready(wlist[k]);
    }
    if ((int)order.size() != N) {
      g.error = "schedule incomplete";
      return g;
    }
    g.sim_ns = now;
  } else {
    order = topo;
  }
  g.tasks.reserve(N);
  for (int t : order) {
    RawTask &rt = tasks[t];
    Task task = rt.t;
    task.seg0 = (int32_t)g.segs.size();
    task.nseg = (int32_t)rt.segs.size();
    for (auto &s : rt.segs) g.segs.push_back(s);
    task.wait0 = (int32_t)g.waits.size();
    task.nwait = (int32_t)(rt.waits.size() + rt.ext.size());  // early (+ external) waits, then nlate late
    task.nlate = (int32_t)rt.late.size();
    const size_t nearly = rt.waits.size() - rt.late.size();
    for (size_t k = 0; k < nearly; ++k) g.waits.push_back(Wait{rt.waits[k], nprod[rt.waits[k]]});
    for (const Wait &w : rt.ext) g.waits.push_back(w);
    for (size_t k = nearly; k < rt.waits.size(); ++k) g.waits.push_back(Wait{rt.waits[k], nprod[rt.waits[k]]});
    task.sig0 = (int32_t)g.sigs.size();
    task.nsig = (int32_t)rt.sigs.size();
    for (int32_t s : rt.sigs) g.sigs.push_back(s);
    g.tasks.push_back(task);
    g.flops += rt.flops;
  }
  {  // compact the critical queue ids (a carried chain leaves its TRSM queue empty)
    std::map<int, int> qmap;
    for (int t : order)
      if (tasks[t].queue > 0 && tasks[t].queue != URGENT_QUEUE) qmap[tasks[t].queue] = 0;
    int k = 0;
    for (auto &kv : qmap) kv.second = ++k;
    for (int t : order)
      if (tasks[t].queue > 0 && tasks[t].queue != URGENT_QUEUE) tasks[t].queue = qmap[tasks[t].queue];
  }
  int ncrit = 0;
  bool has_urgent = false;
  for (int t : order) {
    if (tasks[t].queue == URGENT_QUEUE)
      has_urgent = true;
    else
      ncrit = std::max(ncrit, tasks[t].queue);
  }
  for (int t : order)
    if (tasks[t].queue == URGENT_QUEUE) tasks[t].queue = ncrit + 1;
  g.ncrit = ncrit;
  g.nurgent = has_urgent ? std::max(1, opt.urgent_ctas) : 0;
  int nq = 1;
  for (int t : order) nq = std::max(nq, tasks[t].queue + 1);
  g.qoff.assign(nq + 1, 0);
  for (int t : order) g.qoff[tasks[t].queue + 1]++;
  for (int q = 0; q < nq; ++q) g.qoff[q + 1] += g.qoff[q];
  g.qlist.assign(N, 0);
  {
    std::vector<int32_t> fill(g.qoff.begin(), g.qoff.end() - 1);
    for (int i = 0; i < N; ++i) g.qlist[fill[tasks[order[i]].queue]++] = i;
  }
  g.nctr = nctr;
  g.grid = opt.grid;
  g.ws_doubles = ws_top;
  g.nslots = slot_count;
  for (auto &f : fin) {
    g.fin.push_back(Wait{f.first, nprod[f.first]});
    g.fin_blk.push_back(f.second);
  }
  g.arr_ctr = arr_ctr;
  g.arr_ctr2 = arr_ctr2;
  g.twist_m = twist_m;
  return g;
}

// ---------------------------------------------------------------------------
// Problem constructors
// ---------------------------------------------------------------------------
BlkRef blkref(Loc base, int rows, int cols, bool zero_init = false) {
  BlkRef r;
  r.base = base;
  r.rows = rows;
  r.cols = cols;
  r.zero_init = zero_init;
  r.valid = true;
  return r;
}

// Block families: block i of a family at off + i * stride.
struct Fam {
  int32_t buf;
  int64_t off, stride;
  int32_t ld;
  Loc at(int64_t i) const { return Loc{buf, ld, off + i * stride}; }
};
Fam famD(int64_t b) { return Fam{BUF_DIAG, 0, b * b, (int32_t)b}; }
Fam famL(int64_t b) { return Fam{BUF_LOWER, 0, b * b, (int32_t)b}; }
Fam famA(int64_t b, int64_t a) { return Fam{BUF_ARROW, 0, a * b, (int32_t)b}; }

// The BTA matrix a (nested) partitioned solve works on: block families and the
// global first row of block i (for info); the tip always lives in BUF_TIP.
struct View {
  Fam D, Lo, Ar;
  std::function<int64_t(int64_t)> row;
  int64_t tip_row = 0;
};
View top_view(int64_t n, int64_t b, int64_t a) {
  return View{famD(b), famL(b), famA(b, a), [b](int64_t i) { return i * b; }, n * b};
}

// A BT(A) chain problem: nodes 0..m-1 of size b (diag D(i), lower Lo(i) = (i+1,i),
// arrow Ar(i)), then the arrow node m (size a, storage tip) if a > 0.  Nodes
// [0, elim_upto) are eliminated; the arrow node iff elim_tip.
void chain_problem(Problem &P, int m, int64_t b, int64_t a, std::function<Loc(int)> D, std::function<Loc(int)> Lo,
                   std::function<Loc(int)> Ar, Loc tip, bool tip_zero, int elim_upto, bool elim_tip,
                   std::function<int64_t(int)> rowbase, int64_t tip_rowbase) {
  int nn = m + (a > 0 ? 1 : 0);
  int A = m;
  P.size.assign(nn, (int)b);
  if (a > 0) P.size[A] = (int)a;
  P.elim.assign(nn, 0);
  for (int i = 0; i < elim_upto; ++i) P.elim[i] = 1;
  if (a > 0) P.elim[A] = elim_tip;
  P.accum.assign(nn, 0);
  if (a > 0) P.accum[A] = 1;
  P.rowbase.resize(nn);
  P.rows.assign(nn, {});
  for (int i = 0; i < m; ++i) {
    P.rowbase[i] = rowbase(i);
    P.blk[{i, i}] = blkref(D(i), (int)b, (int)b);
    if (i + 1 < m) {
      P.blk[{i + 1, i}] = blkref(Lo(i), (int)b, (int)b);
      if (i < elim_upto) P.rows[i].push_back(i + 1);
    }
    if (a > 0) {
      P.blk[{A, i}] = blkref(Ar(i), (int)a, (int)b);
      if (i < elim_upto) P.rows[i].push_back(A);
    }
  }
  if (a > 0) {
    P.rowbase[A] = tip_rowbase;
    P.blk[{A, A}] = blkref(tip, (int)a, (int)a, tip_zero);
  }
}

// Middle partition (Alg. 4) on buffers whose block s is at local index ls:
// nodes 0..k-1 = blocks s+1..e-1 (k = e-s-1; node k-1 is the boundary l),
// F = k (block s, moved last by the implicit shifting permutation),
// arrow = k+1.  Bbuf(j) stores the fill-in block (F, node j): rows f, columns j.
void middle_problem(Problem &P, const View &V, int64_t ls, int64_t cnt, int64_t b, int64_t a, Loc U,
                    const Fam &Bbuf, int64_t glob_s) {
  int k = (int)(cnt - 1);
  int F = k, A = k + 1;
  int nn = k + 1 + (a > 0 ? 1 : 0);
  P.size.assign(nn, (int)b);
  if (a > 0) P.size[A] = (int)a;
  P.elim.assign(nn, 0);
  for (int j = 0; j + 1 < k; ++j) P.elim[j] = 1;  // interior s+1..e-2
  P.accum.assign(nn, 0);
  P.accum[F] = 1;
  if (a > 0) P.accum[A] = 1;
  P.rowbase.resize(nn);
  P.rows.assign(nn, {});
  for (int j = 0; j < k; ++j) {
    int64_t li = ls + 1 + j;
    P.rowbase[j] = V.row(glob_s + 1 + j);
    P.blk[{j, j}] = blkref(V.D.at(li), (int)b, (int)b);
    bool el = j + 1 < k;
    if (el) {
      P.blk[{j + 1, j}] = blkref(V.Lo.at(li), (int)b, (int)b);
      P.rows[j].push_back(j + 1);
    }
    // B_{s+1} = A_{s+1,s}^T is copied in; later B_j start as fill-in zeros
    P.blk[{F, j}] = blkref(Bbuf.at(j), (int)b, (int)b, j > 0);
    if (el) P.rows[j].push_back(F);
    if (a > 0) {
      P.blk[{A, j}] = blkref(V.Ar.at(li), (int)a, (int)b);
      if (el) P.rows[j].push_back(A);
    }
  }
  P.rowbase[F] = V.row(glob_s);
  P.blk[{F, F}] = blkref(V.D.at(ls), (int)b, (int)b);
  if (a > 0) {
    P.rowbase[A] = -1;
    P.blk[{A, F}] = blkref(V.Ar.at(ls), (int)a, (int)b);
    P.blk[{A, A}] = blkref(U, (int)a, (int)a, true);
  }
}

int64_t slot_bound(int64_t nblocks, int64_t b, int64_t a) { return nblocks * ntiles(b) + ntiles(a) + 8; }

// Two-sided ("twisted") elimination of the whole BTA matrix, used by the fused
// selinv (kind 2).  Blocks 0..m-1 are eliminated top-down (Alg. 1 as written,
// P:260-271), blocks n-1..m+1 bottom-up (Alg. 1 applied to the block-reversed
// matrix, which is again BTA), the two chains interleaved in one elimination
// order; the meeting block m is eliminated last before the tip.  This is the
// symmetric block permutation [0, n-1, 1, n-2, ..., m, tip] of A: every block
// couples only to its chain successor and the tip, so no fill-in leaves the
// pattern and the flop count is exactly Alg. 1 + Alg. 2; X = A^{-1} on the
// pattern and log det A are permutation invariant (reading R13).  The
// factor L differs from Alg. 1's on the bottom half, so POBTAF alone (kind 0)
// and POBTASI (kind 1) keep the one-sided chain.  The dependent chain is half
// as long: two critical chains run concurrently on their own CTAs.
//
// Bottom-chain couplings A_{j-1,j} = A_{j,j-1}^T (storage lower[j-1]) are
// transposed into workspace T(j) first (row-major factor / inverse storage),
// and X_{j,j-1} = T(j)^T is transposed back into lower[j-1] at the end.
struct Twist {
  int64_t m = 0;
  std::vector<int> pos;           // block -> node
  Fam T{};                        // T(j) at T.at(j - m - 1), j = m+1..n-1
};

// The twisted order pays off where the dependent chain, not the FP64 work, bounds
// the factorisation: the chain has n * b / 64 tile steps of ~30 us, the work
// ~7/3 n b^3 flops (+ the overlapped inversion precompute).  For b >= 2048 the
// one-sided chain already hides under the work (C3), so keep Alg. 1's order.
// scheduler model of the host -> device stream: one unit (diag + lower + arrow
// block) per ~unit bytes / 50 GB/s (PCIe 5 x16, pinned)
double h2d_ns_per_unit(int64_t b, int64_t a) { return (double)(2 * b * b + a * b) * 8.0 / 50.0; }

bool use_twist(int kind, int64_t n, int64_t b, const BuildOptions &opt) {
  return (kind == 2 || kind == 6) && opt.twist_min_n > 0 && n >= std::max(3, opt.twist_min_n) && b <= opt.twist_max_b;
}

// Twisted problem on an arbitrary BTA storage (D, Lo, Ar, tip; row() labels info
// rows): the user matrix (build_twisted_selinv) or an assembled reduced system.
void twisted_problem(Ctx &cx, Problem &P, Twist &tw, int64_t n, int64_t b, int64_t a, const Fam &FD, const Fam &FL,
                     const Fam &FA, Loc tip, const std::function<int64_t(int64_t)> &row, int64_t tip_row) {
  const int64_t m = (n - 1) / 2;
  tw.m = m;
  tw.T = Fam{BUF_WS, cx.alloc((n - 1 - m) * b * b), b * b, (int32_t)b};
  std::vector<int64_t> order;  // node -> block
  for (int64_t k = 0; k < m || k < n - 1 - m; ++k) {
    if (k < m) order.push_back(k);
    if (k < n - 1 - m) order.push_back(n - 1 - k);
  }
  order.push_back(m);
  const int nn = (int)n + (a > 0 ? 1 : 0), A = (int)n;  // node n = tip
  tw.pos.assign(n, 0);
  for (int X = 0; X < (int)n; ++X) tw.pos[order[X]] = X;
  P.size.assign(nn, (int)b);
  if (a > 0) P.size[A] = (int)a;
  P.elim.assign(nn, 1);
  P.accum.assign(nn, 0);
  if (a > 0) P.accum[A] = 1;
  P.rowbase.resize(nn);
  P.rows.assign(nn, {});
  P.nqueue.assign(nn, 1);
  P.nqueue2.assign(nn, 2);
  for (int64_t i = 0; i < n; ++i) {
    const int X = tw.pos[i];
    P.rowbase[X] = row(i);
    P.blk[{X, X}] = blkref(FD.at(i), (int)b, (int)b);
    if (i < m) {  // top chain: successor i+1, L_{i+1,i} in lower[i]
      P.blk[{tw.pos[i + 1], X}] = blkref(FL.at(i), (int)b, (int)b);
      P.rows[X].push_back(tw.pos[i + 1]);
    } else if (i > m) {  // bottom chain: successor i-1, in T(i)
      P.blk[{tw.pos[i - 1], X}] = blkref(tw.T.at(i - m - 1), (int)b, (int)b);
      P.rows[X].push_back(tw.pos[i - 1]);
      P.nqueue[X] = 3;
      P.nqueue2[X] = 4;
    }
    if (a > 0) {
      P.blk[{A, X}] = blkref(FA.at(i), (int)a, (int)b);
      P.rows[X].push_back(A);
    }
  }
  if (a > 0) {
    P.rowbase[A] = tip_row;
    P.blk[{A, A}] = blkref(tip, (int)a, (int)a);
  }
}

// stream_io (kind 6): the host streams units in from both ends (top units
// 0..m on arr_ctr, bottom units n-1..m+1 on arr_ctr2) and each node's outputs
// out as soon as its final-X counter completes (fin, in completion order).
Graph build_twisted_selinv(Ctx &cx, int64_t n, int64_t b, int64_t a, bool stream_io) {
  cx.slot_cap = slot_bound(n, b, a);
  cx.slot_region = cx.alloc(cx.slot_cap);
  Problem P;
  Twist tw;
  twisted_problem(cx, P, tw, n, b, a, famD(b), famL(b), famA(b, a), Loc{BUF_TIP, (int32_t)a, 0},
                  [b](int64_t i) { return i * b; }, n * b);
  Builder bld(cx, P);
  bld.concurrency = 2;
  bld.allocate(true);
  const int nn = (int)P.size.size();
  const int64_t m = tw.m;
  if (stream_io) {
    cx.arr_ctr = cx.new_ext_ctr();
    cx.arr_ctr2 = cx.new_ext_ctr();
    cx.twist_m = m;
    cx.ext_ns[cx.arr_ctr] = cx.ext_ns[cx.arr_ctr2] = 2.0 * h2d_ns_per_unit(b, a);  // the two sides alternate
  }
  // arrival waits: top block i (<= m) present iff arr_ctr >= i + 1, bottom block j
  // (> m, with lower[j-1]) iff arr_ctr2 >= n - j
  auto need = [&](std::vector<Wait> &w, int64_t blk) {
    if (!stream_io) return;
    if (blk <= m) w.push_back(Wait{cx.arr_ctr, (int32_t)(blk + 1)});
    else w.push_back(Wait{cx.arr_ctr2, (int32_t)(n - blk)});
  };
  std::vector<int32_t> tin(n, -1);
  for (int64_t j = m + 1; j < n; ++j) {  // T(j) = A_{j,j-1}^T
    tin[j] = cx.new_ctr();
    cx.ext_default.clear();
    need(cx.ext_default, j);
    cx.copy_block(tw.T.at(j - m - 1), famL(b).at(j - 1), (int)b, (int)b, true, {}, {tin[j]});
  }
  std::vector<int64_t> blk_of(nn, -1);
  for (int64_t i = 0; i < n; ++i) blk_of[tw.pos[i]] = i;
  for (int X = 0; X < nn; ++X) {
    bld.input_waits.clear();
    cx.ext_default.clear();
    const int64_t i = blk_of[X];
    if (i > m) bld.input_waits.push_back(tin[i]);
    if (i >= 0) {  // the column of block i reads blocks i and its chain successor
      need(cx.ext_default, i);
      if (i < m) need(cx.ext_default, i + 1);
      if (i > m) need(cx.ext_default, i - 1);
    } else {
      need(cx.ext_default, m);
    }
    bld.factor_node(X);
  }
  cx.ext_default.clear();
  bld.input_waits.clear();
  cx.logdet(Loc{BUF_LOGDET, 0, 0}, 0, cx.slot_count, Loc{BUF_WS, 0, 0}, 0, 0, {});
  for (int X = 0; X < nn; ++X) bld.precompute_node(X, true);
  for (int X = nn - 1; X >= 0; --X) {
    const int64_t i = blk_of[X];
    if (stream_io) {
      bld.fin_ctr = cx.new_ctr();
      cx.fin.push_back({bld.fin_ctr, (int)i});
    }
    bld.invert_node(X);
    if (i > m) {  // X_{i,i-1} = T(i)^T
      const Loc src = tw.T.at(i - m - 1);
      std::vector<int32_t> w;
      for (int q = 0; q < ntiles(b); ++q) w.push_back(cx.XRC(src, q, 0));
      std::vector<int32_t> s;
      if (bld.fin_ctr >= 0) s.push_back(bld.fin_ctr);
      cx.copy_block(famL(b).at(i - 1), src, (int)b, (int)b, true, w, s);
    }
  }
  return cx.finalize();
}

Graph build_seq_ctx(Ctx &cx, int kind, int64_t n, int64_t b, int64_t a) {
  if (use_twist(kind, n, b, cx.opt)) return build_twisted_selinv(cx, n, b, a, kind == 6);
  bool fact = kind != 1, inv = kind != 0;  // kinds 2 and 6 (selinv, streaming IO) do both
  cx.slot_cap = slot_bound(n, b, a);
  cx.slot_region = cx.alloc(cx.slot_cap);
  Problem P;
  chain_problem(
      P, (int)n, b, a, [&](int i) { return famD(b).at(i); }, [&](int i) { return famL(b).at(i); },
      [&](int i) { return famA(b, a).at(i); }, Loc{BUF_TIP, (int32_t)a, 0}, false, (int)n, true,
      [&](int i) { return (int64_t)i * b; }, n * b);
  P.queue = 1;
  P.queue2 = 2;
  Builder bld(cx, P);
  bld.allocate(inv);
  int nn = (int)P.size.size();
  const bool stream_io = kind == 6;
  if (stream_io) {
    cx.arr_ctr = cx.new_ext_ctr();
    cx.ext_ns[cx.arr_ctr] = h2d_ns_per_unit(b, a);
  }
  if (fact) {
    for (int X = 0; X < nn; ++X) {
      // streaming IO: the column of node X reads blocks X and X+1 (counted in blocks arrived)
      if (stream_io) cx.ext_default = {Wait{cx.arr_ctr, (int32_t)std::min<int64_t>(X + 2, n)}};
      bld.factor_node(X);
    }
    cx.ext_default.clear();
    cx.logdet(Loc{BUF_LOGDET, 0, 0}, 0, cx.slot_count, Loc{BUF_WS, 0, 0}, 0, 0, {});
  }
  if (inv) {
    for (int X = 0; X < nn; ++X) bld.precompute_node(X, fact);
    for (int X = nn - 1; X >= 0; --X) {
      if (stream_io) {
        bld.fin_ctr = cx.new_ctr();
        cx.fin.push_back({bld.fin_ctr, X < (int)n ? X : -1});
      }
      bld.invert_node(X);
    }
  }
  return cx.finalize();
}

// ---------------------------------------------------------------------------
// Partitioned pipeline (shared by the in-process graph and the per-rank graphs)
// ---------------------------------------------------------------------------
struct PartState {
  int p = 0;
  int64_t s = 0, e = 0;  // global block range
  int64_t ls = 0;        // local index of block s in the buffers
  Problem prob;
  std::unique_ptr<Builder> bld;
  Loc U{};                    // a x a tip accumulator
  Fam Bbuf{};                 // fill-in chain (middle partitions)
  std::vector<int32_t> done;  // counters: everything the factor phase wrote
  int nelim = 0;
  int queue = 1;              // critical claim queue of this partition's chain (0: bulk)
  View V;                     // the matrix this partition belongs to
  std::vector<int32_t> inw;   // counters after which the partition's input blocks are ready
  bool bottom = false;        // twisted last partition: eliminated bottom-up, no fill-in (reading R14)
  Fam Tbuf{};                 // bottom: T(j) = A_{j,j-1}^T at Tbuf.at(j - s - 1), j = s+1..e-1
};

// The last partition, eliminated bottom-up (reading R14): the block-reversed
// BTA chain of blocks e-1, e-2, ..., s+1, with block s (its first block) left as
// the boundary node and the arrow node accumulating U_p.  Node k <-> block e-1-k
// (k < cnt-1), node cnt-1 <-> block s, node cnt = arrow.  Couplings A_{j-1,j} =
// A_{j,j-1}^T live transposed in Tbuf (row-major factor / inverse storage).
void bottom_problem(Problem &P, const View &V, int64_t ls, int64_t cnt, int64_t b, int64_t a, Loc U, const Fam &Tb,
                    int64_t glob_s) {
  const int nb = (int)cnt;  // nodes 0..cnt-1 = blocks e-1 .. s
  const int A = nb;
  const int nn = nb + (a > 0 ? 1 : 0);
  P.size.assign(nn, (int)b);
  if (a > 0) P.size[A] = (int)a;
  P.elim.assign(nn, 0);
  for (int k = 0; k + 1 < nb; ++k) P.elim[k] = 1;
  P.accum.assign(nn, 0);
  if (a > 0) P.accum[A] = 1;
  P.rowbase.resize(nn);
  P.rows.assign(nn, {});
  for (int k = 0; k < nb; ++k) {
    const int64_t j = glob_s + (cnt - 1 - k);   // global block of node k
    const int64_t lj = ls + (cnt - 1 - k);      // local index
    P.rowbase[k] = V.row(j);
    P.blk[{k, k}] = blkref(V.D.at(lj), (int)b, (int)b);
    const bool el = k + 1 < nb;
    if (el) {  // successor: block j-1 = node k+1, coupling A_{j-1,j} = T(j)
      P.blk[{k + 1, k}] = blkref(Tb.at(j - glob_s - 1), (int)b, (int)b);
      P.rows[k].push_back(k + 1);
    }
    if (a > 0) {
      P.blk[{A, k}] = blkref(V.Ar.at(lj), (int)a, (int)b);
      if (el) P.rows[k].push_back(A);
    }
  }
  if (a > 0) {
    P.rowbase[A] = -1;
    P.blk[{A, A}] = blkref(U, (int)a, (int)a, true);
  }
}

// PPOBTAF for one partition (Alg. 3 line 3 / line 5): factor the interior and
// flush the Schur updates into the boundary blocks, U_p and (middle) B_{e-1}.
void ppobtaf_part(Ctx &cx, PartState &ps, int64_t b, int64_t a) {
  bool top = ps.p == 0;
  int64_t cnt = ps.e - ps.s;
  ps.U = wsloc(cx.alloc(std::max<int64_t>(a * a, 1)), std::max<int64_t>(a, 1));
  if (ps.bottom) {
    ps.Tbuf = Fam{BUF_WS, cx.alloc(std::max<int64_t>(cnt - 1, 1) * b * b), b * b, (int32_t)b};
    bottom_problem(ps.prob, ps.V, ps.ls, cnt, b, a, ps.U, ps.Tbuf, ps.s);
  } else if (top) {
    int64_t ls = ps.ls;
    const View &V = ps.V;
    chain_problem(
        ps.prob, (int)cnt, b, a, [&](int i) { return V.D.at(ls + i); }, [&](int i) { return V.Lo.at(ls + i); },
        [&](int i) { return V.Ar.at(ls + i); }, ps.U, true, (int)cnt - 1, false,
        [&](int i) { return V.row(ps.s + i); }, -1);
  } else {
    ps.Bbuf = Fam{BUF_WS, cx.alloc((cnt - 1) * b * b), b * b, (int32_t)b};
    middle_problem(ps.prob, ps.V, ps.ls, cnt, b, a, ps.U, ps.Bbuf, ps.s);
  }
  ps.prob.queue = ps.queue;
  ps.prob.queue2 = ps.queue > 0 ? ps.queue + 1 : 0;
  ps.bld.reset(new Builder(cx, ps.prob));
  Builder &B = *ps.bld;
  B.input_waits = ps.inw;
  B.allocate(true);
  std::vector<int32_t> tin;
  if (ps.bottom) {  // T(j) = A_{j,j-1}^T, j = s+1..e-1 (node k = e-1-j needs T(j))
    for (int64_t j = ps.s + 1; j < ps.e; ++j) {
      int32_t c = cx.new_ctr();
      cx.copy_block(ps.Tbuf.at(j - ps.s - 1), ps.V.Lo.at(ps.ls + (j - 1 - ps.s)), (int)b, (int)b, true, ps.inw, {c});
      tin.push_back(c);
      ps.done.push_back(c);
    }
  } else if (!top) {  // B_{s+1} = A_{s+1,s}^T (Alg. 4 line 1, reading R7)
    int32_t c = cx.new_ctr();
    cx.copy_block(ps.Bbuf.at(0), ps.V.Lo.at(ps.ls), (int)b, (int)b, true, ps.inw, {c});
    B.input_waits.push_back(c);
    ps.done.push_back(c);
  }
  for (size_t X = 0; X < ps.prob.size.size(); ++X)
    if (ps.prob.elim[X]) {
      if (ps.bottom) {  // node X = block e-1-X reads T(e-1-X)
        B.input_waits = ps.inw;
        B.input_waits.push_back(tin[(size_t)(ps.e - 1 - (int64_t)X - ps.s - 1)]);
      }
      B.factor_node((int)X);
      ++ps.nelim;
    }
  if (ps.bottom) B.input_waits = ps.inw;
  B.flush_boundary(ps.done);
  if (a > 0 && ps.nelim == 0) {  // U_p = 0 when nothing is eliminated
    int32_t z = cx.new_ctr();
    cx.reduce_block(ps.U, ps.U, 0.0, ps.U, 0, 0, 0.0, (int)a, (int)a, {}, {z});
    ps.done.push_back(z);
  }
  for (auto &kv : B.factordone) ps.done.push_back(kv.second);
}

// one rank's exchange record (doubles): boundary blocks, couplings, U_p, log det
struct XRec {
  int64_t b, a;
  int64_t bd0() const { return 0; }          // A_TT (top) or A_ff (middle)
  int64_t bd1() const { return b * b; }      // A_ll (middle)
  int64_t lw0() const { return 2 * b * b; }  // coupling A_{e,e-1} to the next rank (original)
  int64_t lw1() const { return 3 * b * b; }  // B_{e-1} (rows f, columns l)
  int64_t ar0() const { return 4 * b * b; }
  int64_t ar1() const { return 4 * b * b + a * b; }
  int64_t U() const { return 4 * b * b + 2 * a * b; }
  int64_t ld() const { return 4 * b * b + 2 * a * b + a * a; }
};

// pack partition ps into record `rec` (buffer rbuf, offset r0)
void pack_part(Ctx &cx, PartState &ps, int P, int64_t b, int64_t a, int32_t rbuf, int64_t r0, int32_t sig) {
  XRec x{b, a};
  auto rec = [&](int64_t off, int64_t ld) { return Loc{rbuf, (int32_t)ld, r0 + off}; };
  int64_t cnt = ps.e - ps.s, ls = ps.ls;
  const auto &w = ps.done;
  const View &V = ps.V;
  if (ps.p == 0) {
    cx.copy_block(rec(x.bd0(), b), V.D.at(ls + cnt - 1), (int)b, (int)b, false, w, {sig});
    if (a > 0) cx.copy_block(rec(x.ar0(), b), V.Ar.at(ls + cnt - 1), (int)a, (int)b, false, w, {sig});
  } else if (ps.bottom) {  // boundary block s only
    cx.copy_block(rec(x.bd0(), b), V.D.at(ls), (int)b, (int)b, false, w, {sig});
    if (a > 0) cx.copy_block(rec(x.ar0(), b), V.Ar.at(ls), (int)a, (int)b, false, w, {sig});
  } else {
    cx.copy_block(rec(x.bd0(), b), V.D.at(ls), (int)b, (int)b, false, w, {sig});
    cx.copy_block(rec(x.bd1(), b), V.D.at(ls + cnt - 1), (int)b, (int)b, false, w, {sig});
    cx.copy_block(rec(x.lw1(), b), ps.Bbuf.at(cnt - 2), (int)b, (int)b, false, w, {sig});
    if (a > 0) {
      cx.copy_block(rec(x.ar0(), b), V.Ar.at(ls), (int)a, (int)b, false, w, {sig});
      cx.copy_block(rec(x.ar1(), b), V.Ar.at(ls + cnt - 1), (int)a, (int)b, false, w, {sig});
    }
  }
  if (ps.p < P - 1) cx.copy_block(rec(x.lw0(), b), V.Lo.at(ls + cnt - 1), (int)b, (int)b, false, ps.inw, {sig});
  if (a > 0) cx.copy_block(rec(x.U(), a), ps.U, (int)a, (int)a, false, w, {sig});
}

struct Reduced {
  Fam D, Lo, Ar;
  Loc tip;
  Problem P;
  std::unique_ptr<Builder> B;
  View V;                      // A_r as a BTA matrix (for a nested solve)
  std::vector<int32_t> ready;  // A_r assembled (blocks and reduced tip)
};

// Assemble A_r (2P-1 blocks, reading R9) from the P records at (rbuf, rec0 +
// p*recsz), then POBTARSSI = POBTAF + POBTASI on it (Sec. 3.3).  The reduced tip
// A_nn + U_0 + ... + U_{P-1} (reading R8) is formed in place in BUF_TIP.

void assemble_reduced(Ctx &cx, const View &V0, int P, int64_t b, int64_t a, int32_t rbuf, int64_t rec0,
                      int64_t recsz, const std::vector<int64_t> &starts, const std::vector<int32_t> &inwaits,
                      Reduced &R, bool tw) {
  XRec x{b, a};
  int nr = reduced_size(P, tw);
  R.D = Fam{BUF_WS, cx.alloc(nr * b * b), b * b, (int32_t)b};
  R.Lo = Fam{BUF_WS, cx.alloc(std::max(nr - 1, 1) * b * b), b * b, (int32_t)b};
  R.Ar = Fam{BUF_WS, cx.alloc(std::max<int64_t>(nr * a * b, 1)), a * b, (int32_t)b};
  auto rec = [&](int p, int64_t off, int64_t ld) { return Loc{rbuf, (int32_t)ld, rec0 + p * recsz + off}; };
  int32_t cr = cx.new_ctr();
  std::vector<int32_t> ready{cr};
  cx.copy_block(R.D.at(0), rec(0, x.bd0(), b), (int)b, (int)b, false, inwaits, {cr});
  if (a > 0) cx.copy_block(R.Ar.at(0), rec(0, x.ar0(), b), (int)a, (int)b, false, inwaits, {cr});
  for (int p = 1; p < P; ++p) {
    if (tw && p == P - 1) {  // twisted last partition: its boundary block s only (reading R14)
      cx.copy_block(R.D.at(2 * p - 1), rec(p, x.bd0(), b), (int)b, (int)b, false, inwaits, {cr});
      if (a > 0) cx.copy_block(R.Ar.at(2 * p - 1), rec(p, x.ar0(), b), (int)a, (int)b, false, inwaits, {cr});
      cx.copy_block(R.Lo.at(2 * p - 2), rec(p - 1, x.lw0(), b), (int)b, (int)b, false, inwaits, {cr});
      continue;
    }
    cx.copy_block(R.D.at(2 * p - 1), rec(p, x.bd0(), b), (int)b, (int)b, false, inwaits, {cr});
    cx.copy_block(R.D.at(2 * p), rec(p, x.bd1(), b), (int)b, (int)b, false, inwaits, {cr});
    if (a > 0) {
      cx.copy_block(R.Ar.at(2 * p - 1), rec(p, x.ar0(), b), (int)a, (int)b, false, inwaits, {cr});
      cx.copy_block(R.Ar.at(2 * p), rec(p, x.ar1(), b), (int)a, (int)b, false, inwaits, {cr});
    }
    cx.copy_block(R.Lo.at(2 * p - 2), rec(p - 1, x.lw0(), b), (int)b, (int)b, false, inwaits, {cr});
    cx.copy_block(R.Lo.at(2 * p - 1), rec(p, x.lw1(), b), (int)b, (int)b, true, inwaits, {cr});
  }
  R.tip = Loc{BUF_TIP, (int32_t)std::max<int64_t>(a, 1), 0};
  if (a > 0) {
    int32_t ct = cx.new_ctr();
    cx.reduce_block(R.tip, R.tip, 1.0, rec(0, x.U(), a), recsz, P, 1.0, (int)a, (int)a, inwaits, {ct});
    ready.push_back(ct);
  }
  std::function<int64_t(int64_t)> vrow = V0.row;
  const int64_t tip_row = V0.tip_row;
  std::vector<int64_t> st = starts;
  R.V = View{R.D, R.Lo, R.Ar,
             [st, vrow, b](int64_t i) -> int64_t {
               int64_t blk;
               if (i == 0)
                 blk = st[1] - 1;
               else {
                 int p = (int)((i + 1) / 2);
                 blk = (i & 1) ? st[p] : st[p + 1] - 1;
               }
               // a partition start this rank does not know (distributed): encoded, decoded
               // after the solve from the records' meta (dist_meta.h)
               return blk >= 0 ? vrow(blk) : (int64_t)kEncRow + i * b;
             },
             tip_row};
  R.ready = ready;
}

// POBTARSSI on an assembled A_r: POBTAF + POBTASI as one chain (Sec. 3.3).
void solve_reduced_chain(Ctx &cx, int64_t b, int64_t a, int nr, Reduced &R) {
  chain_problem(
      R.P, nr, b, a, [&](int i) { return R.D.at(i); }, [&](int i) { return R.Lo.at(i); },
      [&](int i) { return R.Ar.at(i); }, R.tip, false, nr, true, [&](int i) { return R.V.row(i); }, R.V.tip_row);
  R.P.queue = 1;
  R.P.queue2 = 2;
  R.B.reset(new Builder(cx, R.P));
  R.B->input_waits = R.ready;
  R.B->allocate(true);
  int nn = (int)R.P.size.size();
  for (int X = 0; X < nn; ++X) R.B->factor_node(X);
  for (int X = 0; X < nn; ++X) R.B->precompute_node(X, true);
  for (int X = nn - 1; X >= 0; --X) R.B->invert_node(X);
}

// POBTARSSI in the twisted order (reading R13): the reduced system is alone on
// the critical path after the exchange, so its chain is split in two (top-down
// and bottom-up towards the middle block).  Bottom couplings live transposed in
// workspace T(j) and are copied back (with their X-ready signals) at the end.
void solve_reduced_twisted(Ctx &cx, int64_t b, int64_t a, int nr, Reduced &R) {
  Twist tw;
  twisted_problem(cx, R.P, tw, nr, b, a, R.D, R.Lo, R.Ar, R.tip, R.V.row, R.V.tip_row);
  R.B.reset(new Builder(cx, R.P));
  Builder &bld = *R.B;
  bld.concurrency = 2;
  bld.allocate(true);
  const int nn = (int)R.P.size.size();
  const int64_t m = tw.m;
  std::vector<int32_t> tin(nr, -1);
  for (int64_t j = m + 1; j < nr; ++j) {  // T(j) = A_{j,j-1}^T
    tin[j] = cx.new_ctr();
    cx.copy_block(tw.T.at(j - m - 1), R.Lo.at(j - 1), (int)b, (int)b, true, R.ready, {tin[j]});
  }
  std::vector<int64_t> blk_of(nn, -1);
  for (int64_t i = 0; i < nr; ++i) blk_of[tw.pos[i]] = i;
  for (int X = 0; X < nn; ++X) {
    bld.input_waits = R.ready;
    if (blk_of[X] > m) bld.input_waits.push_back(tin[blk_of[X]]);
    bld.factor_node(X);
  }
  bld.input_waits = R.ready;
  for (int X = 0; X < nn; ++X) bld.precompute_node(X, true);
  for (int X = nn - 1; X >= 0; --X) {
    bld.invert_node(X);
    const int64_t i = blk_of[X];
    if (i > m) {  // X_{i,i-1} = T(i)^T
      const Loc src = tw.T.at(i - m - 1);
      const Loc dst = R.Lo.at(i - 1);
      std::vector<int32_t> w;
      for (int q = 0; q < ntiles(b); ++q) w.push_back(cx.XRC(src, q, 0));
      cx.copy_block(dst, src, (int)b, (int)b, true, w, {},
                    [&](RawTask &rt, int q, int c) { cx.sig_xblock(rt, dst, q, c); });
    }
  }
}

void solve_reduced(Ctx &cx, int64_t b, int64_t a, int nr, Reduced &R) {
  if (cx.opt.twist_reduced && nr >= 4)
    solve_reduced_twisted(cx, b, a, nr, R);
  else
    solve_reduced_chain(cx, b, a, nr, R);
}

void reduced_from_records(Ctx &cx, const View &V0, int P, int64_t b, int64_t a, int32_t rbuf, int64_t rec0,
                          int64_t recsz, const std::vector<int64_t> &starts, const std::vector<int32_t> &inwaits,
                          Reduced &R, bool tw) {
  assemble_reduced(cx, V0, P, b, a, rbuf, rec0, recsz, starts, inwaits, R, tw);
  solve_reduced(cx, b, a, reduced_size(P, tw), R);
}

// Copy the true-inverse boundary blocks of partition ps from X_r into its
// storage and signal their final-X counters ("POBTARSSI's result is copied to
// PPOBTASI's L and B"; reading R10).
void scatter_xr(Ctx &cx, PartState &ps, int P, int64_t b, int64_t a, const Reduced &R) {
  int p = ps.p;
  Problem &Q = ps.prob;
  auto cp = [&](Loc dst, Loc src, int rows, int cols, bool trans) {
    std::vector<int32_t> w = ps.done;  // WAR on everything the factor phase read / wrote
    int sr = trans ? cols : rows, sc = trans ? rows : cols;
    for (int q = 0; q < ntiles(sr); ++q) w.push_back(cx.XRC(src, q, 0));
    for (int c = 0; c < ntiles(sc); ++c) w.push_back(cx.XRC(src, c, 1));
    cx.copy_block(dst, src, rows, cols, trans, w, {}, [&](RawTask &rt, int q, int c) { cx.sig_xblock(rt, dst, q, c); });
  };
  int nn = (int)Q.size.size();
  if (p == 0) {
    int T = (int)(ps.e - ps.s) - 1;
    cp(Q.blk.at({T, T}).base, R.D.at(0), (int)b, (int)b, false);
    if (a > 0) cp(Q.blk.at({nn - 1, T}).base, R.Ar.at(0), (int)a, (int)b, false);
  } else if (ps.bottom) {  // boundary block s = node cnt-1
    int S = (int)(ps.e - ps.s) - 1;
    cp(Q.blk.at({S, S}).base, R.D.at(2 * p - 1), (int)b, (int)b, false);
    if (a > 0) cp(Q.blk.at({nn - 1, S}).base, R.Ar.at(2 * p - 1), (int)a, (int)b, false);
  } else {
    int k = (int)(ps.e - ps.s) - 1, F = k, L = k - 1;
    cp(Q.blk.at({F, F}).base, R.D.at(2 * p - 1), (int)b, (int)b, false);
    cp(Q.blk.at({L, L}).base, R.D.at(2 * p), (int)b, (int)b, false);
    if (a > 0) {
      cp(Q.blk.at({F + 1, F}).base, R.Ar.at(2 * p - 1), (int)a, (int)b, false);
      cp(Q.blk.at({F + 1, L}).base, R.Ar.at(2 * p), (int)a, (int)b, false);
    }
    cp(Q.blk.at({F, L}).base, R.Lo.at(2 * p - 1), (int)b, (int)b, true);  // Q_{e-1} = X_r(L_p,F_p)^T
  }
  if (p < P - 1)  // coupling to the next partition: X_r(F_{p+1}, L_p)
    cp(ps.V.Lo.at(ps.ls + (ps.e - ps.s) - 1), R.Lo.at(2 * p), (int)b, (int)b, false);
  // the tip node of the partition now stands for the true X_nn (in BUF_TIP)
  if (a > 0) Q.blk[{nn - 1, nn - 1}] = blkref(R.tip, (int)a, (int)a);
}

// PPOBTASI for one partition (Alg. 5 line 3 / line 5).
void ppobtasi_part(Ctx &cx, PartState &ps, int64_t b, bool have_wdiag) {
  Builder &B = *ps.bld;
  int nn = (int)ps.prob.size.size();
  for (int X = 0; X < nn; ++X)
    if (ps.prob.elim[X]) B.precompute_node(X, have_wdiag);
  for (int X = nn - 1; X >= 0; --X)
    if (ps.prob.elim[X]) B.invert_node(X);
  if (ps.bottom) {  // X_{j,j-1} = T(j)^T, j = s+1..e-1
    for (int64_t j = ps.s + 1; j < ps.e; ++j) {
      const Loc src = ps.Tbuf.at(j - ps.s - 1);
      std::vector<int32_t> w;
      for (int q = 0; q < ntiles(b); ++q) w.push_back(cx.XRC(src, q, 0));
      const Loc dst = ps.V.Lo.at(ps.ls + (j - 1 - ps.s));
      cx.copy_block(dst, src, (int)b, (int)b, true, w, {},
                    [&](RawTask &rt, int q, int c) { cx.sig_xblock(rt, dst, q, c); });
    }
  } else if (ps.p > 0) {  // X_{s+1,s} = Q_{s+1}^T (reading R10)
    std::vector<int32_t> w;
    for (int q = 0; q < ntiles(b); ++q) w.push_back(cx.XRC(ps.Bbuf.at(0), q, 0));
    const Loc dst = ps.V.Lo.at(ps.ls);
    cx.copy_block(dst, ps.Bbuf.at(0), (int)b, (int)b, true, w, {},
                  [&](RawTask &rt, int q, int c) { cx.sig_xblock(rt, dst, q, c); });
  }
}

}  // namespace

int64_t sequential_ws_bytes(int kind, int64_t n, int64_t b, int64_t a, const BuildOptions &opt) {
  // replays the allocations of build_seq_ctx (no tasks are built)
  Ctx cx;
  cx.opt = opt;
  bool inv = kind != 0;  // 1, 2, 6
  cx.slot_cap = slot_bound(n, b, a);
  cx.slot_region = cx.alloc(cx.slot_cap);
  Problem P;
  if (use_twist(kind, n, b, opt)) {
    Twist tw;
    twisted_problem(cx, P, tw, n, b, a, famD(b), famL(b), famA(b, a), Loc{BUF_TIP, (int32_t)a, 0},
                    [b](int64_t i) { return i * b; }, n * b);
    Builder bld(cx, P);
    bld.allocate(true);
    return cx.ws_top * 8;
  }
  chain_problem(
      P, (int)n, b, a, [&](int i) { return famD(b).at(i); }, [&](int i) { return famL(b).at(i); },
      [&](int i) { return famA(b, a).at(i); }, Loc{BUF_TIP, (int32_t)a, 0}, false, (int)n, true,
      [&](int i) { return (int64_t)i * b; }, n * b);
  Builder bld(cx, P);
  bld.allocate(inv);
  return cx.ws_top * 8;
}

Graph build_sequential(int kind, int64_t n, int64_t b, int64_t a, const BuildOptions &opt) {
  Ctx cx;
  cx.opt = opt;
  // scheduler cost model per block size (measured, profiles/r02/knobs/): the claim order
  // starts the chain's bulk inputs earlier with a larger GEMM fixed cost at b >= 2048 (C3
  // 936 -> 927 ms) and a lower bulk rate at b = 1024 (C2 56.9 -> 55.6 ms)
  // (not for the streaming-IO graph at b = 1024: its modelled arrivals favour the default;
  // C2 e2e 91.5 vs 115 ms)
  if (!opt.cost_set) {
    if (b >= 2048) cx.opt.cost_gemm_fixed = 7000.0;
    else if (b >= 1024 && kind != 6) cx.opt.cost_gflops = 50.0;
  }
  Graph g = build_seq_ctx(cx, kind, n, b, a);
  if (g.error.empty() && g.ws_doubles * 8 > sequential_ws_bytes(kind, n, b, a, opt))
    g.error = "workspace accounting mismatch";
  return g;
}

void BuildOptions::apply_env() {
  const char *e = getenv("SERINV_OPT");
  if (!e) return;
  std::string s(e);
  size_t i = 0;
  while (i < s.size()) {
    size_t j = s.find(',', i);
    if (j == std::string::npos) j = s.size();
    std::string kv = s.substr(i, j - i);
    size_t eq = kv.find('=');
    if (eq != std::string::npos) {
      std::string k = kv.substr(0, eq);
      long v = strtol(kv.c_str() + eq + 1, nullptr, 10);
      if (k == "update_group") update_group = (int)v;
      else if (k == "critical_queues") critical_queues = v != 0;
      else if (k == "fuse_trsm") fuse_trsm = v != 0;
      else if (k == "fuse_trsm3") fuse_trsm3 = v != 0;
      else if (k == "split_chain") split_chain = v != 0;
      else if (k == "chain_syrk") chain_syrk = v != 0;
      else if (k == "urgent_ctas") urgent_ctas = (int)v;
      else if (k == "si_split") si_split = (int)v;
      else if (k == "rts1_chain") rts1_chain = v != 0;
      else if (k == "max_crit") max_crit = (int)v;
      else if (k == "twist_min_n") twist_min_n = (int)v;
      else if (k == "twist_max_b") twist_max_b = (int)v;
      else if (k == "wide_min_wave") wide_min_wave = (int)v;
      else if (k == "chol8") chol8 = v != 0;
      else if (k == "twist_last") twist_last = v != 0;
      else if (k == "early_sig") early_sig = v != 0;
      else if (k == "carry_chain") carry_chain = v != 0;
      else if (k == "carry_min_b") carry_min_b = (int)v;
      else if (k == "chain_step") chain_step = v != 0;
      else if (k == "dist_len") dist_len = (int)v;
      else if (k == "twist_reduced") twist_reduced = v != 0;
      else if (k == "split_last") split_last = (int)v;
      else if (k == "cost_gemm_fixed") cost_gemm_fixed = (double)v, cost_set = true;
      else if (k == "cost_potrf") cost_potrf = (double)v, cost_set = true;
      else if (k == "cost_gflops") cost_gflops = (double)v, cost_set = true;
    }
    i = j + 1;
  }
}

// Diagnostic graph: ntasks independent 64 x 64 tile GEMMs with K = k (A, B row
// strips, NT) reading/writing disjoint workspace regions -- measures the tile
// engine's throughput without dependencies.
Graph build_gemm_bench(int ntasks, int k, int nseg, const BuildOptions &opt) {
  Ctx cx;
  cx.opt = opt;
  const int64_t strip = (int64_t)TILE * k;
  int64_t A = cx.alloc(strip * 64), Bm = cx.alloc(strip * 64), C = cx.alloc((int64_t)TILE * TILE * 64);
  for (int t = 0; t < ntasks; ++t) {
    RawTask rt;
    rt.t.type = TK_GEMM;
    rt.t.m = rt.t.n = TILE;
    rt.t.out = Loc{BUF_WS, TILE, C + (int64_t)(t % 64) * TILE * TILE};
    rt.t.c0 = rt.t.out;
    rt.t.alpha = -1.0;
    rt.t.beta = 1.0;
    int kk = k / nseg;
    for (int s2 = 0; s2 < nseg; ++s2)
      rt.segs.push_back(mkseg(Loc{BUF_WS, (int32_t)k, A + (t % 64) * strip + s2 * kk}, 0,
                              Loc{BUF_WS, (int32_t)k, Bm + ((t + 7) % 64) * strip + s2 * kk}, 1, kk));
    cx.emit(std::move(rt));
  }
  return cx.finalize();
}

int reduced_size(int P, bool tw) { return tw && P >= 2 ? 2 * P - 2 : 2 * P - 1; }

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

// Plan for the twisted scheme (reading R14): the first and the last partition
// have no fill-in, so both get r times a middle partition's blocks; middles split
// the rest evenly (each >= 2), the remainder to the earliest.  r = 1 gives the
// same partition as plan_partitions.
bool plan_partitions_ends(int64_t n, int P, double r, std::vector<int64_t> &starts) {
  starts.clear();
  if (P < 1 || n < 1) return false;
  if (P == 2 && n >= 2) {  // both partitions are chain ends: equal halves
    starts = {0, n / 2, n};
    return true;
  }
  if (P == 1 || r == 1.0) return plan_partitions(n, P, 1.0, starts);
  if (n < 2 * (int64_t)P - 2) return false;
  const double mid = (double)n / (2.0 * r + (double)(P - 2));
  int64_t end = std::max<int64_t>(1, (int64_t)std::llround(r * mid));
  end = std::min<int64_t>(end, (n - 2 * (int64_t)(P - 2)) / 2);
  if (end < 1) return false;
  int64_t rest = n - 2 * end, base = rest / (P - 2), rem = rest % (P - 2);
  if (base < 2) return false;
  starts.push_back(0);
  int64_t s = end;
  starts.push_back(s);
  for (int p = 1; p < P - 1; ++p) {
    s += base + ((p - 1) < rem ? 1 : 0);
    starts.push_back(s);
  }
  starts.push_back(n);
  return s + end == n;
}

bool plan_partitions_for(int64_t n, int P, double r, bool twist_last, std::vector<int64_t> &starts) {
  return twist_last ? plan_partitions_ends(n, P, r, starts) : plan_partitions(n, P, r, starts);
}

int64_t exchange_meta_offset(int64_t b, int64_t a) { return 4 * b * b + 2 * a * b + a * a; }

// record = boundary blocks + U_p + the dist_meta.h tail (log det partial, info, s, e), padded to 32 doubles
int64_t exchange_doubles(int64_t b, int64_t a) {
  return (4 * b * b + 2 * a * b + a * a + kMetaDoubles + 31) / 32 * 32;
}

// One level of the (nested) partitioned solve of the BTA matrix V (n blocks, tip
// in BUF_TIP): PPOBTAF on Ps[lvl] partitions, A_r (2P-1 blocks) assembled, then
// solved by the next level (Ps[lvl+1] > 1: the same algorithm applied to A_r,
// nested solving, Sec. 4.2) or as one chain (POBTARSSI), X_r scattered,
// PPOBTASI.  Returns false (nothing emitted) if the plan is infeasible.
bool psolve_level(Ctx &cx, const View &V, int64_t n, int64_t b, int64_t a, const std::vector<int> &Ps, size_t lvl,
                  double r, const std::vector<int32_t> &inw) {
  const int P = Ps[lvl];
  std::vector<int64_t> starts;
  const bool ok = plan_partitions_for(n, P, r, cx.opt.twist_last, starts);
  if (P < 1 || (lvl > 0 && P < 2) || !ok) return false;
  const int64_t recsz = exchange_doubles(b, a);
  const int64_t recs = cx.alloc(recsz * P);
  std::vector<PartState> parts(P);
  // exclusive-SM chains only for a few top-level partitions (each takes two SMs)
  const bool crit = lvl == 0 && 2 * P <= cx.opt.max_crit;
  const bool tw = cx.opt.twist_last && P >= 2;
  for (int p = 0; p < P; ++p) {
    parts[p].p = p;
    parts[p].s = starts[p];
    parts[p].e = starts[p + 1];
    parts[p].ls = starts[p];
    parts[p].queue = crit ? 2 * p + 1 : 0;
    parts[p].V = V;
    parts[p].inw = inw;
    parts[p].bottom = tw && p == P - 1;
    ppobtaf_part(cx, parts[p], b, a);
  }
  int32_t packed = cx.new_ctr();
  for (int p = 0; p < P; ++p) pack_part(cx, parts[p], P, b, a, BUF_WS, recs + p * recsz, packed);
  Reduced R;
  assemble_reduced(cx, V, P, b, a, BUF_WS, recs, recsz, starts, {packed}, R, tw);
  const int nr = reduced_size(P, tw);
  bool nested = lvl + 1 < Ps.size() && psolve_level(cx, R.V, nr, b, a, Ps, lvl + 1, r, R.ready);
  if (!nested) solve_reduced(cx, b, a, nr, R);
  for (int p = 0; p < P; ++p) {
    parts[p].done.push_back(packed);  // scatter overwrites what the pack copies read
    scatter_xr(cx, parts[p], P, b, a, R);
    ppobtasi_part(cx, parts[p], b, true);
  }
  return true;
}

Graph build_pselinv(int64_t n, int64_t b, int64_t a, const std::vector<int> &Ps, double r, const BuildOptions &opt) {
  std::vector<int64_t> starts;
  if (Ps.empty() || !plan_partitions_for(n, Ps[0], r, opt.twist_last, starts)) {
    Graph bad;
    bad.error = "infeasible plan";
    return bad;
  }
  Ctx cx;
  cx.opt = opt;
  cx.slot_cap = slot_bound(n + 2 * Ps[0], b, a);
  cx.slot_region = cx.alloc(cx.slot_cap);
  psolve_level(cx, top_view(n, b, a), n, b, a, Ps, 0, r, {});
  cx.logdet(Loc{BUF_LOGDET, 0, 0}, 0, cx.slot_count, Loc{BUF_WS, 0, 0}, 0, 0, {});
  return cx.finalize();
}

Graph build_pselinv(int64_t n, int64_t b, int64_t a, int P, double r, const BuildOptions &opt) {
  return build_pselinv(n, b, a, std::vector<int>{P}, r, opt);
}

int64_t pselinv_ws_bytes(int64_t n, int64_t b, int64_t a, const std::vector<int> &Ps, double r) {
  BuildOptions opt;
  opt.apply_env();  // the layout depends on options (twist_last, wide_min_wave, ...)
  opt.schedule = false;
  Graph g = build_pselinv(n, b, a, Ps, r, opt);
  return g.error.empty() ? g.ws_doubles * 8 : -1;
}

int64_t pselinv_ws_bytes(int64_t n, int64_t b, int64_t a, int P, double r) {
  return pselinv_ws_bytes(n, b, a, std::vector<int>{P}, r);
}

// Default nesting for one device: partitions of about `len` blocks at every level
// until the reduced system is short enough to solve as one chain.  Small blocks
// have latency-bound chains (the per-step work is tiny), so they are cut short.
std::vector<int> auto_partitions(int64_t n, int64_t b) {
  std::vector<int> Ps;
  const int64_t len = b <= 128 ? 64 : (b <= 512 ? 64 : 1 << 30);  // C4 sweep: P = 4 best (35 ms vs 38 ms at P = 8)
  const int64_t chain_max = b <= 128 ? 48 : 16;
  int64_t m = n;
  while (m > chain_max && (int)Ps.size() < 4) {
    int64_t P = std::min<int64_t>((m + len - 1) / len, (m + 1) / 3);
    if (P < 2) break;
    P = std::min<int64_t>(P, 4096);
    Ps.push_back((int)P);
    m = reduced_size((int)P, BuildOptions().twist_last);
  }
  if (Ps.empty()) Ps.push_back(1);
  return Ps;
}

// Nesting plan for the distributed reduced system (solved redundantly on every
// rank, on the critical path of all of them): partitions of about `len` blocks
// per level (len <= 0: the measured default below).
std::vector<int> reduced_plan(int64_t nr, int64_t b, int len) {
  if (len <= 0) {
    // measured (tools/scaling_sim.py, P = 8): nesting in ~16-block partitions at
    // b = 512 (C4: E_weak 57.7 -> 66.6 %), ~32 at b = 64 (C5: 62.8 -> 66.4 %); at
    // b = 1024 the fill-in of a nested level costs more than the chain it cuts
    // (C2: 45.0 -> 41.1 % at len 8), so large blocks keep the single-device plan
    if (b > 512) return auto_partitions(nr, b);
    len = b <= 128 ? 32 : 16;
  }
  std::vector<int> Ps;
  int64_t m = nr;
  while (m > len && (int)Ps.size() < 4) {
    int64_t P = std::min<int64_t>((m + len - 1) / len, (m + 1) / 3);
    if (P < 2) break;
    Ps.push_back((int)P);
    m = reduced_size((int)P, true);
  }
  if (Ps.empty()) Ps.push_back(1);
  return Ps;
}

// Split a rank's blocks [start, start+count) into Q consecutive sub-partitions
// (even sizes, remainder to the earliest).  Every sub-partition needs >= 2
// blocks except a global first one (>= 1).  Returns false if infeasible.
bool split_rank(int64_t start, int64_t count, int Q, std::vector<int64_t> &sub) {
  if (Q < 1 || count < 1) return false;
  sub.assign(Q + 1, start);
  int64_t base = count / Q, rem = count % Q;
  for (int q = 0; q < Q; ++q) sub[q + 1] = sub[q] + base + (q < rem ? 1 : 0);
  for (int q = 0; q < Q; ++q) {
    int64_t c = sub[q + 1] - sub[q];
    if (c < 1 || (c < 2 && !(start == 0 && q == 0) && Q > 1)) return false;
  }
  return true;
}

// Distributed per-rank graphs.  Rank `rank` of P owns the global blocks
// [start, start+count), split into Q sub-partitions (intra-GPU partitioning of
// the rank's chain; Q = 1 is the paper's one partition per process).  Globally
// there are P*Q partitions, rank p owning partitions [pQ, (p+1)Q).
// Phase 0 (ppobtaf): factor the Q local partitions and pack their Q exchange
// records into EXT0.  Phase 1 (ppobtasi): assemble A_r (2PQ-1 blocks, 2PQ-2
// with the twisted last partition) from the all-gathered records in EXT1
// (global order, identical on every rank), solve it redundantly -- nested
// (Sec. 4.2) when it is long, else as one chain (POBTARSSI) -- scatter this
// rank's X_r blocks, backward pass.  Both phases lay the workspace out
// identically (phase 1 replays the factor-phase allocations), so the fill-in
// factor blocks B_i survive between the calls.
Graph build_distributed(int phase, int P, int rank, int64_t n, int64_t start, int64_t count, int64_t b, int64_t a,
                        const BuildOptions &opt, int Q) {
  std::vector<int64_t> sub;
  if (!split_rank(start, count, Q, sub)) {
    Graph bad;
    bad.error = "infeasible rank split";
    return bad;
  }
  const int PQ = P * Q;
  const bool tw = opt.twist_last && PQ >= 2;
  const int nr = reduced_size(PQ, tw);
  std::vector<int> Ps2 = reduced_plan(nr, b, opt.dist_len);
  Ctx cx;
  cx.opt = opt;
  cx.slot_cap = slot_bound(count + 4 * PQ + 8, b, a);
  cx.slot_region = cx.alloc(cx.slot_cap);
  int64_t recsz = exchange_doubles(b, a);
  XRec x{b, a};
  std::vector<PartState> parts(Q);
  const bool crit = 2 * Q <= cx.opt.max_crit;
  for (int q = 0; q < Q; ++q) {
    PartState &ps = parts[q];
    ps.p = rank * Q + q;
    ps.s = sub[q];
    ps.e = sub[q + 1];
    ps.ls = sub[q] - start;
    ps.queue = Q == 1 ? 1 : (crit ? 2 * q + 1 : 0);
    ps.V = top_view(n, b, a);  // local storage (block `start` at index 0), global rows
    ps.bottom = tw && ps.p == PQ - 1;
    ppobtaf_part(cx, ps, b, a);
  }
  if (phase == 0) {
    int32_t packed = cx.new_ctr();
    for (int q = 0; q < Q; ++q) pack_part(cx, parts[q], PQ, b, a, BUF_EXT0, q * recsz, packed);
    // the rank's partial log det travels in its first record
    cx.logdet(Loc{BUF_EXT0, 0, x.ld()}, 0, cx.slot_count, Loc{BUF_WS, 0, 0}, 0, 0, {});
    return cx.finalize();
  }
  // phase 1: the factor tasks ran in phase 0; keep their workspace layout only
  cx.tasks.clear();
  cx.own.clear();
  cx.potrf_ctrs.clear();
  cx.xrc.clear();
  for (auto &ps : parts) {
    Builder &PB = *ps.bld;
    PB.factordone.clear();
    PB.Lprod.clear();
    PB.tstate.clear();
    PB.input_waits.clear();
    PB.wdiag_task.clear();
    ps.done.clear();
  }
  int64_t part_slots = cx.slot_count;
  // partition starts known to this rank (other ranks' inner starts only label info rows)
  std::vector<int64_t> st(PQ + 1, -1);
  for (int q = 0; q <= Q; ++q) st[rank * Q + q] = sub[q];
  st[0] = 0;
  st[PQ] = n;
  Reduced R;
  assemble_reduced(cx, parts[0].V, PQ, b, a, BUF_EXT1, 0, recsz, st, {}, R, tw);
  std::vector<int> lv{0};
  lv.insert(lv.end(), Ps2.begin(), Ps2.end());
  bool nested = Ps2[0] > 1 && psolve_level(cx, R.V, nr, b, a, lv, 1, 1.0, R.ready);
  if (!nested) solve_reduced(cx, b, a, nr, R);
  for (auto &ps : parts) {
    scatter_xr(cx, ps, PQ, b, a, R);
    ppobtasi_part(cx, ps, b, false);  // W tiles recomputed by TRTRI (no fused POTRF here)
  }
  // log det = sum of the ranks' partials (rank order) + 2 sum log diag of POBTAF(A_r)
  cx.logdet(Loc{BUF_LOGDET, 0, 0}, part_slots, cx.slot_count - part_slots, Loc{BUF_EXT1, 0, x.ld()}, P, Q * recsz,
            {});
  return cx.finalize();
}

int64_t distributed_ws_bytes(int P, int rank, int64_t n, int64_t start, int64_t count, int64_t b, int64_t a, int Q) {
  BuildOptions opt;
  opt.apply_env();
  opt.schedule = false;
  Graph g0 = build_distributed(0, P, rank, n, start, count, b, a, opt, Q);
  Graph g1 = build_distributed(1, P, rank, n, start, count, b, a, opt, Q);
  if (!g0.error.empty() || !g1.error.empty()) return -1;
  return std::max(g0.ws_doubles, g1.ws_doubles) * 8;
}

}  // namespace serinv
