// exact_order's capped depth-first search (pkg/src/memplan/ordering.py:183-286)
// for the windows K5 hands back: more order ideals than the node cap, or more
// ops than the GPU DP holds.  Masks are W 64-bit words (a template per width,
// up to 16,384 ops), so windows of any node_limit are served here.  Whether the reference's pruned search reaches
// its cap depends on the exact expansion order, so it is restated node for
// node on the host rather than parallelised:
//
//   _Local           ordering.py:84-123  tracked tensors = outputs of window
//                                        ops + live-in, counted per local
//                                        consumer ENTRY; held = live-out, or
//                                        produced inside with no local consumer
//   input lists      ordering.py:206-211 tracked inputs of each op, distinct,
//                                        one decrement per op (so a tensor an op
//                                        lists twice never frees: hazard h1)
//   search           ordering.py:213-245 memo on the scheduled mask; a node is
//                                        counted when a mask is expanded; branch
//                                        i skipped when live + out[i] >= best
//   budget           node_cap, and the wall-clock deadline every 1024 nodes;
//                                        either returns the greedy incumbent
//   reconstruction   ordering.py:252-279 smallest ready local index whose branch
//                                        value reaches memo[mask]
#include <time.h>

#include <algorithm>
#include <unordered_map>
#include <vector>

#include "roam_internal.h"

namespace roam {
namespace {

struct OrderBudget {};
struct OrderCycle {};

double order_now() {
  timespec ts{};
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return double(ts.tv_sec) + 1e-9 * double(ts.tv_nsec);
}

// scheduled-op masks of W 64-bit words (windows of up to 64 W ops)
template <int W>
struct Mask {
  uint64_t w[W];
  bool operator==(const Mask& o) const {
    for (int k = 0; k < W; ++k)
      if (w[k] != o.w[k]) return false;
    return true;
  }
  bool has(int i) const { return (w[i >> 6] >> (i & 63)) & 1; }
  void set(int i) { w[i >> 6] |= uint64_t(1) << (i & 63); }
  bool covers(const Mask& m) const {  // every bit of m is set here
    for (int k = 0; k < W; ++k)
      if (m.w[k] & ~w[k]) return false;
    return true;
  }
};

template <int W>
struct MaskHash {
  size_t operator()(const Mask<W>& m) const {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (int k = 0; k < W; ++k) {
      h ^= m.w[k] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      h *= 0xbf58476d1ce4e5b9ull;
    }
    return size_t(h ^ (h >> 31));
  }
};

template <int W>
struct OrderDfs {
  using M = Mask<W>;
  int n = 0;
  M full{};
  std::vector<M> pred;
  std::vector<int64_t> out;
  std::vector<std::vector<int>> inputs;  // local tensor indices
  std::vector<int> counts;
  std::vector<uint8_t> held;
  std::vector<int64_t> tsize;
  std::unordered_map<M, int64_t, MaskHash<W>> memo;
  int64_t nodes = 0, node_cap = -1;
  double deadline = 0.0;

  bool ready(const M& mask, int i) const { return !mask.has(i) && mask.covers(pred[i]); }

  int64_t search(M& mask, int64_t live) {
    if (mask == full) return 0;
    auto hit = memo.find(mask);
    if (hit != memo.end()) return hit->second;
    ++nodes;
    if (node_cap >= 0 && nodes > node_cap) throw OrderBudget{};
    if (nodes % 1024 == 0 && deadline > 0.0 && order_now() > deadline) throw OrderBudget{};
    bool have = false;
    int64_t best = 0;
    for (int i = 0; i < n; ++i) {
      if (!ready(mask, i)) continue;
      const int64_t step = live + out[i];
      if (have && step >= best) continue;
      int64_t new_live = step;
      for (int t : inputs[i])
        if (--counts[t] == 0 && !held[t]) new_live -= tsize[t];
      mask.set(i);
      const int64_t sub = search(mask, new_live);
      mask.w[i >> 6] &= ~(uint64_t(1) << (i & 63));
      const int64_t value = step >= sub ? step : sub;
      for (int t : inputs[i]) ++counts[t];
      if (!have || value < best) {
        best = value;
        have = true;
      }
    }
    if (!have) throw OrderCycle{};  // no ready op: the window precedence has a cycle
    memo.emplace(mask, best);
    return best;
  }

  // the reference's search, then its reconstruction walk (ordering.py:252-279):
  // 0 ok, 2 cycle, 4 budget; -1 reconstruction failure
  int run(int64_t start_live, const std::vector<int>& wops, int32_t* order, int64_t* peak) {
    int64_t optimum = 0;
    M mask{};
    try {
      optimum = std::max(search(mask, start_live), start_live);
    } catch (const OrderBudget&) {
      return 4;
    } catch (const OrderCycle&) {
      return 2;
    }
    mask = M{};
    int64_t live = start_live;
    for (int step_i = 0; step_i < n; ++step_i) {
      auto tm = memo.find(mask);
      if (tm == memo.end()) return -1;
      const int64_t target = tm->second;
      int chosen = -1;
      for (int i = 0; i < n && chosen < 0; ++i) {
        if (!ready(mask, i)) continue;
        const int64_t step = live + out[i];
        M nxt = mask;
        nxt.set(i);
        int64_t sub = 0;
        if (!(nxt == full)) {
          auto it = memo.find(nxt);
          if (it == memo.end()) continue;
          sub = it->second;
        }
        if (std::max(step, sub) <= target) chosen = i;
      }
      if (chosen < 0) return -1;
      live += out[chosen];
      for (int t : inputs[chosen])
        if (--counts[t] == 0 && !held[t]) live -= tsize[t];
      mask.set(chosen);
      order[step_i] = wops[chosen];
    }
    *peak = optimum;
    return 0;
  }
};

// the window's _Local state, independent of the mask width
struct LocalState {
  std::vector<std::vector<int>> pred_idx;  // local preds per op
  std::vector<int64_t> out;
  std::vector<std::vector<int>> inputs;
  std::vector<int> counts;
  std::vector<uint8_t> held;
  std::vector<int64_t> tsize;
};

template <int W>
int solve_w(const LocalState& L, int n_ops, int64_t start_live, const std::vector<int>& wops,
            int64_t node_cap, double deadline, int32_t* order, int64_t* peak, int64_t* nodes) {
  OrderDfs<W> S;
  S.n = n_ops;
  for (int i = 0; i < n_ops; ++i) S.full.set(i);
  S.pred.assign(n_ops, Mask<W>{});
  for (int i = 0; i < n_ops; ++i)
    for (int j : L.pred_idx[i]) S.pred[i].set(j);
  S.out = L.out;
  S.inputs = L.inputs;
  S.counts = L.counts;
  S.held = L.held;
  S.tsize = L.tsize;
  S.node_cap = node_cap;
  S.deadline = deadline;
  const int r = S.run(start_live, wops, order, peak);
  *nodes = S.nodes;
  return r;
}

}  // namespace
}  // namespace roam

using namespace roam;

extern "C" int rm_exact_order_search(RmGraph* g, int32_t n_ops, const int32_t* ops, int64_t n_lin,
                                     const int32_t* lin, int64_t n_lout, const int32_t* lout,
                                     int64_t node_cap, double deadline, int32_t* order, int64_t* peak,
                                     int64_t* nodes, int32_t* status, int32_t* bad_tensor) {
  if (!g || n_ops < 0 || n_lin < 0 || n_lout < 0 || !peak || !nodes || !status || !bad_tensor ||
      (n_ops && (!ops || !order)) || (n_lin && !lin) || (n_lout && !lout))
    return fail(RM_ERR_INVALID_ARG, "bad rm_exact_order_search arguments");
  const int n = g->n, T = g->T;
  *status = 0;
  *bad_tensor = -1;
  *nodes = 0;
  std::vector<int> wops(ops, ops + n_ops);
  for (int v : wops)
    if (v < 0 || v >= n) return fail(RM_ERR_INVALID_ARG, "window op out of range");
  std::sort(wops.begin(), wops.end());
  if (std::adjacent_find(wops.begin(), wops.end()) != wops.end())
    return fail(RM_ERR_INVALID_ARG, "window lists an op twice");
  if (n_ops > 64 * 256) return fail(RM_ERR_CAPACITY, "rm_exact_order_search: windows of at most 16384 ops");
  std::vector<int> loc(n, -1);
  for (int i = 0; i < n_ops; ++i) loc[wops[i]] = i;
  std::vector<uint8_t> is_lin(T, 0), is_lout(T, 0);
  for (int64_t k = 0; k < n_lin; ++k) {
    if (lin[k] < 0 || lin[k] >= T) return fail(RM_ERR_INVALID_ARG, "live-in tensor out of range");
    is_lin[lin[k]] = 1;
  }
  for (int64_t k = 0; k < n_lout; ++k) {
    if (lout[k] < 0 || lout[k] >= T) return fail(RM_ERR_INVALID_ARG, "live-out tensor out of range");
    is_lout[lout[k]] = 1;
  }
  // _Local: tracked tensors in ascending id order (ordering.py:100-112)
  std::vector<int> rel;
  for (int v : wops)
    for (int k = g->out_ptr[v]; k < g->out_ptr[v + 1]; ++k) rel.push_back(g->out_idx[k]);
  for (int t = 0; t < T; ++t)
    if (is_lin[t]) rel.push_back(t);
  std::sort(rel.begin(), rel.end());
  rel.erase(std::unique(rel.begin(), rel.end()), rel.end());
  LocalState S;
  std::vector<int> tloc(T, -1);
  int64_t start_live = 0;
  for (int t : rel) {
    int local = 0;
    for (int k = g->cons_ptr[t]; k < g->cons_ptr[t + 1]; ++k) local += loc[g->cons_idx[k]] >= 0;
    const bool produced = loc[g->producer[t]] >= 0;
    bool held = false;
    if (is_lout[t] || (produced && local == 0)) {
      held = true;
    } else if (is_lin[t] && local == 0) {
      *status = 1;  // ConfigError (ordering.py:107-110): smallest such id
      *bad_tensor = t;
      return RM_OK;
    }
    tloc[t] = (int)S.counts.size();
    S.counts.push_back(local);
    S.held.push_back(held ? 1 : 0);
    S.tsize.push_back(g->size[t]);
  }
  for (int t : rel)
    if (is_lin[t]) start_live += g->size[t];
  S.pred_idx.resize(n_ops);
  S.out.assign(n_ops, 0);
  S.inputs.resize(n_ops);
  for (int i = 0; i < n_ops; ++i) {
    const int v = wops[i];
    for (int k = g->out_ptr[v]; k < g->out_ptr[v + 1]; ++k) S.out[i] += g->size[g->out_idx[k]];
    for (int k = g->in_ptr[v]; k < g->in_ptr[v + 1]; ++k) {
      const int t = g->in_idx[k];
      const int pr = g->producer[t];
      if (loc[pr] >= 0 && pr != v) S.pred_idx[i].push_back(loc[pr]);
      const int lt = tloc[t];
      if (lt >= 0 && std::find(S.inputs[i].begin(), S.inputs[i].end(), lt) == S.inputs[i].end())
        S.inputs[i].push_back(lt);
    }
  }
  if (n_ops == 0) {
    *peak = start_live;
    return RM_OK;
  }
  // the narrowest mask that holds the window: one 64-bit word up to 64 ops
  // (the common case), then powers of two up to 256 words
  int r = 0;
  const int words = (n_ops + 63) / 64;
#define RM_ORDER_W(w) \
  else if (words <= w) r = solve_w<w>(S, n_ops, start_live, wops, node_cap, deadline, order, peak, nodes);
  if (false) {
  }
  RM_ORDER_W(1)
  RM_ORDER_W(2)
  RM_ORDER_W(4)
  RM_ORDER_W(8)
  RM_ORDER_W(16)
  RM_ORDER_W(32)
  RM_ORDER_W(64)
  RM_ORDER_W(128)
  RM_ORDER_W(256)
#undef RM_ORDER_W
  if (r < 0) return fail(RM_ERR_INVALID_ARG, "order reconstruction failed");
  *status = r;  // 0 ok, 2 cycle (AssertionError), 4 budget (the greedy incumbent)
  return RM_OK;
}
