// exact_layout's branch-and-bound (pkg/src/memplan/layout.py:153-302) for
// the layout problems K3 cannot decide (some overlap component's long-lived
// first incumbent lies above its lower bound).  Host C++: the search is a
// sequential depth-first walk whose result depends on where its node cap
// stops it, so it is restated node for node rather than parallelised.
//
//   activation block      layout.py:81-97   stacked from 0 in (-len, id) order
//   floors                layout.py:95      block top if the item overlaps an
//                                           activation (bottom mode), else 0
//   components            layout.py:180-197 union-find on time overlap; root =
//                                           smallest tensor id; roots ascending
//   bound                 layout.py:209-217 per probe start: live bytes, and
//                                           block top + floored live bytes
//   incumbent             K3 COMPONENTS offsets (the per-component long-lived
//                                           first placement, layout.py:219-224)
//   search                layout.py:226-282 items ordered by (-size*(len+1),
//                                           id); per node: a key (size, start,
//                                           end, floor) is branched once; the
//                                           lowest fit over the placed,
//                                           time-overlapping spans sorted by
//                                           (lo, hi); prune new_cap >= best
//   budget                node_cap over the nodes of all components together;
//                                           the wall-clock deadline checked every
//                                           4096 nodes, as the reference does
#include <time.h>

#include <algorithm>
#include <array>
#include <numeric>
#include <vector>

#include "roam_internal.h"

namespace roam {
namespace {

struct Budget {};
struct Done {};

double mono_now() {
  timespec ts{};
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return double(ts.tv_sec) + 1e-9 * double(ts.tv_nsec);
}

// item masks of W 64-bit words (components of up to 64 W items)
template <int W>
struct Search {
  int n = 0;
  std::vector<int64_t> size, floor_;
  std::vector<int32_t> st, en;
  std::vector<uint64_t> ov;  // [n][W] overlap bits
  std::vector<int64_t> off, best_off;
  int64_t best_cap = 0, bound = 0;
  int64_t nodes = 0, nodes_before = 0, node_cap = -1;
  double deadline = 0.0;
  uint64_t used[W] = {};

  void run(int depth, int64_t cap) {
    ++nodes;
    if (node_cap >= 0 && nodes_before + nodes > node_cap) throw Budget{};
    if (nodes % 4096 == 0 && deadline > 0.0 && mono_now() > deadline) throw Budget{};
    if (cap >= best_cap) return;
    if (depth == n) {
      best_cap = cap;
      best_off = off;
      if (best_cap <= bound) throw Done{};
      return;
    }
    std::vector<std::array<int64_t, 4>> tried;
    std::vector<std::pair<int64_t, int64_t>> spans;
    for (int i = 0; i < n; ++i) {
      if ((used[i >> 6] >> (i & 63)) & 1) continue;
      const std::array<int64_t, 4> key{size[i], st[i], en[i], floor_[i]};
      if (std::find(tried.begin(), tried.end(), key) != tried.end()) continue;
      tried.push_back(key);
      spans.clear();
      const uint64_t* ovi = ov.data() + size_t(i) * W;
      for (int k = 0; k < W; ++k)
        for (uint64_t m = used[k] & ovi[k]; m; m &= m - 1) {
          const int j = 64 * k + __builtin_ctzll(m);
          spans.emplace_back(off[j], off[j] + size[j]);
        }
      std::sort(spans.begin(), spans.end());
      int64_t o = floor_[i];
      for (const auto& sp : spans) {
        if (o + size[i] <= sp.first) break;
        if (sp.second > o) o = sp.second;
      }
      const int64_t new_cap = cap >= o + size[i] ? cap : o + size[i];
      if (new_cap >= best_cap) continue;
      used[i >> 6] |= uint64_t(1) << (i & 63);
      off[i] = o;
      run(depth + 1, new_cap);
      used[i >> 6] &= ~(uint64_t(1) << (i & 63));
    }
  }
};

// one component's search (items in the reference's branching order);
// returns false when the node cap or the deadline stopped it
template <int W>
bool search_component(const std::vector<int>& order, const int32_t* start, const int32_t* end,
                      const int64_t* size, const std::vector<int64_t>& flo, const int64_t* incumbent,
                      int64_t bound, int64_t node_cap, double deadline, int64_t& nodes_total,
                      int64_t& best_cap, int64_t* offset);

bool overlaps(const int32_t* s, const int32_t* e, int a, int b) { return s[a] <= e[b] && s[b] <= e[a]; }

}  // namespace
}  // namespace roam

using namespace roam;

extern "C" int rm_layout_search(int32_t n, const int32_t* tensor, const int32_t* start, const int32_t* end,
                                const int64_t* size, const uint8_t* is_act, int32_t bottom,
                                const int64_t* incumbent, int64_t node_cap, double deadline,
                                int64_t* offset, int64_t* capacity, int64_t* nodes_out,
                                int32_t* optimal) {
  if (n < 0 || !capacity || !nodes_out || !optimal) return fail(RM_ERR_INVALID_ARG, "bad rm_layout_search arguments");
  if (n > 0 && (!tensor || !start || !end || !size || !is_act || !incumbent || !offset))
    return fail(RM_ERR_INVALID_ARG, "NULL item array");
  *nodes_out = 0;
  *optimal = 1;
  if (n == 0) {
    *capacity = 0;
    return RM_OK;
  }
  // activation block and floors (layout.py:81-97)
  std::vector<int> atvs;
  if (bottom)
    for (int i = 0; i < n; ++i)
      if (is_act[i]) atvs.push_back(i);
  std::sort(atvs.begin(), atvs.end(), [&](int a, int b) {
    const int64_t la = int64_t(end[a]) - start[a], lb = int64_t(end[b]) - start[b];
    return la != lb ? la > lb : tensor[a] < tensor[b];
  });
  int64_t block_top = 0;
  for (int a : atvs) {
    offset[a] = block_top;
    block_top += size[a];
  }
  std::vector<int64_t> flo(n, 0);
  std::vector<int> rest;
  for (int i = 0; i < n; ++i) {
    if (bottom && is_act[i]) continue;
    rest.push_back(i);
    if (bottom)
      for (int a : atvs)
        if (overlaps(start, end, i, a)) {
          flo[i] = block_top;
          break;
        }
  }
  // overlap components of the rest, keyed by their smallest tensor id
  std::vector<int> parent(n);
  std::iota(parent.begin(), parent.end(), 0);
  auto find = [&](int x) {
    while (parent[x] != x) x = parent[x] = parent[parent[x]];
    return x;
  };
  for (size_t a = 0; a < rest.size(); ++a)
    for (size_t b = a + 1; b < rest.size(); ++b)
      if (overlaps(start, end, rest[a], rest[b])) {
        const int ra = find(rest[a]), rb = find(rest[b]);
        if (ra != rb) {
          if (tensor[ra] < tensor[rb]) parent[rb] = ra; else parent[ra] = rb;
        }
      }
  std::vector<std::vector<int>> comps;
  {
    std::vector<int> roots;
    for (int i : rest)
      if (find(i) == i) roots.push_back(i);
    std::sort(roots.begin(), roots.end(), [&](int a, int b) { return tensor[a] < tensor[b]; });
    std::vector<int> slot(n, -1);
    for (size_t k = 0; k < roots.size(); ++k) slot[roots[k]] = (int)k;
    comps.resize(roots.size());
    for (int i : rest) comps[slot[find(i)]].push_back(i);
  }
  int64_t cap_total = block_top, nodes_total = 0;
  bool opt = true;
  for (auto& comp : comps) {
    // bound (layout.py:209-217)
    int64_t bound = 0;
    for (int probe : comp) {
      const int32_t t = start[probe];
      int64_t total = 0, above = 0;
      for (int i : comp)
        if (start[i] <= t && t <= end[i]) {
          total += size[i];
          if (flo[i]) above += size[i];
        }
      bound = std::max({bound, total, above ? block_top + above : int64_t(0)});
    }
    int64_t best_cap = 0;
    for (int i : comp) {
      offset[i] = incumbent[i];
      best_cap = std::max(best_cap, incumbent[i] + size[i]);
    }
    if (best_cap > bound) {
      std::vector<int> order(comp);
      std::sort(order.begin(), order.end(), [&](int a, int b) {
        const int64_t ka = -size[a] * (int64_t(end[a]) - start[a] + 1);
        const int64_t kb = -size[b] * (int64_t(end[b]) - start[b] + 1);
        return ka != kb ? ka < kb : tensor[a] < tensor[b];
      });
      const int words = ((int)order.size() + 63) / 64;
      bool ok = true;
#define RM_LAYOUT_W(w)                                                                            \
  else if (words <= w) ok = search_component<w>(order, start, end, size, flo, incumbent, bound, \
                                                node_cap, deadline, nodes_total, best_cap, offset);
      if (words > 256) return fail(RM_ERR_CAPACITY, "rm_layout_search: components of at most 16384 items");
      RM_LAYOUT_W(1)
      RM_LAYOUT_W(2)
      RM_LAYOUT_W(4)
      RM_LAYOUT_W(8)
      RM_LAYOUT_W(16)
      RM_LAYOUT_W(32)
      RM_LAYOUT_W(64)
      RM_LAYOUT_W(128)
      RM_LAYOUT_W(256)
#undef RM_LAYOUT_W
      if (!ok) opt = false;
    }
    cap_total = std::max(cap_total, best_cap);
  }
  *capacity = cap_total;
  *nodes_out = nodes_total;
  *optimal = opt ? 1 : 0;
  return RM_OK;
}

namespace roam {
namespace {
template <int W>
bool search_component(const std::vector<int>& order, const int32_t* start, const int32_t* end,
                      const int64_t* size, const std::vector<int64_t>& flo, const int64_t* incumbent,
                      int64_t bound, int64_t node_cap, double deadline, int64_t& nodes_total,
                      int64_t& best_cap, int64_t* offset) {
  Search<W> S;
  S.n = (int)order.size();
  S.size.resize(S.n);
  S.floor_.resize(S.n);
  S.st.resize(S.n);
  S.en.resize(S.n);
  S.ov.assign(size_t(S.n) * W, 0);
  S.off.assign(S.n, 0);
  for (int k = 0; k < S.n; ++k) {
    const int i = order[k];
    S.size[k] = size[i];
    S.floor_[k] = flo[i];
    S.st[k] = start[i];
    S.en[k] = end[i];
    S.best_off.push_back(incumbent[i]);
  }
  for (int a = 0; a < S.n; ++a)
    for (int b = a + 1; b < S.n; ++b)
      if (overlaps(start, end, order[a], order[b])) {
        S.ov[size_t(a) * W + (b >> 6)] |= uint64_t(1) << (b & 63);
        S.ov[size_t(b) * W + (a >> 6)] |= uint64_t(1) << (a & 63);
      }
  S.best_cap = best_cap;
  S.bound = bound;
  S.nodes_before = nodes_total;
  S.node_cap = node_cap;
  S.deadline = deadline;
  bool ok = true;
  try {
    S.run(0, 0);
  } catch (const Done&) {
  } catch (const Budget&) {
    ok = false;
  }
  nodes_total += S.nodes;
  best_cap = S.best_cap;
  for (int k = 0; k < S.n; ++k) offset[order[k]] = S.best_off[k];
  return ok;
}
}  // namespace
}  // namespace roam
