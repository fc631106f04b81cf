// place_weight_updates (reference pkg/src/memplan/ordering.py:387-467) in
// libroam, host C++: the weight-update branch placement the planner runs once
// or twice per plan (planner.py:201-207).
//
// The reference re-derives, per branch and per candidate window, the bytes of
// activations alive at a timestep by rescanning every tensor
// (weight_update_cost, ordering.py:310-338).  Here the activation lifetimes
// [asap(producer), max alap(consumers)] (horizon n-1 without consumers) become
// one +size/-size event sweep, so each query is a table lookup; the branch
// loop itself (sort key, ready step, home window, delay rule, first later
// window whose projected use drops back under the activation total) follows
// the reference statement by statement.  Floating point: projected use is
// double(alive) + alpha * double(grad_bytes) and the size ratio
// double(grad_bytes) / mean_size, the expressions Python evaluates (IEEE
// double, no contraction: every operand below 2^53); comparisons against the
// integer activation total are exact in both.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "roam.h"
#include "roam_internal.h"

using namespace roam;

extern "C" int rm_place_weight_updates(
    int32_t n_ops, const int32_t* asap, int64_t n_act, const int32_t* act_start, const int32_t* act_end,
    const int64_t* act_size, double mean_size, int32_t n_slots, const int32_t* slot_kind,
    const int32_t* slot_ref, int32_t n_windows, const int64_t* win_ptr, const int32_t* win_ops,
    int32_t tail_window, int32_t n_branches, const int32_t* br_first, const int64_t* grad_ptr,
    const int32_t* grad_producer, const int64_t* grad_bytes, const double* alpha, double r,
    int32_t force_immediate, int32_t* out_branch, uint8_t* out_delayed, int32_t* out_target,
    int32_t* out_ready, double* out_ratio, double* out_projected, int64_t* activation_total,
    int32_t* missing_op) {
  if (n_ops < 0 || n_act < 0 || n_slots < 0 || n_windows < 0 || n_branches < 0 || !activation_total ||
      !missing_op || (n_ops > 0 && !asap) || (n_act > 0 && (!act_start || !act_end || !act_size)) ||
      (n_slots > 0 && (!slot_kind || !slot_ref)) || !win_ptr ||
      (n_branches > 0 && (!br_first || !grad_ptr || !grad_producer || !grad_bytes || !alpha || !out_branch ||
                          !out_delayed || !out_target || !out_ready || !out_ratio || !out_projected)))
    return fail(RM_ERR_INVALID_ARG, "bad rm_place_weight_updates arguments");
  *missing_op = -1;
  *activation_total = 0;
  // alive[t] for t in [0, n): activations with start <= t <= end
  int64_t total = 0;
  std::vector<int64_t> alive((size_t)n_ops + 1, 0);
  for (int64_t k = 0; k < n_act; ++k) {
    total += act_size[k];
    const int64_t s = act_start[k], e = act_end[k];
    if (s <= e && s < n_ops && e >= 0) {
      alive[size_t(std::max<int64_t>(s, 0))] += act_size[k];
      alive[size_t(std::min<int64_t>(e, n_ops - 1)) + 1] -= act_size[k];
    }
  }
  for (int32_t t = 1; t <= n_ops; ++t) alive[t] += alive[t - 1];
  auto alive_at = [&](int64_t t) -> int64_t { return (t >= 0 && t < n_ops) ? alive[size_t(t)] : 0; };
  auto bad_op = [&](int64_t v) { return v < 0 || v >= n_ops; };
  // _op_slot_positions (ordering.py:360-368): later slots overwrite earlier
  std::vector<int32_t> pos((size_t)n_ops, -1);
  for (int32_t i = 0; i < n_slots; ++i) {
    if (slot_kind[i] == 0) {
      if (bad_op(slot_ref[i])) return fail(RM_ERR_INVALID_ARG, "slot op out of range");
      pos[size_t(slot_ref[i])] = i;
    } else {
      const int32_t w = slot_ref[i];
      if (w < 0 || w >= n_windows) return fail(RM_ERR_INVALID_ARG, "slot window out of range");
      for (int64_t q = win_ptr[w]; q < win_ptr[w + 1]; ++q) {
        if (bad_op(win_ops[q])) return fail(RM_ERR_INVALID_ARG, "window op out of range");
        pos[size_t(win_ops[q])] = i;
      }
    }
  }
  // branch order: (max asap over gradient producers, first op)
  std::vector<int32_t> order((size_t)n_branches);
  std::vector<int64_t> key((size_t)n_branches);
  std::vector<int32_t> prod((size_t)n_branches);
  for (int32_t b = 0; b < n_branches; ++b) {
    if (grad_ptr[b + 1] <= grad_ptr[b]) return fail(RM_ERR_INVALID_ARG, "branch without gradients");
    int32_t best = -1;
    for (int64_t q = grad_ptr[b]; q < grad_ptr[b + 1]; ++q) {
      const int32_t v = grad_producer[q];
      if (bad_op(v)) return fail(RM_ERR_INVALID_ARG, "gradient producer out of range");
      // max by (asap, v), ordering.py:418-421
      if (best < 0 || asap[v] > asap[best] || (asap[v] == asap[best] && v > best)) best = v;
    }
    prod[size_t(b)] = best;
    key[size_t(b)] = asap[best];
  }
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
    if (key[size_t(x)] != key[size_t(y)]) return key[size_t(x)] < key[size_t(y)];
    return br_first[x] < br_first[y];
  });
  const double est = (double)total;
  for (int32_t k = 0; k < n_branches; ++k) {
    const int32_t b = order[size_t(k)];
    const int32_t producer = prod[size_t(b)];
    const int32_t ready_t = asap[producer];
    const double gb = (double)grad_bytes[b];
    const double projected = (double)alive_at(ready_t) + alpha[b] * gb;
    const double ratio = mean_size != 0.0 ? gb / mean_size : 0.0;
    const bool delayed = !force_immediate && ratio > r && projected > est;
    const int32_t home_slot = pos[size_t(producer)];
    if (home_slot < 0) {  // positions[producer] raises KeyError in the reference
      *missing_op = producer;
      return fail(RM_ERR_GRAPH, "gradient producer has no slot");
    }
    int32_t home = -1;
    for (int32_t i = home_slot; i < n_slots; ++i)
      if (slot_kind[i] == 1 && win_ptr[slot_ref[i] + 1] > win_ptr[slot_ref[i]]) {
        home = slot_ref[i];
        break;
      }
    if (home < 0) home = tail_window >= 0 ? tail_window : 0;
    int32_t target = home;
    double chosen = projected;
    if (delayed) {
      target = tail_window >= 0 ? tail_window : home;
      for (int32_t i = home_slot + 1; i < n_slots; ++i) {
        if (slot_kind[i] != 1 || slot_ref[i] == tail_window) continue;
        int64_t t_w = ready_t;
        if (slot_kind[i - 1] == 0) t_w = int64_t(asap[slot_ref[i - 1]]) + 1;
        const double use_w = (double)alive_at(t_w) + alpha[b] * gb;
        if (use_w <= est) {
          target = slot_ref[i];
          chosen = use_w;
          break;
        }
      }
    }
    out_branch[k] = b;
    out_delayed[k] = delayed ? 1 : 0;
    out_target[k] = target;
    out_ready[k] = ready_t;
    out_ratio[k] = ratio;
    out_projected[k] = chosen;
  }
  if (n_branches > 0) *activation_total = total;
  return RM_OK;
}
