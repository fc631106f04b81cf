/*
 * roam.h -- C ABI of libroam, the B200 (sm_100a) implementation of the ROAM
 * planner's data-parallel hot path (arXiv 2310.19295; reference:
 * /root/reference/pkg/src/memplan).
 *
 * Plain C types only: pointers, sizes, int status codes.  Every entry point
 * returns RM_OK (0) or a negative RmStatus; rm_last_error() gives a
 * thread-local message for the last failure on the calling thread.
 *
 * Memory: the caller owns every input and output buffer.  Unless a call
 * takes RM_DEVICE_PTRS in its flags, pointers are HOST pointers (pinned or
 * pageable) and the call stages them through the device itself and returns
 * only after the results are back on the host.  With RM_DEVICE_PTRS all
 * array arguments are device pointers and the call is asynchronous on
 * `stream` (a cudaStream_t; NULL = legacy default stream).
 *
 * The only library-owned memory is the immutable RmGraph handle (graph CSR
 * + derived evaluation metadata, host and device copies).  Calls never share
 * scratch, so they are re-entrant across threads and streams (the reference's
 * ThreadPoolExecutor contract, planner.py:119-124).
 */
#ifndef ROAM_H_
#define ROAM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RM_OK = 0,
  RM_ERR_INVALID_ARG = -1,
  RM_ERR_CUDA = -2,
  RM_ERR_OVERFLOW = -3,
  RM_ERR_NO_DEVICE = -4,
  RM_ERR_CAPACITY = -5,
  RM_ERR_GRAPH = -6
} RmStatus;

enum {
  RM_DEVICE_PTRS = 1u << 0,  /* array arguments are device pointers; async */
  RM_NO_REDUCE = 1u << 1,    /* rm_graph_create: skip transitive reduction */
  RM_ORDERS_U16 = 1u << 2    /* rm_eval_orders/select: rows are uint16[B, n] (n <= 65535):
                                half the bytes to stage and to read */
};

/* ------------------------------------------------------------------ graph */

/* CSR description of a graph with dense ids (reference graph.py:59-135,
 * load_graph 188-278).  cons_idx keeps one entry per input occurrence
 * (graph.py:227-231); in_idx keeps each op's inputs in document order. */
typedef struct {
  int32_t n_ops;
  int32_t n_tensors;
  const int64_t* size;      /* [T] bytes */
  const int32_t* producer;  /* [T] */
  const int32_t* cons_ptr;  /* [T+1] */
  const int32_t* cons_idx;  /* [E] */
  const int32_t* in_ptr;    /* [n+1] */
  const int32_t* in_idx;    /* [E] */
  const int32_t* out_ptr;   /* [n+1] */
  const int32_t* out_idx;   /* [sum outputs] */
} RmGraphDesc;

typedef struct RmGraph RmGraph;

typedef struct {
  int32_t n_ops, n_tensors;
  int64_t n_cons;           /* E */
  int64_t n_pred_edges;     /* P: deduplicated, self-free direct_preds edges */
  int64_t n_check_edges;    /* edges K1 checks (transitive reduction of P) */
  int64_t n_multi;          /* tensors with >= 2 maximal consumers */
  int64_t n_multi_cons;     /* their maximal-consumer entries */
  int64_t n_slots;          /* distinct ops closing a multi-consumer lifetime */
  int64_t n_values;         /* distinct (out_bytes, free_bytes) op classes */
  int32_t reduced;          /* 1 when the reduction ran */
  int32_t wide_index;       /* 1 when ids need int32 (n > 65535) */
  int64_t total_bytes;      /* sum of |size| */
  int32_t k1_variant;       /* default K1: 5 v5 (class bytes), 4 v4, 1 generic */
  int32_t unit_shift;       /* K1 v2 byte unit = 2^unit_shift */
} RmGraphInfo;

/* Validate + marshal a graph; computes the order-evaluation metadata on the
 * host (transitive reduction, maximal consumers, per-op event classes) and,
 * when a device is present, uploads it.  With no CUDA device the handle is
 * host-only: rm_graph_info works, every device entry point fails with
 * RM_ERR_NO_DEVICE. */
int rm_graph_create(const RmGraphDesc* desc, uint32_t flags, RmGraph** out);
int rm_graph_destroy(RmGraph* g);
int rm_graph_info(const RmGraph* g, RmGraphInfo* info);

/* Host copy of the K1 metadata (sizes from rm_graph_info): per-op event class
 * and slot (-1 = none), class table (out_bytes, free_bytes), checked edges,
 * multi-consumer CSR.  Any pointer may be NULL.  Host-only; no device needed. */
int rm_graph_k1_export(const RmGraph* g, int32_t* vidx, int32_t* slot, int64_t* out_tab,
                       int64_t* fs_tab, int32_t* edge_u, int32_t* edge_v, int32_t* mptr,
                       int32_t* mcons, int64_t* msize);

/* Transitive predecessors of every op as bitsets (graph.py:335-347
 * predecessor_masks): rows[v * words + i] bit j set iff op 64*i+j precedes v,
 * words = ceil(n_ops / 64).  Host-only; feeds the vectorised control-plane
 * helpers of the planner plug-in (region filters, linearisation ranks). */
int rm_graph_ancestors(const RmGraph* g, uint64_t* rows);

/* counts[r] = popcount(rows[r] & mask) over `words` 64-bit words per row (mask
 * NULL = all bits): the masked ancestor counts of the plug-in's tree build
 * (segmentation.py:108-117 _mi_over, 408-418 residual ranks).  Host-only. */
int rm_popcount_rows(const uint64_t* rows, int64_t n_rows, int64_t words, const uint64_t* mask,
                     int64_t* counts);

/* Schedule bounds (replaces graph.py:365-372 asap_alap): asap[v] = number of
 * transitive predecessors, alap[v] = n-1 - number of transitive successors,
 * from closure bitsets in C++.  Host-only (no device needed); control-plane
 * code the planner's weight-update placement calls (ordering.py:405). */
int rm_graph_asap_alap(const RmGraph* g, int32_t* asap, int32_t* alap);

/* ----------------------------------------------------- K1: order batches */

/* Evaluate B candidate orders (orders is int32[B, n_ops], row-major), each as
 * peak_memory(g, sequential_schedule(g, order)) (reference graph.py:401-409,
 * 461-468):
 *   valid[b]  = 1 iff the row is a permutation respecting every direct pred
 *               (validate_schedule, graph.py:375-398);
 *   peak[b]   = max over timesteps of live bytes;
 *   argmax[b] = first timestep attaining it.
 * Rows with valid == 0 have unspecified peak/argmax (the reference raises
 * ScheduleError for them).  Replaces graph.py:461 peak_memory in a loop. */
int rm_eval_orders(RmGraph* g, const void* orders, int64_t B, uint32_t flags,
                   int64_t* peak, int32_t* argmax, uint8_t* valid, void* stream);

/* rm_eval_orders followed by rm_argmin in one call: the candidate-plan
 * selection step of the planner (planner.py:209-216) -- best = {peak, id}
 * of the first strict minimum, ids numbered from id_base.  With host
 * pointers the orders are staged through the device in chunks (copy/compute
 * overlap) and every output is back on the host when the call returns. */
int rm_eval_select(RmGraph* g, const void* orders, int64_t B, int64_t id_base, uint32_t flags,
                   int64_t* peak, int32_t* argmax, uint8_t* valid, int64_t* best /* [2] */,
                   void* stream);

/* First strict minimum over valid candidates, i.e. the lexicographic min of
 * (peak, id) -- reference tests/oracles.py:46-56 and planner.py:209-216.
 * out_best = {peak, id + id_base} or {INT64_MAX, -1} when none is valid. */
int rm_argmin(const int64_t* peak, const uint8_t* valid, int64_t B, int64_t id_base,
              uint32_t flags, int64_t* out_best /* [2] */, void* stream);

/* Device-only variant for multi-GPU selection: out_key (device int64[1]) =
 * (peak << id_bits) | (id + id_base) of the first strict minimum, INT64_MAX
 * when none is valid.  Ranks then combine with ONE all_reduce(MIN) of 8 bytes:
 * the packed order equals the lexicographic (peak, id) order.  Fails with
 * RM_ERR_OVERFLOW unless ids < 2^id_bits and max_peak < 2^(63 - id_bits)
 * (max_peak: an upper bound of every peak, e.g. the graph's total bytes). */
int rm_argmin_key(const int64_t* peak, const uint8_t* valid, int64_t B, int64_t id_base,
                  int32_t id_bits, int64_t max_peak, int64_t* out_key, void* stream);

/* K1 + selection in one pass (device pointers only, RM_DEVICE_PTRS): the
 * rm_eval_orders outputs plus out_key = rm_argmin_key's packed key over them
 * (max_peak = the graph's total bytes), reduced inside the K1 launch where the
 * default evaluator runs -- no separate selection kernel. */
int rm_eval_select_key(RmGraph* g, const void* orders, int64_t B, int64_t id_base, int32_t id_bits,
                       uint32_t flags, int64_t* peak, int32_t* argmax, uint8_t* valid,
                       int64_t* out_key, void* stream);

/* Batched live_bytes_by_timestep (graph.py:452-458) over sequential
 * schedules: live[b * n + k] = bytes alive at step k of row b (int64[B, n]),
 * valid[b] = the row is a permutation respecting every direct pred
 * (graph.py:375-398); rows with valid == 0 leave their live row unwritten.
 * max_k live[b, k] and its first index equal rm_eval_orders' peak / argmax.
 * Flags: RM_DEVICE_PTRS, RM_ORDERS_U16.  Graphs whose 12 n bytes exceed one
 * CTA's shared memory fail with RM_ERR_CAPACITY. */
int rm_eval_live(RmGraph* g, const void* orders, int64_t B, uint32_t flags, int64_t* live, uint8_t* valid,
                 void* stream);

/* Multi-GPU selection exchange (one process per GPU): each rank's
 * rm_eval_select_key key (device int64[1], (peak << id_bits) | global id,
 * INT64_MAX when the rank has no valid candidate) becomes the global first
 * strict minimum on every rank with ONE 8-byte ncclAllReduce(MIN), async on
 * stream (replaces the planner's sequential first-strict-min scan,
 * planner.py:209-216, across ranks).  NCCL is dlopen'ed (libnccl.so.2) on
 * first use; the communicator comes from rm_nccl_comm_init (rank 0 makes the
 * id with rm_nccl_unique_id and ships its RM_NCCL_ID_BYTES to the others) or
 * is any ncclComm_t the host already has. */
#define RM_NCCL_ID_BYTES 128
int rm_nccl_unique_id(uint8_t* id, int64_t id_bytes);
int rm_nccl_comm_init(int32_t nranks, const uint8_t* id, int32_t rank, void** comm);
int rm_nccl_comm_destroy(void* comm);
int rm_nccl_select_key(void* comm, int64_t* key_dev, void* stream);

/* Counter-RNG candidate generator: row c is the Kahn topological order that
 * breaks ties by the smallest (splitmix64(seed ^ splitmix64(id)) ^ op, op)
 * key with id = first_id + c (oracle: oracle/memplan_oracle.py kahn_candidate).
 * Always device output (orders_dev int32[B, n]); async on stream. */
int rm_gen_orders(RmGraph* g, uint64_t seed, int64_t first_id, int64_t B,
                  int32_t* orders_dev, void* stream);

/* ------------------------------------------- single schedule (drop-ins) */

typedef struct {
  int32_t status;        /* 0 ok, else RM_SCHED_* below (first failing check) */
  int32_t detail_a;      /* RM_SCHED_PRED: op v */
  int32_t detail_b;      /* RM_SCHED_PRED: predecessor p */
  int32_t n_steps;
  int64_t peak;
  int32_t argmax;
  int32_t _pad;
} RmScheduleResult;

enum {
  RM_SCHED_OK = 0,
  RM_SCHED_NOT_PERMUTATION = 1,   /* graph.py:377-378 */
  RM_SCHED_TIMESTEPS_LEN = 2,     /* graph.py:379-380 */
  RM_SCHED_OPS_PER_STEP = 3,      /* graph.py:381-382 (ConfigError) */
  RM_SCHED_DECREASING = 4,        /* graph.py:385-389 */
  RM_SCHED_STEP_OVERFULL = 5,     /* graph.py:390-394 */
  RM_SCHED_PRED = 6               /* graph.py:395-398 */
};

enum {
  RM_SCHED_VALIDATE = 1u << 8,    /* run validate_schedule first (peak_memory) */
  RM_SCHED_PEAK = 1u << 9         /* compute peak/argmax */
};

/* General schedule evaluation (any timesteps, ops_per_step): validation
 * (graph.py:375-398), tensor_lifetimes (440-449), live_bytes_by_timestep
 * (452-458), peak_memory (461-468).  birth/death (int32[T]) and live
 * (int64[n_steps]) are optional outputs (NULL to skip).  Timesteps must be
 * in [0, 2^31). */
int rm_eval_schedule(RmGraph* g, const int32_t* order, int64_t order_len,
                     const int32_t* timesteps, int64_t ts_len, int32_t ops_per_step,
                     uint32_t flags, RmScheduleResult* res, int32_t* birth, int32_t* death,
                     int64_t* live, void* stream);

/* ------------------------------------------------- K2: layout checks */

/* Items: tensor i has inclusive lifetime [start, end], size, offset and a
 * has_offset flag (layout.py:20-29, 305-329).  Finds every pair i < j of items
 * with offsets overlapping in time AND address; pairs are returned as
 * (i, j) item indices sorted lexicographically (layout_violations order).
 * item_flags[i] bit0 = no offset, bit1 = negative offset, bit2 = extent
 * exceeds capacity.  max_extent = max(off+size) over items with offsets (0 if
 * none), the replay_static actual peak (simulator.py:129-145).  If the
 * number of pairs exceeds max_pairs, n_pairs reports the full count and only
 * the first max_pairs (in sorted order) are written.  Host pointers only. */
int rm_layout_violations(int64_t N, const int32_t* start, const int32_t* end,
                         const int64_t* size, const int64_t* offset, const uint8_t* has_offset,
                         int64_t capacity, uint8_t* item_flags, int64_t* pairs /* [2*max] */,
                         int64_t max_pairs, int64_t* n_pairs, int64_t* max_extent, void* stream);

/* repair_conflicts (layout.py:409-470): items sorted by tensor id, every
 * one with an offset.  Each round finds the conflicting pairs (time AND
 * address overlap) on the device with the items resident, elects one mover
 * per pair (the non-activation side, else the smaller (size, lifetime,
 * -tensor)) and re-places the movers in (size, lifetime, tensor) order on the
 * host: the smallest free gap of the mover's lifetime that fits (lowest on
 * ties), else on top of everything it overlaps in time; capacity grows to
 * fit.  offset[] and *capacity are updated in place; *rounds = rounds that
 * moved something.  After N + 1 rounds a remaining conflict fails with
 * RM_ERR_GRAPH ("conflict repair did not converge", layout.py:468-469).
 * Host pointers; synchronous. */
int rm_repair_conflicts(int64_t N, const int64_t* tensor, const int32_t* start, const int32_t* end,
                        const int64_t* size, const uint8_t* is_act, int64_t* offset,
                        int64_t* capacity, int32_t* rounds, void* stream);

/* The placement step of one repair round alone (layout.py:445-467), host
 * code: movers[] (item indices, in placement order) re-placed one after the
 * other against items with has_offset set. */
int rm_repair_place(int64_t N, const int32_t* start, const int32_t* end, const int64_t* size,
                    const uint8_t* has_offset, int64_t* offset, int64_t* capacity,
                    int64_t n_movers, const int64_t* movers);

/* place_weight_updates (ordering.py:387-467), host C++.  Activation tensors
 * k: lifetime [act_start, act_end] = [asap(producer), max alap(consumers)]
 * (n-1 without consumers), act_size; mean_size = the graph's mean tensor
 * size.  The slot skeleton (Linearization.slots): slot_kind 0 = op slot_ref,
 * 1 = window slot_ref, windows' ops in win_ptr/win_ops CSR, tail_window -1
 * for None.  Branches b (already filtered to floating ones): first op,
 * gradient producers (grad_ptr CSR), grad_bytes, resolved alpha.  Outputs in
 * the reference's placement order k: out_branch[k] (input branch index),
 * delayed, target window, ready_t, size_ratio, projected_use;
 * activation_total (0 without branches).  A gradient producer outside every
 * slot fails with RM_ERR_GRAPH and *missing_op = that op (the reference's
 * KeyError). */
int rm_place_weight_updates(int32_t n_ops, const int32_t* asap, int64_t n_act, const int32_t* act_start,
                            const int32_t* act_end, const int64_t* act_size, double mean_size,
                            int32_t n_slots, const int32_t* slot_kind, const int32_t* slot_ref,
                            int32_t n_windows, const int64_t* win_ptr, const int32_t* win_ops,
                            int32_t tail_window, int32_t n_branches, const int32_t* br_first,
                            const int64_t* grad_ptr, const int32_t* grad_producer, const int64_t* grad_bytes,
                            const double* alpha, double r, int32_t force_immediate, int32_t* out_branch,
                            uint8_t* out_delayed, int32_t* out_target, int32_t* out_ready, double* out_ratio,
                            double* out_projected, int64_t* activation_total, int32_t* missing_op);

/* ---------------------------------------------- K3: batched LLFB packer */

enum {
  RM_LLFB_PLAIN = 0,          /* llfb_layout (layout.py:100-118) */
  RM_LLFB_CONSTRAINED = 1,    /* constrained_llfb_layout (layout.py:121-146) */
  RM_LLFB_COMPONENTS = 2,     /* exact_layout up to its search (layout.py:165-225),
                                 activations_at_bottom=True */
  RM_LLFB_COMPONENTS_FREE = 3 /* the same with activations_at_bottom=False */
};

/* P independent layout problems, one CTA each; problem p owns items
 * [item_ptr[p], item_ptr[p+1]).  Per item: tensor id, inclusive [start, end],
 * size, is_activation.  Outputs: offset[item] (int64) and capacity[p].
 * PLAIN / CONSTRAINED reproduce the reference packers bit-exactly (sort keys,
 * activation stacking and floors, _lowest_fit, capacity).
 * COMPONENTS / COMPONENTS_FREE reproduce exact_layout up to its search:
 * activations pre-placed (bottom mode), overlap-connected components of the
 * rest, each component's long-lived-first incumbent (offset[]) and lower
 * bound.  bound_met[p] = 1 iff every component's incumbent capacity is <= its
 * bound -- then the reference returns exactly this layout without search and
 * capacity[p] is exact_layout's capacity.  comp[item] = the component's
 * smallest tensor id (-1 for pre-placed activations), comp_cap[item] = that
 * component's incumbent capacity.  bound_met/comp/comp_cap may be NULL for
 * PLAIN / CONSTRAINED.  Host pointers; synchronous.  Problems of more than
 * RM_LLFB_MAX_ITEMS items fail with RM_ERR_CAPACITY. */
#define RM_LLFB_MAX_ITEMS 16383
int rm_llfb_batch(int32_t P, const int64_t* item_ptr, const int32_t* tensor,
                  const int32_t* start, const int32_t* end, const int64_t* size,
                  const uint8_t* is_act, int32_t mode, int64_t* offset, int64_t* capacity,
                  uint8_t* bound_met, int32_t* comp, int64_t* comp_cap, void* stream);

/* exact_layout's branch-and-bound (layout.py:226-290) for one problem K3's
 * COMPONENTS pass could not decide: items as for rm_llfb_batch, bottom = the
 * problem's activations_at_bottom, incumbent[item] = K3's COMPONENTS offsets.
 * Components whose incumbent exceeds their bound are searched node for node
 * like the reference (same branching order, same pruning, node_cap counted
 * over all components; node_cap < 0 = none; deadline = CLOCK_MONOTONIC seconds
 * checked every 4096 nodes, <= 0 = none).  Outputs: offset[item], capacity,
 * nodes (the reference's LayoutStats.nodes) and optimal (0 when a budget
 * stopped a search).  Host code (the search is sequential); item masks of
 * as many 64-bit words as a component needs (components of more than 16,384
 * items fail with RM_ERR_CAPACITY). */
int rm_layout_search(int32_t n, const int32_t* tensor, const int32_t* start, const int32_t* end,
                     const int64_t* size, const uint8_t* is_act, int32_t bottom,
                     const int64_t* incumbent, int64_t node_cap, double deadline, int64_t* offset,
                     int64_t* capacity, int64_t* nodes, int32_t* optimal);

/* exact_order's capped depth-first search (ordering.py:183-286) for one
 * window, node for node (memo on the scheduled mask, the reference's branch
 * pruning and reconstruction walk), for the windows rm_exact_windows hands
 * back (status 3: more order ideals than the node cap).  node_cap < 0 = none;
 * deadline = CLOCK_MONOTONIC seconds checked every 1024 nodes (<= 0 = none).
 * status: 0 searched (order[n_ops] global ids, peak, nodes), 1 ConfigError
 * (bad_tensor: live-in tensor without a window consumer), 2 precedence cycle,
 * 4 budget -- the reference then returns its greedy incumbent.  Host code;
 * scheduled-op masks of as many 64-bit words as the window needs (windows
 * of more than 16,384 ops fail with RM_ERR_CAPACITY). */
int rm_exact_order_search(RmGraph* g, int32_t n_ops, const int32_t* ops, int64_t n_lin,
                          const int32_t* lin, int64_t n_lout, const int32_t* lout, int64_t node_cap,
                          double deadline, int32_t* order, int64_t* peak, int64_t* nodes,
                          int32_t* status, int32_t* bad_tensor);

/* ------------------------------------------- K4: batched window greedy */

/* W greedy_order problems (ordering.py:78-180) over one graph.  Window w
 * owns ops win_ops[win_ptr[w] .. win_ptr[w+1]) (sorted ascending) and the
 * live_in / live_out tensor sets lin_idx[lin_ptr[w]..], lout_idx[lout_ptr[w]..].
 * Outputs: order[win_ptr[w]..] (op ids), peak[w].  status[w] = 0 ok, 1 a
 * live-in tensor with no local consumer that is not live-out (ConfigError,
 * ordering.py:107-110), 2 precedence cycle.  Host pointers. */
int rm_greedy_windows(RmGraph* g, int32_t W, const int64_t* win_ptr, const int32_t* win_ops,
                      const int64_t* lin_ptr, const int32_t* lin_idx,
                      const int64_t* lout_ptr, const int32_t* lout_idx,
                      int32_t* order, int64_t* peak, int32_t* status, int32_t* bad_tensor,
                      void* stream);

/* K5: batched exact window ordering (replaces ordering.py:183-286 exact_order
 * for every window whose search provably stays under its node cap), one
 * launch for all windows of a graph.  Same window CSR as rm_greedy_windows;
 * node_cap[w] < 0 means no cap.  Per window: status 0 = exact answer in
 * order[win_ptr[w]..] (global op ids) and peak[w]; 1 = the reference's
 * ConfigError (bad_tensor[w] = the live-in tensor without a local consumer);
 * 2 = no order exists; 3 = the window has more order ideals than
 * node_cap + 1 (or more than 22 ops): the reference's DFS may stop at its cap
 * and return the greedy incumbent, so the caller runs that search.
 * nodes[w] = order ideals - 1 (an upper bound on the DFS's expansions). */
int rm_exact_windows(RmGraph* g, int32_t W, const int64_t* win_ptr, const int32_t* win_ops,
                     const int64_t* lin_ptr, const int32_t* lin_idx,
                     const int64_t* lout_ptr, const int32_t* lout_idx, const int64_t* node_cap,
                     int32_t* order, int64_t* peak, int64_t* nodes, int32_t* status,
                     int32_t* bad_tensor, void* stream);

/* ------------------------------------------------------------- misc */

const char* rm_last_error(void);
int rm_device_count(int* count);
/* Kernel launches made by this process through libroam so far. */
int64_t rm_launch_count(void);
/* Device time (ms) of the last rm_eval_orders K1 launch on this thread when
 * timing was requested through rm_set_timing(1); -1 if unavailable. */
int rm_set_timing(int enable);
/* Force the K1 evaluator variant on this thread: 0 auto (v5, else v4, else
 * generic), 1 the generic evaluator, 4 v4 (sentinel permutation check, SIMD
 * edge checks), 5 v5 (v4's checks, one dynamic class byte per position), 6 v5
 * with rows staged by cp.async.bulk; unsupported choices (and 2, 3: the
 * retired v2/v3) fall back.  For tests and A/B measurement. */
int rm_set_k1_variant(int variant);
/* Leave `sms` SMs idle in every K1 launch of this process (default 0), so a
 * collective issued on another stream (the multi-GPU selection exchange) runs
 * concurrently with the next batch's evaluation instead of after it. */
int rm_set_sm_reserve(int sms);
/* Candidate generator form on this thread: 0 auto (one thread per candidate
 * when the graph qualifies, the rows it cannot finish rewritten by the warp
 * form), 1 the warp form only (one warp per candidate), 40 / 64 the thread
 * form with that heap capacity.  Same rows either way; for tests and A/B
 * measurement. */
int rm_set_gen_form(int form);
/* K3 placement form on this thread: 0 auto (DAG rounds for problems of
 * 1,024 items or more, where they qualify), 1 the placed-list path only,
 * 2 DAG rounds wherever they qualify.  Same offsets either way; for tests
 * and A/B measurement. */
int rm_set_pack_form(int form);
double rm_last_kernel_ms(void);

#ifdef __cplusplus
}
#endif
#endif /* ROAM_H_ */
