// K5: batched exact window ordering -- the planner's exact_order (every window
// with at most node_limit ops, planner.py:127-131) as a dynamic program over
// the window's order ideals, one CTA per window.
//
// Reference (pkg/src/memplan/ordering.py):
//   _Local        78-123  window-local bookkeeping (see k_greedy.cu)
//   exact_order  183-286  memoised DFS over scheduled-set masks with incumbent
//                         pruning; node cap (deterministic) and deadline
//                         (wall clock) return the greedy incumbent; then a walk
//                         from the empty mask picks the smallest local index
//                         whose branch value reaches the optimum.
// Restated exactly (SURVEY §8 hazard h10, oracle/memplan_oracle.py
// exact_order_dp): with live(m) = start_live + sum_{i in m} out[i] - sum of
// freeable tensors whose local consumers are all in m,
//   V[full] = 0,  V[m] = min over ready i of max(live(m) + out[i], V[m | i]);
// the walk takes, from m = 0, the smallest ready i with
// max(live(m) + out[i], V[m | i]) <= V[m]; peak = max(V[0], start_live).
// The DFS memo holds exactly these values (pruning never changes a memo entry)
// and expands each ideal at most once, so whenever (#ideals - 1) <= node_cap
// its cap cannot trigger and this IS its answer.  Windows with more ideals
// than the cap (or more than K5_MAX_N ops) come back with status 3: their
// answer depends on how far the pruned DFS gets, and the caller runs that
// search for them (rm_exact_order_search, order_search.cpp).
//
// Device: per window, one sweep counts the ideals (a mask is an ideal iff
// every member's local preds are in it); then V is filled level by level
// (popcount n-1 .. 0, a barrier between levels), in shared memory up to 2^13
// masks and in a per-CTA global slot beyond; thread 0 walks the order.
#include <algorithm>
#include <climits>

#include "k_common.cuh"

namespace roam {

static constexpr int K5_MAX_N = 22;     // 2^22 masks * 8 B = 32 MB per resident window
static constexpr int K5_SMEM_N = 13;    // V in shared memory up to 2^13 masks (64 KB)

struct K5Args {
  int W;
  const int32_t* nops;        // [W]
  const int64_t* op_base;     // [W] into gop / pred / out
  const int32_t* gop;         // global op id per local op
  const uint32_t* pred;       // local pred masks
  const int64_t* out;         // out bytes
  const int64_t* ten_base;    // [W+1] freeable tensors
  const uint32_t* cmask;      // their local consumer masks
  const int64_t* tsize;
  const int64_t* start_live;  // [W]
  const int64_t* node_cap;    // [W] (-1: none)
  int32_t* order;             // [sum nops] global ids, schedule order
  int64_t* peak;              // [W]
  int64_t* nodes;             // [W] ideals - 1
  int32_t* status;            // [W] 0 ok, 2 no order, 3 caller must search
  long long* vslot;           // [gridDim.x][2^gmax] global V slots
  int gmax;                   // log2 of a global slot's masks
  int max_ten;                // most freeable tensors of any window
};

__device__ __forceinline__ bool k5_ideal(uint32_t m, const uint32_t* pred) {
  for (uint32_t r = m; r; r &= r - 1)
    if (pred[__ffs(r) - 1] & ~m) return false;
  return true;
}

template <int NT>
__global__ void __launch_bounds__(NT) k5_exact(const K5Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long s_cnt;
  __shared__ int s_go;
  long long* vsm = reinterpret_cast<long long*>(smem);                      // [2^K5_SMEM_N]
  int64_t* s_out = reinterpret_cast<int64_t*>(smem + (8u << K5_SMEM_N));  // [K5_MAX_N]
  int64_t* s_tsz = s_out + K5_MAX_N;                                       // [max_ten]
  uint32_t* s_pred = reinterpret_cast<uint32_t*>(s_tsz + a.max_ten);       // [K5_MAX_N]
  uint32_t* s_cm = s_pred + K5_MAX_N;                                      // [max_ten]
  const int tid = threadIdx.x;
  long long* vglob = a.vslot + (size_t(blockIdx.x) << a.gmax);

  for (int w = blockIdx.x; w < a.W; w += gridDim.x) {
    const int n = a.nops[w];
    if (n <= 0 || n > K5_MAX_N) continue;  // handled by the host
    const int64_t ob = a.op_base[w], tb = a.ten_base[w];
    const int nt = (int)(a.ten_base[w + 1] - tb);
    for (int i = tid; i < n; i += NT) {
      s_pred[i] = a.pred[ob + i];
      s_out[i] = a.out[ob + i];
    }
    for (int t = tid; t < nt; t += NT) {
      s_cm[t] = a.cmask[tb + t];
      s_tsz[t] = a.tsize[tb + t];
    }
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    const uint32_t full = n == 32 ? 0xffffffffu : ((1u << n) - 1u);
    const uint32_t nm = full + 1u;  // 2^n masks (n <= 22)
    long long* V = n <= K5_SMEM_N ? vsm : vglob;

    // ---- count the ideals; a cap the DFS could hit sends the window back
    unsigned long long cnt = 0;
    for (uint32_t m = tid; m < nm; m += NT) cnt += k5_ideal(m, s_pred);
    for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    if ((tid & 31) == 0) atomicAdd(&s_cnt, cnt);
    __syncthreads();
    if (tid == 0) {
      const long long cap = a.node_cap[w];
      const unsigned long long ideals = s_cnt;
      a.nodes[w] = (int64_t)ideals - 1;
      s_go = (cap < 0 || (long long)(ideals - 1) <= cap) ? 1 : 0;
      if (!s_go) a.status[w] = 3;
    }
    __syncthreads();
    if (!s_go) continue;

    // ---- V level by level: masks of popcount lev depend on lev + 1 only
    const int64_t start = a.start_live[w];
    for (int lev = n - 1; lev >= 0; --lev) {
      for (uint32_t m = tid; m < nm; m += NT) {
        if (__popc(m) != lev || !k5_ideal(m, s_pred)) continue;
        long long live = start;
        for (uint32_t r = m; r; r &= r - 1) live += s_out[__ffs(r) - 1];
        for (int t = 0; t < nt; ++t)
          if ((s_cm[t] & m) == s_cm[t]) live -= s_tsz[t];
        long long best = LLONG_MAX;
        for (uint32_t r = ~m & full; r; r &= r - 1) {
          const int i = __ffs(r) - 1;
          if (s_pred[i] & ~m) continue;
          const uint32_t nx = m | (1u << i);
          const long long sub = nx == full ? 0 : V[nx];
          const long long step = live + s_out[i];
          const long long val = step >= sub ? step : sub;
          if (val < best) best = val;
        }
        V[m] = best;
      }
      __syncthreads();
    }

    // ---- walk: smallest ready local index whose branch reaches V[m]
    if (tid == 0) {
      int32_t* ord = a.order + ob;
      uint32_t m = 0;
      long long live = start;
      int st = V[0] == LLONG_MAX ? 2 : 0;
      for (int step = 0; step < n && st == 0; ++step) {
        const long long target = V[m];
        int chosen = -1;
        for (int i = 0; i < n; ++i) {
          if ((m >> i & 1u) || (s_pred[i] & ~m)) continue;
          const uint32_t nx = m | (1u << i);
          const long long sub = nx == full ? 0 : V[nx];
          const long long stp = live + s_out[i];
          if ((stp >= sub ? stp : sub) <= target) {
            chosen = i;
            break;
          }
        }
        if (chosen < 0) {
          st = 2;
          break;
        }
        const uint32_t nx = m | (1u << chosen);
        live += s_out[chosen];
        for (int t = 0; t < nt; ++t)  // tensors whose last local consumer this is
          if ((s_cm[t] & nx) == s_cm[t] && (s_cm[t] & m) != s_cm[t]) live -= s_tsz[t];
        m = nx;
        ord[step] = a.gop[ob + chosen];
      }
      a.peak[w] = V[0] > start ? V[0] : start;
      a.status[w] = st;
    }
    __syncthreads();
  }
}

}  // namespace roam

using namespace roam;

extern "C" int rm_exact_windows(RmGraph* g, int32_t W, const int64_t* win_ptr,
                                const int32_t* win_ops, const int64_t* lin_ptr,
                                const int32_t* lin_idx, const int64_t* lout_ptr,
                                const int32_t* lout_idx, const int64_t* node_cap, int32_t* order,
                                int64_t* peak, int64_t* nodes, int32_t* status,
                                int32_t* bad_tensor, void* stream) {
  if (!g) return fail(RM_ERR_INVALID_ARG, "graph handle is NULL");
  if (W < 0 || (W > 0 && (!win_ptr || !lin_ptr || !lout_ptr || !node_cap || !peak || !nodes ||
                          !status || !bad_tensor)))
    return fail(RM_ERR_INVALID_ARG, "bad rm_exact_windows arguments");
  if (W == 0) return RM_OK;
  if (g->device < 0) return fail(RM_ERR_NO_DEVICE, "no CUDA device: libroam has no CPU path");
  const int n = g->n, T = g->T;
  if (win_ptr[0] != 0 || lin_ptr[0] != 0 || lout_ptr[0] != 0)
    return fail(RM_ERR_INVALID_ARG, "CSR pointers must start at 0");
  for (int w = 0; w < W; ++w)
    if (win_ptr[w + 1] < win_ptr[w] || lin_ptr[w + 1] < lin_ptr[w] || lout_ptr[w + 1] < lout_ptr[w])
      return fail(RM_ERR_INVALID_ARG, "CSR pointers must be non-decreasing");
  if ((win_ptr[W] && (!win_ops || !order)) || (lin_ptr[W] && !lin_idx) || (lout_ptr[W] && !lout_idx))
    return fail(RM_ERR_INVALID_ARG, "NULL window array");

  // ---- host: each window's local problem (_Local, ordering.py:84-123) as
  // pred masks, out bytes, start_live and freeable tensors (consumer mask,
  // size): a tracked, non-held tensor frees when its local consumer-ENTRY
  // count reaches 0 with one decrement per distinct consuming op, so a tensor
  // some op lists twice never frees (hazard h1) and is left out.
  std::vector<int32_t> loc(n, -1), lcount(T, 0);
  std::vector<uint8_t> is_lin(T, 0), is_lout(T, 0);
  std::vector<int32_t> nops(W, 0), gop;
  std::vector<int64_t> op_base(W, 0), ten_base(W + 1, 0), start_live(W, 0), out_b, tsize;
  std::vector<uint32_t> pred, cmask;
  std::vector<int32_t> ops, rel;
  int gmax = 0, max_ten = 1;
  for (int w = 0; w < W; ++w) {
    status[w] = 0;
    bad_tensor[w] = -1;
    nodes[w] = 0;
    ops.assign(win_ops + win_ptr[w], win_ops + win_ptr[w + 1]);
    for (int v : ops)
      if (v < 0 || v >= n) return fail(RM_ERR_INVALID_ARG, "window op out of range");
    std::sort(ops.begin(), ops.end());
    if (std::adjacent_find(ops.begin(), ops.end()) != ops.end())
      return fail(RM_ERR_INVALID_ARG, "window lists an op twice");
    const int nw = (int)ops.size();
    for (int i = 0; i < nw; ++i) loc[ops[i]] = i;
    for (int64_t k = lin_ptr[w]; k < lin_ptr[w + 1]; ++k) {
      const int t = lin_idx[k];
      if (t < 0 || t >= T) return fail(RM_ERR_INVALID_ARG, "live-in tensor out of range");
      is_lin[t] = 1;
    }
    for (int64_t k = lout_ptr[w]; k < lout_ptr[w + 1]; ++k) {
      const int t = lout_idx[k];
      if (t < 0 || t >= T) return fail(RM_ERR_INVALID_ARG, "live-out tensor out of range");
      is_lout[t] = 1;
    }
    rel.clear();
    for (int v : ops)
      for (int k = g->out_ptr[v]; k < g->out_ptr[v + 1]; ++k) rel.push_back(g->out_idx[k]);
    for (int64_t k = lin_ptr[w]; k < lin_ptr[w + 1]; ++k) rel.push_back(lin_idx[k]);
    std::sort(rel.begin(), rel.end());
    rel.erase(std::unique(rel.begin(), rel.end()), rel.end());
    int64_t sl = 0;
    const int64_t tb = (int64_t)tsize.size();
    const bool small = nw <= K5_MAX_N;
    for (int t : rel) {
      int local = 0;
      uint32_t cm = 0;
      int distinct = 0;
      for (int k = g->cons_ptr[t]; k < g->cons_ptr[t + 1]; ++k) {
        const int c = loc[g->cons_idx[k]];
        if (c < 0) continue;
        ++local;
        if (small && !(cm >> c & 1u)) {
          cm |= 1u << c;
          ++distinct;
        }
      }
      const bool produced = loc[g->producer[t]] >= 0;
      bool held = false;
      if (is_lout[t] || (produced && local == 0)) {
        held = true;
      } else if (is_lin[t] && local == 0) {
        if (status[w] == 0) {
          status[w] = 1;  // ConfigError (ordering.py:107-110); smallest id first
          bad_tensor[w] = t;
        }
      }
      if (is_lin[t]) sl += g->size[t];
      if (small && !held && local > 0 && distinct == local) {
        cmask.push_back(cm);
        tsize.push_back(g->size[t]);
      }
    }
    start_live[w] = sl;
    op_base[w] = (int64_t)gop.size();
    nops[w] = nw;
    if (small) {
      for (int i = 0; i < nw; ++i) {
        const int v = ops[i];
        int64_t ob = 0;
        for (int k = g->out_ptr[v]; k < g->out_ptr[v + 1]; ++k) ob += g->size[g->out_idx[k]];
        uint32_t pm = 0;
        for (int k = g->in_ptr[v]; k < g->in_ptr[v + 1]; ++k) {
          const int pr = g->producer[g->in_idx[k]];
          if (loc[pr] >= 0 && pr != v) pm |= 1u << loc[pr];
        }
        gop.push_back(v);
        out_b.push_back(ob);
        pred.push_back(pm);
      }
      if (nw > K5_SMEM_N) gmax = std::max(gmax, nw);
    } else {
      status[w] = status[w] ? status[w] : 3;  // too many ops for the GPU DP
    }
    ten_base[w + 1] = (int64_t)tsize.size();
    max_ten = std::max<int>(max_ten, (int)(ten_base[w + 1] - tb));
    for (int v : ops) loc[v] = -1;
    for (int64_t k = lin_ptr[w]; k < lin_ptr[w + 1]; ++k) is_lin[lin_idx[k]] = 0;
    for (int64_t k = lout_ptr[w]; k < lout_ptr[w + 1]; ++k) is_lout[lout_idx[k]] = 0;
  }
  // windows that go to the device: no ConfigError, 1..K5_MAX_N ops
  std::vector<int32_t> nops_dev(nops);
  int64_t n_dev = 0;
  for (int w = 0; w < W; ++w) {
    if (status[w] != 0 || nops[w] == 0) nops_dev[w] = 0;
    if (status[w] == 0 && nops[w] == 0) peak[w] = start_live[w];  // empty window
    n_dev += nops_dev[w] > 0;
  }
  if (n_dev == 0) return RM_OK;

  // ---- device
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = sm_count(dev);
  // persistent CTAs; windows past 2^13 masks keep V in a per-CTA global slot,
  // so their number is bounded by a 1 GiB scratch budget
  int64_t grid64 = std::min<int64_t>(W, int64_t(sms) * 2);
  if (gmax) grid64 = std::min<int64_t>(grid64, std::max<int64_t>(1, (int64_t(1) << 30) >> (gmax + 3)));
  const int grid = (int)grid64;
  Scratch sc(s);
  int32_t *d_nops, *d_gop, *d_ord, *d_st;
  int64_t *d_ob, *d_out, *d_tb, *d_tsz, *d_sl, *d_cap, *d_peak, *d_nodes;
  uint32_t *d_pred, *d_cm;
  long long* d_v = nullptr;
  auto up = [&](auto** d, const auto& v) -> cudaError_t {
    cudaError_t e = sc.alloc(d, std::max<size_t>(v.size(), 1));
    if (e == cudaSuccess && !v.empty())
      e = cudaMemcpyAsync(*d, v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice, s);
    return e;
  };
  std::vector<int64_t> caps(node_cap, node_cap + W), st0(W, 0);
  std::vector<int32_t> st_init(status, status + W);
  RM_CUDA(up(&d_nops, nops_dev));
  RM_CUDA(up(&d_ob, op_base));
  RM_CUDA(up(&d_gop, gop));
  RM_CUDA(up(&d_pred, pred));
  RM_CUDA(up(&d_out, out_b));
  RM_CUDA(up(&d_tb, ten_base));
  RM_CUDA(up(&d_cm, cmask));
  RM_CUDA(up(&d_tsz, tsize));
  RM_CUDA(up(&d_sl, start_live));
  RM_CUDA(up(&d_cap, caps));
  RM_CUDA(up(&d_st, st_init));
  RM_CUDA(up(&d_peak, std::vector<int64_t>(W, 0)));
  RM_CUDA(up(&d_nodes, std::vector<int64_t>(W, 0)));
  RM_CUDA(sc.alloc(&d_ord, std::max<size_t>(gop.size(), 1)));
  if (gmax) RM_CUDA(sc.alloc(&d_v, size_t(grid) << gmax));
  else RM_CUDA(sc.alloc(&d_v, 1));
  K5Args a{W, d_nops, d_ob, d_gop, d_pred, d_out, d_tb, d_cm, d_tsz, d_sl, d_cap,
           d_ord, d_peak, d_nodes, d_st, d_v, gmax, max_ten};
  // + 16 B: the tensor loops' remainder may read s_cm as a pair (LDS.64) one
  // word past its last entry (compute-sanitizer memcheck, k_exact.cu walk)
  const size_t smem = (8u << K5_SMEM_N) + 8 * size_t(K5_MAX_N + max_ten) + 4 * size_t(K5_MAX_N + max_ten) + 16;
  constexpr int NT = 512;
  RM_CUDA(smem_optin(k5_exact<NT>));
  k5_exact<NT><<<grid, NT, smem, s>>>(a);
  RM_LAUNCH_CHECK("k5_exact launch");
  std::vector<int32_t> ord(gop.size()), st(W);
  std::vector<int64_t> pk(W), nd(W);
  if (!gop.empty())
    RM_CUDA(cudaMemcpyAsync(ord.data(), d_ord, gop.size() * 4, cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaMemcpyAsync(st.data(), d_st, size_t(W) * 4, cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaMemcpyAsync(pk.data(), d_peak, size_t(W) * 8, cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaMemcpyAsync(nd.data(), d_nodes, size_t(W) * 8, cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaStreamSynchronize(s));
  for (int w = 0; w < W; ++w) {
    if (nops_dev[w] == 0) continue;
    status[w] = st[w];
    nodes[w] = nd[w];
    if (st[w] == 0) {
      peak[w] = pk[w];
      for (int i = 0; i < nops[w]; ++i) order[win_ptr[w] + i] = ord[op_base[w] + i];
    }
  }
  return RM_OK;
}
