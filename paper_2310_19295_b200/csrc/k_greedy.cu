// K4: batched window greedy (least-memory-increase list scheduling), one CTA
// per window -- the greedy solver the planner runs on every window larger
// than node_limit (planner.py:127-131) and as exact_order's incumbent.
//
// Reference (pkg/src/memplan/ordering.py):
//   _Local          78-123  window-local bookkeeping: ops sorted, tracked
//                           tensors = produced inside U live_in with their
//                           local consumer-ENTRY counts (duplicates count),
//                           held = live_out U produced-and-unconsumed,
//                           start_live = sum(live_in), local precedence
//   greedy_order   126-180  each step scores every ready op by
//                           out_bytes - sum(size of distinct tracked, non-held
//                           inputs whose count is 1), strict < over ascending
//                           local index; then live += out, peak = max, each
//                           distinct tracked input's count -= 1 and frees at 0
//                           unless held.  (Parity hazard h1: an input listed
//                           twice by one op is never freed by this solver.)
//
// Host (C++, this file): builds every window's local problem from the graph
// handle's CSR in O(window + its consumer entries).  Device: one warp per
// window.  Each op's score (out - bytes its inputs would free) is kept in
// shared memory and updated incrementally -- a tracked tensor's count only
// falls when an op runs, and when it reaches 1 the one op still holding an
// entry now frees it -- and the ready ops sit in a compact list, so a step
// compares only the ready ops' scores (a warp (score, index) argmin), then
// applies the pick (counts, score updates, successor pred counts, newly ready
// ops appended): no block barrier per step.  Two identities keep the step's
// dependent chain short:
//   * the bytes the pick frees are out - score: its score counts exactly the
//     distinct tracked inputs whose count is 1, the ones that reach 0 now --
//     no warp reduction of freed bytes;
//   * each tracked tensor carries, beside its count, the XOR of (local index
//     + 1) over its unrun consumer ENTRIES (an op removes its index once per
//     odd multiplicity).  When the count reaches 1 with an unrun entry left,
//     that entry is the only one, so the XOR names the op that now frees the
//     tensor (0: none left) -- no walk of the tensor's consumer list.
// Mutable state lives in shared memory when it fits, else in a per-window
// global scratch.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "roam_internal.h"

namespace roam {

struct K4Args {
  int W;
  const int64_t* op_base;   // [W] window op base in the flat op arrays
  const int32_t* nops;      // [W] ops per window (each window owns nops+1 slots)
  const int64_t* ten_base;  // [W+1] window tensor ranges
  const int32_t* gop;       // [NO] global op id per local op
  const int64_t* out;       // [NO] out_bytes
  const int32_t* npred0;    // [NO] distinct local preds
  const int64_t* in_ptr;    // [NO+1] into in_idx
  const uint32_t* in_idx;   // window-local tensor index | odd-multiplicity bit << 31
  const int64_t* in_sz;     // size of each in_idx entry's tensor (loaded in parallel with it)
  const uint2* in_pk;       // 32-bit score form: {in_idx entry, size >> shift} in one 8-byte load
  const int64_t* succ_ptr;  // [NO+1] into succ_idx (window-local op index)
  const int32_t* succ_idx;
  const uint32_t* cw0;      // [NT_] tracked tensors: consumer-entry count | XOR(local op + 1) << 16
  const int64_t* tsize;     // [NT_]
  const int64_t* start_live;  // [W]
  int32_t* order;           // [NO] global op ids in schedule order
  int64_t* peak;            // [W]
  int32_t* status;          // [W]
  unsigned char* gscratch;
  const int64_t* gscratch_off;  // [W] (-1: shared memory)
  int shift;                // the 32-bit score form keeps scores in units of 2^shift bytes
};

// Working set of one window (all 16-byte aligned): delta int64[n] (or int32
// in units of 2^shift bytes when every op's scores fit: half the bytes, so a
// GPT2-XL window leaves the L1 twice the room), npred
// int16[n], in / succ CSR starts u32[n + 1] each, ready u16[n], tensor words
// u32[nt] (count | XOR << 16).  Compact so that an 8.6k-op window (GPT2-XL's)
// still fits one CTA's shared memory with its CSR starts staged.
struct K4Layout {
  size_t o_delta, o_npred, o_inp, o_sup, o_ready, o_cw, bytes;
  __host__ __device__ K4Layout(int64_t n, int64_t nt, int dbytes) {
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    o_delta = 0;
    o_npred = al(o_delta + size_t(dbytes) * size_t(n));
    o_inp = al(o_npred + 2 * size_t(n));
    o_sup = al(o_inp + 4 * (size_t(n) + 1));
    o_ready = al(o_sup + 4 * (size_t(n) + 1));
    o_cw = al(o_ready + 2 * size_t(n));
    bytes = al(o_cw + 4 * size_t(nt));
  }
};
__host__ __device__ inline size_t k4_bytes(int64_t n_ops, int64_t n_ten, int dbytes) {
  return K4Layout(n_ops, n_ten, dbytes).bytes;
}

// One warp per window.  The ready ops (all predecessors scheduled) sit in a
// compact list -- a training window's ready set is tens of ops, so a step
// scores only those instead of sweeping the whole window -- and everything
// runs inside the warp: no block barrier anywhere on the step's critical path.
// The pick is a REDUX argmin of the packed key (score << 16 | local index:
// |score| < 2^47, local indices < 2^16), and the ops' CSR starts are staged in
// the working set, so a step's first dependent loads are shared-memory ones;
// the pick's input, size and successor entries are then loaded together.
template <bool SH, typename DT>
__global__ void __launch_bounds__(32) k4_greedy(const K4Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int w = blockIdx.x, lane = threadIdx.x;
  // SH: the working set is this CTA's shared memory (a pointer the compiler
  // knows is shared: LDS / STS, not generic loads); else global scratch.  A
  // launch of each form skips the other form's windows.
  if (SH != (a.gscratch_off[w] < 0)) return;
  const int64_t ob = a.op_base[w], tb = a.ten_base[w];
  const int n = a.nops[w];
  const int nt = (int)(a.ten_base[w + 1] - tb);
  const K4Layout L(n, nt, (int)sizeof(DT));
  constexpr bool D32 = sizeof(DT) == 4;
  const int sh = D32 ? a.shift : 0;
  unsigned char* ws = SH ? smem : a.gscratch + a.gscratch_off[w];
  DT* delta = reinterpret_cast<DT*>(ws + L.o_delta);  // out - bytes freed if run now (>> sh)
  short* npred = reinterpret_cast<short*>(ws + L.o_npred);
  uint32_t* inp = reinterpret_cast<uint32_t*>(ws + L.o_inp);
  uint32_t* sup = reinterpret_cast<uint32_t*>(ws + L.o_sup);
  unsigned short* ready = reinterpret_cast<unsigned short*>(ws + L.o_ready);
  uint32_t* cw = reinterpret_cast<uint32_t*>(ws + L.o_cw);
  const int64_t* out = a.out + ob;
  const int64_t* in_ptr = a.in_ptr + ob;
  const int64_t* succ_ptr = a.succ_ptr + ob;
  const int64_t* tsize = a.tsize + tb;
  const uint32_t* cw0 = a.cw0 + tb;
  const unsigned lt = (1u << lane) - 1u;
  int R = 0;
  for (int i0 = 0; i0 <= n; i0 += 32) {
    const int i = i0 + lane;
    if (i <= n) {
      inp[i] = (uint32_t)in_ptr[i];
      sup[i] = (uint32_t)succ_ptr[i];
    }
  }
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    bool rd = false;
    if (i < n) {
      const int np = a.npred0[ob + i];
      npred[i] = (short)np;
      // the score is kept up to date instead of recomputed every step: an
      // input frees when its count is 1, and counts only fall when an op runs
      long long freed = 0;
      for (int64_t k = in_ptr[i]; k < in_ptr[i + 1]; ++k) {
        uint32_t t;
        if constexpr (D32) t = __ldg(a.in_pk + k).x & 0x7fffffffu;
        else t = __ldg(a.in_idx + k) & 0x7fffffffu;
        if ((cw0[t] & 0xffffu) == 1u) freed += tsize[t];
      }
      delta[i] = (DT)((out[i] - freed) >> sh);
      rd = np == 0;
    }
    const unsigned m = __ballot_sync(0xffffffffu, rd);
    if (rd) ready[R + __popc(m & lt)] = (unsigned short)i;
    R += __popc(m);
  }
  for (int t = lane; t < nt; t += 32) cw[t] = cw0[t];
  long long live = a.start_live[w], peak = live;
  __syncwarp();

  // the schedule is written as local indices during the steps (no dependent
  // global load on a step's path) and mapped to global op ids at the end
  int32_t* ord = a.order + ob;
  auto map_order = [&](int steps) {
    __syncwarp();
    for (int i = lane; i < steps; i += 32) ord[i] = a.gop[ob + ord[i]];
  };
  for (int step = 0; step < n; ++step) {
    if (R == 0) {  // no ready op: the window's precedence has a cycle
      map_order(step);
      if (lane == 0) a.status[w] = 2;
      return;
    }
    // ---- score the ready ops: min (delta, local index) -- the reference's
    // strict < over ascending local index -- as one packed key, two REDUX
    long long bk = LLONG_MAX;
    int bs = -1;
    if (lane < R) {  // the common case: at most 32 ready ops
      const int i = ready[lane];
      bk = ((long long)delta[i] << 16) | (long long)i;
      bs = lane;
    }
    for (int j = lane + 32; j < R; j += 32) {
      const int i = ready[j];
      const long long key = ((long long)delta[i] << 16) | (long long)i;
      if (key < bk) {
        bk = key;
        bs = j;
      }
    }
    const int last = ready[R - 1];
    const int khi = (int)(bk >> 32);
    const unsigned klo = (unsigned)bk;
    const int mhi = __reduce_min_sync(0xffffffffu, khi);
    const unsigned mlo = __reduce_min_sync(0xffffffffu, khi == mhi ? klo : 0xffffffffu);
    const unsigned win = __ballot_sync(0xffffffffu, khi == mhi && klo == mlo);
    bs = __shfl_sync(0xffffffffu, bs, __ffs(win) - 1);
    const int bi = (int)(mlo & 0xffffu);
    // the pick's score: out minus exactly the bytes it frees now
    const long long dsel = ((long long)(((unsigned long long)(unsigned)mhi << 32) | mlo) >> 16) << sh;
    // ---- the pick's CSR ranges, then its first 32 input / size / successor
    // entries in one batch of independent loads
    const uint32_t i0 = inp[bi], i1 = inp[bi + 1];
    const uint32_t s0 = sup[bi], s1 = sup[bi + 1];
    const long long ob_bi = out[bi];
    const bool hin = i0 + lane < i1, hsu = s0 + lane < s1;
    // an input entry and its tensor's size (units of 2^sh in the 32-bit form)
    auto ld_in = [&](uint32_t k, uint32_t& e, long long& tsz) {
      if constexpr (D32) {
        const uint2 v = __ldg(a.in_pk + k);
        e = v.x;
        tsz = v.y;
      } else {
        e = __ldg(a.in_idx + k);
        tsz = __ldg(a.in_sz + k);
      }
    };
    uint32_t e = 0u;
    long long tsz = 0;
    if (hin) ld_in(i0 + lane, e, tsz);
    int sv = hsu ? __ldg(a.succ_idx + s0 + lane) : 0;
    // the hole the pick leaves is filled by the list's last entry (unordered
    // list); appends below start at the old last slot, so skip a self-move
    if (lane == 0 && bs != R - 1) ready[bs] = (unsigned short)last;
    --R;
    // ---- inputs: count -= 1, XOR out the pick (odd multiplicity); a count
    // reaching 1 with an unrun entry left moves the free to that op
    const unsigned xb = (unsigned)(bi + 1) << 16;
    for (uint32_t k = i0 + lane;;) {
      if (k < i1) {
        const uint32_t t = e & 0x7fffffffu;
        const uint32_t wv = cw[t];
        const uint32_t c = (wv - 1u) & 0xffffu;  // distinct inputs: no races
        const uint32_t x = (wv ^ ((e >> 31) ? xb : 0u)) & 0xffff0000u;
        cw[t] = x | c;
        if (c == 1u && x != 0u)
        {
          if constexpr (D32)
            atomicAdd(reinterpret_cast<int*>(delta) + ((x >> 16) - 1u), -(int)tsz);
          else
            atomicAdd(reinterpret_cast<unsigned long long*>(delta) + ((x >> 16) - 1u), (unsigned long long)(-tsz));
        }
      }
      k += 32;
      if (k - lane >= i1) break;
      if (k < i1) ld_in(k, e, tsz);
    }
    // ---- successors: predecessor counts, newly ready ops appended
    for (uint32_t k = s0; k < s1; k += 32) {
      bool rd = false;
      if (k + lane < s1) {
        if (k != s0) sv = __ldg(a.succ_idx + k + lane);
        rd = --npred[sv] == 0;  // distinct successors
      }
      const unsigned m = __ballot_sync(0xffffffffu, rd);
      if (rd) ready[R + __popc(m & lt)] = (unsigned short)sv;
      R += __popc(m);
    }
    live += ob_bi;
    peak = max(peak, live);
    live += dsel - ob_bi;
    if (lane == 0) ord[step] = bi;
    __syncwarp();
  }
  map_order(n);
  if (lane == 0) {
    a.peak[w] = peak;
    a.status[w] = 0;
  }
}

template <typename DT>
static int launch_k4_t(const K4Args& a, size_t smem, bool any_global, cudaStream_t s) {
  RM_CUDA(smem_optin(k4_greedy<true, DT>));
  k4_greedy<true, DT><<<a.W, 32, smem, s>>>(a);
  RM_LAUNCH_CHECK("k4_greedy launch");
  if (any_global) k4_greedy<false, DT><<<a.W, 32, 0, s>>>(a);
  RM_LAUNCH_CHECK("k4_greedy launch");
  return RM_OK;
}

}  // namespace roam

using namespace roam;

extern "C" int rm_greedy_windows(RmGraph* g, int32_t W, const int64_t* win_ptr,
                                 const int32_t* win_ops, const int64_t* lin_ptr,
                                 const int32_t* lin_idx, const int64_t* lout_ptr,
                                 const int32_t* lout_idx, int32_t* order, int64_t* peak,
                                 int32_t* status, int32_t* bad_tensor, void* stream) {
  if (!g) return fail(RM_ERR_INVALID_ARG, "graph handle is NULL");
  if (W < 0 || (W > 0 && (!win_ptr || !lin_ptr || !lout_ptr || !peak || !status || !bad_tensor)))
    return fail(RM_ERR_INVALID_ARG, "bad rm_greedy_windows arguments");
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

  // ---- host: build every window's local problem (_Local, ordering.py:84-123)
  std::vector<int32_t> loc(n, -1), tloc(T, -1);
  std::vector<uint8_t> is_lin(T, 0), is_lout(T, 0);
  std::vector<int64_t> op_base(W + 1, 0), ten_base(W + 1, 0), start_live(W, 0);
  std::vector<int32_t> gop, npred0, succ_idx, count0;
  std::vector<uint32_t> in_idx, cw0;
  std::vector<uint8_t> par;  // per local op: odd number of entries in the tensor at hand
  std::vector<int64_t> in_sz;
  std::vector<int64_t> out_b, in_ptr(1, 0), succ_ptr(1, 0), tsize;
  std::vector<int32_t> ops, rel, tmp;
  std::vector<std::vector<int32_t>> succ;
  std::vector<uint8_t> held;
  for (int w = 0; w < W; ++w) {
    status[w] = 0;
    bad_tensor[w] = -1;
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
    // relevant = produced inside U live_in, ascending
    rel.clear();
    for (int v : ops)
      for (int k = g->out_ptr[v]; k < g->out_ptr[v + 1]; ++k) rel.push_back(g->out_idx[k]);
    for (int64_t k = lin_ptr[w]; k < lin_ptr[w + 1]; ++k) rel.push_back(lin_idx[k]);
    std::sort(rel.begin(), rel.end());
    rel.erase(std::unique(rel.begin(), rel.end()), rel.end());
    held.assign(rel.size(), 0);
    int64_t sl = 0;
    const int64_t tb = (int64_t)tsize.size();
    int nt = 0;
    for (size_t r = 0; r < rel.size(); ++r) {
      const int t = rel[r];
      int local = 0;
      for (int k = g->cons_ptr[t]; k < g->cons_ptr[t + 1]; ++k) local += loc[g->cons_idx[k]] >= 0;
      const bool produced = loc[g->producer[t]] >= 0;
      if (is_lout[t] || (produced && local == 0)) {
        held[r] = 1;
      } else if (is_lin[t] && local == 0) {
        if (status[w] == 0) {
          status[w] = 1;  // ConfigError (ordering.py:107-110); smallest id first
          bad_tensor[w] = t;
        }
      }
      if (is_lin[t]) sl += g->size[t];
      if (!held[r]) {  // held tensors never free: the device never needs them
        tloc[t] = nt;
        tsize.push_back(g->size[t]);
        count0.push_back(local);
        // XOR of (local op + 1) over the tensor's local consumer entries
        uint32_t x = 0;
        for (int k = g->cons_ptr[t]; k < g->cons_ptr[t + 1]; ++k) {
          const int j = loc[g->cons_idx[k]];
          if (j < 0) continue;
          x ^= uint32_t(j + 1);
        }
        cw0.push_back(uint32_t(std::min(local, 65535)) | (x << 16));
        ++nt;
      }
    }
    start_live[w] = sl;
    // per op: out_bytes, distinct tracked non-held inputs, local preds
    succ.assign(nw, {});
    for (int i = 0; i < nw; ++i) {
      const int v = ops[i];
      int64_t ob = 0;
      for (int k = g->out_ptr[v]; k < g->out_ptr[v + 1]; ++k) ob += g->size[g->out_idx[k]];
      gop.push_back(v);
      out_b.push_back(ob);
      tmp.clear();
      for (int k = g->in_ptr[v]; k < g->in_ptr[v + 1]; ++k)
        if (tloc[g->in_idx[k]] >= 0) tmp.push_back(tloc[g->in_idx[k]]);
      std::sort(tmp.begin(), tmp.end());
      tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
      for (const int32_t t : tmp) {
        in_idx.push_back(uint32_t(t));  // the parity bit is set below
        in_sz.push_back(tsize[size_t(tb + t)]);
      }
      in_ptr.push_back((int64_t)in_idx.size());
      tmp.clear();
      for (int k = g->in_ptr[v]; k < g->in_ptr[v + 1]; ++k) {
        const int pr = g->producer[g->in_idx[k]];
        if (loc[pr] >= 0 && pr != v) tmp.push_back(loc[pr]);
      }
      std::sort(tmp.begin(), tmp.end());
      tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
      npred0.push_back((int32_t)tmp.size());
      for (int p : tmp) succ[p].push_back(i);
    }
    for (int i = 0; i < nw; ++i) {
      succ_idx.insert(succ_idx.end(), succ[i].begin(), succ[i].end());
      succ_ptr.push_back((int64_t)succ_idx.size());
    }
    op_base[w + 1] = (int64_t)gop.size();
    ten_base[w + 1] = tb + nt;
    // parity bits: an op whose entries in a tracked tensor's consumer list
    // are odd in number flags its input entry for that tensor
    par.assign(nw, 0);
    for (const int t : rel) {
      const int tl = tloc[t];
      if (tl < 0) continue;
      for (int k = g->cons_ptr[t]; k < g->cons_ptr[t + 1]; ++k)
        if (loc[g->cons_idx[k]] >= 0) par[loc[g->cons_idx[k]]] ^= 1;
      for (int k = g->cons_ptr[t]; k < g->cons_ptr[t + 1]; ++k) {
        const int j = loc[g->cons_idx[k]];
        if (j < 0 || !par[j]) continue;
        par[j] = 0;
        const int64_t q = op_base[w] + j;
        for (int64_t e = in_ptr[q]; e < in_ptr[q + 1]; ++e)
          if (in_idx[e] == uint32_t(tl)) in_idx[e] |= 0x80000000u;
      }
    }  // (every par[j] is back to 0: even ones never left it, odd ones were cleared)
    // reset the per-window marks
    for (int v : ops) loc[v] = -1;
    for (int t : rel) tloc[t] = -1;
    for (int64_t k = lin_ptr[w]; k < lin_ptr[w + 1]; ++k) is_lin[lin_idx[k]] = 0;
    for (int64_t k = lout_ptr[w]; k < lout_ptr[w + 1]; ++k) is_lout[lout_idx[k]] = 0;
  }
  // device layout: window w owns nops+1 op slots from opb_dev[w] (the extra
  // slot is the tail entry of its in/succ pointer arrays)
  const int64_t NO = (int64_t)gop.size();
  std::vector<int64_t> in_ptr_w(NO + W), succ_ptr_w(NO + W);
  std::vector<int64_t> opb_dev(W + 1);
  {
    int64_t q = 0;
    for (int w = 0; w < W; ++w) {
      opb_dev[w] = q;
      for (int64_t i = op_base[w]; i <= op_base[w + 1]; ++i, ++q) {
        in_ptr_w[q] = in_ptr[i];
        succ_ptr_w[q] = succ_ptr[i];
      }
    }
    opb_dev[W] = q;
  }

  // ---- device
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  size_t limit = size_t(max_smem) - 1024;
  // test hook: a lower shared-memory budget sends windows to the global-scratch form
  if (const char* e = getenv("RM_K4_SMEM_LIMIT")) limit = std::min(limit, (size_t)strtoull(e, nullptr, 10));
  // 32-bit scores in units of 2^shift (shift = the common power of two of
  // every size the kernel adds) when every op's out bytes and summed tracked
  // input bytes -- the bounds of its score -- stay below 2^30 units
  int shift = 62;
  auto tz = [&](int64_t v) {
    if (v > 0) shift = std::min(shift, __builtin_ctzll((unsigned long long)v));
  };
  for (const int64_t v : out_b) tz(v);
  for (const int64_t v : tsize) tz(v);
  for (const int64_t v : start_live) tz(v);
  if (shift == 62) shift = 0;
  bool d32 = true;
  for (size_t i = 0; i + 1 < in_ptr.size() && d32; ++i) {
    int64_t sin = 0;
    for (int64_t k = in_ptr[i]; k < in_ptr[i + 1]; ++k) sin += in_sz[size_t(k)];
    if ((out_b[i] >> shift) >= (int64_t(1) << 30) || (sin >> shift) >= (int64_t(1) << 30)) d32 = false;
  }
  const int dbytes = d32 ? 4 : 8;
  std::vector<int64_t> goff(W, -1);
  size_t gbytes = 0, smem = 16;
  for (int w = 0; w < W; ++w) {
    const size_t b = k4_bytes(op_base[w + 1] - op_base[w], ten_base[w + 1] - ten_base[w], dbytes);
    if (b <= limit) {
      smem = std::max(smem, b);
    } else {
      goff[w] = (int64_t)gbytes;
      gbytes += b;
    }
  }
  // op arrays are indexed op_base[w] + i on the device; the pointer arrays
  // are indexed opb_dev[w] + i (one extra tail entry per window)
  std::vector<int32_t> gop_w(opb_dev[W], 0), npred_w(opb_dev[W], 0);
  std::vector<int64_t> out_w(opb_dev[W], 0);
  for (int w = 0; w < W; ++w)
    for (int64_t i = 0; i < op_base[w + 1] - op_base[w]; ++i) {
      gop_w[opb_dev[w] + i] = gop[op_base[w] + i];
      npred_w[opb_dev[w] + i] = npred0[op_base[w] + i];
      out_w[opb_dev[w] + i] = out_b[op_base[w] + i];
    }
  Scratch sc(s);
  int64_t *d_ob, *d_tb, *d_out, *d_inp, *d_sup, *d_tsz, *d_sl, *d_peak, *d_goff;
  int32_t *d_gop, *d_np, *d_sui, *d_ord, *d_st;
  uint32_t *d_ini, *d_cw0;
  unsigned char* d_g = nullptr;
  auto up = [&](auto** d, const auto& v) -> cudaError_t {
    cudaError_t e = sc.alloc(d, v.size());
    if (e == cudaSuccess && !v.empty())
      e = cudaMemcpyAsync(*d, v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice, s);
    return e;
  };
  std::vector<int32_t> nops(W);
  for (int w = 0; w < W; ++w) nops[w] = (int32_t)(op_base[w + 1] - op_base[w]);
  // the device's compact working set (K4Layout) and packed argmin key
  for (int w = 0; w < W; ++w)
    if (nops[w] >= 65535) return fail(RM_ERR_CAPACITY, "greedy window above 65,534 ops");
  for (const int32_t c : count0)
    if (c > 65535) return fail(RM_ERR_CAPACITY, "greedy window: a tensor with more than 65,535 local uses");
  for (const int32_t d : npred0)
    if (d > 32767) return fail(RM_ERR_CAPACITY, "greedy window: an op with more than 32,767 local preds");
  if (in_idx.size() >= (size_t(1) << 32) || succ_idx.size() >= (size_t(1) << 32))
    return fail(RM_ERR_CAPACITY, "greedy windows: CSR above 2^32 entries");
  if (g->info.total_bytes >= (int64_t(1) << 46)) return fail(RM_ERR_CAPACITY, "greedy windows: scores above 2^46 bytes");
  int32_t* d_nops;
  RM_CUDA(up(&d_ob, opb_dev));
  RM_CUDA(up(&d_nops, nops));
  RM_CUDA(up(&d_tb, ten_base));
  RM_CUDA(up(&d_gop, gop_w));
  RM_CUDA(up(&d_out, out_w));
  RM_CUDA(up(&d_np, npred_w));
  RM_CUDA(up(&d_inp, in_ptr_w));
  RM_CUDA(up(&d_ini, in_idx));
  RM_CUDA(up(&d_sup, succ_ptr_w));
  RM_CUDA(up(&d_sui, succ_idx));
  RM_CUDA(up(&d_cw0, cw0));
  RM_CUDA(up(&d_tsz, tsize));
  RM_CUDA(up(&d_sl, start_live));
  RM_CUDA(up(&d_goff, goff));
  RM_CUDA(sc.alloc(&d_ord, size_t(std::max<int64_t>(opb_dev[W], 1))));
  RM_CUDA(sc.alloc(&d_peak, size_t(W)));
  RM_CUDA(sc.alloc(&d_st, size_t(W)));
  // a window the kernel abandons (cycle) leaves its peak and the rest of its
  // order unwritten: defined bytes for the read-back (compute-sanitizer initcheck)
  RM_CUDA(cudaMemsetAsync(d_peak, 0, size_t(W) * 8, s));
  RM_CUDA(cudaMemsetAsync(d_st, 0, size_t(W) * 4, s));
  RM_CUDA(cudaMemsetAsync(d_ord, 0xff, size_t(std::max<int64_t>(opb_dev[W], 1)) * 4, s));
  if (gbytes) RM_CUDA(sc.alloc(&d_g, gbytes));
  int64_t* d_insz;
  RM_CUDA(up(&d_insz, in_sz));
  uint32_t* d_inpk = nullptr;
  if (d32) {
    std::vector<uint32_t> pk(2 * in_idx.size());
    for (size_t k = 0; k < in_idx.size(); ++k) {
      pk[2 * k] = in_idx[k];
      pk[2 * k + 1] = uint32_t(in_sz[k] >> shift);
    }
    RM_CUDA(up(&d_inpk, pk));
  }
  K4Args a{W, d_ob, d_nops, d_tb, d_gop, d_out, d_np, d_inp, d_ini, d_insz, reinterpret_cast<const uint2*>(d_inpk),
           d_sup, d_sui, d_cw0, d_tsz, d_sl, d_ord, d_peak, d_st, d_g, d_goff, d32 ? shift : 0};
  int rc = d32 ? launch_k4_t<int>(a, smem, gbytes > 0, s) : launch_k4_t<long long>(a, smem, gbytes > 0, s);
  if (rc) return rc;
  std::vector<int32_t> ord_w(opb_dev[W]), st_dev(W);
  if (opb_dev[W])
    RM_CUDA(cudaMemcpyAsync(ord_w.data(), d_ord, size_t(opb_dev[W]) * 4, cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaMemcpyAsync(peak, d_peak, size_t(W) * 8, cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaMemcpyAsync(st_dev.data(), d_st, size_t(W) * 4, cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaStreamSynchronize(s));
  for (int w = 0; w < W; ++w) {
    if (status[w] == 0 && st_dev[w] != 0) status[w] = st_dev[w];
    const int64_t nw = win_ptr[w + 1] - win_ptr[w];
    for (int64_t i = 0; i < nw; ++i) order[win_ptr[w] + i] = ord_w[opb_dev[w] + i];
  }
  return RM_OK;
}
