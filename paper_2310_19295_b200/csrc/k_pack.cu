// K3: batched long-lived-first (LLFB) offset packer, one CTA per layout
// problem (the independent leaf subtasks the planner's tree decomposition
// produces, planner.py:239-252).
//
// Reference (pkg/src/memplan/layout.py):
//   _lowest_fit             71-78   lowest offset >= floor missing every placed,
//                                   time-overlapping span (spans sorted by lo)
//   _activation_floors      81-97   activations stacked from 0 in (-len, id)
//                                   order; floor = block top if the item
//                                   overlaps any activation, else 0
//   llfb_layout            100-118  sort (-len, -size, id), lowest fit
//   _constrained_incumbent 121-132  + constrained_llfb_layout 135-146
//   exact_layout           153-225  union-find components, per-component
//                                   bound and incumbent (the search itself,
//                                   226-290, runs only when incumbent > bound)
//
// Per problem the CTA: loads the items into shared memory (global scratch
// when they do not fit), bitonic-sorts the placement order, stacks the
// activation block with a block scan, derives the floors, then places items
// one at a time.  _lowest_fit is evaluated in parallel over the placed list
// kept sorted by offset:  with spans sorted by lo and M_k = max(floor,
// max_{j<k} hi_j) over the time-overlapping ones, the sweep breaks at the
// first k with lo_k >= M_k + size and returns M_k (M_last if it never
// breaks); ties in lo never change the result.  So one pass computes chunk
// maxima, a block exclusive max-scan gives each chunk its entry M, a second
// pass finds each chunk's first break, and a block min picks the first one.
// The new item is then inserted at upper_bound(lo) with a register shift.
#include <climits>

#include "roam_internal.h"

namespace roam {

struct K3Args {
  int P;
  const int64_t* item_ptr;
  const int32_t* tensor;
  const int32_t* start;
  const int32_t* end;
  const int64_t* size;
  const uint8_t* is_act;
  int mode;
  int64_t* offset;
  int64_t* capacity;
  uint8_t* bound_met;
  int32_t* comp;
  int64_t* comp_cap;
  unsigned char* gscratch;     // per-problem working set when it exceeds smem
  const int64_t* gscratch_off;  // [P] byte offsets (-1: use shared memory)
  unsigned char* dscratch;      // per-problem obstacle lists of the DAG placement
  const int64_t* dscratch_off;  // [P] byte offsets (-1: the placed-list path)
};

__host__ __device__ inline int k3_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Working-set layout of one problem with N items (all offsets 16-aligned).
struct K3Layout {
  size_t o_sz, o_off, o_flo, o_aux, o_s, o_e, o_tid, o_ord, o_sidx, o_act, bytes;
  __host__ __device__ K3Layout(int N) {
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t n = size_t(N), p2 = size_t(k3_pow2(N));
    o_sz = 0;
    o_off = al(o_sz + 8 * n);
    o_flo = al(o_off + 8 * n);
    o_aux = al(o_flo + 8 * n);
    o_s = al(o_aux + 8 * n);
    o_e = al(o_s + 4 * n);
    o_tid = al(o_e + 4 * n);
    o_ord = al(o_tid + 4 * n);
    o_sidx = al(o_ord + 4 * p2);
    o_act = al(o_sidx + 4 * (n + 1));
    bytes = al(o_act + n);
  }
};

template <int NT>
struct K3Block {
  // block-wide helpers over NT threads (NT multiple of 32, <= 1024)
  static constexpr int NW = NT / 32;
  long long* wv;  // [NW]
  int* wi;        // [NW]

  __device__ long long reduce_max(long long v) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, d));
    __syncthreads();
    if (lane == 0) wv[w] = v;
    __syncthreads();
    long long r = wv[0];
    for (int k = 1; k < NW; ++k) r = max(r, wv[k]);
    return r;
  }
  __device__ long long reduce_sum(long long v) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    __syncthreads();
    if (lane == 0) wv[w] = v;
    __syncthreads();
    long long r = 0;
    for (int k = 0; k < NW; ++k) r += wv[k];
    return r;
  }
  // exclusive max-scan over thread order; *total = inclusive max of all
  __device__ long long excl_max(long long v, long long* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc = max(inc, t);
    }
    long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = LLONG_MIN;
    __syncthreads();
    if (lane == 31) wv[w] = inc;
    __syncthreads();
    long long before = LLONG_MIN, all = LLONG_MIN;
    for (int k = 0; k < NW; ++k) {
      if (k < w) before = max(before, wv[k]);
      all = max(all, wv[k]);
    }
    *total = all;
    return max(before, ex);
  }
  // exclusive sum-scan over thread order; *total = sum of all
  __device__ long long excl_sum(long long v, long long* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += t;
    }
    __syncthreads();
    if (lane == 31) wv[w] = inc;
    __syncthreads();
    long long before = 0, all = 0;
    for (int k = 0; k < NW; ++k) {
      if (k < w) before += wv[k];
      all += wv[k];
    }
    *total = all;
    return before + inc - v;
  }
  // One-barrier forms for the placement loop: each uses its own slots
  // (xw / mk), and between two uses of one form every thread passes the
  // other form's barrier, so no barrier is needed to protect the slots.  The
  // NW per-warp partials are combined with shuffles, not a loop.
  __device__ long long excl_max1(long long v, long long* total, long long* xw) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc = max(inc, t);
    }
    long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = LLONG_MIN;
    if (lane == 31) xw[w] = inc;
    __syncthreads();
    long long q = lane < NW ? xw[lane] : LLONG_MIN;  // inclusive scan over the warps
#pragma unroll
    for (int d = 1; d < NW; d <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, q, d);
      if (lane >= d) q = max(q, t);
    }
    const long long before = __shfl_sync(0xffffffffu, q, w > 0 ? w - 1 : 0);
    *total = __shfl_sync(0xffffffffu, q, NW - 1);
    return w > 0 ? max(before, ex) : ex;
  }
  __device__ int min_key1(int key, long long val, long long* out_val, int* mi, long long* mv) {
    // keys are distinct slot indices (or INT_MAX): one redux.min, and the
    // lane that holds the minimum publishes its value
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int wk = __reduce_min_sync(0xffffffffu, key);
    const unsigned hit = __ballot_sync(0xffffffffu, key == wk);
    if (lane == 0) mi[w] = wk;
    if (key == wk && lane == __ffs(hit) - 1) mv[w] = val;
    __syncthreads();
    key = lane < NW ? mi[lane] : INT_MAX;
    const int bk = __reduce_min_sync(0xffffffffu, key);
    const unsigned bw = __ballot_sync(0xffffffffu, key == bk);
    *out_val = mv[__ffs(bw) - 1];  // every lane: the first warp holding the minimum
    return bk;
  }
  // (min key, its value) over the block; key INT_MAX = none
  __device__ int min_key(int key, long long val, long long* out_val) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const int ok = __shfl_xor_sync(0xffffffffu, key, d);
      const long long ov = __shfl_xor_sync(0xffffffffu, val, d);
      if (ok < key) {
        key = ok;
        val = ov;
      }
    }
    __syncthreads();
    if (lane == 0) {
      wi[w] = key;
      wv[w] = val;
    }
    __syncthreads();
    int k = wi[0];
    long long v = wv[0];
    for (int q = 1; q < NW; ++q)
      if (wi[q] < k) {
        k = wi[q];
        v = wv[q];
      }
    *out_val = v;
    return k;
  }
};

// ---- DAG placement.  _lowest_fit(item, placed, floor) reads only the placed
// items that overlap the item in time, so item u's offset depends only on the
// items before it in the placement order that overlap it (its obstacles), and
// any order respecting that relation gives the reference's offsets.  On the
// planner's leaves the relation is shallow (GPT2-XL's 9,035-item leaf: 8,020
// items to place, at most 11 obstacles each, 18 levels), so the CTA places
// every item whose obstacles are all placed in one round: 18 rounds instead of
// 8,020 dependent placements.
//
// Per item the answer is the smallest candidate c in {floor} U {hi_o >= floor}
// with no obstacle o such that lo_o < c + size and hi_o > c: the sweep's
// candidate only ever takes the floor or an obstacle's hi, every value it
// passes over fails that test against the span that moved it, and the value it
// returns passes it (spans before the break end at or below it, spans after
// start at or above its end).
//
// Obstacle lists: one pass over the earlier items per item (all lanes of a
// warp read the same earlier item: broadcast loads), at most K3_DAG_K per item
// -- a problem with an item over that (or a cycle-free chain too deep to be
// worth rounds) keeps the placed-list path.
constexpr int K3_DAG_K = 48;
constexpr int K3_DAG_SHORT = 32;  // lifetime (end - start) of a short item

struct K3DagLayout {
  size_t o_se, o_lvl, o_cnt, o_lo, o_hi, o_key, o_idx, bytes;
  __host__ __device__ K3DagLayout(int N) {
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t n = size_t(N);
    o_se = 0;                          // int2 {start, end} in placement order
    o_lvl = al(o_se + 8 * n);          // round an item was placed in (-1: not yet)
    o_cnt = al(o_lvl + 4 * n);         // obstacle count
    o_lo = al(o_cnt + 4 * n);          // placed spans
    o_hi = al(o_lo + 8 * n);
    o_key = al(o_hi + 8 * n);          // short items sorted by start: start << 32 | position
    o_idx = al(o_key + 8 * size_t(k3_pow2(N)));  // [n][K3_DAG_K] obstacle positions
    bytes = al(o_idx + 4 * n * size_t(K3_DAG_K));
  }
};

// Places items A..N-1 of the placement order; false (nothing written) when the
// problem does not qualify.  *cap_rest = max(offset + size) over them.
template <int NT>
__device__ bool k3_dag_place(K3Block<NT>& blk, int N, int A, const int* ord, const int* st, const int* en,
                             const long long* sz, const long long* flo, long long* off, unsigned char* ds,
                             long long* cap_rest) {
  const K3DagLayout D(N);
  int2* se = reinterpret_cast<int2*>(ds + D.o_se);
  int* lvl = reinterpret_cast<int*>(ds + D.o_lvl);
  int* cnt = reinterpret_cast<int*>(ds + D.o_cnt);
  long long* LO = reinterpret_cast<long long*>(ds + D.o_lo);
  long long* HI = reinterpret_cast<long long*>(ds + D.o_hi);
  int* idx = reinterpret_cast<int*>(ds + D.o_idx);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int M = N - A;  // local position u = placement index - A
  for (int u = tid; u < M; u += NT) {
    const int q = ord[A + u];
    se[u] = make_int2(st[q], en[q]);
    lvl[u] = -1;
  }
  __syncthreads();
  // Obstacle lists.  The placement order is by lifetime, longest first, so
  // the items longer than K3_DAG_SHORT steps are a prefix [0, NL) and every
  // obstacle of one of them is in it; an obstacle of a short item u is long,
  // or short with its start in [start_u - K3_DAG_SHORT, end_u] -- a window of
  // the short items sorted by start.  A warp takes 32 consecutive targets
  // (lanes) and walks its candidates with every lane reading the same one.
  int NL = 0;
  {
    int c = 0;
    for (int u = tid; u < M; u += NT) c += (se[u].y - se[u].x > K3_DAG_SHORT) ? 1 : 0;
    NL = (int)blk.reduce_sum(c);
  }
  const int NS = M - NL, P2 = k3_pow2(max(NS, 1));
  long long* key = reinterpret_cast<long long*>(ds + D.o_key);
  for (int j = tid; j < P2; j += NT)
    key[j] = j < NS ? ((long long)se[NL + j].x << 32) | (unsigned)(NL + j) : LLONG_MAX;
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < (P2 >> 1); t += NT) {
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int l = i | j;
        const long long x = key[i], y = key[l];
        if (((i & k) == 0) == (y < x)) {
          key[i] = y;
          key[l] = x;
        }
      }
      __syncthreads();
    }
  }
  int over = 0;
  auto add = [&](int& c, int* mine, int i) {
    if (c < K3_DAG_K) mine[c] = i;
    ++c;
  };
  // long targets: the earlier long items
  for (int b = w * 32; b < NL; b += NT) {
    const int u = b + lane;
    const bool have = u < NL;
    const int2 me = have ? se[u] : make_int2(0, 0);
    int* mine = idx + size_t(have ? u : 0) * K3_DAG_K;
    int c = 0;
    const int iend = min(b + 32, NL) - 1;
    for (int i = 0; i < iend; ++i) {
      const int2 o = se[i];
      if (have && i < u && o.x <= me.y && me.x <= o.y) add(c, mine, i);
    }
    if (have) cnt[u] = c;
    over |= c > K3_DAG_K;
  }
  // short targets in start order: every long item, then the start window
  for (int b = w * 32; b < NS; b += NT) {
    const int j = b + lane;
    const bool have = j < NS;
    const int u = have ? (int)(key[j] & 0xffffffffLL) : 0;
    const int2 me = have ? se[u] : make_int2(0, 0);
    int* mine = idx + size_t(u) * K3_DAG_K;
    int c = 0;
    for (int i = 0; i < NL; ++i) {
      const int2 o = se[i];
      if (have && o.x <= me.y && me.x <= o.y) add(c, mine, i);
    }
    const long long lo_s = (long long)__shfl_sync(0xffffffffu, me.x, 0) - K3_DAG_SHORT;  // lane 0: the block's first start
    int hi_e = have ? me.y : INT_MIN;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) hi_e = max(hi_e, __shfl_xor_sync(0xffffffffu, hi_e, d));
    // window [first key with start >= lo_s, first key with start > hi_e)
    int lo = 0, hi = NS;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((key[mid] >> 32) < lo_s) lo = mid + 1;
      else hi = mid;
    }
    int w0 = lo;
    hi = NS;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((key[mid] >> 32) <= hi_e) lo = mid + 1;
      else hi = mid;
    }
    for (int q = w0; q < lo; ++q) {
      const int i = (int)(key[q] & 0xffffffffLL);
      const int2 o = se[i];
      if (have && i < u && o.x <= me.y && me.x <= o.y) add(c, mine, i);
    }
    if (have) cnt[u] = c;
    over |= c > K3_DAG_K;
  }
  if (__syncthreads_or(over)) return false;
  // rounds: every item whose obstacles were all placed in earlier rounds
  long long cmax = LLONG_MIN;
  for (int r = 0;; ++r) {
    int left = 0;
    for (int u = tid; u < M; u += NT) {
      if (lvl[u] >= 0) continue;
      const int* ob = idx + size_t(u) * K3_DAG_K;
      const int k = cnt[u];
      bool ready = true;
      for (int q = 0; q < k && ready; ++q) {
        const int l = lvl[ob[q]];  // -1, or r for an item placed this round: not yet
        ready = l >= 0 && l < r;
      }
      if (!ready) {
        left = 1;
        continue;
      }
      const int qi = ord[A + u];
      const long long s = sz[qi], fl = flo[qi];
      long long best = LLONG_MAX;
      for (int c = -1; c < k; ++c) {
        const long long x = c < 0 ? fl : HI[ob[c]];
        if (x < fl || x >= best) continue;
        bool ok = true;
        for (int q = 0; q < k && ok; ++q) {
          const int o = ob[q];
          ok = !(LO[o] < x + s && HI[o] > x);
        }
        if (ok) best = x;
      }
      LO[u] = best;
      HI[u] = best + s;
      off[qi] = best;
      lvl[u] = r;
      cmax = max(cmax, best + s);
    }
    if (!__syncthreads_or(left)) break;
  }
  *cap_rest = blk.reduce_max(cmax);
  return true;
}

template <int NT, int MAXC, int MS = 0>
__global__ void __launch_bounds__(NT) k3_llfb(const K3Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ long long s_wv[NT / 32];
  __shared__ int s_wi[NT / 32];
  K3Block<NT> blk{s_wv, s_wi};
  const int p = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t base = a.item_ptr[p];
  const int N = (int)(a.item_ptr[p + 1] - base);
  const bool bottom = a.mode == RM_LLFB_CONSTRAINED || a.mode == RM_LLFB_COMPONENTS;
  const bool comps = a.mode == RM_LLFB_COMPONENTS || a.mode == RM_LLFB_COMPONENTS_FREE;
  if (N == 0) {
    if (tid == 0) {
      a.capacity[p] = 0;
      if (a.bound_met) a.bound_met[p] = 1;
    }
    return;
  }
  const K3Layout L(N);
  unsigned char* ws = a.gscratch_off[p] < 0 ? smem : a.gscratch + a.gscratch_off[p];
  long long* sz = reinterpret_cast<long long*>(ws + L.o_sz);
  long long* off = reinterpret_cast<long long*>(ws + L.o_off);
  long long* flo = reinterpret_cast<long long*>(ws + L.o_flo);
  int* st = reinterpret_cast<int*>(ws + L.o_s);
  int* en = reinterpret_cast<int*>(ws + L.o_e);
  int* tn = reinterpret_cast<int*>(ws + L.o_tid);
  int* ord = reinterpret_cast<int*>(ws + L.o_ord);
  int* sidx = reinterpret_cast<int*>(ws + L.o_sidx);
  unsigned char* act = ws + L.o_act;
  const int P2 = k3_pow2(N);

  for (int i = tid; i < N; i += NT) {
    sz[i] = a.size[base + i];
    st[i] = a.start[base + i];
    en[i] = a.end[base + i];
    tn[i] = a.tensor[base + i];
    act[i] = (bottom && a.is_act[base + i]) ? 1 : 0;  // group 0 = stacked activations
    off[i] = 0;
    flo[i] = 0;
  }
  for (int i = tid; i < P2; i += NT) ord[i] = i < N ? i : -1;
  __syncthreads();

  // ---- placement order: activations by (-len, id); the rest by (-len, -size, id)
  auto less = [&](int x, int y) -> bool {
    if (x < 0) return false;
    if (y < 0) return true;
    const int gx = act[x] ? 0 : 1, gy = act[y] ? 0 : 1;
    if (gx != gy) return gx < gy;
    const long long lx = (long long)en[x] - st[x], ly = (long long)en[y] - st[y];
    if (lx != ly) return lx > ly;
    if (gx == 1 && sz[x] != sz[y]) return sz[x] > sz[y];
    if (tn[x] != tn[y]) return tn[x] < tn[y];
    return x < y;
  };
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < (P2 >> 1); t += NT) {
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));  // lower index of the pair
        const int l = i | j;
        const bool up = (i & k) == 0;
        const int x = ord[i], y = ord[l];
        if (up ? less(y, x) : less(x, y)) {
          ord[i] = y;
          ord[l] = x;
        }
      }
      __syncthreads();
    }
  }

  // ---- activation block: stacked from 0 in sorted order (block scan)
  int A = 0;
  {
    long long cnt = 0;
    for (int i = tid; i < N; i += NT) cnt += act[i];
    A = (int)blk.reduce_sum(cnt);
  }
  long long block_top = 0;
  {
    const int C = (A + NT - 1) / NT;
    const int k0 = min(A, tid * C), k1 = min(A, k0 + C);
    long long run = 0;
    for (int k = k0; k < k1; ++k) run += sz[ord[k]];
    long long total;
    long long pre = blk.excl_sum(run, &total);
    for (int k = k0; k < k1; ++k) {
      off[ord[k]] = pre;
      pre += sz[ord[k]];
    }
    block_top = total;
  }
  // floors: block top if the item overlaps any activation (layout.py:95)
  if (A > 0) {
    for (int i = tid; i < N; i += NT) {
      if (act[i]) continue;
      bool hit = false;
      for (int k = 0; k < A && !hit; ++k) {
        const int q = ord[k];
        hit = st[q] <= en[i] && st[i] <= en[q];
      }
      flo[i] = hit ? block_top : 0;
    }
  }
  // placed list sorted by offset: activations first when they are obstacles
  int P = (a.mode == RM_LLFB_CONSTRAINED) ? A : 0;
  for (int k = tid; k < P; k += NT) sidx[k] = ord[k];
  __syncthreads();

  // ---- placement: by DAG rounds where the problem qualifies, else
  // sequential with a parallel _lowest_fit over the placed list
  long long cap_rest = LLONG_MIN;
  bool placed = false;
  if (a.dscratch_off[p] >= 0)
    placed = k3_dag_place<NT>(blk, N, A, ord, st, en, sz, flo, off, a.dscratch + a.dscratch_off[p], &cap_rest);
  if (placed) {
  } else if constexpr (NT * MAXC <= 8192) {
    // Placed list in registers: thread t owns list slots [t*TOT, (t+1)*TOT)
    // as {lo, hi, start, end}; empty slots never overlap and sort last.  An
    // insertion shifts the suffix with lo > res one slot right: within a
    // thread by register selects, across threads by one shuffle (lane 0
    // reads the previous warp's last slot, double-buffered by item parity).
    // NT = 512: start | end << 16 in one register (the host routes problems
    // with timesteps >= 65535 elsewhere), so the list fits 128 registers.
    // MS > 0 (leaves of 8k-16k items): each thread's last MS slots live in
    // shared memory, lane-interleaved ([m][tid]: conflict-free whatever slot
    // a warp touches), the working set in global scratch (the host routes
    // every problem of such a launch there).
    constexpr bool PK = NT > 256;
    constexpr int TOT = MAXC + MS;
    static_assert(MS == 0 || PK, "shared-memory slots use the packed start | end form");
    __shared__ long long s_plo[2][NT / 32], s_phi[2][NT / 32];
    __shared__ long long s_xw[NT / 32], s_mv[NT / 32];
    __shared__ int s_mi[NT / 32];
    __shared__ int s_pst[2][NT / 32], s_pen[2][NT / 32];
    long long* sl_lo = reinterpret_cast<long long*>(smem);            // [MS][NT]
    long long* sl_hi = sl_lo + size_t(MS) * NT;                       // [MS][NT]
    int* sl_se = reinterpret_cast<int*>(sl_hi + size_t(MS) * NT);     // [MS][NT]
    const int lane = tid & 31, w = tid >> 5;
    long long rlo[MAXC], rhi[MAXC];
    int rst[MAXC], ren[PK ? 1 : MAXC];
    // slot m of this thread: registers below MAXC, shared memory above (m is
    // a compile-time constant in every unrolled loop)
    auto g_lo = [&](int m) -> long long { return m < MAXC ? rlo[m < MAXC ? m : 0] : sl_lo[(m - MAXC) * NT + tid]; };
    auto g_hi = [&](int m) -> long long { return m < MAXC ? rhi[m < MAXC ? m : 0] : sl_hi[(m - MAXC) * NT + tid]; };
    auto g_st = [&](int m) -> int { return m < MAXC ? rst[m < MAXC ? m : 0] : sl_se[(m - MAXC) * NT + tid]; };
    auto g_en = [&](int m) -> int { return PK ? 0 : ren[PK ? 0 : m]; };
    auto p_slot = [&](int m, long long lo, long long hi, int se, int en) {
      if (m < MAXC) {
        rlo[m < MAXC ? m : 0] = lo;
        rhi[m < MAXC ? m : 0] = hi;
        rst[m < MAXC ? m : 0] = se;
        if (!PK) ren[PK ? 0 : m] = en;
      } else {
        sl_lo[(m - MAXC) * NT + tid] = lo;
        sl_hi[(m - MAXC) * NT + tid] = hi;
        sl_se[(m - MAXC) * NT + tid] = se;
      }
    };
    auto t_st = [&](int m) { return PK ? (g_st(m) & 0xffff) : g_st(m); };
    auto t_en = [&](int m) { return PK ? ((unsigned)g_st(m) >> 16) : (unsigned)g_en(m); };
#pragma unroll
    for (int m = 0; m < TOT; ++m) {
      const int j = tid * TOT + m;
      int a0 = INT_MAX, a1 = INT_MIN;
      long long lo = LLONG_MAX, hi = LLONG_MIN;
      if (j < P) {
        const int q = ord[j];
        lo = off[q];
        hi = off[q] + sz[q];
        a0 = st[q];
        a1 = en[q];
      }
      // PK: empty slots hold start 65535 > every end
      p_slot(m, lo, hi, PK ? (j < P ? (a0 | (a1 << 16)) : 0xffff) : a0, a1);
    }
    // the next item's record is fetched one placement ahead (the working set
    // of a large leaf lives in global scratch: its loads are the critical path)
    int i_nx = A < N ? ord[A] : 0;
    int si_nx = A < N ? st[i_nx] : 0, ei_nx = A < N ? en[i_nx] : 0;
    long long sz_nx = A < N ? sz[i_nx] : 0, fl_nx = A < N ? flo[i_nx] : 0;
    for (int k = A; k < N; ++k) {
      const int i = i_nx;
      const int si = si_nx, ei = ei_nx;
      const long long szi = sz_nx, fl = fl_nx;
      if (k + 1 < N) {
        i_nx = ord[k + 1];
        si_nx = st[i_nx];
        ei_nx = en[i_nx];
        sz_nx = sz[i_nx];
        fl_nx = flo[i_nx];
      }
      const int buf = k & 1;
      // a warp whose first slot lies past the list's end after this
      // insertion (index P_k) holds only empty slots: it skips the slot work
      // (warp-uniform) and only joins the block reductions -- the list fills
      // from the front, so on average half the warps sit this out
      const bool wlive = w * 32 * TOT <= P + (k - A);
      if (wlive && lane == 31) {
        s_plo[buf][w] = g_lo(TOT - 1);
        s_phi[buf][w] = g_hi(TOT - 1);
        s_pst[buf][w] = g_st(TOT - 1);
        if (!PK) s_pen[buf][w] = g_en(TOT - 1);
      }
      long long mx = LLONG_MIN;
      if (wlive) {
#pragma unroll
        for (int m = 0; m < TOT; ++m)
          if (t_st(m) <= ei && si <= t_en(m)) mx = max(mx, g_hi(m));
      }
      long long all_mx;
      long long M = max(fl, blk.excl_max1(mx, &all_mx, s_xw));
      int brk = INT_MAX;
      long long at = 0;
      if (wlive) {
#pragma unroll
        for (int m = 0; m < TOT; ++m) {
          if (t_st(m) <= ei && si <= t_en(m) && brk == INT_MAX) {
            if (M + szi <= g_lo(m)) {
              brk = tid * TOT + m;
              at = M;
            } else {
              M = max(M, g_hi(m));
            }
          }
        }
      }
      long long res;
      if (blk.min_key1(brk, at, &res, s_mi, s_mv) == INT_MAX) res = max(fl, all_mx);
      if (tid == 0) off[i] = res;
      cap_rest = max(cap_rest, res + szi);
      if (!wlive) continue;
      // the slot before this thread's first one
      long long plo = __shfl_up_sync(0xffffffffu, g_lo(TOT - 1), 1);
      long long phi = __shfl_up_sync(0xffffffffu, g_hi(TOT - 1), 1);
      int pst = __shfl_up_sync(0xffffffffu, g_st(TOT - 1), 1);
      int pen = PK ? 0 : __shfl_up_sync(0xffffffffu, g_en(TOT - 1), 1);
      if (lane == 0) {
        if (w == 0) {
          plo = LLONG_MIN;  // list start: the item goes first if slot 0 moves
        } else {
          plo = s_plo[buf][w - 1];
          phi = s_phi[buf][w - 1];
          pst = s_pst[buf][w - 1];
          if (!PK) pen = s_pen[buf][w - 1];
        }
      }
      const int ist = PK ? (si | (ei << 16)) : si;
#pragma unroll
      for (int m = 0; m < TOT; ++m) {
        // slots with lo <= res stay; the first other slot takes the item, the
        // rest take their predecessor
        const long long olo = g_lo(m), ohi = g_hi(m);
        const int ost = g_st(m), oen = g_en(m);
        if (olo > res) {
          const bool first = plo <= res;
          p_slot(m, first ? res : plo, first ? res + szi : phi, first ? ist : pst, first ? ei : pen);
        }
        plo = olo;
        phi = ohi;
        pst = ost;
        pen = oen;
      }
    }
    __syncthreads();
  } else {
  for (int k = A; k < N; ++k) {
    const int i = ord[k];
    const int si = st[i], ei = en[i];
    const long long szi = sz[i], fl = flo[i];
    const int C = (P + NT) / NT;  // chunk covers [0, P] so index P has an owner
    const int j0 = tid * C, j1 = min(P, j0 + C);
    long long mx = LLONG_MIN;
    for (int j = j0; j < j1; ++j) {
      const int q = sidx[j];
      if (st[q] <= ei && si <= en[q]) mx = max(mx, off[q] + sz[q]);
    }
    long long all_mx;
    long long M = max(fl, blk.excl_max(mx, &all_mx));
    int brk = INT_MAX;
    long long at = 0;
    for (int j = j0; j < j1; ++j) {
      const int q = sidx[j];
      if (st[q] <= ei && si <= en[q]) {
        const long long lo = off[q];
        if (M + szi <= lo) {
          brk = j;
          at = M;
          break;
        }
        M = max(M, lo + sz[q]);
      }
    }
    long long res;
    if (blk.min_key(brk, at, &res) == INT_MAX) res = max(fl, all_mx);
    // insert at upper_bound(lo = res): the elements with lo > res are a
    // suffix of the sorted list and each shifts right by one
    int jm = j1;
    for (int j = j0; j < j1; ++j)
      if (off[sidx[j]] > res) {
        jm = j;
        break;
      }
    const bool owner = jm < j1 && (jm == 0 || off[sidx[jm - 1]] <= res);
    int kv[MAXC];
#pragma unroll
    for (int m = 0; m < MAXC; ++m)
      if (jm + m < j1) kv[m] = sidx[jm + m];
    const bool tail_owner = (P >= j0 && P < j0 + C) && (P == 0 || off[sidx[P - 1]] <= res);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MAXC; ++m)
      if (jm + m < j1) sidx[jm + m + 1] = kv[m];
    if (owner) sidx[jm] = i;
    if (tail_owner) sidx[P] = i;
    if (tid == 0) off[i] = res;
    cap_rest = max(cap_rest, res + szi);
    ++P;
    __syncthreads();
  }
  }
  if (tid == 0) {
    // capacity starts at the activation block (layout.py:127, 199)
    long long cap = max(block_top, cap_rest == LLONG_MIN ? 0 : cap_rest);
    a.capacity[p] = cap;
  }
  for (int i = tid; i < N; i += NT) a.offset[base + i] = off[i];
  if (!comps) return;

  // ---- exact_layout components (layout.py:176-225), O(N^2) per problem.
  // Components of the interval overlap graph are the maximal runs in start
  // order: item i opens a run iff no j has start_j < start_i <= end_j; its
  // label is the largest run-opening start <= start_i.
  int* lab = sidx;  // placement is done: reuse
  __syncthreads();
  for (int i = tid; i < N; i += NT) {
    if (act[i]) continue;
    bool inner = false;
    for (int j = 0; j < N && !inner; ++j)
      inner = !act[j] && st[j] < st[i] && st[i] <= en[j];
    lab[i] = inner ? INT_MIN : st[i];
  }
  __syncthreads();
  for (int i = tid; i < N; i += NT) {
    if (act[i] || lab[i] != INT_MIN) continue;
    int best = INT_MIN;
    for (int j = 0; j < N; ++j)
      if (!act[j] && lab[j] != INT_MIN && st[j] <= st[i] && st[j] > best) best = st[j];
    ord[i] = best;  // stash (ord is free now); label of a non-opening item
  }
  __syncthreads();
  for (int i = tid; i < N; i += NT)
    if (!act[i] && lab[i] == INT_MIN) lab[i] = ord[i];
  __syncthreads();
  // probe value at each item's start: live bytes of its component, and
  // block top + the floored ones (layout.py:209-217)
  long long* probe = reinterpret_cast<long long*>(ws + L.o_aux);
  for (int j = tid; j < N; j += NT) {
    if (act[j]) continue;
    const int lj = lab[j], t = st[j];
    long long total = 0, above = 0;
    for (int q = 0; q < N; ++q) {
      if (act[q] || lab[q] != lj || !(st[q] <= t && t <= en[q])) continue;
      total += sz[q];
      if (flo[q]) above += sz[q];
    }
    probe[j] = max(total, above ? block_top + above : 0LL);
  }
  __syncthreads();
  // per item: root (min id), incumbent capacity and bound of its component
  bool met = true;
  for (int i = tid; i < N; i += NT) {
    if (act[i]) {
      a.comp[base + i] = -1;
      a.comp_cap[base + i] = 0;
      continue;
    }
    const int li = lab[i];
    int root = INT_MAX;
    long long ccap = 0, bound = 0;
    for (int j = 0; j < N; ++j) {
      if (act[j] || lab[j] != li) continue;
      root = min(root, tn[j]);
      ccap = max(ccap, off[j] + sz[j]);
      bound = max(bound, probe[j]);
    }
    a.comp[base + i] = root;
    a.comp_cap[base + i] = ccap;
    if (ccap > bound) met = false;
  }
  const int all_met = __syncthreads_and(met ? 1 : 0);
  if (tid == 0) a.bound_met[p] = all_met ? 1 : 0;
}

static int sm_max_smem(int dev) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

template <int NT, int MAXC, int MS = 0>
static int launch_k3_t(const K3Args& a, int grid, size_t smem, cudaStream_t s) {
  auto kern = k3_llfb<NT, MAXC, MS>;
  RM_CUDA(smem_optin(kern));
  kern<<<grid, NT, smem, s>>>(a);
  RM_LAUNCH_CHECK("k3_llfb launch");
  return RM_OK;
}

static thread_local int t_pack_form = 0;  // 0 auto, 1 placed list only, 2 DAG wherever it qualifies
constexpr int K3_DAG_MIN_ITEMS = 1024;     // auto: DAG rounds for problems from this size

}  // namespace roam

using namespace roam;

extern "C" int rm_set_pack_form(int form) {
  if (form < 0 || form > 2) return fail(RM_ERR_INVALID_ARG, "pack form must be 0 (auto), 1 (list) or 2 (DAG)");
  t_pack_form = form;
  return RM_OK;
}

extern "C" int rm_llfb_batch(int32_t P, const int64_t* item_ptr, const int32_t* tensor,
                             const int32_t* start, const int32_t* end, const int64_t* size,
                             const uint8_t* is_act, int32_t mode, int64_t* offset,
                             int64_t* capacity, uint8_t* bound_met, int32_t* comp,
                             int64_t* comp_cap, void* stream) {
  if (P < 0 || !item_ptr || !capacity || mode < 0 || mode > 3)
    return fail(RM_ERR_INVALID_ARG, "bad rm_llfb_batch arguments");
  if (P == 0) return RM_OK;
  if (item_ptr[0] != 0) return fail(RM_ERR_INVALID_ARG, "item_ptr[0] must be 0");
  int maxN = 0;
  for (int p = 0; p < P; ++p) {
    const int64_t n = item_ptr[p + 1] - item_ptr[p];
    if (n < 0) return fail(RM_ERR_INVALID_ARG, "item_ptr must be non-decreasing");
    if (n > RM_LLFB_MAX_ITEMS) return fail(RM_ERR_CAPACITY, "layout problem exceeds RM_LLFB_MAX_ITEMS");
    maxN = std::max<int>(maxN, (int)n);
  }
  const int64_t NI = item_ptr[P];
  if (NI > 0 && (!tensor || !start || !end || !size || !is_act || !offset))
    return fail(RM_ERR_INVALID_ARG, "NULL item array");
  const bool comps = mode >= RM_LLFB_COMPONENTS;
  if (comps && (!bound_met || !comp || !comp_cap))
    return fail(RM_ERR_INVALID_ARG, "component outputs are required for COMPONENTS modes");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(RM_ERR_NO_DEVICE, "no CUDA device: libroam has no CPU path");
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // shared memory holds any problem up to the opt-in limit; larger ones work
  // out of a global scratch region (L1/L2 cached)
  const size_t limit = (size_t)sm_max_smem(dev) - 1024;
  // NT = 512 / 1024 pack start | end << 16 per placed item
  bool times16 = true;
  for (int64_t k = 0; k < NI && times16; ++k)
    times16 = start[k] >= 0 && end[k] >= 0 && start[k] < 65535 && end[k] < 65535;
  // leaves of 8k-10k items: a 1024-thread list with 4 register and 6
  // shared-memory slots per thread; shared memory then holds the list and
  // every working set goes to global scratch
  constexpr int kHyNT = 1024, kHyMR = 4, kHyMS = 6;
  const bool hybrid = maxN >= 8192 && maxN < kHyNT * (kHyMR + kHyMS) && times16;
  std::vector<int64_t> goff(P, -1);
  size_t gbytes = 0, smem = hybrid ? size_t(kHyMS) * kHyNT * 20 : 0;
  for (int p = 0; p < P; ++p) {
    const int n = (int)(item_ptr[p + 1] - item_ptr[p]);
    if (n == 0) continue;
    const size_t b = K3Layout(n).bytes;
    if (b <= limit && !hybrid) {
      smem = std::max(smem, b);
    } else {
      goff[p] = (int64_t)gbytes;
      gbytes += b;
    }
  }
  // DAG placement scratch (obstacle lists) for the problems that try it
  std::vector<int64_t> doff(P, -1);
  size_t dbytes = 0;
  for (int p = 0; p < P; ++p) {
    const int n = (int)(item_ptr[p + 1] - item_ptr[p]);
    if (n == 0 || t_pack_form == 1 || (t_pack_form == 0 && n < K3_DAG_MIN_ITEMS)) continue;
    doff[p] = (int64_t)dbytes;
    dbytes += K3DagLayout(n).bytes;
  }
  Scratch sc(s);
  int64_t *d_ptr, *d_sz, *d_off, *d_cap, *d_goff, *d_doff, *d_ccap = nullptr;
  unsigned char* d_ds = nullptr;
  int32_t *d_t, *d_s, *d_e, *d_comp = nullptr;
  uint8_t *d_act, *d_met = nullptr;
  unsigned char* d_g = nullptr;
  const size_t ni = size_t(std::max<int64_t>(NI, 1));
  RM_CUDA(sc.alloc(&d_ptr, size_t(P) + 1));
  RM_CUDA(sc.alloc(&d_t, ni));
  RM_CUDA(sc.alloc(&d_s, ni));
  RM_CUDA(sc.alloc(&d_e, ni));
  RM_CUDA(sc.alloc(&d_sz, ni));
  RM_CUDA(sc.alloc(&d_act, ni));
  RM_CUDA(sc.alloc(&d_off, ni));
  RM_CUDA(sc.alloc(&d_cap, size_t(P)));
  RM_CUDA(sc.alloc(&d_goff, size_t(P)));
  if (comps) {
    RM_CUDA(sc.alloc(&d_met, size_t(P)));
    RM_CUDA(sc.alloc(&d_comp, ni));
    RM_CUDA(sc.alloc(&d_ccap, ni));
  }
  if (gbytes) RM_CUDA(sc.alloc(&d_g, gbytes));
  RM_CUDA(sc.alloc(&d_doff, size_t(P)));
  if (dbytes) RM_CUDA(sc.alloc(&d_ds, dbytes));
  RM_CUDA(cudaMemcpyAsync(d_doff, doff.data(), size_t(P) * 8, cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaMemcpyAsync(d_ptr, item_ptr, (size_t(P) + 1) * 8, cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaMemcpyAsync(d_goff, goff.data(), size_t(P) * 8, cudaMemcpyHostToDevice, s));
  if (NI > 0) {
    RM_CUDA(cudaMemcpyAsync(d_t, tensor, size_t(NI) * 4, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaMemcpyAsync(d_s, start, size_t(NI) * 4, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaMemcpyAsync(d_e, end, size_t(NI) * 4, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaMemcpyAsync(d_sz, size, size_t(NI) * 8, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaMemcpyAsync(d_act, is_act, size_t(NI), cudaMemcpyHostToDevice, s));
  }
  K3Args a{P, d_ptr, d_t, d_s, d_e, d_sz, d_act, mode, d_off, d_cap, d_met, d_comp, d_ccap, d_g,
           d_goff, d_ds, d_doff};
  int rc;
  // the register-resident placed list holds NT * MAXC - 1 placed items; fewer
  // slots per thread shorten the per-item chain between the block barriers
  if (maxN < 4096 && times16)
    rc = launch_k3_t<512, 8>(a, P, smem, s);
  else if (maxN < 4096)
    rc = launch_k3_t<256, 16>(a, P, smem, s);
  else if (maxN < 8192 && times16)
    rc = launch_k3_t<512, 16>(a, P, smem, s);
  else if (hybrid)
    rc = launch_k3_t<kHyNT, kHyMR, kHyMS>(a, P, smem, s);
  else
    rc = launch_k3_t<1024, 16>(a, P, smem, s);
  if (rc) return rc;
  RM_CUDA(cudaMemcpyAsync(capacity, d_cap, size_t(P) * 8, cudaMemcpyDeviceToHost, s));
  if (NI > 0) RM_CUDA(cudaMemcpyAsync(offset, d_off, size_t(NI) * 8, cudaMemcpyDeviceToHost, s));
  if (comps) {
    RM_CUDA(cudaMemcpyAsync(bound_met, d_met, size_t(P), cudaMemcpyDeviceToHost, s));
    if (NI > 0) {
      RM_CUDA(cudaMemcpyAsync(comp, d_comp, size_t(NI) * 4, cudaMemcpyDeviceToHost, s));
      RM_CUDA(cudaMemcpyAsync(comp_cap, d_ccap, size_t(NI) * 8, cudaMemcpyDeviceToHost, s));
    }
  }
  RM_CUDA(cudaStreamSynchronize(s));
  return RM_OK;
}
