// Device-side candidate generator: one warp per candidate runs Kahn's
// algorithm with counter-based random priorities, so B candidate orders are
// materialised in HBM without a host round trip.
//
//   mix(x)   = splitmix64 finaliser of x + 0x9E3779B97F4A7C15
//   h(id)    = mix(seed ^ mix(id))
//   key(op)  = mix(h(id) ^ op)
//   row(id)  = Kahn order over direct_preds popping the ready op with the
//              smallest (key(op), op)
// Python restatement (the checker): oracle/memplan_oracle.py kahn_candidate.
#include <algorithm>
#include <climits>

#include "roam_internal.h"

namespace roam {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

template <class IdxT>
__global__ void __launch_bounds__(256) k_gen_orders(int n, uint64_t seed, int64_t first_id, int64_t B,
                                                    const int32_t* __restrict__ pred_ptr,
                                                    const int32_t* __restrict__ succ_ptr,
                                                    const int32_t* __restrict__ succ_idx,
                                                    int32_t* __restrict__ out, int warps_per_block,
                                                    const int32_t* __restrict__ redo,
                                                    const unsigned* __restrict__ n_redo) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = ((2 * size_t(n) * sizeof(IdxT)) + 15) & ~size_t(15);
  IdxT* indeg = reinterpret_cast<IdxT*>(smem + per_warp * warp);
  IdxT* ready = indeg + n;
  const int64_t stride = int64_t(gridDim.x) * warps_per_block;
  if (redo) B = *n_redo;  // rows the thread form handed over (candidate indices)
  for (int64_t i = int64_t(blockIdx.x) * warps_per_block + warp; i < B; i += stride) {
    const int64_t c = redo ? int64_t(redo[i]) : i;
    const uint64_t h = mix64(seed ^ mix64((uint64_t)(first_id + c)));
    int32_t* row = out + c * int64_t(n);
    int nready = 0;
    for (int base = 0; base < n; base += 32) {
      const int v = base + lane;
      int d = 1;
      if (v < n) {
        d = __ldg(pred_ptr + v + 1) - __ldg(pred_ptr + v);
        indeg[v] = (IdxT)d;
      }
      const unsigned m = __ballot_sync(0xffffffffu, v < n && d == 0);
      if (v < n && d == 0) ready[nready + __popc(m & ((1u << lane) - 1))] = (IdxT)v;
      nready += __popc(m);
    }
    __syncwarp();
    int keep = 0;
    int step = 0;
    for (; step < n && nready > 0; ++step) {
      uint64_t bk = ~0ull;
      int bv = INT_MAX, bi = -1;
      for (int i = lane; i < nready; i += 32) {
        const int v = (int)ready[i];
        const uint64_t k = mix64(h ^ (uint64_t)v);
        if (k < bk || (k == bk && v < bv)) {
          bk = k;
          bv = v;
          bi = i;
        }
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        const uint64_t ok = __shfl_xor_sync(0xffffffffu, bk, d);
        const int ov = __shfl_xor_sync(0xffffffffu, bv, d);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, d);
        if (ok < bk || (ok == bk && ov < bv)) {
          bk = ok;
          bv = ov;
          bi = oi;
        }
      }
      const int v = bv;
      __syncwarp();
      if (lane == 0) ready[bi] = ready[nready - 1];
      --nready;
      if ((step & 31) == lane) keep = v;
      if ((step & 31) == 31) row[step - 31 + lane] = keep;
      const int s0 = __ldg(succ_ptr + v), s1 = __ldg(succ_ptr + v + 1);
      __syncwarp();
      for (int k0 = s0; k0 < s1; k0 += 32) {
        const int k = k0 + lane;
        int w = -1;
        if (k < s1) {
          w = __ldg(succ_idx + k);
          const int d = (int)indeg[w] - 1;
          indeg[w] = (IdxT)d;
          if (d != 0) w = -1;
        }
        const unsigned m = __ballot_sync(0xffffffffu, w >= 0);
        if (w >= 0) ready[nready + __popc(m & ((1u << lane) - 1))] = (IdxT)w;
        nready += __popc(m);
      }
      __syncwarp();
    }
    // flush the partial tail; a cycle leaves -1 (rejected later as invalid)
    const int tail0 = step - (step & 31);
    if (lane < (step & 31)) row[tail0 + lane] = keep;
    for (int i = step + lane; i < n; i += 32) row[i] = -1;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Thread-per-candidate form (the default when the graph qualifies, GenMeta):
// each thread runs one candidate's Kahn order alone, its ready set a 4-ary
// min-heap of full 64-bit keys and its predecessor-arrival counters
// lane-interleaved in shared memory (word k of lane l at [k * 32 + l]):
// whatever heap slot or counter each thread of a warp touches, the warp's
// access is the minimum number of wavefronts -- divergent heap walks never
// bank-conflict.  mix64 is a bijection, so keys never tie and the popped op is
// recovered by inverting it (unmix64); the heap walks are predicated moves
// over the levels the heap's size implies, so a warp's threads stay together.
// Counters return to zero when an op becomes ready (a toggle bit sees its
// second arrival; an arrival counter is cleared at its last), so nothing is
// reset between candidates.
//
// Heap entries per candidate: GEN_CAP (a template parameter, 32-64) in a
// 4-ary heap, walked with GEN_DEPTH = 3 unrolled predicated levels.  A ready set above GEN_CAP (or a
// cycle) hands the candidate to the warp form, which rewrites its row.

__device__ __forceinline__ uint64_t unmix64(uint64_t y) {
  y ^= (y >> 31) ^ (y >> 62);
  y *= 0x319642b2d24d8ec3ull;  // inverse of 0x94D049BB133111EB mod 2^64
  y ^= (y >> 27) ^ (y >> 54);
  y *= 0x96de1b173f119089ull;  // inverse of 0xBF58476D1CE4E5B9
  y ^= (y >> 30) ^ (y >> 60);
  return y - 0x9E3779B97F4A7C15ull;
}

// The successor table (eptr as PtrT, edges as u32) is staged in shared memory
// once per CTA: the per-step lookups are dependent loads, which from L2 would
// cost ~700 cycles each (the per-thread state leaves L1 almost no room).
template <typename PtrT, int GEN_CAP, int GEN_DEPTH = 3>
__global__ void __launch_bounds__(1024) k_gen_thread(int n, uint64_t seed, int64_t first_id, int64_t B,
                                                     const uint32_t* __restrict__ eptr_g,
                                                     const uint32_t* __restrict__ edges_g, int n_edges,
                                                     const uint16_t* __restrict__ zero, int n_zero,
                                                     int words, size_t table_bytes, int32_t* __restrict__ out,
                                                     int32_t* __restrict__ redo, unsigned* __restrict__ n_redo) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* edges = reinterpret_cast<uint32_t*>(smem);
  PtrT* eptr = reinterpret_cast<PtrT*>(smem + 4 * size_t(n_edges));
  for (int i = threadIdx.x; i < n_edges; i += blockDim.x) edges[i] = __ldg(edges_g + i);
  for (int i = threadIdx.x; i <= n; i += blockDim.x) eptr[i] = (PtrT)__ldg(eptr_g + i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = (size_t(words) * 4 + size_t(GEN_CAP) * 8) * 32;
  unsigned char* wbase = smem + table_bytes + per_warp * warp;
  uint32_t* ctr = reinterpret_cast<uint32_t*>(wbase) + lane;
  uint64_t* heap = reinterpret_cast<uint64_t*>(wbase + size_t(words) * 128) + lane;
  const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
  const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int k = 0; k < words; ++k) ctr[k * 32] = 0u;
  for (int64_t c = gtid; c < B; c += nthreads) {
    const uint64_t h = mix64(seed ^ mix64((uint64_t)(first_id + c)));
    int32_t* row = out + c * int64_t(n);
    int R = 0;
    bool over = false;
    // 4-ary min-heap (children of i: 4i+1 .. 4i+4): GEN_DEPTH = 3 levels hold
    // 85 entries, half the levels of a binary heap on every walk
    // insert key x at slot R and sift it up (predicated moves)
    auto push = [&](uint64_t x) {
      over |= R == GEN_CAP;
      int i = min(R, GEN_CAP - 1);
      R = min(R + 1, GEN_CAP);
      bool go = true;
#pragma unroll
      for (int L = 0; L < GEN_DEPTH; ++L) {
        const int p = (i - 1) >> 2;
        const uint64_t e = heap[max(p, 0) * 32];
        go = go && i > 0 && x < e;
        if (go) {
          heap[i * 32] = e;
          i = p;
        }
      }
      heap[i * 32] = x;
    };
    for (int k = 0; k < n_zero; ++k) push(mix64(h ^ __ldg(zero + k)));
    int step = 0;
    for (; step < n && R > 0 && !over; ++step) {
      const uint64_t top = heap[0];
      --R;
      if (R > 0) {  // move the last entry down from the root (predicated moves)
        const uint64_t x = heap[R * 32];
        int i = 0;
        bool go = true;
#pragma unroll
        for (int L = 0; L < GEN_DEPTH; ++L) {
          const int ch = 4 * i + 1;  // children may pass R (or the heap) on the last level
          const uint64_t a0 = heap[min(ch, GEN_CAP - 1) * 32];
          const uint64_t a1 = heap[min(ch + 1, GEN_CAP - 1) * 32];
          const uint64_t a2 = heap[min(ch + 2, GEN_CAP - 1) * 32];
          const uint64_t a3 = heap[min(ch + 3, GEN_CAP - 1) * 32];
          // min of the children below R, as a two-level tree
          const bool t1 = ch + 1 < R && a1 < a0;
          const uint64_t m01 = t1 ? a1 : a0;
          const int i01 = t1 ? 1 : 0;
          const bool v2 = ch + 2 < R, t3 = ch + 3 < R && a3 < a2;
          const uint64_t m23 = t3 ? a3 : a2;
          const int i23 = t3 ? 3 : 2;
          const bool tr = v2 && m23 < m01;
          const uint64_t m = tr ? m23 : m01;
          go = go && ch < R && m < x;
          if (go) {
            heap[i * 32] = m;
            i = ch + (tr ? i23 : i01);
          }
        }
        heap[i * 32] = x;
      }
      const uint32_t v = (uint32_t)(unmix64(top) ^ h);
      row[step] = (int32_t)v;
      const uint32_t e1 = eptr[v + 1];
      for (uint32_t q = eptr[v]; q < e1; ++q) {
        const uint32_t e = edges[q];
        const uint32_t w = e & 0xffffu, kind = e >> 29, bo = (e >> 16) & 0x1fffu;
        bool ready = true;
        if (kind != 0) {
          uint32_t* cw = ctr + (bo >> 5) * 32;
          const uint32_t word = *cw, sh = bo & 31u;
          if (kind == 1) {  // two predecessors: a toggle bit
            *cw = word ^ (1u << sh);
            ready = (word >> sh) & 1u;
          } else {          // kind + 1 predecessors: count the earlier arrivals
            const uint32_t m = kind <= 3u ? 3u : 7u;  // field width 2 or 3 bits
            ready = ((word >> sh) & m) == kind;
            *cw = ready ? (word & ~(m << sh)) : word + (1u << sh);
          }
        }
        if (ready) push(mix64(h ^ w));
      }
    }
    if (step < n) {  // overflow or a cycle: clear the counters, hand the row over
      for (int k = 0; k < words; ++k) ctr[k * 32] = 0u;
      redo[atomicAdd(n_redo, 1u)] = (int32_t)c;
    }
  }
}

void build_gen_meta(RmGraph& g) {
  // Over the checked edges (the transitive reduction of direct_preds when
  // rm_graph_create reduced): a redundant edge p -> w (p already an ancestor
  // of another predecessor of w) never decides when w becomes ready, so
  // Kahn's order is unchanged and most multi-predecessor ops need no counter
  // (GPT2-XL: 2,224 -> 871 of them).
  GenMeta& m = g.gen;
  m.ok = 0;
  const int n = g.n;
  if (n <= 0 || n > 65536) return;
  const size_t E = g.h_edge_u.size();
  std::vector<int> indeg(size_t(n), 0);
  for (size_t e = 0; e < E; ++e) indeg[size_t(g.h_edge_v[e])]++;
  // counter bit offsets: toggles (two predecessors) and 2/3-bit arrival
  // counters, packed so that no field straddles a 32-bit word
  std::vector<uint32_t> code(size_t(n), 0);  // bitoff << 16 | kind << 29 (w added per edge)
  uint32_t bit = 0;
  auto alloc = [&](uint32_t width) {
    if ((bit & 31u) + width > 32u) bit = (bit + 31u) & ~31u;
    const uint32_t at = bit;
    bit += width;
    return at;
  };
  for (int v = 0; v < n; ++v) {
    const int d = indeg[size_t(v)];
    if (d <= 1) continue;
    if (d > 8) return;
    const uint32_t kind = uint32_t(d - 1);
    const uint32_t at = alloc(d == 2 ? 1u : d <= 4 ? 2u : 3u);
    code[size_t(v)] = (at << 16) | (kind << 29);
  }
  if (bit > 8192u) return;
  m.words = int((bit + 31u) / 32u);
  m.h_eptr.assign(size_t(n) + 1, 0);
  m.h_edges.clear();
  m.h_zero.clear();
  size_t e = 0;  // edges come grouped by source, ascending
  for (int v = 0; v < n; ++v) {
    for (; e < E && g.h_edge_u[e] == v; ++e) {
      const int w = g.h_edge_v[e];
      m.h_edges.push_back(code[size_t(w)] | uint32_t(w));
    }
    m.h_eptr[size_t(v) + 1] = (uint32_t)m.h_edges.size();
    if (indeg[size_t(v)] == 0) m.h_zero.push_back((uint16_t)v);
  }
  if (e != E) return;  // not grouped by source: keep the warp form
  m.n_zero = (int)m.h_zero.size();
  if (m.h_edges.empty()) m.h_edges.push_back(0);
  if (m.h_zero.empty()) m.h_zero.push_back(0);
  m.ok = 1;
}

static thread_local int t_gen_form = 0;  // 0 auto, 1 warp form only
static thread_local int t_gen_cap = 0;   // thread form heap entries: 40 or 64; 0 = by graph size

static int launch_gen_warp(RmGraph* g, uint64_t seed, int64_t first_id, int64_t B, int32_t* out,
                           const int32_t* redo, const unsigned* n_redo, cudaStream_t s) {
  const int n = g->n;
  const bool wide = g->info.wide_index != 0;
  const size_t per_warp = ((2 * size_t(n) * (wide ? 4 : 2)) + 15) & ~size_t(15);
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device);
  int wpb = (int)std::min<size_t>(8, per_warp ? size_t(max_smem) / per_warp : 8);
  if (wpb < 1) return fail(RM_ERR_CAPACITY, "generator: graph too large for shared memory");
  const size_t smem = per_warp * wpb;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
  const int64_t blocks_needed = (B + wpb - 1) / wpb;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks_needed, int64_t(sms) * 8));
  if (wide) {
    RM_CUDA(smem_optin(k_gen_orders<int32_t>));
    k_gen_orders<int32_t><<<grid, 32 * wpb, smem, s>>>(
        n, seed, first_id, B, g->d_pred_ptr.as<int32_t>(), g->d_succ_ptr.as<int32_t>(),
        g->d_succ_idx.as<int32_t>(), out, wpb, redo, n_redo);
  } else {
    RM_CUDA(smem_optin(k_gen_orders<uint16_t>));
    k_gen_orders<uint16_t><<<grid, 32 * wpb, smem, s>>>(
        n, seed, first_id, B, g->d_pred_ptr.as<int32_t>(), g->d_succ_ptr.as<int32_t>(),
        g->d_succ_idx.as<int32_t>(), out, wpb, redo, n_redo);
  }
  RM_LAUNCH_CHECK("k_gen_orders launch");
  return RM_OK;
}

int launch_gen(RmGraph* g, uint64_t seed, int64_t first_id, int64_t B, int32_t* out, cudaStream_t s) {
  if (B <= 0) return RM_OK;
  const GenMeta& m = g->gen;
  int max_smem = 0, sms = 148;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
  const int n_edges = (int)m.h_edges.size();
  const bool narrow = n_edges < 65536;
  auto a16 = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t table = a16(4 * size_t(n_edges)) + a16((narrow ? 2 : 4) * (size_t(g->n) + 1));
  // heap capacity (rm_set_gen_form 40/64 for A/B).  Default 40 below
  // 8k ops (GPT-2 small / BERT-large: ready sets reach ~37), 64 above (the
  // 11k-op GPT2-XL's reach further: 40 entries hand ~1 % of its rows to the
  // slow warp form, 3.25 vs 3.50 M/s measured); a candidate that outgrows the
  // heap is rewritten by the warp form
  const int cap = t_gen_cap > 0 ? t_gen_cap : (g->n >= 8192 ? 64 : 40);
  const size_t per_warp = (size_t(m.words) * 4 + size_t(cap) * 8) * 32;
  const int warps = m.ok && size_t(max_smem) > table ? (int)std::min<size_t>(32, (size_t(max_smem) - table) / per_warp) : 0;
  if (t_gen_form == 1 || warps < 4 || B > INT32_MAX)
    return launch_gen_warp(g, seed, first_id, B, out, nullptr, nullptr, s);
  // one CTA per SM, as many warps as shared memory holds
  const int threads = 32 * warps;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, (B + threads - 1) / threads));
  Scratch sc(s);
  int32_t* redo;
  unsigned* n_redo;
  RM_CUDA(sc.alloc(&redo, size_t(B)));
  RM_CUDA(sc.alloc(&n_redo, 1));
  RM_CUDA(cudaMemsetAsync(n_redo, 0, sizeof(unsigned), s));
  const size_t smem = table + per_warp * warps;
#define RM_GEN_CASE(PT, CAP)                                                                            \
  if (cap == CAP) {                                                                                     \
    RM_CUDA(smem_optin(k_gen_thread<PT, CAP>));                                                         \
    k_gen_thread<PT, CAP><<<grid, threads, smem, s>>>(g->n, seed, first_id, B, m.eptr.as<uint32_t>(),     \
                                                      m.edges.as<uint32_t>(), n_edges, m.zero.as<uint16_t>(), \
                                                      m.n_zero, m.words, table, out, redo, n_redo);     \
  }
  if (narrow) {
    RM_GEN_CASE(uint16_t, 40) RM_GEN_CASE(uint16_t, 64)
  } else {
    RM_GEN_CASE(uint32_t, 40) RM_GEN_CASE(uint32_t, 64)
  }
#undef RM_GEN_CASE
  RM_LAUNCH_CHECK("k_gen_thread launch");
  // the rows the thread form handed over (a ready set above GEN_CAP entries,
  // or a cycle): the warp form rewrites them; a no-op launch when there are none
  return launch_gen_warp(g, seed, first_id, std::min<int64_t>(B, int64_t(sms) * 8), out, redo, n_redo, s);
}

}  // namespace roam

extern "C" int rm_set_gen_form(int form) {
  // 0 auto, 1 warp form; 40/64 = auto with that heap capacity (A/B)
  if (form == 40 || form == 64) {
    roam::t_gen_form = 0;
    roam::t_gen_cap = form;
    return RM_OK;
  }
  if (form < 0 || form > 1) return roam::fail(RM_ERR_INVALID_ARG, "gen form must be 0 (auto) or 1 (warp)");
  roam::t_gen_form = form;
  if (form == 0) roam::t_gen_cap = 0;
  return RM_OK;
}

extern "C" int rm_gen_orders(RmGraph* g, uint64_t seed, int64_t first_id, int64_t B,
                             int32_t* orders_dev, void* stream) {
  using namespace roam;
  if (!g) return fail(RM_ERR_INVALID_ARG, "graph handle is NULL");
  if (g->device < 0) return fail(RM_ERR_NO_DEVICE, "no CUDA device: libroam has no CPU path");
  if (B < 0 || (B > 0 && !orders_dev)) return fail(RM_ERR_INVALID_ARG, "bad rm_gen_orders arguments");
  return launch_gen(g, seed, first_id, B, orders_dev, static_cast<cudaStream_t>(stream));
}
