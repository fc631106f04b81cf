// K1: batched candidate-order evaluator + argmin, and the general single
// schedule evaluator (validate_schedule / tensor_lifetimes /
// live_bytes_by_timestep / peak_memory) for sm_100a.
//
// Reference: pkg/src/memplan/graph.py:375-468 (validate_schedule,
// sequential_schedule, tensor_lifetimes, live_bytes_by_timestep, peak_memory),
// tests/oracles.py:46-56 and planner.py:209-216 (first strict minimum).
//
// K1 layout (one persistent CTA per SM, G candidate groups of NT threads,
// each group evaluates one candidate at a time with named barriers):
//   smem (shared by groups): opmeta[n] {class, slot} (IdxT pairs),
//                            table[U] {out_bytes, free_bytes} (longlong2)
//   smem (per group):        stage[n] order row (IdxT), pos[n] inverse (IdxT),
//                            mfree[K] int64 multi-consumer frees per slot,
//                            group-reduction scratch
// Phase 1  coalesced row load -> stage[k] = o, pos[o] = k, range check
// Phase 2  checked edges (pos[u] < pos[v]); multi-consumer tensors:
//          argmax_c pos[c] over maximal consumers -> mfree[slot(c)] += size
// Phase 3  blocked scan over positions: x_k = out[o_k] - freed_after(o_{k-1}),
//          readback pos[o_k] == k (permutation), running max/first argmax,
//          group exclusive scan of chunk totals, (max, min-index) reduction.
#include <climits>
#include <cstring>
#include <map>

#include <cstdlib>

#include "k_common.cuh"

namespace roam {

thread_local bool g_timing = false;
thread_local int g_sm_reserve = 0;
thread_local double g_last_ms = -1.0;

struct K1Args {
  const int32_t* orders;
  int64_t B;
  int n;
  int C;  // positions per thread in the blocked scan, ceil(n / NT)
  int NT, G;
  const void* opmeta;
  const longlong2* table;
  int U;
  const void* edges;
  int64_t n_edges;
  const int32_t* mptr;
  const void* mcons;
  const int64_t* msize;
  int64_t n_multi;
  int K;
  int64_t* peak;
  int32_t* argmax;
  uint8_t* valid;
  size_t off_table, off_groups, group_bytes, off_pos, off_mfree, off_red;
};

template <class IdxT>
struct Pair;
template <>
struct Pair<uint16_t> {
  using T = uint32_t;  // two u16 in one 32-bit word
  __device__ static void split(T w, int& a, int& b) { a = w & 0xffff; b = w >> 16; }
};
template <>
struct Pair<int32_t> {
  using T = int2;
  __device__ static void split(T w, int& a, int& b) { a = w.x; b = w.y; }
};

template <class IdxT, int MAXC>
__global__ void __launch_bounds__(1024, 1) k1_eval_orders(const K1Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  using PW = typename Pair<IdxT>::T;
  constexpr IdxT NONE = (IdxT)-1;
  const int n = a.n;

  // ---- stage graph metadata once per CTA
  {
    const size_t meta_words = (2 * size_t(n) * sizeof(IdxT) + 3) / 4;
    const uint32_t* src = static_cast<const uint32_t*>(a.opmeta);
    uint32_t* dst = reinterpret_cast<uint32_t*>(smem);
    for (size_t i = threadIdx.x; i < meta_words; i += blockDim.x) dst[i] = __ldg(src + i);
    longlong2* tab = reinterpret_cast<longlong2*>(smem + a.off_table);
    for (int i = threadIdx.x; i < a.U; i += blockDim.x) tab[i] = a.table[i];
  }
  __syncthreads();
  const PW* opm = reinterpret_cast<const PW*>(smem);
  const longlong2* tab = reinterpret_cast<const longlong2*>(smem + a.off_table);

  const int gid = threadIdx.x / a.NT;
  const int tid = threadIdx.x - gid * a.NT;
  if (gid >= a.G) return;
  const int bar_id = 1 + gid;
  const int NT = a.NT;
  unsigned char* gbase = smem + a.off_groups + size_t(gid) * a.group_bytes;
  IdxT* stage = reinterpret_cast<IdxT*>(gbase);
  IdxT* pos = reinterpret_cast<IdxT*>(gbase + a.off_pos);
  long long* mfree = reinterpret_cast<long long*>(gbase + a.off_mfree);
  long long* red_v = reinterpret_cast<long long*>(gbase + a.off_red);  // [NT/32]
  int* red_i = reinterpret_cast<int*>(red_v + 32);                      // [NT/32]
  const PW* edges = static_cast<const PW*>(a.edges);
  const IdxT* mcons = static_cast<const IdxT*>(a.mcons);
  const int lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;

  for (int64_t c = int64_t(blockIdx.x) * a.G + gid; c < a.B; c += int64_t(gridDim.x) * a.G) {
    const int32_t* row = a.orders + c * int64_t(n);
    int bad = 0;
    // ---- phase 1: load row (all loads in flight first), scatter positions
    constexpr int BATCH = MAXC < 8 ? MAXC : 8;  // loads in flight per thread
#pragma unroll
    for (int j0 = 0; j0 < MAXC; j0 += BATCH) {
      int32_t v[BATCH];
#pragma unroll
      for (int j = 0; j < BATCH; ++j) {
        const int k = tid + (j0 + j) * NT;
        v[j] = k < n ? __ldcs(row + k) : 0;  // streamed once: evict-first
      }
#pragma unroll
      for (int j = 0; j < BATCH; ++j) {
        const int k = tid + (j0 + j) * NT;
        if (k < n) {
          int o = v[j];
          if ((unsigned)o >= (unsigned)n) {
            bad = 1;
            o = 0;
          }
          stage[k] = (IdxT)o;
          pos[o] = (IdxT)k;
        }
      }
    }
    for (int s = tid; s < a.K; s += NT) mfree[s] = 0;
    gbar(bar_id, NT);

    // ---- phase 2: precedence edges, multi-consumer frees
    for (int64_t e = tid; e < a.n_edges; e += NT) {
      int u, w;
      Pair<IdxT>::split(__ldg(edges + e), u, w);
      bad |= (int)pos[u] >= (int)pos[w];
    }
    for (int64_t m = tid; m < a.n_multi; m += NT) {
      const int b0 = __ldg(a.mptr + m), b1 = __ldg(a.mptr + m + 1);
      int best = -1, bc = 0;
      for (int q = b0; q < b1; ++q) {
        const int cc = (int)__ldg(mcons + q);
        const int p = (int)pos[cc];
        if (p > best) {
          best = p;
          bc = cc;
        }
      }
      int s0, s1;
      Pair<IdxT>::split(opm[bc], s0, s1);
      atomicAdd(reinterpret_cast<unsigned long long*>(mfree + s1),
                (unsigned long long)__ldg(a.msize + m));
    }
    gbar(bar_id, NT);

    // ---- phase 3: blocked scan of x_k = out[o_k] - freed_after(o_{k-1})
    const int k0 = tid * a.C;
    const int k1 = min(n, k0 + a.C);
    long long carry = 0;
    if (k0 > 0 && k0 < n) {
      int cls, slot;
      Pair<IdxT>::split(opm[stage[k0 - 1]], cls, slot);
      carry = tab[cls].y + ((IdxT)slot != NONE ? mfree[slot] : 0);
    }
    long long run = 0, best = LLONG_MIN;
    int bestk = INT_MAX;
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
      const int o = (int)stage[k];
      bad |= (int)pos[o] != k;
      int cls, slot;
      Pair<IdxT>::split(opm[o], cls, slot);
      const longlong2 e = tab[cls];
      run += e.x - carry;
      if (run > best) {
        best = run;
        bestk = k;
      }
      carry = e.y + ((IdxT)slot != NONE ? mfree[slot] : 0);
    }
    // group exclusive scan of chunk totals
    long long incl = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane == 31) red_v[warp] = incl;
    bad = gbar_or(bar_id, NT, bad);
    long long off = incl - run;
    for (int w = 0; w < warp; ++w) off += red_v[w];
    long long cand = bestk == INT_MAX ? LLONG_MIN : off + best;
    int ck = bestk;
    // (max value, min index) reduction
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const long long ov = __shfl_down_sync(0xffffffffu, cand, d);
      const int oi = __shfl_down_sync(0xffffffffu, ck, d);
      if (ov > cand || (ov == cand && oi < ck)) {
        cand = ov;
        ck = oi;
      }
    }
    // red_v is re-used: everyone has read the warp totals before this barrier
    gbar(bar_id, NT);
    if (lane == 0) {
      red_v[warp] = cand;
      red_i[warp] = ck;
    }
    gbar(bar_id, NT);
    if (tid == 0) {
      long long bv = red_v[0];
      int bi = red_i[0];
      for (int w = 1; w < nwarps; ++w)
        if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bi)) {
          bv = red_v[w];
          bi = red_i[w];
        }
      if (n == 0) {
        bv = 0;
        bi = 0;
      }
      a.peak[c] = bv;
      a.argmax[c] = bi;
      a.valid[c] = bad ? 0 : 1;
    }
  }
}

// ---------------------------------------------------------------- argmin
// Lexicographic min of (peak, id) over valid rows; last-block-done finish.
// With out_key, also the packed key (peak << id_bits) | id (INT64_MAX when
// none is valid) so that ranks can combine with one all_reduce(MIN).
__global__ void k_argmin(const int64_t* __restrict__ peak, const uint8_t* __restrict__ valid,
                         int64_t B, int64_t id_base, long long* partial, unsigned* counter,
                         int64_t* out, int64_t* out_key, int id_bits) {
  __shared__ long long sv[32], si[32];
  __shared__ bool last;
  long long bv = LLONG_MAX, bi = LLONG_MAX;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < B;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (valid[i]) {
      const long long p = peak[i];
      if (p < bv || (p == bv && i < bi)) {
        bv = p;
        bi = i;
      }
    }
  }
  auto wred = [&](long long& v, long long& ix) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const long long ov = __shfl_down_sync(0xffffffffu, v, d);
      const long long oi = __shfl_down_sync(0xffffffffu, ix, d);
      if (ov < v || (ov == v && oi < ix)) {
        v = ov;
        ix = oi;
      }
    }
  };
  wred(bv, bi);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) {
    sv[warp] = bv;
    si[warp] = bi;
  }
  __syncthreads();
  if (warp == 0) {
    bv = lane < nw ? sv[lane] : LLONG_MAX;
    bi = lane < nw ? si[lane] : LLONG_MAX;
    wred(bv, bi);
    if (lane == 0) {
      partial[2 * blockIdx.x] = bv;
      partial[2 * blockIdx.x + 1] = bi;
      __threadfence();
      last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (last && warp == 0) {
    __threadfence();
    bv = LLONG_MAX;
    bi = LLONG_MAX;
    for (unsigned b = lane; b < gridDim.x; b += 32) {
      const long long v = ((volatile long long*)partial)[2 * b];
      const long long ix = ((volatile long long*)partial)[2 * b + 1];
      if (v < bv || (v == bv && ix < bi)) {
        bv = v;
        bi = ix;
      }
    }
    wred(bv, bi);
    if (lane == 0) {
      if (out) {
        out[0] = bi == LLONG_MAX ? LLONG_MAX : bv;
        out[1] = bi == LLONG_MAX ? -1 : bi + id_base;
      }
      if (out_key)
        out_key[0] = bi == LLONG_MAX ? LLONG_MAX : (bv << id_bits) | (bi + id_base);
    }
  }
}

// ------------------------------------------------- single-schedule kernels
struct SchedArgs {
  int n, T, steps;
  int64_t order_len;
  const int32_t* order;
  const int32_t* ts;
  int32_t* pos;
  int32_t* cnt;
  int32_t* cnt_ts;
  int* flags;  // [0] not-perm, [1] decreasing, [2] overfull
  unsigned long long* first_pred;  // min (v * n + p)
  int ops_per_step;
};

__global__ void k_sched_scatter(SchedArgs a) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.order_len;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int v = a.order[i];
    if ((unsigned)v >= (unsigned)a.n) {
      a.flags[0] = 1;
      continue;
    }
    atomicAdd(a.cnt + v, 1);
    a.pos[v] = (int)i;
  }
}

__global__ void k_sched_check(SchedArgs a, const int32_t* __restrict__ pred_ptr,
                              const int32_t* __restrict__ pred_idx) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * blockDim.x) {
    if (a.cnt[v] != 1) a.flags[0] = 1;
    const int t = a.ts[v];
    if (t < 0 || t >= a.steps) {
      a.flags[3] = 1;  // padding of a short timesteps vector: reported as such
      continue;
    }
    if (atomicAdd(a.cnt_ts + t, 1) + 1 > a.ops_per_step) a.flags[2] = 1;
  }
}

__global__ void k_sched_order(SchedArgs a, const int32_t* __restrict__ pred_ptr,
                              const int32_t* __restrict__ pred_idx) {
  // only launched for permutations: pos[] is the inverse permutation
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * blockDim.x) {
    const int i = a.pos[v];
    if (i > 0 && a.ts[v] < a.ts[a.order[i - 1]]) a.flags[1] = 1;
    for (int k = pred_ptr[v]; k < pred_ptr[v + 1]; ++k) {
      const int p = pred_idx[k];
      if (a.pos[p] > i || a.ts[p] > a.ts[v]) {
        atomicMin(a.first_pred, (unsigned long long)v * (unsigned long long)a.n + p);
        break;  // pred lists are sorted: the first hit is this v's smallest p
      }
    }
  }
}

// tensor_lifetimes (graph.py:440-449) + +/- size events
__global__ void k_lifetimes(int T, int steps, const int32_t* __restrict__ ts,
                            const int32_t* __restrict__ producer, const int32_t* __restrict__ cons_ptr,
                            const int32_t* __restrict__ cons_idx, const int64_t* __restrict__ size,
                            int32_t* birth, int32_t* death, unsigned long long* delta) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    const int b = ts[producer[t]];
    int d = INT_MIN;
    for (int k = cons_ptr[t]; k < cons_ptr[t + 1]; ++k) d = max(d, ts[cons_idx[k]]);
    if (d == INT_MIN) d = steps - 1;
    d = max(b, d);
    if (birth) birth[t] = b;
    if (death) death[t] = d;
    if (delta) {
      atomicAdd(delta + b, (unsigned long long)size[t]);
      atomicAdd(delta + d + 1, (unsigned long long)(-size[t]));
    }
  }
}

// one block: inclusive scan of delta -> live, max + first argmax
__global__ void __launch_bounds__(1024) k_live_scan(int steps, const long long* __restrict__ delta,
                                                    long long* live, long long* out_peak,
                                                    int* out_arg) {
  __shared__ long long wsum[32], wv[32];
  __shared__ int wi[32];
  const int NT = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int C = (steps + NT - 1) / NT;
  const int k0 = tid * C, k1 = min(steps, k0 + C);
  long long run = 0, best = LLONG_MIN;
  int bk = INT_MAX;
  for (int k = k0; k < k1; ++k) run += delta[k];
  long long incl = run;
  for (int d = 1; d < 32; d <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  long long acc = incl - run;
  for (int w = 0; w < warp; ++w) acc += wsum[w];
  for (int k = k0; k < k1; ++k) {
    acc += delta[k];
    if (live) live[k] = acc;
    if (acc > best) {
      best = acc;
      bk = k;
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    const long long ov = __shfl_down_sync(0xffffffffu, best, d);
    const int oi = __shfl_down_sync(0xffffffffu, bk, d);
    if (ov > best || (ov == best && oi < bk)) {
      best = ov;
      bk = oi;
    }
  }
  if (lane == 0) {
    wv[warp] = best;
    wi[warp] = bk;
  }
  __syncthreads();
  if (tid == 0) {
    best = wv[0];
    bk = wi[0];
    for (int w = 1; w < NT / 32; ++w)
      if (wv[w] > best || (wv[w] == best && wi[w] < bk)) {
        best = wv[w];
        bk = wi[w];
      }
    *out_peak = steps ? best : 0;
    *out_arg = steps ? bk : 0;
  }
}

// ----------------------------------------------------------- host launch

template <class IdxT, int MAXC>
static int launch_k1_t(K1Args& a, int grid, size_t smem, cudaStream_t s) {
  auto kern = k1_eval_orders<IdxT, MAXC>;
  RM_CUDA(smem_optin(kern));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  kern<<<grid, a.NT * a.G, smem, s>>>(a);
  RM_LAUNCH_CHECK("k1_eval_orders launch");
  if (g_timing) {
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    g_last_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return RM_OK;
}

template <class IdxT>
static int launch_k1_idx(K1Args& a, int maxc, int grid, size_t smem, cudaStream_t s) {
  switch (maxc) {
    case 4: return launch_k1_t<IdxT, 4>(a, grid, smem, s);
    case 8: return launch_k1_t<IdxT, 8>(a, grid, smem, s);
    case 16: return launch_k1_t<IdxT, 16>(a, grid, smem, s);
    case 32: return launch_k1_t<IdxT, 32>(a, grid, smem, s);
    case 64: return launch_k1_t<IdxT, 64>(a, grid, smem, s);
  }
  return fail(RM_ERR_CAPACITY, "K1: positions per thread exceed 64");
}

static thread_local int t_force_variant = 0;  // 0 auto, 1 generic, 4 v4, 5 v5, 6 v5 with bulk-copied rows

// Launch geometry: NT threads per candidate group, G groups per CTA, one
// CTA per SM.  Shared memory bounds G; NT keeps ~8-16 positions per thread.
__global__ void k_widen_rows(const uint16_t* __restrict__ in, int32_t* __restrict__ out, int64_t count) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

static int launch_k1_int32(RmGraph* g, const int32_t* orders_dev, int64_t B, int64_t* peak,
                           int32_t* argmax, uint8_t* valid, cudaStream_t s);

// orders_dev: int32[B, n], or uint16[B, n] with u16_rows (n < 65536).
int launch_k1(RmGraph* g, const void* orders_dev, int64_t B, int64_t* peak, int32_t* argmax,
              uint8_t* valid, cudaStream_t s, bool u16_rows, const K1KeySel* sel = nullptr,
              bool* fused = nullptr) {
  if (fused) *fused = false;
  if (B <= 0) return RM_OK;
  if (g->k5v.ok && (t_force_variant == 0 || t_force_variant >= 5)) {
    const int rc = launch_k1v5(g, orders_dev, B, peak, argmax, valid, s, u16_rows, sel, t_force_variant == 6);
    if (rc != 1) {
      if (fused) *fused = sel != nullptr && rc == RM_OK;
      return rc;
    }
  }
  if (g->k4v.ok && (t_force_variant == 0 || t_force_variant >= 4)) {
    const int rc = launch_k1v4(g, orders_dev, B, peak, argmax, valid, s, u16_rows, sel);
    if (rc != 1) {
      if (fused) *fused = sel != nullptr && rc == RM_OK;
      return rc;
    }
  }
  if (!u16_rows)
    return launch_k1_int32(g, static_cast<const int32_t*>(orders_dev), B, peak, argmax, valid, s);
  // the generic evaluator reads int32 rows: widen into scratch
  Scratch sc(s);
  int32_t* wide_rows;
  const int64_t count = B * int64_t(g->n);
  RM_CUDA(sc.alloc(&wide_rows, size_t(std::max<int64_t>(count, 1))));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (count + 255) / 256));
  k_widen_rows<<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(orders_dev), wide_rows, count);
  RM_LAUNCH_CHECK("k_widen_rows launch");
  return launch_k1_int32(g, wide_rows, B, peak, argmax, valid, s);
}

static int launch_k1_int32(RmGraph* g, const int32_t* orders_dev, int64_t B, int64_t* peak,
                           int32_t* argmax, uint8_t* valid, cudaStream_t s) {
  const int n = g->n;
  const bool wide = g->info.wide_index != 0;
  const size_t isz = wide ? 4 : 2;
  K1Args a{};
  a.orders = orders_dev;
  a.B = B;
  a.n = n;
  a.opmeta = g->k1.opmeta.p;
  a.table = g->k1.table.as<longlong2>();
  a.U = (int)g->info.n_values;
  a.edges = g->k1.edges.p;
  a.n_edges = g->info.n_check_edges;
  a.mptr = g->k1.mptr.as<int32_t>();
  a.mcons = g->k1.mcons.p;
  a.msize = g->k1.msize.as<int64_t>();
  a.n_multi = g->info.n_multi;
  a.K = (int)g->info.n_slots;
  a.peak = peak;
  a.argmax = argmax;
  a.valid = valid;

  int NT = n <= 1024 ? 64 : n <= 2048 ? 128 : n <= 8192 ? 256 : 512;
  int C = (n + NT - 1) / NT;
  if (C < 1) C = 1;
  int maxc = C <= 4 ? 4 : C <= 8 ? 8 : C <= 16 ? 16 : C <= 32 ? 32 : 64;
  if (C > 64) return fail(RM_ERR_CAPACITY, "K1: graph too large for the shared-memory kernel");
  a.NT = NT;
  a.C = C;
  a.off_table = align16(2 * size_t(n) * isz);
  a.off_groups = align16(a.off_table + 16 * size_t(a.U));
  a.off_pos = align16(size_t(n) * isz);
  a.off_mfree = align16(a.off_pos + size_t(n) * isz);
  a.off_red = align16(a.off_mfree + 8 * size_t(a.K));
  a.group_bytes = align16(a.off_red + 32 * 8 + 32 * 4);
  int dev = g->device;
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t avail = max_smem > (int)a.off_groups ? size_t(max_smem) - a.off_groups : 0;
  int G = (int)(avail / a.group_bytes);
  G = std::min(G, 1024 / NT);
  G = std::min(G, 15);  // named barriers 1..15
  if (G < 1) return fail(RM_ERR_CAPACITY, "K1: graph metadata does not fit in shared memory");
  // don't launch more groups than candidates
  const int64_t sms = k1_sms(dev);
  if (int64_t(G) * sms > B) G = (int)std::max<int64_t>(1, (B + sms - 1) / sms);
  a.G = G;
  const size_t smem = a.off_groups + size_t(G) * a.group_bytes;
  const int grid = (int)std::min<int64_t>(sms, (B + G - 1) / G);
  return wide ? launch_k1_idx<int32_t>(a, maxc, grid, smem, s)
              : launch_k1_idx<uint16_t>(a, maxc, grid, smem, s);
}

int launch_argmin(const int64_t* peak_dev, const uint8_t* valid_dev, int64_t B, int64_t id_base,
                  int64_t* out_dev, cudaStream_t s, int64_t* key_dev = nullptr, int id_bits = 0) {
  Scratch sc(s);
  long long* partial;
  unsigned* counter;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148, (B + 1023) / 1024));
  RM_CUDA(sc.alloc(&partial, 2 * size_t(grid)));
  RM_CUDA(sc.alloc(&counter, 1));
  RM_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), s));
  k_argmin<<<grid, 1024, 0, s>>>(peak_dev, valid_dev, B, id_base, partial, counter, out_dev,
                                 key_dev, id_bits);
  RM_LAUNCH_CHECK("k_argmin launch");
  return RM_OK;
}

static int need_device(RmGraph* g) {
  if (!g) return fail(RM_ERR_INVALID_ARG, "graph handle is NULL");
  if (g->device < 0) return fail(RM_ERR_NO_DEVICE, "no CUDA device: libroam has no CPU path");
  return RM_OK;
}

}  // namespace roam

using namespace roam;

extern "C" {

int rm_set_timing(int enable) {
  g_timing = enable != 0;
  return RM_OK;
}
int rm_set_sm_reserve(int sms) {
  if (sms < 0 || sms > 64) return fail(RM_ERR_INVALID_ARG, "SM reserve must be 0..64");
  g_sm_reserve = sms;
  return RM_OK;
}
int rm_set_k1_variant(int variant) {
  if (variant < 0 || variant > 6) return fail(RM_ERR_INVALID_ARG, "variant must be 0..6");
  t_force_variant = variant;
  return RM_OK;
}
double rm_last_kernel_ms(void) { return g_last_ms; }

static int eval_impl(RmGraph* g, const void* orders, int64_t B, uint32_t flags, int64_t* peak,
                     int32_t* argmax, uint8_t* valid, int64_t id_base, int64_t* best,
                     void* stream) {
  int st = need_device(g);
  if (st) return st;
  if (B < 0) return fail(RM_ERR_INVALID_ARG, "negative batch");
  if (B > 0 && ((!orders && g->n > 0) || !peak || !argmax || !valid))
    return fail(RM_ERR_INVALID_ARG, "NULL array argument");
  const bool u16 = (flags & RM_ORDERS_U16) != 0;
  if (u16 && g->n > 65535) return fail(RM_ERR_INVALID_ARG, "uint16 rows need n_ops <= 65535");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (flags & RM_DEVICE_PTRS) {
    int rc = launch_k1(g, orders, B, peak, argmax, valid, s, u16);
    if (rc || !best) return rc;
    if (B == 0) {
      const int64_t none[2] = {INT64_MAX, -1};
      RM_CUDA(cudaMemcpyAsync(best, none, 16, cudaMemcpyHostToDevice, s));
      RM_CUDA(cudaStreamSynchronize(s));
      return RM_OK;
    }
    return launch_argmin(peak, valid, B, id_base, best, s);
  }

  // Host buffers: chunked pipeline -- every chunk's H2D is queued back to back
  // on a copy stream (device rows for the whole batch, no buffer reuse waits),
  // K1 on chunk i waits only for chunk i's copy; results come back through a
  // pinned staging buffer in one D2H each.
  const int64_t n = g->n;
  const int64_t esz = u16 ? 2 : 4;
  const int64_t row_bytes = std::max<int64_t>(esz * n, 4);
  // chunks of ~16 MB, halving towards the end of the batch so that the K1
  // launch left after the last copy is short (ROAM_STAGE_CHUNK_KB overrides
  // the first size, for measurement)
  static const int64_t chunk_bytes = [] {
    const char* e = std::getenv("ROAM_STAGE_CHUNK_KB");
    const long long kb = e ? std::atoll(e) : 0;
    return kb > 0 ? int64_t(kb) << 10 : int64_t(16) << 20;
  }();
  std::vector<std::pair<int64_t, int64_t>> chunks;  // (first row, rows)
  {
    int64_t cur = std::max<int64_t>(1, chunk_bytes / row_bytes);
    const int64_t floor_rows = std::max<int64_t>(1, (int64_t(1) << 20) / row_bytes);
    for (int64_t b0 = 0; b0 < B;) {
      const int64_t rem = B - b0;
      while (rem < 2 * cur && cur > floor_rows) cur = std::max(floor_rows, cur / 2);
      const int64_t nb = std::min(cur, rem);
      chunks.emplace_back(b0, nb);
      b0 += nb;
    }
  }
  const int64_t n_chunks = (int64_t)chunks.size();
  // per-thread copy stream, events and pinned result staging, created once
  // (re-entrant: calls on different threads never share them)
  struct CopyCtx {
    int dev = -1;
    cudaStream_t cs = nullptr;
    std::vector<cudaEvent_t> ev;
    unsigned char* pinned = nullptr;
    size_t pinned_bytes = 0;
  };
  static thread_local CopyCtx ctx;
  if (ctx.dev != g->device) {
    RM_CUDA(cudaStreamCreateWithFlags(&ctx.cs, cudaStreamNonBlocking));
    ctx.ev.clear();
    ctx.dev = g->device;
  }
  while ((int64_t)ctx.ev.size() < n_chunks + 1) {
    cudaEvent_t e;
    RM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx.ev.push_back(e);
  }
  const size_t res_bytes = size_t(B) * 13 + 16;  // peak, argmax, valid, best
  if (ctx.pinned_bytes < res_bytes) {
    if (ctx.pinned) cudaFreeHost(ctx.pinned);
    ctx.pinned = nullptr;
    ctx.pinned_bytes = 0;
    RM_CUDA(cudaMallocHost(&ctx.pinned, res_bytes));
    ctx.pinned_bytes = res_bytes;
  }
  cudaStream_t cs = ctx.cs;
  Scratch sc(s);
  unsigned char* d_ord;
  int64_t* d_peak;
  int32_t* d_arg;
  uint8_t* d_val;
  RM_CUDA(sc.alloc(&d_ord, size_t(std::max<int64_t>(B, 1) * n * esz)));
  RM_CUDA(sc.alloc(&d_peak, size_t(B)));
  RM_CUDA(sc.alloc(&d_arg, size_t(B)));
  RM_CUDA(sc.alloc(&d_val, size_t(B)));
  int64_t* d_best;
  RM_CUDA(sc.alloc(&d_best, 2));
  // the allocations above are ordered on s; the copy stream must see them
  RM_CUDA(cudaEventRecord(ctx.ev[n_chunks], s));
  RM_CUDA(cudaStreamWaitEvent(cs, ctx.ev[n_chunks], 0));
  for (int64_t k = 0; k < n_chunks; ++k) {
    const int64_t b0 = chunks[k].first, nb = chunks[k].second;
    RM_CUDA(cudaMemcpyAsync(d_ord + b0 * n * esz, static_cast<const unsigned char*>(orders) + b0 * n * esz,
                            size_t(nb * n * esz), cudaMemcpyHostToDevice, cs));
    RM_CUDA(cudaEventRecord(ctx.ev[k], cs));
  }
  int rc = RM_OK;
  for (int64_t k = 0; k < n_chunks && rc == RM_OK; ++k) {
    const int64_t b0 = chunks[k].first, nb = chunks[k].second;
    cudaStreamWaitEvent(s, ctx.ev[k], 0);
    rc = launch_k1(g, d_ord + b0 * n * esz, nb, d_peak + b0, d_arg + b0, d_val + b0, s, u16);
  }
  unsigned char* hp = ctx.pinned;
  if (rc == RM_OK && best && B > 0) {
    rc = launch_argmin(d_peak, d_val, B, id_base, d_best, s);
    if (rc == RM_OK) cudaMemcpyAsync(hp + size_t(B) * 13, d_best, 16, cudaMemcpyDeviceToHost, s);
  }
  if (rc == RM_OK && B > 0) {
    cudaMemcpyAsync(hp, d_peak, size_t(B) * 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hp + size_t(B) * 8, d_arg, size_t(B) * 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hp + size_t(B) * 12, d_val, size_t(B), cudaMemcpyDeviceToHost, s);
  }
  cudaError_t e = cudaStreamSynchronize(s);
  cudaError_t e2 = cudaStreamSynchronize(cs);
  if (e == cudaSuccess) e = e2;
  if (rc != RM_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "rm_eval_orders");
  if (B > 0) {
    std::memcpy(peak, hp, size_t(B) * 8);
    std::memcpy(argmax, hp + size_t(B) * 8, size_t(B) * 4);
    std::memcpy(valid, hp + size_t(B) * 12, size_t(B));
    if (best) std::memcpy(best, hp + size_t(B) * 13, 16);
  } else if (best) {
    best[0] = INT64_MAX;
    best[1] = -1;
  }
  return RM_OK;
}

int rm_eval_orders(RmGraph* g, const void* orders, int64_t B, uint32_t flags, int64_t* peak,
                   int32_t* argmax, uint8_t* valid, void* stream) {
  return eval_impl(g, orders, B, flags, peak, argmax, valid, 0, nullptr, stream);
}

int rm_eval_select(RmGraph* g, const void* orders, int64_t B, int64_t id_base, uint32_t flags,
                   int64_t* peak, int32_t* argmax, uint8_t* valid, int64_t* best, void* stream) {
  if (!best) return fail(RM_ERR_INVALID_ARG, "best is NULL");
  return eval_impl(g, orders, B, flags, peak, argmax, valid, id_base, best, stream);
}

int rm_argmin(const int64_t* peak, const uint8_t* valid, int64_t B, int64_t id_base,
              uint32_t flags, int64_t* out_best, void* stream) {
  if (B < 0 || !out_best || (B > 0 && (!peak || !valid)))
    return fail(RM_ERR_INVALID_ARG, "bad rm_argmin arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (flags & RM_DEVICE_PTRS) {
    if (B == 0) {
      const int64_t none[2] = {INT64_MAX, -1};
      RM_CUDA(cudaMemcpyAsync(out_best, none, 16, cudaMemcpyHostToDevice, s));
      return cudaStreamSynchronize(s) == cudaSuccess ? RM_OK : fail(RM_ERR_CUDA, "sync");
    }
    return launch_argmin(peak, valid, B, id_base, out_best, s);
  }
  if (B == 0) {
    out_best[0] = INT64_MAX;
    out_best[1] = -1;
    return RM_OK;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(RM_ERR_NO_DEVICE, "no CUDA device: libroam has no CPU path");
  }
  Scratch sc(s);
  int64_t *d_peak, *d_out;
  uint8_t* d_val;
  RM_CUDA(sc.alloc(&d_peak, size_t(B)));
  RM_CUDA(sc.alloc(&d_val, size_t(B)));
  RM_CUDA(sc.alloc(&d_out, 2));
  RM_CUDA(cudaMemcpyAsync(d_peak, peak, size_t(B) * 8, cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaMemcpyAsync(d_val, valid, size_t(B), cudaMemcpyHostToDevice, s));
  int rc = launch_argmin(d_peak, d_val, B, id_base, d_out, s);
  if (rc) return rc;
  RM_CUDA(cudaMemcpyAsync(out_best, d_out, 16, cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaStreamSynchronize(s));
  return RM_OK;
}

int rm_argmin_key(const int64_t* peak, const uint8_t* valid, int64_t B, int64_t id_base,
                  int32_t id_bits, int64_t max_peak, int64_t* out_key, void* stream) {
  if (B < 0 || !out_key || (B > 0 && (!peak || !valid)) || id_bits < 1 || id_bits > 62 ||
      max_peak < 0)
    return fail(RM_ERR_INVALID_ARG, "bad rm_argmin_key arguments");
  if ((id_base + B) > (int64_t(1) << id_bits) || id_base < 0)
    return fail(RM_ERR_OVERFLOW, "candidate ids do not fit id_bits");
  if (max_peak >= (int64_t(1) << (63 - id_bits)))
    return fail(RM_ERR_OVERFLOW, "peak bytes do not fit beside the id bits");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (B == 0) {
    const int64_t none = INT64_MAX;
    RM_CUDA(cudaMemcpyAsync(out_key, &none, 8, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaStreamSynchronize(s));
    return RM_OK;
  }
  return launch_argmin(peak, valid, B, id_base, nullptr, s, out_key, id_bits);
}

int rm_eval_select_key(RmGraph* g, const void* orders, int64_t B, int64_t id_base, int32_t id_bits,
                       uint32_t flags, int64_t* peak, int32_t* argmax, uint8_t* valid,
                       int64_t* out_key, void* stream) {
  int st = need_device(g);
  if (st) return st;
  if (!(flags & RM_DEVICE_PTRS)) return fail(RM_ERR_INVALID_ARG, "rm_eval_select_key takes device pointers");
  if (B < 0 || !out_key || (B > 0 && ((!orders && g->n > 0) || !peak || !argmax || !valid)) ||
      id_bits < 1 || id_bits > 62 || id_base < 0)
    return fail(RM_ERR_INVALID_ARG, "bad rm_eval_select_key arguments");
  const bool u16 = (flags & RM_ORDERS_U16) != 0;
  if (u16 && g->n > 65535) return fail(RM_ERR_INVALID_ARG, "uint16 rows need n_ops <= 65535");
  if ((id_base + B) > (int64_t(1) << id_bits))
    return fail(RM_ERR_OVERFLOW, "candidate ids do not fit id_bits");
  if (g->info.total_bytes >= (int64_t(1) << (63 - id_bits)))
    return fail(RM_ERR_OVERFLOW, "peak bytes do not fit beside the id bits");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (B == 0) {
    const int64_t none = INT64_MAX;
    RM_CUDA(cudaMemcpyAsync(out_key, &none, 8, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaStreamSynchronize(s));
    return RM_OK;
  }
  // partials and a counter the kernel leaves at zero, one set per (device,
  // stream): launches on one stream are ordered (PDL waits before touching
  // them), launches on different streams never share a counter
  struct SelCtx {
    long long* partial = nullptr;
    unsigned* counter = nullptr;
  };
  static thread_local std::map<std::pair<int, cudaStream_t>, SelCtx> ctxs;
  SelCtx& ctx = ctxs[{g->device, s}];
  if (!ctx.counter) {
    RM_CUDA(cudaMalloc(&ctx.partial, sizeof(long long) * 4096));
    RM_CUDA(cudaMalloc(&ctx.counter, sizeof(unsigned)));
    RM_CUDA(cudaMemsetAsync(ctx.counter, 0, sizeof(unsigned), s));
  }
  const K1KeySel sel{out_key, ctx.partial, ctx.counter, id_base, id_bits};
  bool fused = false;
  int rc = launch_k1(g, orders, B, peak, argmax, valid, s, u16, &sel, &fused);
  if (rc != RM_OK || fused) return rc;
  return launch_argmin(peak, valid, B, id_base, nullptr, s, out_key, id_bits);
}

int rm_eval_schedule(RmGraph* g, const int32_t* order, int64_t order_len, const int32_t* timesteps,
                     int64_t ts_len, int32_t ops_per_step, uint32_t flags, RmScheduleResult* res,
                     int32_t* birth, int32_t* death, int64_t* live, void* stream) {
  int st = need_device(g);
  if (st) return st;
  if (!res || order_len < 0 || ts_len < 0) return fail(RM_ERR_INVALID_ARG, "bad arguments");
  if ((order_len && !order) || (ts_len && !timesteps))
    return fail(RM_ERR_INVALID_ARG, "NULL order/timesteps");
  const int n = g->n, T = g->T;
  *res = RmScheduleResult{};
  const bool dev = (flags & RM_DEVICE_PTRS) != 0;
  if (dev) return fail(RM_ERR_INVALID_ARG, "rm_eval_schedule takes host pointers");
  // host-side length checks mirror graph.py:377-382 ordering
  int32_t max_ts = -1;
  for (int64_t i = 0; i < std::min<int64_t>(ts_len, n); ++i) {
    if (timesteps[i] < 0) return fail(RM_ERR_INVALID_ARG, "negative timestep");
    max_ts = std::max(max_ts, timesteps[i]);
  }
  for (int64_t i = n; i < ts_len; ++i) max_ts = std::max(max_ts, timesteps[i]);
  const int steps = ts_len ? max_ts + 1 : 0;  // Schedule.n_steps (graph.py:165-167)
  res->n_steps = steps;
  // a short timesteps vector is a validation failure (graph.py:379-380) that
  // the reference reports only after the permutation check
  if (ts_len < n && !(flags & RM_SCHED_VALIDATE))
    return fail(RM_ERR_INVALID_ARG, "timesteps shorter than n_ops");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  int32_t *d_ts, *d_order = nullptr, *d_pos, *d_cnt, *d_cnt_ts, *d_flags, *d_birth = nullptr,
                 *d_death = nullptr, *d_arg;
  unsigned long long *d_first, *d_delta = nullptr;
  long long *d_live = nullptr, *d_peak;
  RM_CUDA(sc.alloc(&d_ts, size_t(n)));
  RM_CUDA(cudaMemsetAsync(d_ts, 0, size_t(n) * 4, s));
  const int64_t ts_copy = std::min<int64_t>(ts_len, n);
  if (ts_copy)
    RM_CUDA(cudaMemcpyAsync(d_ts, timesteps, size_t(ts_copy) * 4, cudaMemcpyHostToDevice, s));
  const int TB = 256;
  auto blocks = [&](int64_t work) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(4096, (work + TB - 1) / TB));
  };
  if (flags & RM_SCHED_VALIDATE) {
    int status = 0;
    if (order_len != n) status = RM_SCHED_NOT_PERMUTATION;
    RM_CUDA(sc.alloc(&d_order, size_t(std::max<int64_t>(order_len, 1))));
    RM_CUDA(sc.alloc(&d_pos, size_t(n)));
    RM_CUDA(sc.alloc(&d_cnt, size_t(n)));
    RM_CUDA(sc.alloc(&d_cnt_ts, size_t(std::max(steps, 1))));
    RM_CUDA(sc.alloc(&d_flags, 4));
    RM_CUDA(sc.alloc(&d_first, 1));
    if (order_len)
      RM_CUDA(cudaMemcpyAsync(d_order, order, size_t(order_len) * 4, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaMemsetAsync(d_cnt, 0, size_t(n) * 4, s));
    RM_CUDA(cudaMemsetAsync(d_cnt_ts, 0, size_t(std::max(steps, 1)) * 4, s));
    RM_CUDA(cudaMemsetAsync(d_flags, 0, 16, s));
    RM_CUDA(cudaMemsetAsync(d_first, 0xff, 8, s));
    SchedArgs sa{n, T, steps, order_len, d_order, d_ts, d_pos, d_cnt, d_cnt_ts, d_flags, d_first,
                 ops_per_step};
    int h_flags[4] = {0, 0, 0, 0};
    unsigned long long h_first = ~0ull;
    if (!status) {
      k_sched_scatter<<<blocks(order_len), TB, 0, s>>>(sa);
      RM_LAUNCH_CHECK("k_sched_scatter");
      k_sched_check<<<blocks(n), TB, 0, s>>>(sa, g->d_pred_ptr.as<int32_t>(),
                                             g->d_pred_idx.as<int32_t>());
      RM_LAUNCH_CHECK("k_sched_check");
      RM_CUDA(cudaMemcpyAsync(h_flags, d_flags, 16, cudaMemcpyDeviceToHost, s));
      RM_CUDA(cudaStreamSynchronize(s));
      if (h_flags[0]) status = RM_SCHED_NOT_PERMUTATION;
    }
    if (!status && ts_len != n) status = RM_SCHED_TIMESTEPS_LEN;
    if (!status && ops_per_step < 1) status = RM_SCHED_OPS_PER_STEP;
    if (!status) {
      k_sched_order<<<blocks(n), TB, 0, s>>>(sa, g->d_pred_ptr.as<int32_t>(),
                                             g->d_pred_idx.as<int32_t>());
      RM_LAUNCH_CHECK("k_sched_order");
      RM_CUDA(cudaMemcpyAsync(h_flags, d_flags, 16, cudaMemcpyDeviceToHost, s));
      RM_CUDA(cudaMemcpyAsync(&h_first, d_first, 8, cudaMemcpyDeviceToHost, s));
      RM_CUDA(cudaStreamSynchronize(s));
      if (h_flags[1]) status = RM_SCHED_DECREASING;
      else if (h_flags[2]) status = RM_SCHED_STEP_OVERFULL;
      else if (h_first != ~0ull) {
        status = RM_SCHED_PRED;
        res->detail_a = (int32_t)(h_first / (unsigned long long)n);
        res->detail_b = (int32_t)(h_first % (unsigned long long)n);
      }
    }
    res->status = status;
    if (status) return RM_OK;
  }
  const bool want_peak = (flags & RM_SCHED_PEAK) || live;
  if (birth || death) {
    RM_CUDA(sc.alloc(&d_birth, size_t(T)));
    RM_CUDA(sc.alloc(&d_death, size_t(T)));
  }
  if (want_peak) {
    RM_CUDA(sc.alloc(&d_delta, size_t(steps) + 1));
    RM_CUDA(cudaMemsetAsync(d_delta, 0, (size_t(steps) + 1) * 8, s));
  }
  if (T > 0 && (birth || death || want_peak)) {
    k_lifetimes<<<blocks(T), TB, 0, s>>>(T, steps, d_ts, g->d_producer.as<int32_t>(),
                                         g->d_cons_ptr.as<int32_t>(), g->d_cons_idx.as<int32_t>(),
                                         g->d_size.as<int64_t>(), d_birth, d_death, d_delta);
    RM_LAUNCH_CHECK("k_lifetimes");
  }
  if (want_peak) {
    if (live) RM_CUDA(sc.alloc(&d_live, size_t(std::max(steps, 1))));
    RM_CUDA(sc.alloc(&d_peak, 1));
    RM_CUDA(sc.alloc(&d_arg, 1));
    k_live_scan<<<1, 1024, 0, s>>>(steps, reinterpret_cast<long long*>(d_delta), d_live, d_peak,
                                   d_arg);
    RM_LAUNCH_CHECK("k_live_scan");
    RM_CUDA(cudaMemcpyAsync(&res->peak, d_peak, 8, cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaMemcpyAsync(&res->argmax, d_arg, 4, cudaMemcpyDeviceToHost, s));
    if (live && steps)
      RM_CUDA(cudaMemcpyAsync(live, d_live, size_t(steps) * 8, cudaMemcpyDeviceToHost, s));
  }
  if (birth && T) RM_CUDA(cudaMemcpyAsync(birth, d_birth, size_t(T) * 4, cudaMemcpyDeviceToHost, s));
  if (death && T) RM_CUDA(cudaMemcpyAsync(death, d_death, size_t(T) * 4, cudaMemcpyDeviceToHost, s));
  RM_CUDA(cudaStreamSynchronize(s));
  return RM_OK;
}

}  // extern "C"
