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
#include <climits>

#include "roam_internal.h"

namespace roam {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Per warp (one candidate at a time): indeg[n], the ready set as op ids
// ready[] plus the high 32 bits of their keys rk[] (computed once, when an op
// becomes ready).  Each step selects the minimum (key, op) with warp
// min-reductions (REDUX) on the key's high word; only ties on it (rare)
// recompute the full 64-bit keys of the tied ops.
template <class IdxT>
__global__ void __launch_bounds__(1024) k_gen_orders(int n, int n_succ, uint64_t seed, int64_t first_id,
                                                     int64_t B, const int32_t* __restrict__ pred_ptr,
                                                     const int32_t* __restrict__ succ_ptr,
                                                     const int32_t* __restrict__ succ_idx,
                                                     int32_t* __restrict__ out, int warps_per_block,
                                                     size_t meta_bytes) {
  extern __shared__ __align__(16) unsigned char smem[];
  // CTA-shared graph: initial in-degrees and the successor CSR (each Kahn
  // step reads them on its critical path: shared memory, not L2)
  IdxT* s_indeg0 = reinterpret_cast<IdxT*>(smem);
  IdxT* s_sptr = s_indeg0 + n;          // [n + 1]
  IdxT* s_sidx = s_sptr + (n + 1);      // [n_succ]
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    s_indeg0[v] = (IdxT)(__ldg(pred_ptr + v + 1) - __ldg(pred_ptr + v));
    s_sptr[v] = (IdxT)__ldg(succ_ptr + v);
  }
  if (threadIdx.x == 0) s_sptr[n] = (IdxT)__ldg(succ_ptr + n);
  for (int k = threadIdx.x; k < n_succ; k += blockDim.x) s_sidx[k] = (IdxT)__ldg(succ_idx + k);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = ((size_t(n) * (2 * sizeof(IdxT) + 4)) + 15) & ~size_t(15);
  unsigned char* wbase = smem + meta_bytes + per_warp * warp;
  uint32_t* rk = reinterpret_cast<uint32_t*>(wbase);          // [n] key high words
  IdxT* indeg = reinterpret_cast<IdxT*>(rk + n);                // [n]
  IdxT* ready = indeg + n;                                      // [n]
  const unsigned lt = (1u << lane) - 1;
  const int64_t stride = int64_t(gridDim.x) * warps_per_block;
  for (int64_t c = int64_t(blockIdx.x) * warps_per_block + warp; c < B; c += stride) {
    const uint64_t h = mix64(seed ^ mix64((uint64_t)(first_id + c)));
    int32_t* row = out + c * int64_t(n);
    int nready = 0;
    for (int base = 0; base < n; base += 32) {
      const int v = base + lane;
      int d = 1;
      if (v < n) {
        d = (int)s_indeg0[v];
        indeg[v] = (IdxT)d;
      }
      const bool r = v < n && d == 0;
      const unsigned m = __ballot_sync(0xffffffffu, r);
      if (r) {
        const int slot = nready + __popc(m & lt);
        ready[slot] = (IdxT)v;
        rk[slot] = (uint32_t)(mix64(h ^ (uint64_t)v) >> 32);
      }
      nready += __popc(m);
    }
    __syncwarp();
    int keep = 0;
    int step = 0;
    for (; step < n && nready > 0; ++step) {
      // this lane's best among its strided ready entries (high key word, op)
      uint32_t bk = 0xffffffffu;
      int bv = INT_MAX, bi = -1;
      bool dup = false;  // two of this lane's entries share the best high word
      for (int i = lane; i < nready; i += 32) {
        const uint32_t k = rk[i];
        const int v = (int)ready[i];
        dup = k < bk ? false : (dup || k == bk);
        if (k < bk || (k == bk && v < bv)) {
          bk = k;
          bv = v;
          bi = i;
        }
      }
      const uint32_t mk = __reduce_min_sync(0xffffffffu, bk);
      const unsigned tied = __ballot_sync(0xffffffffu, bi >= 0 && bk == mk);
      const unsigned dups = __ballot_sync(0xffffffffu, bi >= 0 && bk == mk && dup);
      int win;
      if (__popc(tied) == 1 && !dups) {
        win = __ffs(tied) - 1;  // a unique minimal high word decides
      } else {
        // general case: full 64-bit keys of every entry whose high word ties
        uint64_t fk = ~0ull;
        int fv = INT_MAX, fi = -1;
        for (int i = lane; i < nready; i += 32) {
          if (rk[i] != mk) continue;
          const int v = (int)ready[i];
          const uint64_t k = mix64(h ^ (uint64_t)v);
          if (k < fk || (k == fk && v < fv)) {
            fk = k;
            fv = v;
            fi = i;
          }
        }
        const uint32_t mlo = __reduce_min_sync(0xffffffffu, fi >= 0 ? (uint32_t)fk : 0xffffffffu);
        const unsigned t2 = __ballot_sync(0xffffffffu, fi >= 0 && (uint32_t)fk == mlo);
        const int mv = (int)__reduce_min_sync(0xffffffffu, (t2 >> lane) & 1u ? (unsigned)fv : 0xffffffffu);
        const unsigned t3 = __ballot_sync(0xffffffffu, ((t2 >> lane) & 1u) && fv == mv);
        win = __ffs(t3) - 1;
        bv = fv;
        bi = fi;
      }
      const int v = __shfl_sync(0xffffffffu, bv, win);
      const int vi = __shfl_sync(0xffffffffu, bi, win);
      __syncwarp();
      if (lane == 0) {
        ready[vi] = ready[nready - 1];
        rk[vi] = rk[nready - 1];
      }
      --nready;
      if ((step & 31) == lane) keep = v;
      if ((step & 31) == 31) row[step - 31 + lane] = keep;
      const int s0 = (int)s_sptr[v], s1 = (int)s_sptr[v + 1];
      __syncwarp();
      for (int k0 = s0; k0 < s1; k0 += 32) {
        const int k = k0 + lane;
        int w = -1;
        if (k < s1) {
          w = (int)s_sidx[k];
          const int d = (int)indeg[w] - 1;
          indeg[w] = (IdxT)d;
          if (d != 0) w = -1;
        }
        const unsigned m = __ballot_sync(0xffffffffu, w >= 0);
        if (w >= 0) {
          const int slot = nready + __popc(m & lt);
          ready[slot] = (IdxT)w;
          rk[slot] = (uint32_t)(mix64(h ^ (uint64_t)w) >> 32);
        }
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

int launch_gen(RmGraph* g, uint64_t seed, int64_t first_id, int64_t B, int32_t* out, cudaStream_t s) {
  if (B <= 0) return RM_OK;
  const int n = g->n;
  const int n_succ = (int)g->succ_idx.size();
  // u16 ids and successor offsets when both fit
  const bool wide = n > 65535 || n_succ > 65535;
  const size_t isz = wide ? 4 : 2;
  const size_t meta = ((isz * (size_t(n) * 2 + 1 + size_t(n_succ))) + 15) & ~size_t(15);
  const size_t per_warp = ((size_t(n) * (2 * isz + 4)) + 15) & ~size_t(15);
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device);
  if (size_t(max_smem) < meta + per_warp)
    return fail(RM_ERR_CAPACITY, "generator: graph too large for shared memory");
  const int wpb = (int)std::min<size_t>(32, (size_t(max_smem) - meta) / per_warp);
  const size_t smem = meta + per_warp * wpb;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
  const int64_t blocks_needed = (B + wpb - 1) / wpb;
  const int grid = (int)std::min<int64_t>(blocks_needed, int64_t(sms));
  if (wide) {
    RM_CUDA(cudaFuncSetAttribute(k_gen_orders<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    k_gen_orders<int32_t><<<grid, 32 * wpb, smem, s>>>(
        n, n_succ, seed, first_id, B, g->d_pred_ptr.as<int32_t>(), g->d_succ_ptr.as<int32_t>(),
        g->d_succ_idx.as<int32_t>(), out, wpb, meta);
  } else {
    RM_CUDA(cudaFuncSetAttribute(k_gen_orders<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    k_gen_orders<uint16_t><<<grid, 32 * wpb, smem, s>>>(
        n, n_succ, seed, first_id, B, g->d_pred_ptr.as<int32_t>(), g->d_succ_ptr.as<int32_t>(),
        g->d_succ_idx.as<int32_t>(), out, wpb, meta);
  }
  RM_LAUNCH_CHECK("k_gen_orders launch");
  return RM_OK;
}

}  // namespace roam

extern "C" int rm_gen_orders(RmGraph* g, uint64_t seed, int64_t first_id, int64_t B,
                             int32_t* orders_dev, void* stream) {
  using namespace roam;
  if (!g) return fail(RM_ERR_INVALID_ARG, "graph handle is NULL");
  if (g->device < 0) return fail(RM_ERR_NO_DEVICE, "no CUDA device: libroam has no CPU path");
  if (B < 0 || (B > 0 && !orders_dev)) return fail(RM_ERR_INVALID_ARG, "bad rm_gen_orders arguments");
  return launch_gen(g, seed, first_id, B, orders_dev, static_cast<cudaStream_t>(stream));
}
