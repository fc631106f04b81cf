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

template <class IdxT>
__global__ void __launch_bounds__(256) k_gen_orders(int n, uint64_t seed, int64_t first_id, int64_t B,
                                                    const int32_t* __restrict__ pred_ptr,
                                                    const int32_t* __restrict__ succ_ptr,
                                                    const int32_t* __restrict__ succ_idx,
                                                    int32_t* __restrict__ out, int warps_per_block) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = ((2 * size_t(n) * sizeof(IdxT)) + 15) & ~size_t(15);
  IdxT* indeg = reinterpret_cast<IdxT*>(smem + per_warp * warp);
  IdxT* ready = indeg + n;
  const int64_t stride = int64_t(gridDim.x) * warps_per_block;
  for (int64_t c = int64_t(blockIdx.x) * warps_per_block + warp; c < B; c += stride) {
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

int launch_gen(RmGraph* g, uint64_t seed, int64_t first_id, int64_t B, int32_t* out, cudaStream_t s) {
  if (B <= 0) return RM_OK;
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
  const int grid = (int)std::min<int64_t>(blocks_needed, int64_t(sms) * 8);
  if (wide) {
    RM_CUDA(smem_optin(k_gen_orders<int32_t>));
    k_gen_orders<int32_t><<<grid, 32 * wpb, smem, s>>>(
        n, seed, first_id, B, g->d_pred_ptr.as<int32_t>(), g->d_succ_ptr.as<int32_t>(),
        g->d_succ_idx.as<int32_t>(), out, wpb);
  } else {
    RM_CUDA(smem_optin(k_gen_orders<uint16_t>));
    k_gen_orders<uint16_t><<<grid, 32 * wpb, smem, s>>>(
        n, seed, first_id, B, g->d_pred_ptr.as<int32_t>(), g->d_succ_ptr.as<int32_t>(),
        g->d_succ_idx.as<int32_t>(), out, wpb);
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
