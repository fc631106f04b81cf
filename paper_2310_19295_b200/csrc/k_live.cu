// Batched live_bytes_by_timestep (reference pkg/src/memplan/graph.py:452-458)
// over sequential schedules: live[c, k] = bytes alive at step k of candidate
// c's order, every tensor alive from its producer's step to the last step of
// any consumer (the horizon n-1 without consumers; tensor_lifetimes,
// graph.py:440-449), plus valid[c] = the row is a permutation respecting every
// direct predecessor (validate_schedule, graph.py:375-398).
//
// The per-position output K1 does not write: max_k live[c, k]
// and its first index are K1's peak / argmax, and a segmented max over a
// window's step range is that window's order peak.  One CTA per candidate
// (grid-stride): the row's inverse permutation in shared memory, each
// tensor's +size / -size events added to a shared delta array by 64-bit
// shared atomics, one block scan writing the n live values.  The output is
// 8 bytes per position against the row's 4: HBM-bound by the write.
#include <algorithm>
#include <climits>

#include "roam_internal.h"

namespace roam {

constexpr int KL_NT = 256;

static int kl_max_smem(int dev) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

template <typename RowT>
__global__ void __launch_bounds__(KL_NT) k_live_batch(int n, int T, int64_t B, const RowT* __restrict__ orders,
                                                      const int32_t* __restrict__ producer,
                                                      const int32_t* __restrict__ cons_ptr,
                                                      const int32_t* __restrict__ cons_idx,
                                                      const int64_t* __restrict__ size,
                                                      const int32_t* __restrict__ pred_ptr,
                                                      const int32_t* __restrict__ pred_idx,
                                                      long long* __restrict__ live, uint8_t* __restrict__ valid) {
  extern __shared__ __align__(16) unsigned char smem[];
  long long* delta = reinterpret_cast<long long*>(smem);               // [n + 1]
  int* pos = reinterpret_cast<int*>(smem + 8 * (size_t(n) + 1));        // [n]
  __shared__ long long wsum[KL_NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t c = blockIdx.x; c < B; c += gridDim.x) {
    const RowT* row = orders + c * int64_t(n);
    for (int k = tid; k < n; k += KL_NT) pos[k] = -1;
    for (int k = tid; k <= n; k += KL_NT) delta[k] = 0;
    __syncthreads();
    int bad = 0;
    for (int k = tid; k < n; k += KL_NT) {
      const long long o = (long long)row[k];
      if (o < 0 || o >= n) bad = 1;
      else if (atomicExch(pos + o, k) != -1) bad = 1;  // a duplicate: some id stays -1
    }
    bad = __syncthreads_or(bad);
    // every direct predecessor strictly earlier (pos -1 = missing id: invalid)
    if (!bad) {
      for (int v = tid; v < n && !bad; v += KL_NT) {
        const int pv = pos[v];
        if (pv < 0) {
          bad = 1;
          break;
        }
        for (int q = pred_ptr[v]; q < pred_ptr[v + 1]; ++q)
          if (pos[pred_idx[q]] >= pv) bad = 1;
      }
    }
    bad = __syncthreads_or(bad);
    const bool ok = !bad;
    if (tid == 0) valid[c] = ok ? 1 : 0;
    if (ok) {
      for (int t = tid; t < T; t += KL_NT) {
        const int b = pos[producer[t]];
        int d = INT_MIN;
        for (int q = cons_ptr[t]; q < cons_ptr[t + 1]; ++q) d = max(d, pos[cons_idx[q]]);
        if (d == INT_MIN) d = n - 1;
        d = max(b, d);
        atomicAdd(reinterpret_cast<unsigned long long*>(delta + b), (unsigned long long)size[t]);
        atomicAdd(reinterpret_cast<unsigned long long*>(delta + d + 1), (unsigned long long)(-size[t]));
      }
    }
    __syncthreads();
    if (ok) {  // blocked inclusive scan: thread t owns steps [t*C, t*C + C)
      const int C = (n + KL_NT - 1) / KL_NT;
      const int k0 = min(n, tid * C), k1 = min(n, k0 + C);
      long long run = 0;
      for (int k = k0; k < k1; ++k) run += delta[k];
      long long incl = run;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const long long x = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += x;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      long long acc = incl - run;
      for (int w = 0; w < warp; ++w) acc += wsum[w];
      long long* out = live + c * int64_t(n);
      for (int k = k0; k < k1; ++k) {
        acc += delta[k];
        __stcs(out + k, acc);  // streamed out once
      }
    }
    __syncthreads();
  }
}

}  // namespace roam

using namespace roam;

extern "C" int rm_eval_live(RmGraph* g, const void* orders, int64_t B, uint32_t flags, int64_t* live,
                            uint8_t* valid, void* stream) {
  if (!g) return fail(RM_ERR_INVALID_ARG, "graph handle is NULL");
  if (B < 0 || (B > 0 && (!orders || !live || !valid))) return fail(RM_ERR_INVALID_ARG, "bad rm_eval_live arguments");
  if (g->device < 0) return fail(RM_ERR_NO_DEVICE, "no CUDA device: libroam has no CPU path");
  const bool u16 = flags & RM_ORDERS_U16;
  if (u16 && g->n > 65535) return fail(RM_ERR_INVALID_ARG, "uint16 rows need n <= 65535");
  const int n = g->n, T = g->T;
  if (B == 0) return RM_OK;
  if (n == 0) {  // the empty schedule is valid and has no steps
    if (flags & RM_DEVICE_PTRS) RM_CUDA(cudaMemsetAsync(valid, 1, size_t(B), static_cast<cudaStream_t>(stream)));
    else std::fill(valid, valid + B, uint8_t(1));
    return RM_OK;
  }
  const size_t smem = 8 * (size_t(n) + 1) + 4 * size_t(n);
  if (smem > size_t(kl_max_smem(g->device)) - 2048)
    return fail(RM_ERR_CAPACITY, "rm_eval_live: graph too large for one CTA's shared memory");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  const void* d_ord = orders;
  long long* d_live = reinterpret_cast<long long*>(live);
  uint8_t* d_val = valid;
  const size_t esz = u16 ? 2 : 4;
  if (!(flags & RM_DEVICE_PTRS)) {
    void* o;
    RM_CUDA(sc.alloc(reinterpret_cast<unsigned char**>(&o), size_t(B) * n * esz));
    RM_CUDA(cudaMemcpyAsync(o, orders, size_t(B) * n * esz, cudaMemcpyHostToDevice, s));
    d_ord = o;
    RM_CUDA(sc.alloc(&d_live, size_t(B) * n));
    RM_CUDA(sc.alloc(&d_val, size_t(B)));
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
  const int per_sm = std::max<int>(1, std::min<int>(8, int(size_t(kl_max_smem(g->device)) / (smem + 2048))));
  const int grid = (int)std::min<int64_t>(B, int64_t(sms) * per_sm);
  if (u16) {
    RM_CUDA(smem_optin(k_live_batch<uint16_t>));
    k_live_batch<uint16_t><<<grid, KL_NT, smem, s>>>(
        n, T, B, static_cast<const uint16_t*>(d_ord), g->d_producer.as<int32_t>(), g->d_cons_ptr.as<int32_t>(),
        g->d_cons_idx.as<int32_t>(), g->d_size.as<int64_t>(), g->d_pred_ptr.as<int32_t>(),
        g->d_pred_idx.as<int32_t>(), d_live, d_val);
  } else {
    RM_CUDA(smem_optin(k_live_batch<int32_t>));
    k_live_batch<int32_t><<<grid, KL_NT, smem, s>>>(
        n, T, B, static_cast<const int32_t*>(d_ord), g->d_producer.as<int32_t>(), g->d_cons_ptr.as<int32_t>(),
        g->d_cons_idx.as<int32_t>(), g->d_size.as<int64_t>(), g->d_pred_ptr.as<int32_t>(),
        g->d_pred_idx.as<int32_t>(), d_live, d_val);
  }
  RM_LAUNCH_CHECK("k_live_batch launch");
  if (!(flags & RM_DEVICE_PTRS)) {
    RM_CUDA(cudaMemcpyAsync(live, d_live, size_t(B) * n * 8, cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaMemcpyAsync(valid, d_val, size_t(B), cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaStreamSynchronize(s));
  }
  return RM_OK;
}
