// Device and host helpers shared by the K1 translation units.
#pragma once

#include <algorithm>
#include <climits>

#include "roam_internal.h"

namespace roam {

extern thread_local bool g_timing;     // rm_set_timing
extern thread_local int g_sm_reserve;  // rm_set_sm_reserve: SMs K1 leaves free (this thread's calls)
extern thread_local double g_last_ms;  // rm_last_kernel_ms

__device__ __forceinline__ void gbar(int id, int nt) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nt) : "memory");
}
__device__ __forceinline__ int gbar_or(int id, int nt, int pred) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.s32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\t"
      "selp.s32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(pred), "r"(id), "r"(nt)
      : "memory");
  return r;
}

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

inline int sm_count(int dev) {
  static int cached[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int c = 0;
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = c > 0 ? c : 148;
  }
  return cached[dev];
}



// SMs the persistent K1 grids use: all but rm_set_sm_reserve()'s count, so a
// collective launched on another stream finds an idle SM while K1 runs
inline int64_t k1_sms(int dev) { return std::max<int64_t>(1, sm_count(dev) - g_sm_reserve); }

// K1 v4 (k_eval_v4.cu): returns 1 when g->k4v.ok == 0 (the caller falls
// back to the generic evaluator).  u16_rows: orders are uint16[B, n] instead
// of int32[B, n].
// Fused selection: K1 v4 also reduces the packed key (peak << id_bits) |
// (id_base + c) of the first strict minimum over valid candidates into
// *key_out (INT64_MAX when none is valid), via per-group partials and a
// last-group reduction; partial / counter are per-thread scratch (counter
// zero between launches, reset by the last group).
struct K1KeySel {
  int64_t* key_out;
  long long* partial;
  unsigned* counter;
  int64_t id_base;
  int id_bits;
};
int launch_k1v4(RmGraph* g, const void* orders_dev, int64_t B, int64_t* peak, int32_t* argmax,
                uint8_t* valid, cudaStream_t s, bool u16_rows, const K1KeySel* sel = nullptr);

// K1 v5 (k_eval_v5.cu): same contract; returns 1 when g->k5v.ok == 0.
// bulk_rows: stage rows with cp.async.bulk instead of the register prefetch.
int launch_k1v5(RmGraph* g, const void* orders_dev, int64_t B, int64_t* peak, int32_t* argmax,
                uint8_t* valid, cudaStream_t s, bool u16_rows, const K1KeySel* sel = nullptr,
                bool bulk_rows = false);

}  // namespace roam
