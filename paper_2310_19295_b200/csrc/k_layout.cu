// K2: pairwise time x address interference over a layout's items
// (layout_violations / repair_conflicts.conflicts / validate_layout /
// replay_static), tiled over the upper triangle of the N x N pair matrix.
//
// Reference: pkg/src/memplan/layout.py:20-29 (inclusive overlap), 305-329
// (layout_violations), 420-429 (conflicts), simulator.py:129-145 (replay_static:
// the actual peak equals max(off + size) over items with offsets, since every
// item is live at its own start).
#include <algorithm>
#include <climits>

#include "roam_internal.h"

namespace roam {

constexpr int K2_TILE = 128;

struct K2Args {
  int64_t N;
  const int32_t* start;
  const int32_t* end;
  const int64_t* size;
  const int64_t* off;
  const uint8_t* has;
  int64_t capacity;
  uint8_t* flags;
  unsigned long long* pairs;  // (i << 32) | j
  unsigned long long cap_pairs;
  unsigned long long* count;
  long long* max_extent;
};

__global__ void k2_items(K2Args a) {
  long long mx = 0;
  bool any = false;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.N;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint8_t f = 0;
    if (!a.has[i]) {
      f = 1;
    } else {
      const long long o = a.off[i], top = o + a.size[i];
      if (o < 0) f |= 2;
      if (top > a.capacity) f |= 4;
      mx = any ? max(mx, top) : top;
      any = true;
    }
    a.flags[i] = f;
  }
  if (any) atomicMax(a.max_extent, mx);
}

// One CTA per (bi <= bj) tile pair; thread r owns row i = bi*T + r and scans
// the j tile staged in shared memory.
__global__ void __launch_bounds__(K2_TILE) k2_pairs(K2Args a, int tiles) {
  __shared__ int sj_s[K2_TILE], sj_e[K2_TILE];
  __shared__ long long sj_lo[K2_TILE], sj_hi[K2_TILE];
  __shared__ unsigned char sj_h[K2_TILE];
  // linear tile id -> (bi, bj) with bi <= bj
  int64_t t = blockIdx.x;
  int bi = 0;
  while (t >= tiles - bi) {
    t -= tiles - bi;
    ++bi;
  }
  const int bj = bi + (int)t;
  const int64_t j0 = int64_t(bj) * K2_TILE;
  const int r = threadIdx.x;
  if (j0 + r < a.N) {
    const int64_t j = j0 + r;
    sj_s[r] = a.start[j];
    sj_e[r] = a.end[j];
    sj_lo[r] = a.off[j];
    sj_hi[r] = a.off[j] + a.size[j];
    sj_h[r] = a.has[j];
  }
  __syncthreads();
  const int64_t i = int64_t(bi) * K2_TILE + r;
  if (i >= a.N || !a.has[i]) return;
  const int is = a.start[i], ie = a.end[i];
  const long long ilo = a.off[i], ihi = ilo + a.size[i];
  const int64_t rem = a.N - j0;
  const int jn = rem < K2_TILE ? (int)rem : K2_TILE;
  const int jbeg = bi == bj ? r + 1 : 0;
  for (int q = jbeg; q < jn; ++q) {
    if (sj_h[q] && is <= sj_e[q] && sj_s[q] <= ie && ilo < sj_hi[q] && sj_lo[q] < ihi) {
      const unsigned long long slot = atomicAdd(a.count, 1ull);
      if (slot < a.cap_pairs)
        a.pairs[slot] = ((unsigned long long)i << 32) | (unsigned long long)(j0 + q);
    }
  }
}

}  // namespace roam

using namespace roam;

extern "C" int rm_layout_violations(int64_t N, const int32_t* start, const int32_t* end,
                                    const int64_t* size, const int64_t* offset,
                                    const uint8_t* has_offset, int64_t capacity,
                                    uint8_t* item_flags, int64_t* pairs, int64_t max_pairs,
                                    int64_t* n_pairs, int64_t* max_extent, void* stream) {
  if (N < 0 || N >= (int64_t(1) << 31) || !n_pairs || !max_extent || max_pairs < 0)
    return fail(RM_ERR_INVALID_ARG, "bad rm_layout_violations arguments");
  if (N > 0 && (!start || !end || !size || !offset || !has_offset || !item_flags))
    return fail(RM_ERR_INVALID_ARG, "NULL item array");
  if (max_pairs > 0 && !pairs) return fail(RM_ERR_INVALID_ARG, "pairs is NULL");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(RM_ERR_NO_DEVICE, "no CUDA device: libroam has no CPU path");
  }
  *n_pairs = 0;
  *max_extent = 0;
  if (N == 0) return RM_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int tiles = (int)((N + K2_TILE - 1) / K2_TILE);
  const int64_t ntile_pairs = int64_t(tiles) * (tiles + 1) / 2;
  unsigned long long cap = (unsigned long long)std::max<int64_t>(max_pairs, 4096);
  for (int attempt = 0; attempt < 2; ++attempt) {
    Scratch sc(s);
    int32_t *d_s, *d_e;
    int64_t *d_sz, *d_off;
    uint8_t *d_has, *d_flags;
    unsigned long long *d_pairs, *d_count;
    long long* d_mx;
    RM_CUDA(sc.alloc(&d_s, size_t(N)));
    RM_CUDA(sc.alloc(&d_e, size_t(N)));
    RM_CUDA(sc.alloc(&d_sz, size_t(N)));
    RM_CUDA(sc.alloc(&d_off, size_t(N)));
    RM_CUDA(sc.alloc(&d_has, size_t(N)));
    RM_CUDA(sc.alloc(&d_flags, size_t(N)));
    RM_CUDA(sc.alloc(&d_pairs, size_t(cap)));
    RM_CUDA(sc.alloc(&d_count, 1));
    RM_CUDA(sc.alloc(&d_mx, 1));
    RM_CUDA(cudaMemcpyAsync(d_s, start, size_t(N) * 4, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaMemcpyAsync(d_e, end, size_t(N) * 4, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaMemcpyAsync(d_sz, size, size_t(N) * 8, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaMemcpyAsync(d_off, offset, size_t(N) * 8, cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaMemcpyAsync(d_has, has_offset, size_t(N), cudaMemcpyHostToDevice, s));
    RM_CUDA(cudaMemsetAsync(d_count, 0, 8, s));
    RM_CUDA(cudaMemsetAsync(d_mx, 0, 8, s));
    K2Args a{N, d_s, d_e, d_sz, d_off, d_has, capacity, d_flags, d_pairs, cap, d_count, d_mx};
    const int ib = (int)std::min<int64_t>(1184, (N + 255) / 256);
    k2_items<<<ib, 256, 0, s>>>(a);
    RM_LAUNCH_CHECK("k2_items");
    k2_pairs<<<(unsigned)ntile_pairs, K2_TILE, 0, s>>>(a, tiles);
    RM_LAUNCH_CHECK("k2_pairs");
    unsigned long long cnt = 0;
    long long mx = 0;
    RM_CUDA(cudaMemcpyAsync(&cnt, d_count, 8, cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaMemcpyAsync(&mx, d_mx, 8, cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaMemcpyAsync(item_flags, d_flags, size_t(N), cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaStreamSynchronize(s));
    *max_extent = mx;
    *n_pairs = (int64_t)cnt;
    if (cnt > cap) {  // buffer too small: rerun once with room for every pair
      cap = cnt;
      continue;
    }
    if (max_pairs > 0 && cnt > 0) {
      std::vector<unsigned long long> h(cnt);
      RM_CUDA(cudaMemcpy(h.data(), d_pairs, size_t(cnt) * 8, cudaMemcpyDeviceToHost));
      std::sort(h.begin(), h.end());  // lexicographic (i, j) = reference emission order
      const int64_t m = std::min<int64_t>((int64_t)cnt, max_pairs);
      for (int64_t k = 0; k < m; ++k) {
        pairs[2 * k] = (int64_t)(h[k] >> 32);
        pairs[2 * k + 1] = (int64_t)(h[k] & 0xffffffffull);
      }
    }
    return RM_OK;
  }
  return fail(RM_ERR_CAPACITY, "pair buffer overflow");
}

