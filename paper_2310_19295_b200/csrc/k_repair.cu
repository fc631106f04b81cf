// repair_conflicts (reference pkg/src/memplan/layout.py:409-470) in libroam:
// conflict detection and mover election on the device (K2's tiled pair test,
// items resident for every round), mover placement in host C++.
//
// Per round the reference (1) lists every conflicting pair of items sorted by
// tensor id (layout.py:420-429), (2) elects one mover per pair -- the
// non-activation side, else the smaller (size, lifetime, -tensor)
// (layout.py:431-436) -- and (3) re-places the distinct movers in
// (size, lifetime, tensor) order, each into the smallest free gap of its
// lifetime that fits (the lowest such gap on ties: strict <), or on top of
// everything it overlaps in time (layout.py:438-467), growing capacity.
// At most N + 1 rounds, then a final check (layout.py:468-469).
//
// Only the mover SET matters for (3), so the device writes one flag per
// elected item instead of materialising the pairs: the round's D2H traffic is
// N bytes plus a counter, its H2D traffic the N offsets the host moved.
#include <algorithm>
#include <vector>

#include "roam_internal.h"

namespace roam {

constexpr int KR_TILE = 128;

struct KRArgs {
  int64_t N;
  const int32_t* start;
  const int32_t* end;
  const int64_t* size;
  const int64_t* tensor;
  const uint8_t* is_act;
  const int64_t* off;
  uint8_t* mover;                 // [N] 1 = elected by some conflicting pair
  unsigned long long* count;      // conflicting pairs this round
};

// mover(a, b), layout.py:431-436: a and b are item indices
__device__ __forceinline__ int64_t kr_elect(const KRArgs& a, int64_t i, int64_t j) {
  const uint8_t ai = a.is_act[i], aj = a.is_act[j];
  if (ai != aj) return ai ? j : i;
  const int64_t si = a.size[i], sj = a.size[j];
  if (si != sj) return si < sj ? i : j;
  const int64_t di = int64_t(a.end[i]) - a.start[i], dj = int64_t(a.end[j]) - a.start[j];
  if (di != dj) return di < dj ? i : j;
  return -a.tensor[i] < -a.tensor[j] ? i : j;
}

// One CTA per (bi <= bj) tile pair of the upper triangle; thread r owns row
// i = bi * T + r against the staged j tile (the k2_pairs geometry).
__global__ void __launch_bounds__(KR_TILE) kr_movers(KRArgs a, int tiles) {
  __shared__ int sj_s[KR_TILE], sj_e[KR_TILE];
  __shared__ long long sj_lo[KR_TILE], sj_hi[KR_TILE];
  int64_t t = blockIdx.x;
  int bi = 0;
  while (t >= tiles - bi) {
    t -= tiles - bi;
    ++bi;
  }
  const int bj = bi + (int)t;
  const int64_t j0 = int64_t(bj) * KR_TILE;
  const int r = threadIdx.x;
  if (j0 + r < a.N) {
    const int64_t j = j0 + r;
    sj_s[r] = a.start[j];
    sj_e[r] = a.end[j];
    sj_lo[r] = a.off[j];
    sj_hi[r] = a.off[j] + a.size[j];
  }
  __syncthreads();
  const int64_t i = int64_t(bi) * KR_TILE + r;
  if (i >= a.N) return;
  const int is = a.start[i], ie = a.end[i];
  const long long ilo = a.off[i], ihi = ilo + a.size[i];
  const int64_t rem = a.N - j0;
  const int jn = rem < KR_TILE ? (int)rem : KR_TILE;
  unsigned hits = 0;
  for (int q = bi == bj ? r + 1 : 0; q < jn; ++q) {
    if (is <= sj_e[q] && sj_s[q] <= ie && ilo < sj_hi[q] && sj_lo[q] < ihi) {
      a.mover[kr_elect(a, i, j0 + q)] = 1;  // idempotent: any writer wins
      ++hits;
    }
  }
  if (hits) atomicAdd(a.count, (unsigned long long)hits);
}

// Step (3) for one round's movers, in order, on host copies of the offsets
// (layout.py:445-467).  Items overlapping the mover in time (inclusive
// lifetimes, layout.py:28-29) and holding an offset give the occupied spans
// [off, off + size) sorted by (lo, hi); gaps open wherever a span starts
// above the running top edge.
static void place_movers(int64_t N, const int32_t* start, const int32_t* end, const int64_t* size,
                         const uint8_t* has, int64_t* off, int64_t* capacity,
                         const std::vector<int64_t>& movers) {
  std::vector<std::pair<int64_t, int64_t>> spans;
  spans.reserve(size_t(N));
  int64_t cap = *capacity;
  for (const int64_t m : movers) {
    spans.clear();
    const int32_t ms = start[m], me = end[m];
    for (int64_t o = 0; o < N; ++o)
      if (o != m && has[o] && start[o] <= me && ms <= end[o]) spans.emplace_back(off[o], off[o] + size[o]);
    std::sort(spans.begin(), spans.end());
    int64_t edge = 0, best_w = -1, best_lo = 0;
    auto gap = [&](int64_t lo, int64_t hi) {
      const int64_t w = hi - lo;
      if (w >= size[m] && (best_w < 0 || w < best_w)) {
        best_w = w;
        best_lo = lo;
      }
    };
    for (const auto& sp : spans) {
      if (sp.first > edge) gap(edge, sp.first);
      edge = std::max(edge, sp.second);
    }
    if (cap > edge) gap(edge, cap);
    const int64_t at = best_w >= 0 ? best_lo : edge;
    off[m] = at;
    cap = std::max(cap, at + size[m]);
  }
  *capacity = cap;
}

}  // namespace roam

using namespace roam;

extern "C" int rm_repair_place(int64_t N, const int32_t* start, const int32_t* end, const int64_t* size,
                               const uint8_t* has_offset, int64_t* offset, int64_t* capacity,
                               int64_t n_movers, const int64_t* movers) {
  if (N < 0 || n_movers < 0 || !capacity || (N > 0 && (!start || !end || !size || !has_offset || !offset)) ||
      (n_movers > 0 && !movers))
    return fail(RM_ERR_INVALID_ARG, "bad rm_repair_place arguments");
  std::vector<int64_t> mv(movers, movers + n_movers);
  for (const int64_t m : mv)
    if (m < 0 || m >= N) return fail(RM_ERR_INVALID_ARG, "mover index out of range");
  place_movers(N, start, end, size, has_offset, offset, capacity, mv);
  return RM_OK;
}

extern "C" int rm_repair_conflicts(int64_t N, const int64_t* tensor, const int32_t* start,
                                   const int32_t* end, const int64_t* size, const uint8_t* is_act,
                                   int64_t* offset, int64_t* capacity, int32_t* rounds,
                                   void* stream) {
  if (N < 0 || N >= (int64_t(1) << 31) || !capacity || !rounds ||
      (N > 0 && (!tensor || !start || !end || !size || !is_act || !offset)))
    return fail(RM_ERR_INVALID_ARG, "bad rm_repair_conflicts arguments");
  *rounds = 0;
  if (N < 2) return RM_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(RM_ERR_NO_DEVICE, "no CUDA device: libroam has no CPU path");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  int32_t *d_s, *d_e;
  int64_t *d_sz, *d_t, *d_off;
  uint8_t *d_act, *d_mv;
  unsigned long long* d_cnt;
  RM_CUDA(sc.alloc(&d_s, size_t(N)));
  RM_CUDA(sc.alloc(&d_e, size_t(N)));
  RM_CUDA(sc.alloc(&d_sz, size_t(N)));
  RM_CUDA(sc.alloc(&d_t, size_t(N)));
  RM_CUDA(sc.alloc(&d_off, size_t(N)));
  RM_CUDA(sc.alloc(&d_act, size_t(N)));
  RM_CUDA(sc.alloc(&d_mv, size_t(N)));
  RM_CUDA(sc.alloc(&d_cnt, 1));
  RM_CUDA(cudaMemcpyAsync(d_s, start, size_t(N) * 4, cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaMemcpyAsync(d_e, end, size_t(N) * 4, cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaMemcpyAsync(d_sz, size, size_t(N) * 8, cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaMemcpyAsync(d_t, tensor, size_t(N) * 8, cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaMemcpyAsync(d_off, offset, size_t(N) * 8, cudaMemcpyHostToDevice, s));
  RM_CUDA(cudaMemcpyAsync(d_act, is_act, size_t(N), cudaMemcpyHostToDevice, s));
  const int tiles = (int)((N + KR_TILE - 1) / KR_TILE);
  const int64_t ntile = int64_t(tiles) * (tiles + 1) / 2;
  KRArgs a{N, d_s, d_e, d_sz, d_t, d_act, d_off, d_mv, d_cnt};
  std::vector<uint8_t> flag((size_t)N);
  std::vector<uint8_t> has((size_t)N, 1);
  std::vector<int64_t> movers;
  // one detection pass: the mover flags and the pair count of the current offsets
  auto detect = [&](unsigned long long& cnt) -> int {
    RM_CUDA(cudaMemsetAsync(d_mv, 0, size_t(N), s));
    RM_CUDA(cudaMemsetAsync(d_cnt, 0, 8, s));
    kr_movers<<<(unsigned)ntile, KR_TILE, 0, s>>>(a, tiles);
    RM_LAUNCH_CHECK("kr_movers");
    RM_CUDA(cudaMemcpyAsync(&cnt, d_cnt, 8, cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaMemcpyAsync(flag.data(), d_mv, size_t(N), cudaMemcpyDeviceToHost, s));
    RM_CUDA(cudaStreamSynchronize(s));
    return RM_OK;
  };
  unsigned long long cnt = 0;
  for (int64_t round = 0; round <= N; ++round) {
    int rc = detect(cnt);
    if (rc != RM_OK) return rc;
    if (cnt == 0) return RM_OK;
    movers.clear();
    for (int64_t i = 0; i < N; ++i)
      if (flag[size_t(i)]) movers.push_back(i);
    std::sort(movers.begin(), movers.end(), [&](int64_t x, int64_t y) {
      if (size[x] != size[y]) return size[x] < size[y];
      const int64_t dx = int64_t(end[x]) - start[x], dy = int64_t(end[y]) - start[y];
      if (dx != dy) return dx < dy;
      return tensor[x] < tensor[y];
    });
    place_movers(N, start, end, size, has.data(), offset, capacity, movers);
    *rounds = (int32_t)(round + 1);
    RM_CUDA(cudaMemcpyAsync(d_off, offset, size_t(N) * 8, cudaMemcpyHostToDevice, s));
  }
  int rc = detect(cnt);
  if (rc != RM_OK) return rc;
  if (cnt != 0) return fail(RM_ERR_GRAPH, "conflict repair did not converge");
  return RM_OK;
}
