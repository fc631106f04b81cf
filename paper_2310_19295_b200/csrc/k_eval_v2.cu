// K1 v2 / v3: the default candidate-order evaluators (see k_eval.cu for the
// generic one and DESIGN.md section 4 for the design).
//
// Reference: pkg/src/memplan/graph.py:375-468 (validate_schedule,
// sequential_schedule, tensor_lifetimes, live_bytes_by_timestep, peak_memory).
#include "k_common.cuh"

namespace roam {

// ------------------------------------------------------------- K1 v2
// Unit-packed, interleaved evaluator (the default when the graph qualifies,
// see K1V2Meta).  One persistent CTA per SM holds the graph metadata in
// shared memory; G groups of NT threads each evaluate one candidate at a time.
// Candidate rows are near-topological, so ops at consecutive positions have
// nearby ids: per-op gathers run with consecutive positions on consecutive
// lanes (position k = t + j*NT), which keeps them close to conflict-free.
//   P1  pos[o_k] = k (u16) from the row held in registers; range check
//   P2a checked edges pos[u] < pos[v]; per position: readback pos[o_k] == k
//       (permutation), xs[k] = (out units of o_k) << 32 | (single-consumer
//       free units of o_k); then the NEXT candidate's row is loaded into
//       registers (it lands while P2b/P3 run)
//   P2b per multi-consumer tensor: k* = latest position among its maximal
//       consumers; 32-bit shared atomicAdd of its size units into the free
//       field of xs[k*] (the host bounds every position's frees below 2^32)
//   P3  blocked scan over xs (padded, LDS.128): live[k] = sum_{j<k}(out-free)
//       + out_k, running max / first argmax, group scan of chunk totals
struct K1V2Args {
  const void* orders;  // int32 or uint16 rows [B, n]
  int64_t B;
  int n, G;
  int shift;
  const void* opv;  // int2 {fs, out} units per op, zero beyond n
  const uint32_t* edges;
  int n_edges;
  const uint32_t* mpair;
  const uint32_t* mptr;
  const uint16_t* mcons;
  const uint32_t* msz;
  int n_pair, n_gen, n_mcons;
  int64_t* peak;
  int32_t* argmax;
  uint8_t* valid;
  size_t off_edges, off_mpair, off_mptr, off_mcons, off_msz, off_groups, group_bytes, off_xs, off_red;
  int64_t xs_words;  // int64 words of one candidate's xs (v3 keeps two)
  int C;             // v2: rounds of NT positions (ceil(n / NT))
};

// P3 chunk geometry: C3 = MAXC positions per thread (power of two); the
// stride pads each chunk so that (stride / 2) is odd, which keeps the 16-byte
// reads of 8 consecutive threads on distinct bank groups.
template <int MAXC>
struct XsGeom {
  static constexpr int C3 = MAXC;
  static constexpr int C3L = MAXC == 4 ? 2 : MAXC == 8 ? 3 : 4;
  static constexpr int STRIDE = ((MAXC / 2) % 2 == 1) ? MAXC : MAXC + 2;
};

__device__ __forceinline__ unsigned pos_at(const uint16_t* pos, unsigned i) { return pos[i]; }

template <typename RowT, int NT, int MAXC>
__global__ void __launch_bounds__(1024, 1) k1v2_eval_orders(const K1V2Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  // SL = C * NT positions per group (C = ceil(n / NT) <= MAXC rounds of NT):
  // the row plus padding slots; padding slot k holds op id k (zero bytes, its
  // own position), so no slot needs a bounds predicate -- only the round
  // index is tested, against the group-uniform C.  Ids SL and SL+1 have
  // pinned positions 0 and 0xffff and form the dummy edge of the edge loop.
  const int n = a.n;
  const int C = a.C;
  const int SL = C * NT;
  const RowT* orders = static_cast<const RowT*>(a.orders);
  // ---- stage the graph metadata once per CTA
  {
    auto cp16 = [&](const void* g, size_t off, size_t bytes) {
      const uint4* src = static_cast<const uint4*>(g);
      uint4* dst = reinterpret_cast<uint4*>(smem + off);
      for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    };
    cp16(a.opv, 0, align16(8 * size_t(SL)));
    cp16(a.edges, a.off_edges, align16(4 * size_t(a.n_edges)));
    cp16(a.mpair, a.off_mpair, align16(4 * size_t(a.n_pair)));
    cp16(a.mptr, a.off_mptr, align16(4 * size_t(a.n_gen + 1)));
    cp16(a.mcons, a.off_mcons, align16(2 * size_t(a.n_mcons)));
    cp16(a.msz, a.off_msz, align16(4 * size_t(a.n_pair + a.n_gen)));
  }
  __syncthreads();
  const long long* opv = reinterpret_cast<const long long*>(smem);  // fs | out << 32
  const uint32_t* edges = reinterpret_cast<const uint32_t*>(smem + a.off_edges);
  const uint32_t* mpair = reinterpret_cast<const uint32_t*>(smem + a.off_mpair);
  const uint32_t* mptr = reinterpret_cast<const uint32_t*>(smem + a.off_mptr);
  const uint16_t* mcons = reinterpret_cast<const uint16_t*>(smem + a.off_mcons);
  const uint32_t* msz = reinterpret_cast<const uint32_t*>(smem + a.off_msz);

  const int gid = threadIdx.x / NT;
  const int tid = threadIdx.x - gid * NT;
  if (gid >= a.G) return;
  const int bar_id = 1 + gid;
  unsigned char* gbase = smem + a.off_groups + size_t(gid) * a.group_bytes;
  uint16_t* pos = reinterpret_cast<uint16_t*>(gbase);  // [SL + 2]
  long long* xs = reinterpret_cast<long long*>(gbase + a.off_xs);
  long long* red_v = reinterpret_cast<long long*>(gbase + a.off_red);  // [32]
  int* red_i = reinterpret_cast<int*>(red_v + 32);                      // [32]
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NWARPS = NT / 32;
  const int64_t cstride = int64_t(gridDim.x) * a.G;
  // position k lives at xs[(k >> C3L) * STRIDE + (k & (C3-1))]; NT is a
  // multiple of C3, so P2a's slot j is xs_w + j * XS_STEP (compile-time)
  using X = XsGeom<MAXC>;
  constexpr int XS_STEP = (NT / X::C3) * X::STRIDE;
  long long* xs_w = xs + (tid >> X::C3L) * X::STRIDE + (tid & (X::C3 - 1));
  const int n_edges = a.n_edges, n_pair = a.n_pair, n_gen = a.n_gen;
  for (int i = tid; i < SL; i += NT) pos[i] = 0;  // no stale garbage for P2b
  if (tid == 0) {
    pos[SL] = 0;
    pos[SL + 1] = 0xffffu;
  }
  gbar(bar_id, NT);
  const uint32_t dummy_edge = (uint32_t)SL | ((uint32_t)(SL + 1) << 16);

  int32_t v[MAXC];
  // the raw row goes straight into registers; nothing reads it until the
  // next P1, so the loads stay in flight behind P2b / P3
  auto load_row = [&](int64_t cc) {
    const RowT* row = orders + cc * int64_t(n);
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
      const int k = tid + j * NT;
      v[j] = k < n ? (int32_t)__ldcs(row + k) : k;
    }
  };
  int64_t c = int64_t(blockIdx.x) * a.G + gid;
  if (c < a.B) load_row(c);
  for (; c < a.B; c += cstride) {
    unsigned bad = 0;
    // ---- P1: range check (an out-of-range id is clamped so the row stays in
    // bounds, and flagged), scatter positions
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
      if (j < C) {
        const int k = tid + j * NT;
        const unsigned r = (unsigned)v[j];
        bad |= (r >= (unsigned)n) & (k < n);
        v[j] = (int32_t)min(r, (unsigned)(SL - 1));
        pos[v[j]] = (uint16_t)k;
      }
    }
    gbar(bar_id, NT);
    // ---- P2a: checked edges (pv - pu - 1 < 0 marks a violation; OR keeps the sign)
    int edge_acc = 0;
    for (int e0 = tid; e0 < n_edges; e0 += 4 * NT) {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = e0 + i * NT < n_edges ? edges[e0 + i * NT] : dummy_edge;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        edge_acc |= (int)pos_at(pos, w[i] >> 16) - (int)pos_at(pos, w[i] & 0xffffu) - 1;
    }
    // ---- P2a: per position: permutation readback, (single frees, out) units
    unsigned diff = 0;
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
      if (j < C) {
        const int o = v[j];
        diff |= pos_at(pos, o) ^ (unsigned)(tid + j * NT);
        xs_w[j * XS_STEP] = opv[o];
      }
    }
    bad |= (diff != 0) | (edge_acc < 0);
    // prefetch the next candidate's row; it lands while P2b / P3 run
    const int64_t cn = c + cstride;
    if (cn < a.B) load_row(cn);
    gbar(bar_id, NT);
    // ---- P2b: multi-consumer tensors free after their latest maximal consumer
    auto add_free = [&](int kmax, unsigned units) {
      atomicAdd(reinterpret_cast<unsigned*>(xs + (kmax >> X::C3L) * X::STRIDE + (kmax & (X::C3 - 1))),
                units);
    };
    for (int m = tid; m < n_pair; m += NT) {
      const uint32_t w = mpair[m];
      add_free(max((int)pos_at(pos, w & 0xffffu), (int)pos_at(pos, w >> 16)), msz[m]);
    }
    for (int m = tid; m < n_gen; m += NT) {
      const int q0 = mptr[m], q1 = mptr[m + 1];
      int kmax = 0;
      for (int q = q0; q < q1; ++q) kmax = max(kmax, (int)pos_at(pos, mcons[q]));
      add_free(kmax, msz[n_pair + m]);
    }
    gbar(bar_id, NT);
    // ---- P3: blocked scan over this thread's chunk of xs (padding slots
    // carry zero bytes: they never raise the running max); threads past the
    // last chunk hold none
    const int k0 = tid << X::C3L;
    const long long* xr = xs + tid * X::STRIDE;
    long long run = 0, best = LLONG_MIN;
    int bi = INT_MAX;
    if (k0 < SL) {
#pragma unroll
      for (int i = 0; i < X::C3; i += 2) {
        const longlong2 pr = *reinterpret_cast<const longlong2*>(xr + i);
        long long live = run + (long long)((unsigned long long)pr.x >> 32);
        if (live > best) {
          best = live;
          bi = i;
        }
        run = live - (long long)(unsigned)pr.x;
        live = run + (long long)((unsigned long long)pr.y >> 32);
        if (live > best) {
          best = live;
          bi = i + 1;
        }
        run = live - (long long)(unsigned)pr.y;
      }
    }
    const int bestk = bi == INT_MAX ? INT_MAX : k0 + bi;
    long long incl = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane == 31) red_v[warp] = incl;
    bad = gbar_or(bar_id, NT, bad);
    long long off = incl - run;
#pragma unroll
    for (int w = 0; w < NWARPS - 1; ++w)
      if (w < warp) off += red_v[w];
    long long cand = bestk == INT_MAX ? LLONG_MIN : off + best;
    int ck = bestk;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const long long ov = __shfl_down_sync(0xffffffffu, cand, d);
      const int oi = __shfl_down_sync(0xffffffffu, ck, d);
      if (ov > cand || (ov == cand && oi < ck)) {
        cand = ov;
        ck = oi;
      }
    }
    gbar(bar_id, NT);
    if (lane == 0) {
      red_v[warp] = cand;
      red_i[warp] = ck;
    }
    gbar(bar_id, NT);
    if (tid == 0) {
      long long bv = red_v[0];
      int bk = red_i[0];
#pragma unroll
      for (int w = 1; w < NWARPS; ++w)
        if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bk)) {
          bv = red_v[w];
          bk = red_i[w];
        }
      if (n == 0) {
        bv = 0;
        bk = 0;
      }
      a.peak[c] = (int64_t)bv << a.shift;
      a.argmax[c] = bk;
      a.valid[c] = bad ? 0 : 1;
    }
  }
}

// ------------------------------------------------------------- K1 v3
// Two candidates per group (the default when n < 32767): positions of the
// pair (A, B) share one 32-bit word per op (A in the low, B in the high
// half), so every edge check and every multi-consumer lookup is ONE gather
// for both candidates and the two comparisons run as one SIMD-within-a-word
// subtraction: with positions < 2^15,
//   ((pv | 0x80008000) - pu - 0x00010001) keeps bit 15 / bit 31 set
// exactly when pv > pu in the low / high half (no borrow crosses halves).
// Per-position work (scatter, readback, out/free units, blocked scan) stays
// per candidate; barriers and the group scan are shared by the pair.
template <typename RowT, int NT, int MAXC>
__global__ void __launch_bounds__(1024, 1) k1v3_eval_orders(const K1V2Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n;
  const RowT* orders = static_cast<const RowT*>(a.orders);
  {
    auto cp16 = [&](const void* g, size_t off, size_t bytes) {
      const uint4* src = static_cast<const uint4*>(g);
      uint4* dst = reinterpret_cast<uint4*>(smem + off);
      for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    };
    cp16(a.opv, 0, align16(8 * size_t(n + 1)));
    cp16(a.edges, a.off_edges, align16(4 * size_t(a.n_edges)));
    cp16(a.mpair, a.off_mpair, align16(4 * size_t(a.n_pair)));
    cp16(a.mptr, a.off_mptr, align16(4 * size_t(a.n_gen + 1)));
    cp16(a.mcons, a.off_mcons, align16(2 * size_t(a.n_mcons)));
    cp16(a.msz, a.off_msz, align16(4 * size_t(a.n_pair + a.n_gen)));
  }
  __syncthreads();
  const long long* opv = reinterpret_cast<const long long*>(smem);  // fs | out << 32
  const uint32_t* edges = reinterpret_cast<const uint32_t*>(smem + a.off_edges);
  const uint32_t* mpair = reinterpret_cast<const uint32_t*>(smem + a.off_mpair);
  const uint32_t* mptr = reinterpret_cast<const uint32_t*>(smem + a.off_mptr);
  const uint16_t* mcons = reinterpret_cast<const uint16_t*>(smem + a.off_mcons);
  const uint32_t* msz = reinterpret_cast<const uint32_t*>(smem + a.off_msz);

  const int gid = threadIdx.x / NT;
  const int tid = threadIdx.x - gid * NT;
  if (gid >= a.G) return;
  const int D = n;
  const int bar_id = 1 + gid;
  using X = XsGeom<MAXC>;
  constexpr int XS_STEP = (NT / X::C3) * X::STRIDE;
  constexpr int NWARPS = NT / 32;
  unsigned char* gbase = smem + a.off_groups + size_t(gid) * a.group_bytes;
  uint32_t* pos2 = reinterpret_cast<uint32_t*>(gbase);        // [n + 3] (A | B << 16)
  uint16_t* posh = reinterpret_cast<uint16_t*>(gbase);        // halves: 2*o (A), 2*o+1 (B)
  long long* xsA = reinterpret_cast<long long*>(gbase + a.off_xs);
  long long* xsB = xsA + size_t(a.xs_words);
  long long* red_v = reinterpret_cast<long long*>(gbase + a.off_red);  // [2 * NWARPS]
  int* red_i = reinterpret_cast<int*>(red_v + 2 * NWARPS);              // [2 * NWARPS]
  unsigned* red_f = reinterpret_cast<unsigned*>(red_i + 2 * NWARPS);    // [NWARPS]
  const int lane = tid & 31, warp = tid >> 5;
  const int xw_off = (tid >> X::C3L) * X::STRIDE + (tid & (X::C3 - 1));
  const int n_edges = a.n_edges, n_pair = a.n_pair, n_gen = a.n_gen;
  for (int i = tid; i < n; i += NT) pos2[i] = 0;
  if (tid == 0) {
    pos2[D + 1] = 0;            // dummy edge (D+1 -> D+2) of the predicated loop
    pos2[D + 2] = 0x7fff7fffu;  // always passes in both halves
  }
  gbar(bar_id, NT);
  const uint32_t dummy_edge = (uint32_t)(D + 1) | ((uint32_t)(D + 2) << 16);

  const int64_t npairs = (a.B + 1) / 2;
  const int64_t pstride = int64_t(gridDim.x) * a.G;
  uint32_t v[MAXC];
  unsigned pend = 0;  // out-of-range ids seen while loading: bit0 A, bit1 B
  auto load_pair = [&](int64_t pp) {
    const int64_t cA = 2 * pp, cB = cA + 1 < a.B ? cA + 1 : cA;
    const RowT* rA = orders + cA * int64_t(n);
    const RowT* rB = orders + cB * int64_t(n);
    pend = 0;
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
      const int k = tid + j * NT;
      uint32_t oa = D, ob = D;
      if (k < n) {
        const int32_t ra = (int32_t)__ldcs(rA + k), rb = (int32_t)__ldcs(rB + k);
        const bool ba = (unsigned)ra >= (unsigned)n, bb = (unsigned)rb >= (unsigned)n;
        pend |= (unsigned)ba | ((unsigned)bb << 1);
        oa = ba ? D : ra;
        ob = bb ? D : rb;
      }
      v[j] = oa | (ob << 16);
    }
  };
  int64_t pp = int64_t(blockIdx.x) * a.G + gid;
  if (pp < npairs) load_pair(pp);
  for (; pp < npairs; pp += pstride) {
    unsigned bad = pend;
    // ---- P1: scatter both candidates' positions
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
      const int k = tid + j * NT;
      posh[2 * (v[j] & 0xffffu)] = (uint16_t)k;
      posh[2 * (v[j] >> 16) + 1] = (uint16_t)k;
    }
    gbar(bar_id, NT);
    // ---- P2a: checked edges for both candidates at once
    uint32_t ok = 0xffffffffu;
    for (int e0 = tid; e0 < n_edges; e0 += 4 * NT) {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = e0 + i * NT < n_edges ? edges[e0 + i * NT] : dummy_edge;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        ok &= (pos2[w[i] >> 16] | 0x80008000u) - pos2[w[i] & 0xffffu] - 0x00010001u;
    }
    bad |= ((~ok >> 15) & 1u) | ((~ok >> 30) & 2u);
    // ---- P2a: per position: readback, (out, single frees) for A and B
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
      const int k = tid + j * NT;
      const unsigned oa = v[j] & 0xffffu, ob = v[j] >> 16;
      if (k < n) {
        bad |= ((unsigned)posh[2 * oa] != (unsigned)k) | (((unsigned)posh[2 * ob + 1] != (unsigned)k) << 1);
        xsA[xw_off + j * XS_STEP] = opv[oa];  // fs | out << 32
        xsB[xw_off + j * XS_STEP] = opv[ob];
      }
    }
    const int64_t pn = pp + pstride;
    const int64_t cA = 2 * pp;
    const bool hasB = cA + 1 < a.B;
    if (pn < npairs) load_pair(pn);
    gbar(bar_id, NT);
    // ---- P2b: multi-consumer tensors, both candidates per gather
    auto add_free = [&](long long* xs, unsigned kmax, unsigned units) {
      if ((int)kmax < n)
        atomicAdd(reinterpret_cast<unsigned*>(xs + (kmax >> X::C3L) * X::STRIDE + (kmax & (X::C3 - 1))),
                  units);
    };
    for (int m = tid; m < n_pair; m += NT) {
      const uint32_t w = mpair[m];
      const uint32_t p1 = pos2[w & 0xffffu], p2 = pos2[w >> 16];
      const unsigned u = msz[m];
      add_free(xsA, max(p1 & 0xffffu, p2 & 0xffffu), u);
      add_free(xsB, max(p1 >> 16, p2 >> 16), u);
    }
    for (int m = tid; m < n_gen; m += NT) {
      const int q0 = mptr[m], q1 = mptr[m + 1];
      unsigned ka = 0, kb = 0;
      for (int q = q0; q < q1; ++q) {
        const uint32_t pq = pos2[mcons[q]];
        ka = max(ka, pq & 0xffffu);
        kb = max(kb, pq >> 16);
      }
      const unsigned u = msz[n_pair + m];
      add_free(xsA, ka, u);
      add_free(xsB, kb, u);
    }
    gbar(bar_id, NT);
    // ---- P3: blocked scans of both candidates' chunks
    const int k0 = tid << X::C3L;
    const int mc = n - k0;
    const long long* xa = xsA + tid * X::STRIDE;
    const long long* xb = xsB + tid * X::STRIDE;
    long long runA = 0, bestA = LLONG_MIN, runB = 0, bestB = LLONG_MIN;
    int biA = INT_MAX, biB = INT_MAX;
#pragma unroll
    for (int i = 0; i < X::C3; i += 2) {
      if (i < mc) {
        const longlong2 pa = *reinterpret_cast<const longlong2*>(xa + i);
        const longlong2 pb = *reinterpret_cast<const longlong2*>(xb + i);
        long long la = runA + (long long)((unsigned long long)pa.x >> 32);
        long long lb = runB + (long long)((unsigned long long)pb.x >> 32);
        if (la > bestA) { bestA = la; biA = i; }
        if (lb > bestB) { bestB = lb; biB = i; }
        runA = la - (long long)(unsigned)pa.x;
        runB = lb - (long long)(unsigned)pb.x;
        if (i + 1 < mc) {
          la = runA + (long long)((unsigned long long)pa.y >> 32);
          lb = runB + (long long)((unsigned long long)pb.y >> 32);
          if (la > bestA) { bestA = la; biA = i + 1; }
          if (lb > bestB) { bestB = lb; biB = i + 1; }
          runA = la - (long long)(unsigned)pa.y;
          runB = lb - (long long)(unsigned)pb.y;
        }
      }
    }
    long long incA = runA, incB = runB;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long ta = __shfl_up_sync(0xffffffffu, incA, d);
      const long long tb = __shfl_up_sync(0xffffffffu, incB, d);
      if (lane >= d) {
        incA += ta;
        incB += tb;
      }
    }
    const unsigned wbad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 31) {
      red_v[warp] = incA;
      red_v[NWARPS + warp] = incB;
    }
    if (lane == 0) red_f[warp] = wbad;
    gbar(bar_id, NT);
    long long offA = incA - runA, offB = incB - runB;
    unsigned gbad = 0;
#pragma unroll
    for (int w = 0; w < NWARPS; ++w) {
      if (w < warp) {
        offA += red_v[w];
        offB += red_v[NWARPS + w];
      }
      gbad |= red_f[w];
    }
    long long candA = biA == INT_MAX ? LLONG_MIN : offA + bestA;
    long long candB = biB == INT_MAX ? LLONG_MIN : offB + bestB;
    int ckA = biA == INT_MAX ? INT_MAX : k0 + biA;
    int ckB = biB == INT_MAX ? INT_MAX : k0 + biB;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const long long oa = __shfl_down_sync(0xffffffffu, candA, d);
      const int ia = __shfl_down_sync(0xffffffffu, ckA, d);
      const long long ob = __shfl_down_sync(0xffffffffu, candB, d);
      const int ib = __shfl_down_sync(0xffffffffu, ckB, d);
      if (oa > candA || (oa == candA && ia < ckA)) {
        candA = oa;
        ckA = ia;
      }
      if (ob > candB || (ob == candB && ib < ckB)) {
        candB = ob;
        ckB = ib;
      }
    }
    gbar(bar_id, NT);
    if (lane == 0) {
      red_v[warp] = candA;
      red_i[warp] = ckA;
      red_v[NWARPS + warp] = candB;
      red_i[NWARPS + warp] = ckB;
    }
    gbar(bar_id, NT);
    if (tid < 2 && (tid == 0 || hasB)) {
      const int base = tid * NWARPS;
      long long bv = red_v[base];
      int bk = red_i[base];
#pragma unroll
      for (int w = 1; w < NWARPS; ++w)
        if (red_v[base + w] > bv || (red_v[base + w] == bv && red_i[base + w] < bk)) {
          bv = red_v[base + w];
          bk = red_i[base + w];
        }
      if (n == 0) {
        bv = 0;
        bk = 0;
      }
      const int64_t c = cA + tid;
      a.peak[c] = (int64_t)bv << a.shift;
      a.argmax[c] = bk;
      a.valid[c] = ((gbad >> tid) & 1u) ? 0 : 1;
    }
  }
}

template <bool PAIRS, typename RowT, int NT, int MAXC>
static int launch_k1v2_t(K1V2Args& a, int grid, size_t smem, cudaStream_t s) {
  auto kern = PAIRS ? k1v3_eval_orders<RowT, NT, MAXC> : k1v2_eval_orders<RowT, NT, MAXC>;
  RM_CUDA(smem_optin(kern));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  kern<<<grid, NT * a.G, smem, s>>>(a);
  RM_LAUNCH_CHECK(PAIRS ? "k1v3_eval_orders launch" : "k1v2_eval_orders launch");
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

template <bool PAIRS, typename RowT>
static int launch_k1v2_nt(K1V2Args& a, int NT, int MAXC, int grid, size_t smem, cudaStream_t s) {
#define RM_K1V2_CASE(nt, mc) \
  if (NT == nt && MAXC == mc) return launch_k1v2_t<PAIRS, RowT, nt, mc>(a, grid, smem, s);
  RM_K1V2_CASE(64, 4)
  RM_K1V2_CASE(64, 8)
  RM_K1V2_CASE(64, 16)
  RM_K1V2_CASE(128, 8)
  RM_K1V2_CASE(128, 16)
  RM_K1V2_CASE(256, 8)
  RM_K1V2_CASE(256, 16)
  RM_K1V2_CASE(512, 8)
  RM_K1V2_CASE(512, 16)
  RM_K1V2_CASE(1024, 8)
  RM_K1V2_CASE(1024, 16)
#undef RM_K1V2_CASE
  return 1;
}

// K1 v2/v3 geometry: NT threads per group (<= 16 positions per thread in
// P1/P2), as many groups per CTA as shared memory allows (<= 15 named
// barriers).  v3 (pairs) evaluates two candidates per group.  Returns 1 when
// the graph does not fit the layout (caller falls back).
int launch_k1v2(RmGraph* g, const void* orders_dev, int64_t B, int64_t* peak, int32_t* argmax,
                uint8_t* valid, cudaStream_t s, bool pairs, bool u16_rows) {
  const int n = g->n;
  if (pairs && n > 32766) return 1;  // 15-bit positions for the SIMD compare
  K1V2Args a{};
  a.orders = orders_dev;
  a.B = B;
  a.n = n;
  a.shift = g->k2v.shift;
  a.opv = g->k2v.opv.p;
  a.edges = g->k2v.edges.as<uint32_t>();
  a.n_edges = (int)g->info.n_check_edges;
  a.mpair = g->k2v.mpair.as<uint32_t>();
  a.mptr = g->k2v.mptr.as<uint32_t>();
  a.mcons = g->k2v.mcons.as<uint16_t>();
  a.msz = g->k2v.msz.as<uint32_t>();
  a.n_pair = (int)g->k2v.n_pair;
  a.n_gen = (int)g->k2v.n_gen;
  a.n_mcons = (int)g->k2v.n_mcons;
  a.peak = peak;
  a.argmax = argmax;
  a.valid = valid;
  int dev = g->device;
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // <= 16 positions per thread (v2) or <= 8 (v3: a pair's two scans keep
  // twice the state, and twice the threads per group restores occupancy)
  const int per = pairs ? 8 : 16;
  int best_nt = 64;
  while (best_nt < 1024 && best_nt * per < n) best_nt *= 2;
  const int NT = best_nt;
  const int C = std::max(1, (n + NT - 1) / NT);
  const int MAXC = C <= 4 && NT == 64 ? 4 : C <= 8 ? 8 : 16;
  const int C3 = MAXC;
  const int stride = ((C3 / 2) % 2 == 1) ? C3 : C3 + 2;  // XsGeom<MAXC>::STRIDE
  if (C > 16) return 1;  // > 16384 ops: the generic evaluator
  a.C = C;
  const size_t slots = size_t(NT) * C;  // v2: row + padding slots (padding slot k = op id k)
  a.off_edges = align16(8 * (pairs ? size_t(n + 1) : slots));
  a.off_mpair = align16(a.off_edges + 4 * size_t(a.n_edges));
  a.off_mptr = align16(a.off_mpair + 4 * size_t(a.n_pair));
  a.off_mcons = align16(a.off_mptr + 4 * size_t(a.n_gen + 1));
  a.off_msz = align16(a.off_mcons + 2 * size_t(a.n_mcons));
  a.off_groups = align16(a.off_msz + 4 * size_t(a.n_pair + a.n_gen));
  a.xs_words = int64_t(pairs ? (n + C3 - 1) / C3 : (slots + C3 - 1) / C3) * stride;
  a.off_xs = align16(pairs ? 4 * size_t(n + 3) : 2 * (slots + 2));
  a.off_red = align16(a.off_xs + 8 * size_t(a.xs_words) * (pairs ? 2 : 1));
  a.group_bytes = align16(a.off_red + 64 * 8 + 64 * 4 + 32 * 4);
  const size_t avail = max_smem > (int)a.off_groups ? size_t(max_smem) - a.off_groups : 0;
  int G = (int)(avail / a.group_bytes);
  G = std::min(G, 1024 / NT);
  G = std::min(G, 15);
  if (G < 1) return 1;
  const int64_t sms = k1_sms(dev);
  const int64_t units = pairs ? (B + 1) / 2 : B;  // what one group evaluates at a time
  if (int64_t(G) * sms > units) G = (int)std::max<int64_t>(1, (units + sms - 1) / sms);
  a.G = G;
  const size_t smem = a.off_groups + size_t(G) * a.group_bytes;
  const int grid = (int)std::min<int64_t>(sms, (units + G - 1) / G);
  if (u16_rows)
    return pairs ? launch_k1v2_nt<true, uint16_t>(a, NT, MAXC, grid, smem, s)
                 : launch_k1v2_nt<false, uint16_t>(a, NT, MAXC, grid, smem, s);
  return pairs ? launch_k1v2_nt<true, int32_t>(a, NT, MAXC, grid, smem, s)
               : launch_k1v2_nt<false, int32_t>(a, NT, MAXC, grid, smem, s);
}

}  // namespace roam
