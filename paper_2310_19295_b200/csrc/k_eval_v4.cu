// K1 v4: the candidate-order evaluator for unit-packed graphs whose classes
// do not fit v5's one-byte form (the layered DAG).
//
// Reference: pkg/src/memplan/graph.py:375-468 (validate_schedule,
// sequential_schedule, tensor_lifetimes, live_bytes_by_timestep, peak_memory).
//
// live[k] = sum_{j<k}(out - free)(o_j) + out(o_k) over unit-packed {fs, out}
// words (K1V2Meta's opv: byte counts in units of 2^shift), multi-consumer
// frees added at the latest maximal consumer's position.  Against the generic
// evaluator (k_eval.cu) what changes is how little each position costs:
//   * compile-time geometry: SL = NT * C slots, every thread owns exactly C
//     positions (padding slot k >= n holds op id k, zero bytes), so no loop
//     carries a runtime guard;
//   * permutation check by sentinel: pos[] holds 0x8000 for every id before
//     the scatter; an out-of-range id is clamped to the sink slot SL, so any
//     duplicate or out-of-range entry leaves some id in [0, SL) at 0x8000 --
//     one OR per id instead of a range check and a readback per position;
//   * the edges (u, u+1) and (u, u+2) of the transitive reduction (77 % of a
//     training graph's) are checked for two ids per 32-bit word in an id-major
//     pass over pos[] (LDS.128 of 8 ids): with positions < 2^15,
//     ((pv | 0x80008000) - pu - 0x00010001) keeps bit 15 / 31 iff pv > pu;
//   * the remaining edges and the two-consumer tensors come as pre-scaled byte
//     offsets, padded so the loops have a uniform trip count;
//   * the group's (max, first argmax) is three warp REDUX operations;
//   * the edge masks of a thread's chunks are register words (build_k1_em).
#include "k_common.cuh"

namespace roam {

struct K1V4Args {
  const void* orders;  // int32 or uint16 rows [B, n]
  int64_t B;
  int n, G, shift;
  const void* opv;  // int2 {fs, out} units per id [SL + 1]
  const uint8_t* cls;  // CLS mode: class per id [SL + 1] ...
  const void* tab;     // ... and int2 {fs, out} units per class [ncls]
  int ncls;
  size_t off_tab;
  const uint32_t* em;  // SIMD edge-mask word per 8-id chunk (roam_graph.cpp build_k1_em)
  const uint32_t* edges;
  int n_edges;  // multiple of 4 * NT
  const uint32_t* mpair;
  int n_pair;  // multiple of NT
  const uint32_t* mptr;
  const uint16_t* mcons;
  const uint32_t* msz;
  int n_gen, n_mcons;
  int64_t* peak;
  int32_t* argmax;
  uint8_t* valid;
  K1KeySel sel;  // sel.key_out == nullptr: no fused selection
  size_t off_edges, off_mpair, off_mptr, off_mcons, off_msz;
  size_t off_groups, group_bytes, off_xs, off_red;
};

template <int C>
struct V4Geom {
  static constexpr int L = C == 4 ? 2 : C == 8 ? 3 : C == 16 ? 4 : C == 32 ? 5 : 6;
  static constexpr int STRIDE = C + 2;  // (STRIDE / 2) odd: conflict-free LDS.128 rows
};

__device__ __forceinline__ unsigned lds_u16(const unsigned char* base, unsigned byte_off) {
  return *reinterpret_cast<const uint16_t*>(base + byte_off);
}

// ((v | 0x80008000) - u - 0x00010001) | nm: bit 15 / 31 set iff the half's
// edge holds (pv > pu) or is not checked
__device__ __forceinline__ unsigned simd_gt(unsigned v, unsigned u, unsigned nm) {
  return ((v | 0x80008000u) - u - 0x00010001u) | nm;
}

// C = 32 instances cap the CTA at 512 threads: 128 registers hold the
// 32-position row and the other register-resident lists
__host__ __device__ constexpr int v4_cta_cap(int c) { return c == 64 ? 256 : c == 32 ? 512 : 1024; }

// scan-layout word offset of position tid + j*NT relative to that of tid
// (NT a multiple of C, or C a multiple of NT)
template <int NT, int C>
__device__ constexpr int v4_xs_off(int j) {
  return ((j * NT) >> V4Geom<C>::L) * V4Geom<C>::STRIDE + ((j * NT) & (C - 1));
}

// group barrier; a one-warp group only needs the warp's own
template <int NT>
__device__ __forceinline__ void v4_bar(int id) {
  if constexpr (NT == 32) __syncwarp(); else gbar(id, NT);
}
template <int NT>
__device__ __forceinline__ unsigned v4_bar_or(int id, unsigned p) {
  if constexpr (NT == 32) return __any_sync(0xffffffffu, p) ? 1u : 0u;
  else return (unsigned)gbar_or(id, NT, (int)p);
}

// CLS: per-op {fs, out} as a one-byte class into a small table (graphs with
// at most 255 distinct {out, fs} pairs): the per-id table shrinks 8x, which
// buys a second resident group on large graphs at the cost of a dependent
// table lookup per position
template <typename RowT, int NT, int C, bool CLS = false>
__global__ void __launch_bounds__((v4_cta_cap(C) / NT) * NT, 1) k1v4_eval_orders(const K1V4Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  asm volatile("griddepcontrol.launch_dependents;");  // the next launch may start its prologue
  constexpr int SL = NT * C;
  constexpr int Q = SL / 8;                 // 8-id chunks
  constexpr int QR = (Q + NT - 1) / NT;     // chunk rounds per thread
  constexpr bool QFULL = (Q % NT) == 0;
  constexpr int NWARPS = NT / 32;
  using X = V4Geom<C>;
  const int n = a.n;
  const RowT* orders = static_cast<const RowT*>(a.orders);
  {
    auto cp16 = [&](const void* g, size_t off, size_t bytes) {
      const uint4* src = static_cast<const uint4*>(g);
      uint4* dst = reinterpret_cast<uint4*>(smem + off);
      for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    };
    if (CLS) {
      cp16(a.cls, 0, align16(size_t(SL + 1)));
      cp16(a.tab, a.off_tab, align16(8 * size_t(a.ncls)));
    } else {
      cp16(a.opv, 0, align16(8 * size_t(SL + 1)));
    }
    if (a.n_edges > (C / 4) * NT) cp16(a.edges, a.off_edges, 4 * size_t(a.n_edges));
    cp16(a.mpair, a.off_mpair, align16(4 * size_t(a.n_pair)));
    cp16(a.mptr, a.off_mptr, align16(4 * size_t(a.n_gen + 1)));
    cp16(a.mcons, a.off_mcons, align16(2 * size_t(a.n_mcons)));
    cp16(a.msz, a.off_msz, align16(4 * size_t(a.n_pair + a.n_gen)));
  }
  __syncthreads();
  const long long* opv = reinterpret_cast<const long long*>(smem);  // fs | out << 32
  const uint8_t* cls8 = smem;                                         // CLS: class per id
  const long long* tab = reinterpret_cast<const long long*>(smem + a.off_tab);
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
  uint16_t* pos = reinterpret_cast<uint16_t*>(gbase);  // [SL + 8]: ids, sink SL, lookahead
  const unsigned char* posb = gbase;
  long long* xs = reinterpret_cast<long long*>(gbase + a.off_xs);
  long long* red_t = reinterpret_cast<long long*>(gbase + a.off_red);  // [NWARPS] warp totals
  long long* red_c = red_t + NWARPS;                                    // [NWARPS] warp maxima
  int* red_i = reinterpret_cast<int*>(red_c + NWARPS);                  // [NWARPS] their indices
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t cstride = int64_t(gridDim.x) * a.G;
  long long* xs_w = xs + (tid >> X::L) * X::STRIDE + (tid & (C - 1));
  const int n_edges = a.n_edges, n_pair = a.n_pair, n_gen = a.n_gen;
  // the generic edges stay in registers when there are exactly 4 per thread
  constexpr int ER = C / 4;  // list entries per thread kept in registers
  const int ek = n_edges / NT;         // a multiple of 4
  const bool ereg = ek <= ER;
  uint32_t er[ER];
#pragma unroll
  for (int i = 0; i < ER; ++i) er[i] = (ereg && i < ek) ? __ldg(a.edges + tid + i * NT) : 0u;
  // likewise the two-consumer tensors when there are at most 4 per thread
  const int pk = n_pair / NT;
  const bool preg = pk <= ER;
  uint32_t pw[ER], pu[ER];
#pragma unroll
  for (int i = 0; i < ER; ++i) {
    pw[i] = (preg && i < pk) ? __ldg(a.mpair + tid + i * NT) : 0u;
    pu[i] = (preg && i < pk) ? __ldg(a.msz + tid + i * NT) : 0u;
  }
  uint32_t em[QR];  // edge masks of this thread's chunks (ids 8q..8q+9)
#pragma unroll
  for (int r = 0; r < QR; ++r) {
    const int q = tid + r * NT;
    em[r] = (QFULL || q < Q) ? __ldg(a.em + q) : 0xff00ff00u;
  }
  for (int i = tid; i < (SL + 8) / 2; i += NT) reinterpret_cast<uint32_t*>(pos)[i] = 0x80008000u;
  v4_bar<NT>(bar_id);
  // programmatic dependent launch: everything above reads only the graph's
  // read-only metadata, so it may overlap the previous launch's tail; rows,
  // outputs and the selection counter are touched only after that launch has
  // completed (a no-op for a normal launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");

  uint32_t v[C];
  auto load_row = [&](int64_t cc) {
    const RowT* row = orders + cc * int64_t(n);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int k = tid + j * NT;
      v[j] = k < n ? (uint32_t)__ldcs(row + k) : (uint32_t)k;
    }
  };
  long long kbest = LLONG_MAX;  // fused selection: this group's best key (thread 0)
  int64_t c = int64_t(blockIdx.x) * a.G + gid;
  if (c < a.B) load_row(c);
  for (; c < a.B; c += cstride) {
    // ---- P1: scatter positions; out-of-range ids land in the sink slot
#pragma unroll
    for (int j = 0; j < C; ++j) {
      v[j] = min(v[j], (uint32_t)SL);
      pos[v[j]] = (uint16_t)(tid + j * NT);
    }
    v4_bar<NT>(bar_id);
    // ---- P2a (id-major): missing ids (sentinel) and the (u, u+1), (u, u+2) edges
    unsigned sent = 0, ok = 0xffffffffu;
#pragma unroll
    for (int r = 0; r < QR; ++r) {
      const int q = tid + r * NT;
      // the next chunk's first word comes from the next lane (same round)
      const uint4 w = (QFULL || q < Q) ? *reinterpret_cast<const uint4*>(pos + 8 * q)
                                       : make_uint4(0, 0, 0, 0);
      unsigned w4 = __shfl_down_sync(0xffffffffu, w.x, 1);
      if (lane == 31 && (QFULL || q < Q)) w4 = *reinterpret_cast<const uint32_t*>(pos + 8 * q + 8);
      const unsigned m = em[r];
      sent |= w.x | w.y | w.z | w.w;
      ok &= simd_gt(__byte_perm(w.x, w.y, 0x5432), w.x, m);
      ok &= simd_gt(__byte_perm(w.y, w.z, 0x5432), w.y, m << 1);
      ok &= simd_gt(__byte_perm(w.z, w.w, 0x5432), w.z, m << 2);
      ok &= simd_gt(__byte_perm(w.w, w4, 0x5432), w.w, m << 3);
      ok &= simd_gt(w.y, w.x, m << 4);
      ok &= simd_gt(w.z, w.y, m << 5);
      ok &= simd_gt(w.w, w.z, m << 6);
      ok &= simd_gt(w4, w.w, m << 7);
    }
    // ---- P2a: the other checked edges (pv - pu - 1 < 0 marks a violation)
    int eacc = 0;
    int e_first = tid;
    if (ereg) {
      // every slot loads (unused ones read pos[0]: a broadcast) so the loads
      // issue back to back; unused slots are masked out of the result
#pragma unroll
      for (int i = 0; i < ER; ++i) {
        const int d = (int)lds_u16(posb, er[i] >> 16) - (int)lds_u16(posb, er[i] & 0xffffu) - 1;
        eacc |= i < ek ? d : 0;
      }
      e_first = n_edges;
    }
    for (int e0 = e_first; e0 < n_edges; e0 += 4 * NT) {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = edges[e0 + i * NT];
#pragma unroll
      for (int i = 0; i < 4; ++i) eacc |= (int)lds_u16(posb, w[i] >> 16) - (int)lds_u16(posb, w[i] & 0xffffu) - 1;
    }
    // ---- P2a (position-major): {fs, out} units of the op at each position
    // class form: the two dependent lookups are batched 8 deep (GPT2-XL 0.187 ->
    // 0.180 ms); the plain table keeps the compiler's own interleave (GPT-2
    // small 0.080 ms vs 0.082 batched)
    constexpr int GB = CLS ? (C < 8 ? C : 8) : 1;
#pragma unroll
    for (int j0 = 0; j0 < C; j0 += GB) {  // GB gathers in flight before their stores
      long long gv[GB];
#pragma unroll
      for (int j = 0; j < GB; ++j) gv[j] = CLS ? tab[cls8[v[j0 + j]]] : opv[v[j0 + j]];
#pragma unroll
      for (int j = 0; j < GB; ++j) xs_w[v4_xs_off<NT, C>(j0 + j)] = gv[j];
    }
    unsigned bad = ((sent & 0x80008000u) != 0) | ((ok & 0x80008000u) != 0x80008000u) | (eacc < 0);
    // prefetch the next candidate's row; it lands while P2b / P3 run
    const int64_t cn = c + cstride;
    if (cn < a.B) load_row(cn);
    v4_bar<NT>(bar_id);
    // ---- P2b: multi-consumer tensors free after their latest maximal consumer
    // (positions of a broken row may be the sentinel: clamp into the group)
    // unconditional shared reduction: the zero-size padding pairs add 0 to a
    // real slot, which is cheaper than branching around their atomics
    auto add_free = [&](unsigned kmax, unsigned units) {
      kmax = min(kmax, (unsigned)(SL - 1));
      atomicAdd(reinterpret_cast<unsigned*>(xs + (kmax >> X::L) * X::STRIDE + (kmax & (C - 1))), units);
    };
    int m_first = tid;
    if (preg) {
      // gathers first (independent, back to back), then the atomics of the
      // slots in use (pk is uniform)
      unsigned km[ER];
#pragma unroll
      for (int i = 0; i < ER; ++i) km[i] = max(lds_u16(posb, pw[i] & 0xffffu), lds_u16(posb, pw[i] >> 16));
#pragma unroll
      for (int i = 0; i < ER; ++i)
        if (i < pk) add_free(km[i], pu[i]);
      m_first = n_pair;
    }
    for (int m = m_first; m < n_pair; m += NT) {
      const uint32_t w = mpair[m];
      add_free(max(lds_u16(posb, w & 0xffffu), lds_u16(posb, w >> 16)), msz[m]);
    }
    for (int m = tid; m < n_gen; m += NT) {
      const int q0 = mptr[m], q1 = mptr[m + 1];
      unsigned kmax = 0;
      for (int q = q0; q < q1; ++q) kmax = max(kmax, (unsigned)pos[mcons[q]]);
      add_free(kmax, msz[n_pair + m]);
    }
    v4_bar<NT>(bar_id);
    // ---- P3: reset this thread's ids to the sentinel for the next candidate
#pragma unroll
    for (int r = 0; r < QR; ++r) {
      const int q = tid + r * NT;
      if (QFULL || q < Q)
        *reinterpret_cast<uint4*>(pos + 8 * q) = make_uint4(0x80008000u, 0x80008000u, 0x80008000u, 0x80008000u);
    }
    // ---- P3: blocked scan over this thread's C positions (padding slots
    // carry zero bytes: they never raise the running max above a real slot)
    const int k0 = tid * C;
    const long long* xr = xs + tid * X::STRIDE;
    // the running sum is one dependent chain; the (max, first index) over the
    // C live values is a pairwise tree (depth log2 C instead of C)
    long long run = 0;
    long long lv[C];
#pragma unroll
    for (int i = 0; i < C; i += 2) {
      const longlong2 pr = *reinterpret_cast<const longlong2*>(xr + i);
      lv[i] = run + (long long)((unsigned long long)pr.x >> 32);
      run = lv[i] - (long long)(unsigned)pr.x;
      lv[i + 1] = run + (long long)((unsigned long long)pr.y >> 32);
      run = lv[i + 1] - (long long)(unsigned)pr.y;
    }
    int ix[C / 2];
#pragma unroll
    for (int p = 0; p < C / 2; ++p) {  // strict >: ties keep the earlier position
      const bool t = lv[2 * p + 1] > lv[2 * p];
      lv[p] = t ? lv[2 * p + 1] : lv[2 * p];
      ix[p] = 2 * p + (t ? 1 : 0);
    }
#pragma unroll
    for (int w = C / 2; w > 1; w >>= 1) {
#pragma unroll
      for (int p = 0; p < w / 2; ++p) {
        const bool t = lv[2 * p + 1] > lv[2 * p];
        lv[p] = t ? lv[2 * p + 1] : lv[2 * p];
        ix[p] = t ? ix[2 * p + 1] : ix[2 * p];
      }
    }
    const long long best = lv[0];
    const int bi = ix[0];
    long long incl = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane == 31) red_t[warp] = incl;
    bad = v4_bar_or<NT>(bar_id, bad);
    long long off = incl - run;
#pragma unroll
    for (int w = 0; w < NWARPS - 1; ++w)
      if (w < warp) off += red_t[w];
    // warp (max, first index): REDUX on the high word, then the low word among
    // the lanes holding the maximal high word, then the smallest index
    const long long cand = off + best;
    const int hi = (int)(cand >> 32);
    const unsigned lo = (unsigned)cand;
    const int mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    const unsigned mi = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? (unsigned)(k0 + bi) : 0xffffffffu);
    if (lane == 0) {
      red_c[warp] = (long long)(((unsigned long long)(unsigned)mh << 32) | ml);
      red_i[warp] = (int)mi;
    }
    v4_bar<NT>(bar_id);
    if (tid == 0) {
      long long bv = red_c[0];
      int bk = red_i[0];
#pragma unroll
      for (int w = 1; w < NWARPS; ++w)
        if (red_c[w] > bv) {  // warps hold increasing index ranges: strict > keeps the first
          bv = red_c[w];
          bk = red_i[w];
        }
      if (n == 0) {
        bv = 0;
        bk = 0;
      }
      a.peak[c] = (int64_t)bv << a.shift;
      a.argmax[c] = bk;
      a.valid[c] = bad ? 0 : 1;
      if (!bad) kbest = min(kbest, (((long long)bv << a.shift) << a.sel.id_bits) | (a.sel.id_base + c));
    }
  }
  if (a.sel.key_out) {
    // fused selection: each group leaves its best key; the last group to
    // finish reduces them all (threadfence + counter), then resets the counter
    int* s_last = red_i + NWARPS;
    if (tid == 0) {
      a.sel.partial[blockIdx.x * a.G + gid] = kbest;
      __threadfence();
      *s_last = atomicAdd(a.sel.counter, 1u) == gridDim.x * (unsigned)a.G - 1u;
    }
    v4_bar<NT>(bar_id);
    if (*s_last) {
      __threadfence();
      const int total = gridDim.x * a.G;
      long long m = LLONG_MAX;
      for (int i = tid; i < total; i += NT) m = min(m, ((volatile long long*)a.sel.partial)[i]);
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, d));
      if (lane == 0) red_c[warp] = m;
      v4_bar<NT>(bar_id);
      if (tid == 0) {
        for (int w = 1; w < NWARPS; ++w) m = min(m, red_c[w]);
        *a.sel.key_out = m;
        *a.sel.counter = 0u;
      }
    }
  }
}

template <typename RowT, int NT, int C, bool CLS = false>
static int launch_k1v4_t(K1V4Args& a, int grid, size_t smem, cudaStream_t s) {
  auto kern = k1v4_eval_orders<RowT, NT, C, CLS>;
  RM_CUDA(smem_optin(kern));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT * a.G);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RM_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  RM_LAUNCH_CHECK("k1v4_eval_orders launch");
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

// the instance table must list every (NT, C) k1v4_geometry (roam_graph.cpp) picks
template <typename RowT>
static int launch_k1v4_nt(K1V4Args& a, int NT, int C, bool cls, int grid, size_t smem, cudaStream_t s) {
#define RM_K1V4_CLS(nt, cc) \
  if (cls && NT == nt && C == cc) return launch_k1v4_t<RowT, nt, cc, true>(a, grid, smem, s);
  RM_K1V4_CLS(256, 16)
  RM_K1V4_CLS(320, 16)
  RM_K1V4_CLS(384, 16)
  RM_K1V4_CLS(512, 16)
  RM_K1V4_CLS(640, 16)
  RM_K1V4_CLS(768, 16)
  RM_K1V4_CLS(1024, 16)
  RM_K1V4_CLS(128, 32)
  RM_K1V4_CLS(256, 32)
  RM_K1V4_CLS(512, 32)
#undef RM_K1V4_CLS
  if (cls) return 1;
#define RM_K1V4_CASE(nt, cc) \
  if (NT == nt && C == cc) return launch_k1v4_t<RowT, nt, cc>(a, grid, smem, s);
  RM_K1V4_CASE(32, 4)
  RM_K1V4_CASE(32, 8)
  RM_K1V4_CASE(64, 8)
  RM_K1V4_CASE(96, 8)
  RM_K1V4_CASE(128, 8)
  RM_K1V4_CASE(64, 16)
  RM_K1V4_CASE(96, 16)
  RM_K1V4_CASE(128, 16)
  RM_K1V4_CASE(160, 16)
  RM_K1V4_CASE(192, 16)
  RM_K1V4_CASE(256, 16)
  RM_K1V4_CASE(320, 16)
  RM_K1V4_CASE(384, 16)
  RM_K1V4_CASE(512, 16)
  RM_K1V4_CASE(640, 16)
  RM_K1V4_CASE(768, 16)
  RM_K1V4_CASE(1024, 16)
  RM_K1V4_CASE(32, 32)
  RM_K1V4_CASE(64, 32)
  RM_K1V4_CASE(128, 32)
  RM_K1V4_CASE(256, 32)
  RM_K1V4_CASE(512, 32)
  RM_K1V4_CASE(32, 64)
  RM_K1V4_CASE(64, 64)
  RM_K1V4_CASE(128, 64)
#undef RM_K1V4_CASE
  return 1;
}

int launch_k1v4(RmGraph* g, const void* orders_dev, int64_t B, int64_t* peak, int32_t* argmax,
                uint8_t* valid, cudaStream_t s, bool u16_rows, const K1KeySel* sel) {
  const K1V4Meta& m = g->k4v;
  if (!m.ok) return 1;
  const int NT = m.NT, C = m.C, SL = m.SL;
  K1V4Args a{};
  a.orders = orders_dev;
  a.B = B;
  a.n = g->n;
  a.shift = g->k2v.shift;
  a.opv = g->k2v.opv.p;
  a.em = m.em.as<uint32_t>();
  a.edges = m.edges.as<uint32_t>();
  a.n_edges = (int)m.n_edges;
  a.mpair = m.mpair.as<uint32_t>();
  a.n_pair = (int)m.n_pair;
  a.mptr = g->k2v.mptr.as<uint32_t>();
  a.mcons = g->k2v.mcons.as<uint16_t>();
  a.msz = m.msz.as<uint32_t>();
  a.n_gen = (int)g->k2v.n_gen;
  a.n_mcons = (int)g->k2v.n_mcons;
  a.peak = peak;
  a.argmax = argmax;
  a.valid = valid;
  if (sel) a.sel = *sel;
  a.cls = m.cls.as<uint8_t>();
  a.tab = m.tab.p;
  a.ncls = m.ncls;
  const int stride = C + 2;  // V4Geom<C>::STRIDE
  int dev = g->device;
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int cap = (C == 64 ? 256 : C == 32 ? 512 : 1024) / NT;
  // layout with the per-id table (cls = false) or the class form; the class
  // form is used only where it fits more groups per SM
  auto layout = [&](bool cls) {
    K1V4Args b = a;
    const size_t table = cls ? align16(size_t(SL + 1)) + align16(8 * size_t(a.ncls)) : align16(8 * size_t(SL + 1));
    b.off_tab = align16(size_t(SL + 1));
    b.off_edges = table;
    b.off_mpair = align16(b.off_edges + 4 * size_t(b.n_edges));
    b.off_mptr = align16(b.off_mpair + 4 * size_t(b.n_pair));
    b.off_mcons = align16(b.off_mptr + 4 * size_t(b.n_gen + 1));
    b.off_msz = align16(b.off_mcons + 2 * size_t(b.n_mcons));
    b.off_groups = align16(b.off_msz + 4 * size_t(b.n_pair + b.n_gen));
    b.off_xs = align16(2 * size_t(SL + 8));
    b.off_red = align16(b.off_xs + 8 * size_t(SL / C) * stride);
    b.group_bytes = align16(b.off_red + 3 * 8 * size_t(NT / 32) + 16);
    const size_t avail = max_smem > (int)b.off_groups ? size_t(max_smem) - b.off_groups : 0;
    b.G = std::min({(int)(avail / b.group_bytes), cap, 15});
    return b;
  };
  K1V4Args plain = layout(false);
  bool use_cls = false;
  if (m.ncls > 0 && ((C == 16 && NT >= 256) || (C == 32 && NT >= 128))) {
    K1V4Args c = layout(true);
    if (c.G > plain.G) {
      plain = c;
      use_cls = true;
    }
  }
  a = plain;
  int G = a.G;
  if (G < 1) return 1;
  const int64_t sms = k1_sms(dev);
  if (int64_t(G) * sms > B) G = (int)std::max<int64_t>(1, (B + sms - 1) / sms);
  a.G = G;
  const size_t smem = a.off_groups + size_t(G) * a.group_bytes;
  const int grid = (int)std::min<int64_t>(sms, (B + G - 1) / G);
  return u16_rows ? launch_k1v4_nt<uint16_t>(a, NT, C, use_cls, grid, smem, s)
                  : launch_k1v4_nt<int32_t>(a, NT, C, use_cls, grid, smem, s);
}

}  // namespace roam
