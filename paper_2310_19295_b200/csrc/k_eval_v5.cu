// K1 v5: the candidate-order evaluator for graphs whose per-op events fit a
// one-byte DYNAMIC class.
//
// Reference: pkg/src/memplan/graph.py:375-468 (validate_schedule,
// sequential_schedule, tensor_lifetimes, live_bytes_by_timestep, peak_memory).
//
// Same arithmetic and validity checks as v4 (k_eval_v4.cu): live[k] =
// sum_{j<k}(out - free)(o_j) + out(o_k), a tensor with several maximal
// consumers freed after the latest of them.  What changes is what crosses
// shared memory per position.  v4 gathers an 8-byte {fs, out} word per
// position and transposes it (strided -> blocked) through an 8-byte xs array;
// multi-consumer frees are atomics into xs.  Here every op's events --
// including which of its multi-consumer tensors it closes in THIS candidate --
// are one byte:
//
//   class(v, mask) = base[v] + mask,  mask bit i = v is the latest maximal
//                    consumer of its i-th multi-consumer tensor
//
// (roam_graph.cpp build_k1v5_host gives every op signature -- static frees,
// outputs, multi-consumer sizes -- a block of 2^m classes; training graphs
// need 75-83; a graph that needs more than 255 runs v4).  Per candidate:
//   P1  restore the group's class bytes cls'[] from base[] (id-major), clamp
//       the row, scatter pos[o_k] = k;
//   P2  v4's sentinel / SIMD edge checks and generic edges; each
//       multi-consumer tensor adds its bit to the winner's class byte (one
//       32-bit shared atomic per tensor);
//   P3  gather cls'[o_k] (1 byte, strided: consecutive positions on
//       consecutive lanes) and store it position-major into the blocked
//       layout xc (1 byte per position instead of v4's 8);
//   P4  each thread reads its C class bytes (LDS.128), looks up {fs, out}
//       units in a lane-replicated class table (ltab[c][lane]: every lookup
//       conflict-free) and runs v4's blocked scan and (max, first argmax).
#include "k_common.cuh"

namespace roam {

struct K1V5Args {
  const void* orders;  // int32 or uint16 rows [B, n]
  int64_t B;
  int n, G, shift;
  const uint8_t* base;  // base class per id [SL + 16]
  const void* tab;      // int2 {fs, out} units per class [ncls]
  int ncls;
  const uint32_t* em;  // SIMD edge-mask word per 8-id chunk (shared with v4)
  const uint32_t* edges;
  int n_edges;  // multiple of 4 * NT
  // WIDE (more than 8,192 slots): every id / target field below doubles
  // to 16 bits + its shift: g4 four u32, gcons u32, dtgt {ta, tb} u32 pairs
  const uint32_t* dpair;  // two-consumer tensors: pos byte offsets 2a | 2b << 16 ...
  const void* dtgt;       // ... and class-bit targets ta | tb << 16, t = word | shift << 11
  int n_pair;             // multiple of NT (padding: target 0xffffffff)
  const void* g4;         // 3-4 consumer tensors: four u16 (id | bit index << 13),
  int n_g4;               // a short list repeating its first; multiple of NT, pads 0xe000
  const uint32_t* gptr;   // >= 5 consumer tensors: CSR of consumer id | bit index << 13
  const void* gcons;
  int n_gen, n_gcons;
  int64_t* peak;
  int32_t* argmax;
  uint8_t* valid;
  K1KeySel sel;
  size_t off_base, off_edges, off_dpair, off_dtgt, off_g4, off_gptr, off_gcons;
  size_t off_groups, group_bytes, off_cls, off_xc, off_red, off_rbuf, off_mbar;
};

static constexpr uint32_t K1V5_PAD = 0xffffffffu;  // padding pair target

template <int C>
struct V5Geom {
  // byte stride of a thread's C class bytes in xc: the blocked LDS.128 /
  // LDS.64 / LDS.32 reads of a quarter / half / full warp hit distinct banks
  static constexpr int XS = C >= 32 ? C + 16 : C == 16 ? 48 : C;
  static constexpr int L = C == 4 ? 2 : C == 8 ? 3 : C == 16 ? 4 : C == 32 ? 5 : 6;
};

__device__ __forceinline__ unsigned v5_lds_u16(const unsigned char* base, unsigned byte_off) {
  return *reinterpret_cast<const uint16_t*>(base + byte_off);
}
__device__ __forceinline__ unsigned v5_simd_gt(unsigned v, unsigned u, unsigned nm) {
  return ((v | 0x80008000u) - u - 0x00010001u) | nm;
}
// threads per CTA: the register-held row prefetch of the LDG form needs 128
// registers at C >= 32 (512 threads); the bulk-copy form stages rows in shared
// memory instead and fits 640
__host__ __device__ constexpr int v5_cta_cap(int c, bool bulk) { return c >= 32 ? (bulk ? 640 : 512) : 1024; }

template <int NT>
__device__ __forceinline__ void v5_bar(int id) {
  if constexpr (NT == 32) __syncwarp(); else gbar(id, NT);
}
template <int NT>
__device__ __forceinline__ unsigned v5_bar_or(int id, unsigned p) {
  if constexpr (NT == 32) return __any_sync(0xffffffffu, p) ? 1u : 0u;
  else return (unsigned)gbar_or(id, NT, (int)p);
}

// the id / target encodings of one geometry: 13-bit ids (up to 8,192 slots)
// or 16-bit ids (WIDE) with the fields widened
template <bool WIDE>
struct V5Enc {
  using G4 = uint2;        // four u16 consumer entries
  using GC = uint16_t;
  using TG = uint32_t;     // ta | tb << 16
  static constexpr unsigned IDB = 13, G4PAD = 0xe000u;
  __device__ static unsigned pick(TG t2, bool b) { return __byte_perm(t2, 0u, b ? 0x4432u : 0x4410u); }
  __device__ static bool pad(TG t2) { return t2 == 0xffffffffu; }
  static constexpr unsigned TWB = 11;  // target: word | shift << TWB
};
template <>
struct V5Enc<true> {
  using G4 = uint4;        // four u32 consumer entries
  using GC = uint32_t;
  using TG = uint2;        // {ta, tb}
  static constexpr unsigned IDB = 16, G4PAD = 0x70000u;
  __device__ static unsigned pick(TG t2, bool b) { return b ? t2.y : t2.x; }
  __device__ static bool pad(TG t2) { return t2.x == 0xffffffffu; }
  static constexpr unsigned TWB = 16;
};

template <typename RowT, int NT, int C, bool BULK, bool WIDE = false>
__global__ void __launch_bounds__((v5_cta_cap(C, BULK) / NT) * NT, 1) k1v5_eval_orders(const K1V5Args a) {
  using E = V5Enc<WIDE>;
  using G4T = typename E::G4;
  using GCT = typename E::GC;
  using TGT = typename E::TG;
  constexpr unsigned IDM = (1u << E::IDB) - 1u;
  extern __shared__ __align__(16) unsigned char smem[];
  asm volatile("griddepcontrol.launch_dependents;");
  constexpr int SL = NT * C;
  constexpr int Q = SL / 8;              // 8-id chunks
  constexpr int QR = (Q + NT - 1) / NT;  // chunk rounds per thread
  constexpr bool QFULL = (Q % NT) == 0;
  constexpr int NWARPS = NT / 32;
  constexpr int XS = V5Geom<C>::XS;
  // positions j*NT + tid with j < JSAFE are always < n: the launcher runs the
  // C >= 32 instances only when n > SL / 2
  constexpr int JSAFE = (C >= 32 && NT >= 64) ? C / 2 : 0;
  // two-consumer tensors per thread kept in registers (WIDE: 8-byte targets)
  constexpr int PR = C >= 32 ? (WIDE ? 4 : 6) : C / 4;
  const int n = a.n;
  const RowT* orders = static_cast<const RowT*>(a.orders);
  const int lane = threadIdx.x & 31;
  {
    auto cp16 = [&](const void* g, size_t off, size_t bytes) {
      const uint4* src = static_cast<const uint4*>(g);
      uint4* dst = reinterpret_cast<uint4*>(smem + off);
      for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    };
    cp16(a.base, a.off_base, align16(size_t(SL + 16)));
    // lane-replicated class table: entry (c, l) at ltab[c * 32 + l]
    const long long* tab = static_cast<const long long*>(a.tab);
    long long* lt = reinterpret_cast<long long*>(smem);
    for (int i = threadIdx.x; i < a.ncls * 32; i += blockDim.x) lt[i] = __ldg(tab + (i >> 5));
    if (a.n_edges > (C / 4) * NT) cp16(a.edges, a.off_edges, 4 * size_t(a.n_edges));
    if (a.n_pair > PR * NT) {
      cp16(a.dpair, a.off_dpair, 4 * size_t(a.n_pair));
      cp16(a.dtgt, a.off_dtgt, sizeof(TGT) * size_t(a.n_pair));
    }
    cp16(a.g4, a.off_g4, sizeof(G4T) * size_t(a.n_g4));
    cp16(a.gptr, a.off_gptr, align16(4 * size_t(a.n_gen + 1)));
    cp16(a.gcons, a.off_gcons, align16(sizeof(GCT) * size_t(a.n_gcons)));
  }
  __syncthreads();
  const uint8_t* base8 = smem + a.off_base;
  // the class table sits at the start of shared memory: entry (c, l) at byte
  // c * 256 + l * 8, so a lookup is [PRMT result + the window base]
  const unsigned char* ltab_b = smem;
  const unsigned lane8 = (unsigned)lane * 8u;
  const uint32_t* edges = reinterpret_cast<const uint32_t*>(smem + a.off_edges);
  const uint32_t* dpair = reinterpret_cast<const uint32_t*>(smem + a.off_dpair);
  const TGT* dtgt = reinterpret_cast<const TGT*>(smem + a.off_dtgt);
  const G4T* g4 = reinterpret_cast<const G4T*>(smem + a.off_g4);
  const uint32_t* gptr = reinterpret_cast<const uint32_t*>(smem + a.off_gptr);
  const GCT* gcons = reinterpret_cast<const GCT*>(smem + a.off_gcons);

  const int gid = threadIdx.x / NT;
  const int tid = threadIdx.x - gid * NT;
  if (gid >= a.G) return;
  const int bar_id = 1 + gid;
  unsigned char* gbase = smem + a.off_groups + size_t(gid) * a.group_bytes;
  uint16_t* pos = reinterpret_cast<uint16_t*>(gbase);  // [SL + 8]: ids, sink SL, lookahead
  const unsigned char* posb = gbase;
  unsigned char* clsp = gbase + a.off_cls;              // [SL + 16] this candidate's classes
  unsigned char* xc = gbase + a.off_xc;                 // [NT * XS] blocked class bytes
  long long* red_t = reinterpret_cast<long long*>(gbase + a.off_red);
  long long* red_c = red_t + NWARPS;
  int* red_i = reinterpret_cast<int*>(red_c + NWARPS);
  const int warp = tid >> 5;
  const int64_t cstride = int64_t(gridDim.x) * a.G;
  const int n_edges = a.n_edges, n_pair = a.n_pair, n_gen = a.n_gen, n_g4 = a.n_g4;
  constexpr int ER = C / 4;  // list entries per thread kept in registers
  const int ek = n_edges / NT;
  const bool ereg = ek <= ER;
  uint32_t er[ER];
#pragma unroll
  for (int i = 0; i < ER; ++i) er[i] = (ereg && i < ek) ? __ldg(a.edges + tid + i * NT) : 0u;
  const int pk = n_pair / NT;
  const bool preg = pk <= PR;
  uint32_t pw[PR];
  TGT pt[PR];
  const TGT* gdtgt = static_cast<const TGT*>(a.dtgt);
#pragma unroll
  for (int i = 0; i < PR; ++i) {
    pw[i] = (preg && i < pk) ? __ldg(a.dpair + tid + i * NT) : 0u;
    if (preg && i < pk) pt[i] = gdtgt[tid + i * NT];
    else if constexpr (WIDE) pt[i] = make_uint2(K1V5_PAD, K1V5_PAD);
    else pt[i] = K1V5_PAD;
  }
  uint32_t em[QR];
#pragma unroll
  for (int r = 0; r < QR; ++r) {
    const int q = tid + r * NT;
    em[r] = (QFULL || q < Q) ? __ldg(a.em + q) : 0xff00ff00u;
  }
  for (int i = tid; i < (SL + 8) / 2; i += NT) reinterpret_cast<uint32_t*>(pos)[i] = 0x80008000u;
  // the class bytes past the last chunk (the sink id SL) never change
  for (int i = SL + tid; i < SL + 16; i += NT) clsp[i] = base8[i];
  // xc byte of position k = tid + j*NT: (k / C) * XS + k % C; every instance
  // has NT % C == 0, so that is xc0 + j * (NT / C) * XS (immediate offsets)
  static_assert(NT % C == 0, "v5 geometry: NT must be a multiple of C");
  unsigned char* const xc0 = xc + (tid / C) * XS + (tid % C);
  // BULK: the group's row buffer and its mbarrier; rows arrive by
  // cp.async.bulk (one elected thread issues, the copy engine writes shared
  // memory), so no register holds a prefetched row
  const unsigned rbuf_s = (unsigned)__cvta_generic_to_shared(gbase + a.off_rbuf);
  const unsigned mbar_s = (unsigned)__cvta_generic_to_shared(gbase + a.off_mbar);
  if (BULK && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_s) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  v5_bar<NT>(bar_id);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int ES = (int)sizeof(RowT);
  const uintptr_t ord0 = reinterpret_cast<uintptr_t>(orders);
  const uintptr_t ord_end16 = (ord0 + uintptr_t(a.B) * uintptr_t(n) * ES) & ~uintptr_t(15);
  // the 16-byte-aligned span holding row cc (never past the batch's last
  // aligned byte: a row's last elements beyond it are read from global)
  auto span = [&](int64_t cc, uintptr_t& a0, unsigned& bytes) {
    const uintptr_t g0 = ord0 + uintptr_t(cc) * uintptr_t(n) * ES;
    a0 = g0 & ~uintptr_t(15);
    uintptr_t a1 = (g0 + uintptr_t(n) * ES + 15) & ~uintptr_t(15);
    if (a1 > ord_end16) a1 = ord_end16 > a0 ? ord_end16 : a0;
    bytes = (unsigned)(a1 - a0);
  };
  auto issue = [&](int64_t cc) {  // one thread of the group
    uintptr_t a0;
    unsigned bytes;
    span(cc, a0, bytes);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar_s), "r"(bytes) : "memory");
    if (bytes)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(rbuf_s), "l"(a0), "r"(bytes), "r"(mbar_s) : "memory");
  };
  unsigned phase = 0;

  uint32_t v[C];
  auto load_row = [&](int64_t cc) {
    const RowT* row = orders + cc * int64_t(n);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int k = tid + j * NT;
      v[j] = (j < JSAFE || k < n) ? (uint32_t)__ldcs(row + k) : (uint32_t)k;
    }
  };
  // add `bit` to the class byte of id w (32-bit shared atomic on its word)
  auto add_bit = [&](unsigned w, unsigned bit) {
    atomicAdd(reinterpret_cast<unsigned*>(clsp + (w & ~3u)), bit << (8 * (w & 3u)));
  };
  long long kbest = LLONG_MAX;
  int64_t c = int64_t(blockIdx.x) * a.G + gid;
  if (c < a.B) {
    if constexpr (BULK) {
      if (tid == 0) issue(c);
    } else {
      load_row(c);
    }
  }
  for (; c < a.B; c += cstride) {
    if constexpr (BULK) {  // this candidate's row: wait for its copy, read it
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "W%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra W%=;\n\t}" ::"r"(mbar_s), "r"(phase) : "memory");
      phase ^= 1u;
      uintptr_t a0;
      unsigned bytes;
      span(c, a0, bytes);
      const uintptr_t g0 = ord0 + uintptr_t(c) * uintptr_t(n) * ES;
      const int head = (int)((g0 - a0) / ES);
      const int ncop = (int)((a0 + bytes - g0) / ES);  // elements in the buffer
      const RowT* rb = reinterpret_cast<const RowT*>(gbase + a.off_rbuf) + head;
      const RowT* row = orders + c * int64_t(n);
#pragma unroll
      for (int j = 0; j < C; ++j) {
        const int k = tid + j * NT;
        // padding slots k >= n hold op id k (the span may run past the row)
        v[j] = j < JSAFE ? (uint32_t)rb[k]
                         : (k < n ? (k < ncop ? (uint32_t)rb[k] : (uint32_t)__ldcs(row + k)) : (uint32_t)k);
      }
    }
    // ---- P1: restore this candidate's class bytes; scatter positions
#pragma unroll
    for (int r = 0; r < QR; ++r) {
      const int q = tid + r * NT;
      if (QFULL || q < Q)
        reinterpret_cast<uint2*>(clsp)[q] = reinterpret_cast<const uint2*>(base8)[q];
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
      v[j] = min(v[j], (uint32_t)SL);
      pos[v[j]] = (uint16_t)(tid + j * NT);
    }
    v5_bar<NT>(bar_id);
    if constexpr (BULK) {  // every thread has read the row buffer: refill it
      if (tid == 0 && c + cstride < a.B) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(c + cstride);
      }
    }
    // ---- P2 (id-major): missing ids (sentinel) and the (u, u+1), (u, u+2) edges
    unsigned sent = 0, ok = 0xffffffffu;
#pragma unroll
    for (int r = 0; r < QR; ++r) {
      const int q = tid + r * NT;
      const uint4 w = (QFULL || q < Q) ? *reinterpret_cast<const uint4*>(pos + 8 * q)
                                       : make_uint4(0, 0, 0, 0);
      unsigned w4 = __shfl_down_sync(0xffffffffu, w.x, 1);
      if (lane == 31 && (QFULL || q < Q)) w4 = *reinterpret_cast<const uint32_t*>(pos + 8 * q + 8);
      const unsigned m = em[r];
      sent |= w.x | w.y | w.z | w.w;
      ok &= v5_simd_gt(__byte_perm(w.x, w.y, 0x5432), w.x, m);
      ok &= v5_simd_gt(__byte_perm(w.y, w.z, 0x5432), w.y, m << 1);
      ok &= v5_simd_gt(__byte_perm(w.z, w.w, 0x5432), w.z, m << 2);
      ok &= v5_simd_gt(__byte_perm(w.w, w4, 0x5432), w.w, m << 3);
      ok &= v5_simd_gt(w.y, w.x, m << 4);
      ok &= v5_simd_gt(w.z, w.y, m << 5);
      ok &= v5_simd_gt(w.w, w.z, m << 6);
      ok &= v5_simd_gt(w4, w.w, m << 7);
    }
    // ---- P2: the other checked edges (pv - pu - 1 < 0 marks a violation)
    int eacc = 0;
    int e_first = tid;
    if (ereg) {
#pragma unroll
      for (int i = 0; i < ER; ++i) {
        const int d = (int)v5_lds_u16(posb, er[i] >> 16) - (int)v5_lds_u16(posb, er[i] & 0xffffu) - 1;
        eacc |= i < ek ? d : 0;
      }
      e_first = n_edges;
    }
    for (int e0 = e_first; e0 < n_edges; e0 += 4 * NT) {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = edges[e0 + i * NT];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        eacc |= (int)v5_lds_u16(posb, w[i] >> 16) - (int)v5_lds_u16(posb, w[i] & 0xffffu) - 1;
    }
    // ---- P2: multi-consumer tensors: the latest maximal consumer's class
    // byte gains the tensor's bit (positions of a broken row may be the
    // sentinel; the bits stay in range either way)
    // pair (a, b): the later consumer's class byte gains the tensor's bit;
    // the target half t = class word | bit shift << 11 is picked by one PRMT
    auto pair_free = [&](TGT t2, unsigned pa, unsigned pbv) {
      const unsigned t = E::pick(t2, pbv > pa);
      if (!E::pad(t2))
        atomicAdd(reinterpret_cast<unsigned*>(clsp) + (t & ((1u << E::TWB) - 1u)), 1u << (t >> E::TWB));
    };
    int m_first = tid;
    if (preg) {
      unsigned pa[PR], pbv[PR];
#pragma unroll
      for (int i = 0; i < PR; ++i) {
        pa[i] = v5_lds_u16(posb, pw[i] & 0xffffu);
        pbv[i] = v5_lds_u16(posb, pw[i] >> 16);
      }
#pragma unroll
      for (int i = 0; i < PR; ++i) pair_free(pt[i], pa[i], pbv[i]);
      m_first = n_pair;
    }
    for (int m = m_first; m < n_pair; m += NT) {
      const uint32_t w = dpair[m];
      pair_free(dtgt[m], v5_lds_u16(posb, w & 0xffffu), v5_lds_u16(posb, w >> 16));
    }
    for (int m = tid; m < n_g4; m += NT) {
      const G4T e = g4[m];
      unsigned e0, e1, e2, e3;
      if constexpr (WIDE) {
        e0 = e.x, e1 = e.y, e2 = e.z, e3 = e.w;
      } else {
        e0 = e.x & 0xffffu, e1 = e.x >> 16, e2 = e.y & 0xffffu, e3 = e.y >> 16;
      }
      const unsigned p0 = pos[e0 & IDM], p1 = pos[e1 & IDM], p2 = pos[e2 & IDM], p3 = pos[e3 & IDM];
      // first maximum, in list order (ties only in broken rows)
      const unsigned b01 = p1 > p0 ? e1 : e0, q01 = max(p0, p1);
      const unsigned b23 = p3 > p2 ? e3 : e2, q23 = max(p2, p3);
      const unsigned bw = q23 > q01 ? b23 : b01;
      if (e0 != E::G4PAD) add_bit(bw & IDM, 1u << (bw >> E::IDB));
    }
    for (int m = tid; m < n_gen; m += NT) {
      const int q0 = gptr[m], q1 = gptr[m + 1];
      unsigned best = 0, bw = 0;
      for (int q = q0; q < q1; ++q) {
        const unsigned e = gcons[q], p = pos[e & IDM];
        if (q == q0 || p > best) {
          best = p;
          bw = e;
        }
      }
      add_bit(bw & IDM, 1u << (bw >> E::IDB));
    }
    unsigned bad = ((sent & 0x80008000u) != 0) | ((ok & 0x80008000u) != 0x80008000u) | (eacc < 0);
    v5_bar<NT>(bar_id);
    // ---- P3: this candidate's class byte per position, blocked layout
#pragma unroll
    for (int j = 0; j < C; ++j) xc0[j * (NT / C) * XS] = clsp[v[j]];
#pragma unroll
    for (int r = 0; r < QR; ++r) {
      const int q = tid + r * NT;
      if (QFULL || q < Q)
        *reinterpret_cast<uint4*>(pos + 8 * q) = make_uint4(0x80008000u, 0x80008000u, 0x80008000u, 0x80008000u);
    }
    if constexpr (!BULK) {
      const int64_t cn = c + cstride;
      if (cn < a.B) load_row(cn);
    }
    v5_bar<NT>(bar_id);
    // ---- P4: blocked scan over this thread's C positions
    const int k0 = tid * C;
    const unsigned char* xr = xc + tid * XS;
    // per 16-position piece: live values, their (max, first index) by a
    // pairwise tree, folded into the thread's running (max, first index)
    // with strict > (pieces come in position order); one piece of live
    // values in registers at a time
    long long run = 0, best = LLONG_MIN;
    int bi = 0;
    constexpr int PIECE = C >= 16 ? 16 : C;  // class bytes per shared load
#pragma unroll
    for (int p0 = 0; p0 < C; p0 += PIECE) {
      uint32_t cw[PIECE / 4];
      if constexpr (PIECE == 16) {
        const uint4 t = *reinterpret_cast<const uint4*>(xr + p0);
        cw[0] = t.x;
        cw[1] = t.y;
        cw[2] = t.z;
        cw[3] = t.w;
      } else if constexpr (PIECE == 8) {
        const uint2 t = *reinterpret_cast<const uint2*>(xr);
        cw[0] = t.x;
        cw[1] = t.y;
      } else {
        cw[0] = *reinterpret_cast<const uint32_t*>(xr);
      }
      long long lv[PIECE];
#pragma unroll
      for (int i = 0; i < PIECE; ++i) {
        // byte offset class * 256 + lane * 8 in one PRMT (byte 0 <- lane8,
        // byte 1 <- the class byte, bytes 2-3 <- 0)
        const unsigned off = __byte_perm(cw[i >> 2], lane8, 0x7704u | ((i & 3) << 4));
        const long long e = *reinterpret_cast<const long long*>(ltab_b + off);
        lv[i] = run + (long long)((unsigned long long)e >> 32);
        run = lv[i] - (long long)(unsigned)e;
      }
      int ix[PIECE / 2];
#pragma unroll
      for (int p = 0; p < PIECE / 2; ++p) {  // strict >: ties keep the earlier position
        const bool t = lv[2 * p + 1] > lv[2 * p];
        lv[p] = t ? lv[2 * p + 1] : lv[2 * p];
        ix[p] = 2 * p + (t ? 1 : 0);
      }
#pragma unroll
      for (int w = PIECE / 2; w > 1; w >>= 1) {
#pragma unroll
        for (int p = 0; p < w / 2; ++p) {
          const bool t = lv[2 * p + 1] > lv[2 * p];
          lv[p] = t ? lv[2 * p + 1] : lv[2 * p];
          ix[p] = t ? ix[2 * p + 1] : ix[2 * p];
        }
      }
      if (p0 == 0 || lv[0] > best) {
        best = lv[0];
        bi = p0 + ix[0];
      }
    }
    long long incl = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane == 31) red_t[warp] = incl;
    bad = v5_bar_or<NT>(bar_id, bad);
    long long off = incl - run;
#pragma unroll
    for (int w = 0; w < NWARPS - 1; ++w)
      if (w < warp) off += red_t[w];
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
    v5_bar<NT>(bar_id);
    if (tid == 0) {
      long long bv = red_c[0];
      int bk = red_i[0];
#pragma unroll
      for (int w = 1; w < NWARPS; ++w)
        if (red_c[w] > bv) {
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
    int* s_last = red_i + NWARPS;
    if (tid == 0) {
      a.sel.partial[blockIdx.x * a.G + gid] = kbest;
      __threadfence();
      *s_last = atomicAdd(a.sel.counter, 1u) == gridDim.x * (unsigned)a.G - 1u;
    }
    v5_bar<NT>(bar_id);
    if (*s_last) {
      __threadfence();
      const int total = gridDim.x * a.G;
      long long m = LLONG_MAX;
      for (int i = tid; i < total; i += NT) m = min(m, ((volatile long long*)a.sel.partial)[i]);
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, d));
      if (lane == 0) red_c[warp] = m;
      v5_bar<NT>(bar_id);
      if (tid == 0) {
        for (int w = 1; w < NWARPS; ++w) m = min(m, red_c[w]);
        *a.sel.key_out = m;
        *a.sel.counter = 0u;
      }
    }
  }
}

template <typename RowT, int NT, int C, bool BULK, bool WIDE = false>
static int launch_k1v5_t(K1V5Args& a, int grid, size_t smem, cudaStream_t s) {
  auto kern = k1v5_eval_orders<RowT, NT, C, BULK, WIDE>;
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
  RM_LAUNCH_CHECK("k1v5_eval_orders launch");
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

// the instance table must list every (NT, C) k1v4_geometry (roam_graph.cpp)
// picks for a class-form graph
template <typename RowT>
static int launch_k1v5_nt(K1V5Args& a, int NT, int C, bool bulk, bool wide, int grid, size_t smem,
                          cudaStream_t s) {
  if (wide) {  // 8,192 < slots <= 16,384: one 512-thread group per CTA
    if (NT == 512 && C == 32 && !bulk) return launch_k1v5_t<RowT, 512, 32, false, true>(a, grid, smem, s);
    return 1;
  }
#define RM_K1V5_CASE(nt, cc)                                                      \
  if (NT == nt && C == cc)                                                        \
    return bulk ? launch_k1v5_t<RowT, nt, cc, true>(a, grid, smem, s)             \
                : launch_k1v5_t<RowT, nt, cc, false>(a, grid, smem, s);
  RM_K1V5_CASE(32, 4)
  RM_K1V5_CASE(32, 8)
  RM_K1V5_CASE(64, 8)
  RM_K1V5_CASE(96, 8)
  RM_K1V5_CASE(128, 8)
  RM_K1V5_CASE(32, 32)
  RM_K1V5_CASE(64, 32)
  RM_K1V5_CASE(128, 32)
  RM_K1V5_CASE(256, 32)
#undef RM_K1V5_CASE
  return 1;
}

int launch_k1v5(RmGraph* g, const void* orders_dev, int64_t B, int64_t* peak, int32_t* argmax,
                uint8_t* valid, cudaStream_t s, bool u16_rows, const K1KeySel* sel, bool bulk_rows) {
  const K1V5Meta& m = g->k5v;
  const K1V4Meta& m4 = g->k4v;
  if (!m.ok || !m4.ok) return 1;
  const int NT = m4.NT, C = m4.C, SL = m4.SL;
  K1V5Args a{};
  a.orders = orders_dev;
  a.B = B;
  a.n = g->n;
  a.shift = g->k2v.shift;
  a.base = m.base.as<uint8_t>();
  a.tab = m.tab.p;
  a.ncls = m.ncls;
  a.em = m4.em.as<uint32_t>();
  a.edges = m4.edges.as<uint32_t>();
  a.n_edges = (int)m4.n_edges;
  a.dpair = m.dpair.as<uint32_t>();
  a.dtgt = m.dtgt.p;
  a.n_pair = (int)m.n_pair;
  a.g4 = m.g4.p;
  a.n_g4 = (int)m.n_g4;
  a.gptr = m.gptr.as<uint32_t>();
  a.gcons = m.gcons.p;
  a.n_gen = (int)m.n_gen;
  a.n_gcons = (int)m.n_gcons;
  a.peak = peak;
  a.argmax = argmax;
  a.valid = valid;
  if (sel) a.sel = *sel;
  const int xs = C >= 32 ? C + 16 : C == 16 ? 48 : C;  // V5Geom<C>::XS
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device);
  a.off_base = 256 * size_t(a.ncls);
  a.off_edges = align16(a.off_base + size_t(SL + 16));
  a.off_dpair = align16(a.off_edges + 4 * size_t(a.n_edges));
  const bool wide = SL > 8192;
  const size_t fw = wide ? 2 : 1;  // WIDE doubles the target / entry fields
  a.off_dtgt = align16(a.off_dpair + 4 * size_t(a.n_pair));
  a.off_g4 = align16(a.off_dtgt + 4 * fw * size_t(a.n_pair));
  a.off_gptr = align16(a.off_g4 + 8 * fw * size_t(a.n_g4));
  a.off_gcons = align16(a.off_gptr + 4 * size_t(a.n_gen + 1));
  a.off_groups = align16(a.off_gcons + 2 * fw * size_t(a.n_gcons));
  a.off_cls = align16(2 * size_t(SL + 8));
  a.off_xc = align16(a.off_cls + size_t(SL + 16));
  a.off_red = align16(a.off_xc + size_t(NT) * xs);
  if (C >= 32 && NT >= 64 && a.n <= SL / 2) return 1;  // the kernel's JSAFE
  // bulk-copied rows (rm_set_k1_variant(6); C >= 32 geometries): the first
  // half of a row must lie in the copied span (n >= SL/2 + 8).  Measured
  // slower than the register prefetch on GPT-2 small (0.0735 vs 0.0670 ms per
  // 16k candidates): 640 threads at 96 registers raise warps per SM 24 -> 30 %,
  // but the kernel is issue-bound and the shared-memory reads of the staged
  // row add 14 % instructions
  const bool bulk = bulk_rows && C >= 32 && NT >= 64 && a.n >= SL / 2 + 8;
  const int esz = u16_rows ? 2 : 4;
  a.off_rbuf = align16(a.off_red + 3 * 8 * size_t(NT / 32) + 16);
  a.off_mbar = bulk ? align16(a.off_rbuf + size_t(esz) * a.n + 32) : a.off_rbuf;
  a.group_bytes = bulk ? align16(a.off_mbar + 8) : a.off_rbuf;
  const size_t avail = max_smem > (int)a.off_groups ? size_t(max_smem) - a.off_groups : 0;
  const int cap = v5_cta_cap(C, bulk) / NT;
  int G = std::min({(int)(avail / a.group_bytes), cap, 15});
  if (G < 1) return 1;
  const int64_t sms = k1_sms(g->device);
  if (int64_t(G) * sms > B) G = (int)std::max<int64_t>(1, (B + sms - 1) / sms);
  a.G = G;
  const size_t smem = a.off_groups + size_t(G) * a.group_bytes;
  const int grid = (int)std::min<int64_t>(sms, (B + G - 1) / G);
  return u16_rows ? launch_k1v5_nt<uint16_t>(a, NT, C, bulk, wide, grid, smem, s)
                  : launch_k1v5_nt<int32_t>(a, NT, C, bulk, wide, grid, smem, s);
}

}  // namespace roam
