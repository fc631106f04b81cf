// Internal declarations shared by the libroam translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/roam.h"

namespace roam {

// ---- thread-local error reporting ----------------------------------------
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void note_launch(int64_t k = 1);

#define RM_CUDA(call)                                         \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return ::roam::cuda_fail(e_, #call); \
  } while (0)

#define RM_LAUNCH_CHECK(what)                                  \
  do {                                                         \
    ::roam::note_launch();                                     \
    cudaError_t e_ = cudaGetLastError();                       \
    if (e_ != cudaSuccess) return ::roam::cuda_fail(e_, what); \
  } while (0)

// ---- dynamic shared memory opt-in -------------------------------------------
// Always the largest value the kernel can take (device opt-in limit minus its
// static shared memory), never the size of the launch at hand: the library is
// re-entrant, and a per-launch value set by one host thread could shrink the
// limit between another thread's set and launch ("too many resources").
// Done once per (device, kernel); later calls are a locked set lookup.
cudaError_t smem_optin_raw(const void* kern);
template <class Kern>
inline cudaError_t smem_optin(Kern kern) {
  return smem_optin_raw(reinterpret_cast<const void*>(kern));
}

// ---- device buffer owned by a handle --------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf();
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  cudaError_t upload(const void* host, size_t nbytes);
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// Per-call scratch: stream-ordered device allocation freed on scope exit.
struct Scratch {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t st) : s(st) {}
  ~Scratch();
  template <class T>
  cudaError_t alloc(T** out, size_t count) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, count ? count * sizeof(T) : 16, s);
    if (e == cudaSuccess) ptrs.push_back(p);
    *out = static_cast<T*>(p);
    return e;
  }
};

// K1 metadata: the order evaluator never touches the raw CSR.  For a valid
// sequential order o (pos = inverse permutation):
//   live[i] = sum_{j<=i} ( out[o_j] - freed_after[o_{j-1}] )
//   freed_after[v] = fs[v] + sum{ size_t : t multi, argmax_{c in maxC(t)} pos[c] == v }
// where maxC(t) = consumers of t that are not transitive predecessors of
// another consumer (their positions bound every consumer's), fs[v] = summed
// size of tensors with maxC(t) == {v}; zero-consumer tensors are never freed.
// Validity: the permutation plus every edge of the transitive reduction of
// direct_preds (equivalent to all edges for a linear extension).
struct K1Meta {
  int wide = 0;              // 0: uint16 ids, 1: int32 ids
  int64_t n_edges = 0;       // checked edges
  int64_t n_multi = 0;
  int64_t n_multi_cons = 0;
  int64_t n_slots = 0;
  int64_t n_values = 0;
  DevBuf opmeta;             // per op {vidx, slot} (IdxT pair)
  DevBuf table;              // longlong2 {out, fs} [n_values]
  DevBuf edges;              // IdxT pairs (u, v) [n_edges]
  DevBuf mptr;               // int32 [n_multi + 1]
  DevBuf mcons;              // IdxT [n_multi_cons]
  DevBuf msize;              // int64 [n_multi]
};

// K1 v2 metadata (the default order evaluator when the graph qualifies:
// n < 65535, sizes >= 0, per-op byte counts < 2^31 units of 2^shift and the
// frees that can land on one position < 2^32 units).
//   opv[v]  = {out[v] >> shift, fs[v] >> shift} (int2), plus a zero padding op
//   edges   = checked pred edges packed u | v << 16
//   multi-consumer tensors (freed after their latest maximal consumer):
//             mpair = the two-consumer ones as packed u16 pairs; mptr/mcons =
//             the rest as a CSR; msz = size units, pairs first.
struct K1V2Meta {
  int ok = 0;
  int shift = 0;
  int64_t n_pair = 0, n_gen = 0, n_mcons = 0;
  DevBuf opv, edges, mpair, mptr, mcons, msz;
};

// K1 v4 metadata (k_eval_v4.cu; on top of K1V2Meta's opv and generic
// multi-consumer CSR).  Geometry fixed per graph: NT threads per candidate,
// C positions per thread, SL = NT * C slots (ids n..SL-1 are zero-byte
// padding ops, id SL the sink for out-of-range row values).
//   em      = one register word per 8-id chunk: the "not-checked" masks of the SIMD edge checks (u, u+1)
//             and (u, u+2) (roam_graph.cpp build_k1_em)
//   edges   = every other checked edge as byte offsets (2u | 2v << 16), padded
//             with copies of the first one to a multiple of 4*NT
//   mpair   = two-consumer tensors as byte offsets, padded to a multiple of NT
//             with zero-size dummies; msz = their size units, then the
//             generic (>= 3 consumer) tensors' (K1V2Meta mptr/mcons order)
struct K1V4Meta {
  int ok = 0;
  int NT = 0, C = 0, SL = 0;
  int64_t n_edges = 0, n_pair = 0;
  DevBuf em, edges, mpair, msz;
  // class form (ncls > 0 when the graph has <= 255 distinct {out, fs} pairs):
  // cls = class per id [SL + 1] (padding ids: a zero class), tab = int2
  // {fs, out} units per class
  int ncls = 0;
  DevBuf cls, tab;
};

// K1 v5 metadata (k_eval_v5.cu; on top of K1V4Meta's geometry, em and
// generic edges).  One byte per op per candidate: class(v, mask) = base[v] +
// mask, mask bit i set when v is the latest maximal consumer of its i-th
// multi-consumer tensor (build_k1v5_host); ok = 0 when a graph needs more
// than 255 classes or an op has more than 7 multi-consumer tensors.
//   base  = base class per id [SL + 16] (padding ids and the sink: a zero class)
//   tab   = int2 {fs, out} units per class [ncls]
//   dpair = two-consumer tensors as pos byte offsets 2a | 2b << 16, dtgt =
//           their class-bit targets ta | tb << 16 (t = class word index |
//           (8 * (id & 3) + bit index) << 11); lane-interleaved (slot tid +
//           i*NT holds the thread's i-th pair, consecutive lanes far apart),
//           padded to a multiple of NT with target 0xffffffff
//   g4    = the 3-4 consumer tensors, four u16 (id | bit index << 13) each
//           (a short list repeats its first entry), padded to a multiple of
//           NT with 0xe000 entries
//   gptr / gcons = the >= 5 consumer tensors as a CSR of the same u16 entries
struct K1V5Meta {
  int ok = 0;
  int ncls = 0;
  int64_t n_pair = 0, n_g4 = 0, n_gen = 0, n_gcons = 0;
  DevBuf base, tab, dpair, dtgt, g4, gptr, gcons;
};

// Thread-per-candidate generator metadata (k_gen.cu, k_gen_thread): per op
// its direct successors as one u32 each, w | bitoff << 16 | kind << 29, where
// kind 0 = w has one predecessor (ready at once), 1 = two (a toggle bit at
// bitoff of the thread's counter words), k >= 2 = k + 1 predecessors (an
// arrival counter of ceil(log2(k + 1)) bits at bitoff, never straddling a
// word); zero = the ops without predecessors.  ok = 0 when n > 65536, an op
// has more than 8 predecessors or the counters need more than 8192 bits.
struct GenMeta {
  int ok = 0;
  int words = 0;   // counter words per candidate
  int n_zero = 0;
  std::vector<uint32_t> h_eptr, h_edges;
  std::vector<uint16_t> h_zero;
  DevBuf eptr, edges, zero;
};
void build_gen_meta(RmGraph& g);

}  // namespace roam

struct RmGraph {
  int32_t n = 0, T = 0;
  RmGraphInfo info{};
  // host CSR
  std::vector<int64_t> size;
  std::vector<int32_t> producer, cons_ptr, cons_idx, in_ptr, in_idx, out_ptr, out_idx;
  std::vector<int32_t> pred_ptr, pred_idx;   // direct_preds (dedup, sorted, no self)
  std::vector<int32_t> succ_ptr, succ_idx;   // direct_succs
  // host copies of K1 metadata (kept for tests / introspection)
  std::vector<int32_t> h_vidx, h_slot;
  std::vector<int64_t> h_out, h_fs;          // per value class
  std::vector<int32_t> h_edge_u, h_edge_v;
  std::vector<int32_t> h_mptr, h_mcons;
  std::vector<int64_t> h_msize;
  // device side
  int device = -1;
  roam::K1Meta k1;
  roam::K1V2Meta k2v;
  roam::K1V4Meta k4v;
  roam::K1V5Meta k5v;
  roam::GenMeta gen;
  std::vector<int32_t> h2_opv;     // 2n
  std::vector<uint32_t> h2_edges, h2_mpair, h2_mptr, h2_msz;
  std::vector<uint16_t> h2_mcons;
  std::vector<uint32_t> h4_em, h4_edges, h4_mpair, h4_msz;
  std::vector<uint8_t> h4_cls;
  std::vector<int32_t> h4_tab;
  std::vector<uint8_t> h5_base;
  std::vector<int32_t> h5_tab;
  std::vector<uint32_t> h5_dpair, h5_dtgt, h5_gptr, h5_g4;
  std::vector<uint16_t> h5_gcons;
  std::vector<uint32_t> h5_gcons32;  // WIDE v5 (more than 8,192 slots)
  roam::DevBuf d_size, d_producer, d_cons_ptr, d_cons_idx, d_in_ptr, d_in_idx, d_out_ptr,
      d_out_idx, d_pred_ptr, d_pred_idx, d_succ_ptr, d_succ_idx;
};
