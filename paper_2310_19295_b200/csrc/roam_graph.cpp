// Host half of libroam: error plumbing, graph validation/marshalling, and
// the once-per-graph K1 metadata (transitive reduction of direct_preds,
// maximal consumer sets, per-op event classes) described in roam_internal.h.
//
// Reference semantics being restated (pkg/src/memplan/graph.py):
//   direct_preds  97-104  producers of inputs, dedup, self discarded
//   tensor_lifetimes 440-449  birth = ts[producer], death = max ts[consumers]
//                              (horizon if none), clamped >= birth
//   validate_schedule 375-398 permutation + preds-before
#include <algorithm>
#include <array>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <unordered_map>

#include "roam_internal.h"

namespace roam {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return RM_ERR_CUDA;
}
void note_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

cudaError_t smem_optin_raw(const void* kern) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, kern})) return cudaSuccess;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, kern);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done.insert({dev, kern});
  return e;
}

DevBuf::~DevBuf() {
  if (p) cudaFree(p);
}
cudaError_t DevBuf::upload(const void* host, size_t nbytes) {
  // padded to 16 bytes (zeroed) so kernels may stage it with 16-byte loads
  bytes = nbytes;
  const size_t padded = (nbytes + 15) & ~size_t(15);
  cudaError_t e = cudaMalloc(&p, padded ? padded : 16);
  if (e != cudaSuccess) return e;
  if (padded != nbytes || !nbytes) e = cudaMemset(p, 0, padded ? padded : 16);
  if (e == cudaSuccess && nbytes) e = cudaMemcpy(p, host, nbytes, cudaMemcpyHostToDevice);
  return e;
}

Scratch::~Scratch() {
  for (void* p : ptrs) cudaFreeAsync(p, s);
}

static const int kReduceLimit = 20000;  // ops; n^2/8 bytes of reachability bitsets

// Reachability bitsets desc[v] (strict descendants) over direct_succs, in
// reverse topological order.  Returns false on a cycle.
static bool descendants(const RmGraph& g, std::vector<uint64_t>& desc, size_t& words) {
  const int n = g.n;
  words = (size_t(n) + 63) / 64;
  std::vector<int32_t> indeg(n), topo;
  topo.reserve(n);
  for (int v = 0; v < n; ++v) indeg[v] = g.pred_ptr[v + 1] - g.pred_ptr[v];
  for (int v = 0; v < n; ++v)
    if (!indeg[v]) topo.push_back(v);
  for (size_t h = 0; h < topo.size(); ++h) {
    int u = topo[h];
    for (int k = g.succ_ptr[u]; k < g.succ_ptr[u + 1]; ++k)
      if (--indeg[g.succ_idx[k]] == 0) topo.push_back(g.succ_idx[k]);
  }
  if ((int)topo.size() != n) return false;
  desc.assign(words * size_t(n), 0);
  for (int h = n - 1; h >= 0; --h) {
    int u = topo[h];
    uint64_t* du = &desc[size_t(u) * words];
    for (int k = g.succ_ptr[u]; k < g.succ_ptr[u + 1]; ++k) {
      int w = g.succ_idx[k];
      const uint64_t* dw = &desc[size_t(w) * words];
      for (size_t i = 0; i < words; ++i) du[i] |= dw[i];
      du[w >> 6] |= 1ull << (w & 63);
    }
  }
  return true;
}

// K1 v2 metadata (see roam_internal.h).  Leaves g.k2v.ok = 0 when the graph
// does not qualify; the generic evaluator then runs.
static void build_k1v2_host(RmGraph& g, const std::vector<int64_t>& out,
                            const std::vector<int64_t>& fs) {
  const int n = g.n, T = g.T;
  g.k2v.ok = 0;
  if (n > 65532) return;  // ids and the three dummy ops fit 16 bits
  int shift = 62;
  for (int t = 0; t < T; ++t) {
    if (g.size[t] < 0) return;
    if (g.size[t] > 0) shift = std::min(shift, __builtin_ctzll((unsigned long long)g.size[t]));
  }
  if (shift == 62) shift = 0;
  const int64_t lim = INT32_MAX;
  // {fs, out} units per op (one 64-bit word: fs | out << 32), zero-byte
  // entries beyond n for the evaluators' padding ids (<= max(2n, 1024))
  g.h2_opv.assign(2 * (size_t(std::max(2 * n, 1024)) + 4), 0);
  for (int v = 0; v < n; ++v) {
    if ((out[v] >> shift) > lim || (fs[v] >> shift) > lim) return;
    g.h2_opv[2 * v] = (int32_t)(fs[v] >> shift);
    g.h2_opv[2 * v + 1] = (int32_t)(out[v] >> shift);
  }
  g.h2_edges.resize(g.h_edge_u.size());
  for (size_t e = 0; e < g.h_edge_u.size(); ++e)
    g.h2_edges[e] = (uint32_t)g.h_edge_u[e] | ((uint32_t)g.h_edge_v[e] << 16);
  // multi-consumer tensors: two-consumer ones first as packed pairs (the
  // common case), the rest as a CSR; sizes in units
  const size_t M = g.h_msize.size();
  std::vector<int64_t> worst(n);
  for (int v = 0; v < n; ++v) worst[v] = fs[v] >> shift;
  g.h2_mpair.clear();
  g.h2_mptr.assign(1, 0);
  g.h2_mcons.clear();
  std::vector<uint32_t> sz_pair, sz_gen;
  for (size_t m = 0; m < M; ++m) {
    const int64_t u = g.h_msize[m] >> shift;
    if (u > (int64_t)UINT32_MAX) return;
    const int q0 = g.h_mptr[m], q1 = g.h_mptr[m + 1];
    for (int q = q0; q < q1; ++q) worst[g.h_mcons[q]] += u;
    if (q1 - q0 == 2) {
      g.h2_mpair.push_back((uint32_t)g.h_mcons[q0] | ((uint32_t)g.h_mcons[q0 + 1] << 16));
      sz_pair.push_back((uint32_t)u);
    } else {
      for (int q = q0; q < q1; ++q) g.h2_mcons.push_back((uint16_t)g.h_mcons[q]);
      g.h2_mptr.push_back((uint32_t)g.h2_mcons.size());
      sz_gen.push_back((uint32_t)u);
    }
  }
  // sizes: pairs first, then the generic tensors
  g.h2_msz = sz_pair;
  g.h2_msz.insert(g.h2_msz.end(), sz_gen.begin(), sz_gen.end());
  // the frees that land on one position are added into a 32-bit field:
  // bound each op's worst case (its single-consumer frees plus every
  // multi-consumer tensor it may close)
  for (int v = 0; v < n; ++v)
    if (worst[v] > (int64_t)UINT32_MAX) return;
  g.k2v.n_pair = (int64_t)g.h2_mpair.size();
  g.k2v.n_gen = (int64_t)sz_gen.size();
  g.k2v.shift = shift;
  g.k2v.n_mcons = (int64_t)g.h2_mcons.size();
  g.k2v.ok = 1;
}

// K1 v4 geometry: the smallest slot count SL = NT * C >= n among the compiled
// instances (k_eval_v4.cu launch table).  C positions per thread: 8 up to 1k
// ops; 32 up to 2k (two-warp groups, 128 registers: GPT-2 small 0.082 vs
// 0.090 ms per 16k candidates at C = 16) and up to 8k when the per-op table
// has a class form (GPT2-XL 0.197 vs 0.209 ms per 8k); 16 otherwise (32
// would halve the resident warps once a group's shared memory grows).
// ROAM_K1_C=16|32|64 forces C where an instance exists (A/B runs).
static bool k1v4_geometry(int n, bool classes, int& NT, int& C) {
  static const int cenv = [] {
    const char* e = std::getenv("ROAM_K1_C");
    return e ? std::atoi(e) : 0;
  }();
  const int want = cenv ? cenv : (n > 1024 && (n <= 2048 || (classes && n <= 16384)) ? 32 : 0);
  if (want == 32 || want == 64) {
    static const int nts[] = {32, 64, 128, 256, 512};
    for (int nt : nts)
      if (nt * want >= n && (want == 32 || nt <= 128)) {
        NT = nt;
        C = want;
        return true;
      }
  }
  static const int nt8[] = {32, 64, 96, 128};
  static const int nt16[] = {64, 96, 128, 160, 192, 256, 320, 384, 512, 640, 768, 1024};
  if (n <= 128) {
    NT = 32;
    C = 4;
    return true;
  }
  for (int nt : nt8)
    if (nt * 8 >= n) {
      NT = nt;
      C = 8;
      return true;
    }
  for (int nt : nt16)
    if (nt * 16 >= n) {
      NT = nt;
      C = 16;
      return true;
    }
  return false;
}

// Bank-aware lane assignment for the per-candidate gather lists (v4/v5):
// entry e of a list sits at slot tid + i * NT, and the 32 slots of one
// (warp, i) are one shared-memory instruction per address they touch.
// bank[e][c] = the bank (address class) entry e touches in access c of that
// instruction; lanes sharing a bank with different words serialise.  Groups
// of 32 are filled greedily with the entry adding the fewest collisions
// (ties: the lowest index), then laid out group by group.  Order never
// matters to the kernels (every entry's result is OR-ed / atomically added).
template <int NC>
static std::vector<size_t> bank_aware_order(const std::vector<std::array<int, NC>>& bank, int NT) {
  const size_t E = bank.size();
  std::vector<size_t> out;
  if (E == 0 || NT % 32) {
    for (size_t e = 0; e < E; ++e) out.push_back(e);
    return out;
  }
  const size_t rounds = (E + NT - 1) / NT, warps = size_t(NT) / 32;
  std::vector<std::vector<size_t>> groups(rounds * warps);
  std::vector<char> used(E, 0);
  size_t left = E;
  for (size_t gi = 0; gi < groups.size() && left; ++gi) {
    int cnt[NC][32] = {};
    for (int lane = 0; lane < 32 && left; ++lane) {
      size_t best = E;
      int best_cost = 1 << 30;
      for (size_t e = 0; e < E; ++e) {
        if (used[e]) continue;
        int cost = 0;
        for (int c = 0; c < NC; ++c) cost += bank[e][c] >= 0 ? cnt[c][bank[e][c]] : 0;
        if (cost < best_cost) {
          best_cost = cost;
          best = e;
          if (cost == 0) break;
        }
      }
      used[best] = 1;
      --left;
      for (int c = 0; c < NC; ++c)
        if (bank[best][c] >= 0) cnt[c][bank[best][c]]++;
      groups[gi].push_back(best);
    }
  }
  // group (i, w) -> slots w*32 + lane + i*NT
  out.assign(rounds * size_t(NT), E);
  for (size_t i = 0; i < rounds; ++i)
    for (size_t w = 0; w < warps; ++w) {
      const auto& gr = groups[i * warps + w];
      for (size_t l = 0; l < gr.size(); ++l) out[w * 32 + l + i * size_t(NT)] = gr[l];
    }
  return out;  // E marks an empty slot
}

// K1 v4 metadata (see roam_internal.h); needs the v2 layout (unit-packed
// opv, 32-bit free fields) and 15-bit positions.
static void build_k1v4_host(RmGraph& g) {
  g.k4v.ok = 0;
  const int n = g.n;
  int NT = 0, C = 0;
  if (!g.k2v.ok || !k1v4_geometry(n, g.h_out.size() < 255, NT, C)) return;
  const int SL = NT * C;
  if (SL + 8 > 32768) return;
  if (g.h2_opv.size() < 2 * size_t(SL + 1)) g.h2_opv.resize(2 * size_t(SL + 1), 0);
  std::vector<uint32_t> gen;  // edges the SIMD masks (build_k1_em) do not cover
  for (size_t e = 0; e < g.h_edge_u.size(); ++e) {
    const int u = g.h_edge_u[e], v = g.h_edge_v[e];
    if (v - u != 1 && v - u != 2) gen.push_back((uint32_t)(2 * u) | ((uint32_t)(2 * v) << 16));
  }
  if (!gen.empty()) {
    // lanes of one gather instruction on distinct banks (pos is u16: id u at
    // byte 2u, bank (u >> 1) & 31); empty slots repeat the first edge (a
    // broadcast, no conflict); the list is padded to a multiple of 4 * NT
    std::vector<std::array<int, 2>> bank(gen.size());
    for (size_t e = 0; e < gen.size(); ++e)
      bank[e] = {int(((gen[e] & 0xffffu) >> 2) & 31), int(((gen[e] >> 16) >> 2) & 31)};
    const std::vector<size_t> ord = bank_aware_order<2>(bank, NT);
    std::vector<uint32_t> laid(ord.size());
    for (size_t k = 0; k < ord.size(); ++k) laid[k] = ord[k] < gen.size() ? gen[ord[k]] : gen[0];
    gen = laid;
    const size_t pad = 4 * size_t(NT);
    const uint32_t first = gen[0];
    while (gen.size() % pad) gen.push_back(first);
  }
  g.h4_edges = gen;
  g.h4_mpair.clear();
  g.h4_msz.clear();
  for (size_t m = 0; m < g.h2_mpair.size(); ++m) {
    const uint32_t w = g.h2_mpair[m];
    g.h4_mpair.push_back(((w & 0xffffu) << 1) | ((w >> 16) << 17));
    g.h4_msz.push_back(g.h2_msz[m]);
  }
  // padding pairs (zero size) name one id twice, a different id each, so
  // their free atomics land on distinct slots: a padding list that all
  // pointed at id 0 serialised its 32 lanes on one address (ncu: 40
  // wavefronts per candidate for that one ATOMS)
  for (uint32_t i = 0; g.h4_mpair.size() % NT; ++i) {
    const uint32_t id = n > 0 ? i % (uint32_t)n : 0u;
    g.h4_mpair.push_back((id << 1) | (id << 17));
    g.h4_msz.push_back(0);
  }
  g.h4_msz.insert(g.h4_msz.end(), g.h2_msz.begin() + g.h2_mpair.size(), g.h2_msz.end());
  // class form: one byte per id into a table of {fs, out} units
  g.k4v.ncls = 0;
  g.h4_cls.clear();
  g.h4_tab.clear();
  if (g.h_out.size() < 255) {
    int zero = -1;
    for (size_t c = 0; c < g.h_out.size(); ++c) {
      g.h4_tab.push_back((int32_t)(g.h_fs[c] >> g.k2v.shift));
      g.h4_tab.push_back((int32_t)(g.h_out[c] >> g.k2v.shift));
      if (g.h_out[c] == 0 && g.h_fs[c] == 0) zero = (int)c;
    }
    if (zero < 0) {
      zero = (int)g.h_out.size();
      g.h4_tab.push_back(0);
      g.h4_tab.push_back(0);
    }
    g.h4_cls.assign(size_t(SL + 1), (uint8_t)zero);
    for (int v = 0; v < n; ++v) g.h4_cls[v] = (uint8_t)g.h_vidx[v];
    g.k4v.ncls = (int)(g.h4_tab.size() / 2);
  }
  g.k4v.NT = NT;
  g.k4v.C = C;
  g.k4v.SL = SL;
  g.k4v.n_edges = (int64_t)g.h4_edges.size();
  g.k4v.n_pair = (int64_t)g.h4_mpair.size();
  g.k4v.ok = 1;
}

// K1 v5 metadata (see roam_internal.h K1V5Meta).  An op's events in one
// candidate are its static frees and outputs plus, for each multi-consumer
// tensor it is a maximal consumer of, whether it is the latest one: every
// distinct signature (fs, out, those tensors' sizes) gets a block of 2^m
// consecutive classes, class = block base + mask.
static void build_k1v5_host(RmGraph& g) {
  g.k5v.ok = 0;
  if (!g.k4v.ok || !g.k2v.ok) return;
  const int n = g.n, SL = g.k4v.SL, NT = g.k4v.NT;
  if (SL > 16384) return;
  // up to 8,192 slots a consumer id and its 3-bit bit index share 16 bits;
  // beyond (WIDE) every entry is 32 bits: id | bit << 16, word | shift << 16
  const bool wide = SL > 8192;
  const uint32_t IDB = wide ? 16 : 13, TWB = wide ? 16 : 11;
  const int shift = g.k2v.shift;
  const size_t M = g.h_msize.size();
  std::vector<std::vector<int>> dyn(n);
  for (size_t m = 0; m < M; ++m)
    for (int q = g.h_mptr[m]; q < g.h_mptr[m + 1]; ++q) dyn[g.h_mcons[q]].push_back((int)m);
  std::map<std::vector<int64_t>, int> blocks;
  std::vector<int32_t> tab;
  auto block = [&](const std::vector<int64_t>& sig) -> int {
    auto it = blocks.find(sig);
    if (it != blocks.end()) return it->second;
    const int b = (int)(tab.size() / 2), m = (int)sig.size() - 2;
    for (int mask = 0; mask < (1 << m); ++mask) {
      int64_t f = sig[0];
      for (int i = 0; i < m; ++i)
        if (mask >> i & 1) f += sig[2 + i];
      tab.push_back((int32_t)(uint32_t)f);  // <= UINT32_MAX (build_k1v2_host's bound)
      tab.push_back((int32_t)sig[1]);
    }
    blocks.emplace(sig, b);
    return b;
  };
  std::vector<uint8_t> base(size_t(SL + 16), 0);
  const int zero = block({0, 0});
  std::fill(base.begin(), base.end(), (uint8_t)zero);
  for (int v = 0; v < n; ++v) {
    const int m = (int)dyn[v].size();
    if (m > 7) return;
    std::vector<int64_t> sig = {g.h_fs[g.h_vidx[v]] >> shift, g.h_out[g.h_vidx[v]] >> shift};
    for (int t : dyn[v]) sig.push_back(g.h_msize[t] >> shift);
    const int b = block(sig);
    if (b + (1 << m) > 256) return;
    base[v] = (uint8_t)b;
  }
  auto idx_of = [&](int v, int t) {
    return (uint32_t)(std::find(dyn[v].begin(), dyn[v].end(), t) - dyn[v].begin());
  };
  std::vector<uint32_t> pw;
  auto target = [&](int v, int t) {  // class word of v | bit shift << TWB
    return (uint32_t)(v >> 2) | ((uint32_t)(8 * (v & 3)) + idx_of(v, t)) << TWB;
  };
  g.h5_gptr.assign(1, 0);
  g.h5_gcons.clear();
  g.h5_gcons32.clear();
  g.h5_g4.clear();
  std::vector<uint64_t> pt;  // {ta, tb} per pair (packed ta | tb << 16 narrow, a u32 pair WIDE)
  for (size_t m = 0; m < M; ++m) {
    const int q0 = g.h_mptr[m], q1 = g.h_mptr[m + 1];
    if (q1 - q0 == 2) {
      const int a = g.h_mcons[q0], b = g.h_mcons[q0 + 1];
      pw.push_back((uint32_t)(2 * a) | ((uint32_t)(2 * b) << 16));
      pt.push_back((uint64_t)target(a, (int)m) | ((uint64_t)target(b, (int)m) << 32));
    } else if (q1 - q0 <= 4) {
      uint32_t e[4];
      for (int q = q0; q < q0 + 4; ++q) {
        const int c = g.h_mcons[q < q1 ? q : q0];
        e[q - q0] = (uint32_t)c | (idx_of(c, (int)m) << IDB);
      }
      if (wide) {
        for (int q = 0; q < 4; ++q) g.h5_g4.push_back(e[q]);
      } else {
        g.h5_g4.push_back(e[0] | (e[1] << 16));
        g.h5_g4.push_back(e[2] | (e[3] << 16));
      }
    } else {
      for (int q = q0; q < q1; ++q) {
        const int c = g.h_mcons[q];
        const uint32_t e = (uint32_t)c | (idx_of(c, (int)m) << IDB);
        if (wide) g.h5_gcons32.push_back(e);
        else g.h5_gcons.push_back((uint16_t)e);
      }
      g.h5_gptr.push_back((uint32_t)(wide ? g.h5_gcons32.size() : g.h5_gcons.size()));
    }
  }
  const size_t g4w = wide ? 4 : 2;  // u32 words per 3-4-consumer tensor
  while ((g.h5_g4.size() / g4w) % NT) {
    if (wide) g.h5_g4.insert(g.h5_g4.end(), 4, 0x70000u);  // id 0 | bit 7: never a real entry
    else g.h5_g4.push_back(0xe000e000u);
  }
  // bank-aware lanes: the lanes of one instruction gather pos[a], pos[b]
  // from distinct banks and add to distinct class words / banks (same-word
  // atomics from one instruction serialise); padding slots read pos[0] and
  // hold target 0xffffffff, which the kernel predicates off
  const size_t P = pw.size();
  const uint32_t wmask = (1u << TWB) - 1u;
  std::vector<std::array<int, 4>> bank(P);
  for (size_t e = 0; e < P; ++e)
    bank[e] = {int(((pw[e] & 0xffffu) >> 2) & 31), int(((pw[e] >> 16) >> 2) & 31),
               int(((uint32_t)pt[e] & wmask) & 31), int(((uint32_t)(pt[e] >> 32) & wmask) & 31)};
  const std::vector<size_t> ord = bank_aware_order<4>(bank, NT);
  g.h5_dpair.assign(ord.size(), 0u);
  g.h5_dtgt.assign(ord.size() * (wide ? 2 : 1), 0xffffffffu);
  for (size_t k = 0; k < ord.size(); ++k)
    if (ord[k] < P) {
      const uint64_t t = pt[ord[k]];
      g.h5_dpair[k] = pw[ord[k]];
      if (wide) {
        g.h5_dtgt[2 * k] = (uint32_t)t;
        g.h5_dtgt[2 * k + 1] = (uint32_t)(t >> 32);
      } else {
        g.h5_dtgt[k] = (uint32_t)t | ((uint32_t)(t >> 32) << 16);
      }
    }
  g.h5_base = base;
  g.h5_tab = tab;
  g.k5v.ncls = (int)(tab.size() / 2);
  g.k5v.n_pair = (int64_t)g.h5_dpair.size();
  g.k5v.n_g4 = (int64_t)(g.h5_g4.size() / g4w);
  g.k5v.n_gen = (int64_t)g.h5_gptr.size() - 1;
  g.k5v.n_gcons = (int64_t)(wide ? g.h5_gcons32.size() : g.h5_gcons.size());
  g.k5v.ok = 1;
}

// SIMD edge-mask words of K1 v4, em[q] (one per 8-id chunk q, held in a
// register by the thread owning the chunk): bit 15-m / 31-m = edge
// (8q+2m, 8q+2m+1) / (8q+2m+1, 8q+2m+2) NOT checked, bit 11-m / 27-m = the
// same for (8q+2m, 8q+2m+2) / (8q+2m+1, 8q+2m+3), so (em << m) and
// (em << (m + 4)) put word m's masks on bits 15 and 31.  Sized for every
// chunk either geometry reads.
static void build_k1_em(RmGraph& g) {
  const size_t chunks = g.k4v.ok ? size_t(g.k4v.SL / 8) : 0;
  g.h4_em.assign(chunks, 0xff00ff00u);
  if (!chunks) return;
  for (size_t e = 0; e < g.h_edge_u.size(); ++e) {
    const int u = g.h_edge_u[e], v = g.h_edge_v[e];
    const int d = v - u, m = (u & 7) >> 1, hi = u & 1;
    if (d == 1) g.h4_em[u >> 3] &= ~(1u << (15 - m + 16 * hi));
    if (d == 2) g.h4_em[u >> 3] &= ~(1u << (11 - m + 16 * hi));
  }
}

static int build_k1_host(RmGraph& g, bool allow_reduce) {
  const int n = g.n, T = g.T;
  std::vector<uint64_t> desc;
  size_t words = 0;
  bool reduced = allow_reduce && n <= kReduceLimit && n > 0 && descendants(g, desc, words);
  auto reach = [&](int a, int b) {  // b is a strict descendant of a
    return (desc[size_t(a) * words + (b >> 6)] >> (b & 63)) & 1ull;
  };

  // checked edges: transitive reduction of direct_preds (or all of them)
  g.h_edge_u.clear();
  g.h_edge_v.clear();
  std::vector<uint64_t> R(reduced ? words : 0);
  for (int u = 0; u < n; ++u) {
    if (reduced) {
      std::fill(R.begin(), R.end(), 0);
      for (int k = g.succ_ptr[u]; k < g.succ_ptr[u + 1]; ++k) {
        const uint64_t* dw = &desc[size_t(g.succ_idx[k]) * words];
        for (size_t i = 0; i < words; ++i) R[i] |= dw[i];
      }
    }
    for (int k = g.succ_ptr[u]; k < g.succ_ptr[u + 1]; ++k) {
      int v = g.succ_idx[k];
      if (reduced && ((R[v >> 6] >> (v & 63)) & 1ull)) continue;
      g.h_edge_u.push_back(u);
      g.h_edge_v.push_back(v);
    }
  }

  // births and frees
  std::vector<int64_t> out(n, 0), fs(n, 0);
  for (int t = 0; t < T; ++t) out[g.producer[t]] += g.size[t];
  g.h_mptr.assign(1, 0);
  g.h_mcons.clear();
  g.h_msize.clear();
  std::vector<int32_t> C, maxc;
  for (int t = 0; t < T; ++t) {
    C.assign(g.cons_idx.begin() + g.cons_ptr[t], g.cons_idx.begin() + g.cons_ptr[t + 1]);
    if (C.empty()) continue;  // graph output: live to the horizon, never freed
    std::sort(C.begin(), C.end());
    C.erase(std::unique(C.begin(), C.end()), C.end());
    maxc.clear();
    for (int c : C) {
      bool dominated = false;
      if (reduced)
        for (int c2 : C)
          if (c2 != c && reach(c, c2)) { dominated = true; break; }
      if (!dominated) maxc.push_back(c);
    }
    if (maxc.size() == 1) {
      fs[maxc[0]] += g.size[t];
    } else {
      for (int c : maxc) g.h_mcons.push_back(c);
      g.h_mptr.push_back((int32_t)g.h_mcons.size());
      g.h_msize.push_back(g.size[t]);
    }
  }

  // per-op event classes (distinct (out, fs) pairs, first-appearance order)
  std::map<std::pair<int64_t, int64_t>, int32_t> cls;
  g.h_vidx.assign(n, 0);
  g.h_out.clear();
  g.h_fs.clear();
  for (int v = 0; v < n; ++v) {
    auto key = std::make_pair(out[v], fs[v]);
    auto it = cls.find(key);
    if (it == cls.end()) {
      it = cls.emplace(key, (int32_t)g.h_out.size()).first;
      g.h_out.push_back(out[v]);
      g.h_fs.push_back(fs[v]);
    }
    g.h_vidx[v] = it->second;
  }
  // slots: ops that can close a multi-consumer lifetime
  g.h_slot.assign(n, -1);
  int32_t K = 0;
  for (int32_t c : g.h_mcons)
    if (g.h_slot[c] < 0) g.h_slot[c] = K++;

  build_k1v2_host(g, out, fs);
  build_k1v4_host(g);
  build_k1_em(g);
  build_k1v5_host(g);

  RmGraphInfo& I = g.info;
  I.k1_variant = g.k5v.ok ? 5 : g.k4v.ok ? 4 : 1;
  I.unit_shift = g.k2v.shift;
  I.n_check_edges = (int64_t)g.h_edge_u.size();
  I.n_multi = (int64_t)g.h_msize.size();
  I.n_multi_cons = (int64_t)g.h_mcons.size();
  I.n_slots = K;
  I.n_values = (int64_t)g.h_out.size();
  I.reduced = reduced ? 1 : 0;
  I.wide_index = n > 65535 ? 1 : 0;
  return RM_OK;
}

template <class IdxT>
static cudaError_t upload_k1(RmGraph& g) {
  const int n = g.n;
  const IdxT none = (IdxT)-1;
  std::vector<IdxT> om(2 * size_t(n));
  for (int v = 0; v < n; ++v) {
    om[2 * v] = (IdxT)g.h_vidx[v];
    om[2 * v + 1] = g.h_slot[v] < 0 ? none : (IdxT)g.h_slot[v];
  }
  std::vector<int64_t> tab(2 * g.h_out.size());
  for (size_t i = 0; i < g.h_out.size(); ++i) {
    tab[2 * i] = g.h_out[i];
    tab[2 * i + 1] = g.h_fs[i];
  }
  std::vector<IdxT> ed(2 * g.h_edge_u.size());
  for (size_t i = 0; i < g.h_edge_u.size(); ++i) {
    ed[2 * i] = (IdxT)g.h_edge_u[i];
    ed[2 * i + 1] = (IdxT)g.h_edge_v[i];
  }
  std::vector<IdxT> mc(g.h_mcons.begin(), g.h_mcons.end());
  cudaError_t e;
  if ((e = g.k1.opmeta.upload(om.data(), om.size() * sizeof(IdxT)))) return e;
  if ((e = g.k1.table.upload(tab.data(), tab.size() * sizeof(int64_t)))) return e;
  if ((e = g.k1.edges.upload(ed.data(), ed.size() * sizeof(IdxT)))) return e;
  if ((e = g.k1.mptr.upload(g.h_mptr.data(), g.h_mptr.size() * sizeof(int32_t)))) return e;
  if ((e = g.k1.mcons.upload(mc.data(), mc.size() * sizeof(IdxT)))) return e;
  if ((e = g.k1.msize.upload(g.h_msize.data(), g.h_msize.size() * sizeof(int64_t)))) return e;
  return cudaSuccess;
}

template <class V>
static cudaError_t up(DevBuf& b, const std::vector<V>& v) {
  return b.upload(v.data(), v.size() * sizeof(V));
}

}  // namespace roam

using namespace roam;

extern "C" {

const char* rm_last_error(void) { return g_last_error.c_str(); }
int64_t rm_launch_count(void) { return g_launches.load(); }

int rm_device_count(int* count) {
  if (!count) return fail(RM_ERR_INVALID_ARG, "count is NULL");
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *count = c;
  return RM_OK;
}

static bool csr_ok(const int32_t* ptr, int32_t rows, int64_t* total) {
  if (rows < 0) return false;
  if (!ptr) return rows == 0 ? (*total = 0, true) : false;
  if (ptr[0] != 0) return false;
  for (int32_t i = 0; i < rows; ++i)
    if (ptr[i + 1] < ptr[i]) return false;
  *total = ptr[rows];
  return true;
}

int rm_graph_create(const RmGraphDesc* d, uint32_t flags, RmGraph** out) {
  if (!d || !out) return fail(RM_ERR_INVALID_ARG, "desc/out is NULL");
  *out = nullptr;
  const int32_t n = d->n_ops, T = d->n_tensors;
  if (n < 0 || T < 0) return fail(RM_ERR_INVALID_ARG, "negative op/tensor count");
  if (T > 0 && (!d->size || !d->producer)) return fail(RM_ERR_INVALID_ARG, "size/producer NULL");
  int64_t E = 0, Ein = 0, Eout = 0;
  if (!csr_ok(d->cons_ptr, T, &E) || !csr_ok(d->in_ptr, n, &Ein) || !csr_ok(d->out_ptr, n, &Eout))
    return fail(RM_ERR_INVALID_ARG, "malformed CSR pointer array");
  if ((E && !d->cons_idx) || (Ein && !d->in_idx) || (Eout && !d->out_idx))
    return fail(RM_ERR_INVALID_ARG, "CSR index array NULL");

  RmGraph* g = new RmGraph();
  g->n = n;
  g->T = T;
  g->size.assign(d->size, d->size + T);
  g->producer.assign(d->producer, d->producer + T);
  g->cons_ptr.assign(d->cons_ptr, d->cons_ptr + T + 1);
  g->cons_idx.assign(d->cons_idx, d->cons_idx + E);
  g->in_ptr.assign(d->in_ptr, d->in_ptr + n + 1);
  g->in_idx.assign(d->in_idx, d->in_idx + Ein);
  g->out_ptr.assign(d->out_ptr, d->out_ptr + n + 1);
  g->out_idx.assign(d->out_idx, d->out_idx + Eout);
  if (T == 0) g->cons_ptr.assign(1, 0);
  auto bad = [&](const std::string& m) {
    delete g;
    return fail(RM_ERR_GRAPH, m);
  };
  int64_t total = 0;
  for (int t = 0; t < T; ++t) {
    if (g->producer[t] < 0 || g->producer[t] >= n) return bad("producer out of range");
    int64_t s = g->size[t];
    uint64_t a = s < 0 ? 0ull - (uint64_t)s : (uint64_t)s;
    if (a >= (1ull << 62) || (uint64_t)total + a >= (1ull << 62)) {
      delete g;
      return fail(RM_ERR_OVERFLOW, "summed tensor sizes exceed 2^62 bytes");
    }
    total += (int64_t)a;
  }
  for (int64_t k = 0; k < E; ++k)
    if (g->cons_idx[k] < 0 || g->cons_idx[k] >= n) return bad("consumer out of range");
  for (int64_t k = 0; k < Ein; ++k)
    if (g->in_idx[k] < 0 || g->in_idx[k] >= T) return bad("input tensor out of range");
  for (int64_t k = 0; k < Eout; ++k)
    if (g->out_idx[k] < 0 || g->out_idx[k] >= T) return bad("output tensor out of range");

  // direct_preds (graph.py:97-104) and its transpose
  g->pred_ptr.assign(n + 1, 0);
  std::vector<int32_t> tmp;
  for (int v = 0; v < n; ++v) {
    tmp.clear();
    for (int k = g->in_ptr[v]; k < g->in_ptr[v + 1]; ++k) {
      int p = g->producer[g->in_idx[k]];
      if (p != v) tmp.push_back(p);
    }
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    g->pred_idx.insert(g->pred_idx.end(), tmp.begin(), tmp.end());
    g->pred_ptr[v + 1] = (int32_t)g->pred_idx.size();
  }
  g->succ_ptr.assign(n + 1, 0);
  for (int32_t p : g->pred_idx) g->succ_ptr[p + 1]++;
  for (int v = 0; v < n; ++v) g->succ_ptr[v + 1] += g->succ_ptr[v];
  g->succ_idx.resize(g->pred_idx.size());
  {
    std::vector<int32_t> cur(g->succ_ptr.begin(), g->succ_ptr.end() - 1);
    for (int v = 0; v < n; ++v)  // ascending v keeps each succ list sorted
      for (int k = g->pred_ptr[v]; k < g->pred_ptr[v + 1]; ++k) g->succ_idx[cur[g->pred_idx[k]]++] = v;
  }

  RmGraphInfo& I = g->info;
  I.n_ops = n;
  I.n_tensors = T;
  I.n_cons = E;
  I.n_pred_edges = (int64_t)g->pred_idx.size();
  I.total_bytes = total;
  int st = build_k1_host(*g, !(flags & RM_NO_REDUCE));
  if (st != RM_OK) {
    delete g;
    return st;
  }

  build_gen_meta(*g);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
    cudaGetLastError();
    ndev = 0;
  }
  if (ndev > 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    g->device = dev;
    // keep freed stream-ordered scratch cached in the device's default pool
    // (every call allocates its scratch with cudaMallocAsync)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    cudaError_t e = g->info.wide_index ? upload_k1<int32_t>(*g) : upload_k1<uint16_t>(*g);
    if (!e && g->k2v.ok) e = up(g->k2v.opv, g->h2_opv);
    if (!e && g->k2v.ok) e = up(g->k2v.edges, g->h2_edges);
    if (!e && g->k2v.ok) e = up(g->k2v.mpair, g->h2_mpair);
    if (!e && g->k2v.ok) e = up(g->k2v.mptr, g->h2_mptr);
    if (!e && g->k2v.ok) e = up(g->k2v.mcons, g->h2_mcons);
    if (!e && g->k2v.ok) e = up(g->k2v.msz, g->h2_msz);
    if (!e && g->k4v.ok) e = up(g->k4v.edges, g->h4_edges);
    if (!e && g->k4v.ok) e = up(g->k4v.mpair, g->h4_mpair);
    if (!e && g->k4v.ok) e = up(g->k4v.msz, g->h4_msz);
    if (!e && g->k4v.ok) e = up(g->k4v.em, g->h4_em);
    if (!e && g->k4v.ok && g->k4v.ncls) e = up(g->k4v.cls, g->h4_cls);
    if (!e && g->k4v.ok && g->k4v.ncls) e = up(g->k4v.tab, g->h4_tab);
    if (!e && g->k5v.ok) e = up(g->k5v.base, g->h5_base);
    if (!e && g->k5v.ok) e = up(g->k5v.tab, g->h5_tab);
    if (!e && g->k5v.ok) e = up(g->k5v.dpair, g->h5_dpair);
    if (!e && g->k5v.ok) e = up(g->k5v.dtgt, g->h5_dtgt);
    if (!e && g->k5v.ok) e = up(g->k5v.g4, g->h5_g4);
    if (!e && g->k5v.ok) e = up(g->k5v.gptr, g->h5_gptr);
    if (!e && g->k5v.ok) e = g->h5_gcons32.empty() ? up(g->k5v.gcons, g->h5_gcons) : up(g->k5v.gcons, g->h5_gcons32);
    if (!e && g->gen.ok) e = up(g->gen.eptr, g->gen.h_eptr);
    if (!e && g->gen.ok) e = up(g->gen.edges, g->gen.h_edges);
    if (!e && g->gen.ok) e = up(g->gen.zero, g->gen.h_zero);
    if (!e) e = up(g->d_size, g->size);
    if (!e) e = up(g->d_producer, g->producer);
    if (!e) e = up(g->d_cons_ptr, g->cons_ptr);
    if (!e) e = up(g->d_cons_idx, g->cons_idx);
    if (!e) e = up(g->d_in_ptr, g->in_ptr);
    if (!e) e = up(g->d_in_idx, g->in_idx);
    if (!e) e = up(g->d_out_ptr, g->out_ptr);
    if (!e) e = up(g->d_out_idx, g->out_idx);
    if (!e) e = up(g->d_pred_ptr, g->pred_ptr);
    if (!e) e = up(g->d_pred_idx, g->pred_idx);
    if (!e) e = up(g->d_succ_ptr, g->succ_ptr);
    if (!e) e = up(g->d_succ_idx, g->succ_idx);
    if (e) {
      delete g;
      return cuda_fail(e, "rm_graph_create upload");
    }
  }
  *out = g;
  return RM_OK;
}

int rm_graph_destroy(RmGraph* g) {
  delete g;
  return RM_OK;
}

int rm_graph_info(const RmGraph* g, RmGraphInfo* info) {
  if (!g || !info) return fail(RM_ERR_INVALID_ARG, "NULL argument");
  *info = g->info;
  return RM_OK;
}

int rm_graph_k1_export(const RmGraph* g, int32_t* vidx, int32_t* slot, int64_t* out_tab,
                       int64_t* fs_tab, int32_t* edge_u, int32_t* edge_v, int32_t* mptr,
                       int32_t* mcons, int64_t* msize) {
  if (!g) return fail(RM_ERR_INVALID_ARG, "NULL graph");
  auto cp = [](auto* dst, const auto& src) {
    if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(src[0]));
  };
  cp(vidx, g->h_vidx);
  cp(slot, g->h_slot);
  cp(out_tab, g->h_out);
  cp(fs_tab, g->h_fs);
  cp(edge_u, g->h_edge_u);
  cp(edge_v, g->h_edge_v);
  cp(mptr, g->h_mptr);
  cp(mcons, g->h_mcons);
  cp(msize, g->h_msize);
  return RM_OK;
}

int rm_popcount_rows(const uint64_t* rows, int64_t n_rows, int64_t words, const uint64_t* mask,
                     int64_t* counts) {
  if (n_rows < 0 || words < 0 || (n_rows > 0 && (!rows || !counts)))
    return fail(RM_ERR_INVALID_ARG, "bad rm_popcount_rows arguments");
  for (int64_t r = 0; r < n_rows; ++r) {
    const uint64_t* row = rows + r * words;
    int64_t c = 0;
    if (mask)
      for (int64_t i = 0; i < words; ++i) c += __builtin_popcountll(row[i] & mask[i]);
    else
      for (int64_t i = 0; i < words; ++i) c += __builtin_popcountll(row[i]);
    counts[r] = c;
  }
  return RM_OK;
}

int rm_graph_ancestors(const RmGraph* g, uint64_t* rows) {
  // rows[v * words + i]: bit j of word i set iff op 64*i+j is a transitive
  // predecessor of v (graph.py:335-347 predecessor_masks as bitsets), words =
  // ceil(n / 64); ancestors accumulate over direct_preds in topological order
  if (!g || (g->n > 0 && !rows)) return fail(RM_ERR_INVALID_ARG, "NULL argument");
  const int n = g->n;
  if (n == 0) return RM_OK;
  if (n > 60000) return fail(RM_ERR_CAPACITY, "ancestors: closure bitsets above 60k ops");
  const size_t words = (size_t(n) + 63) / 64;
  std::vector<int32_t> indeg(n), topo;
  topo.reserve(n);
  for (int v = 0; v < n; ++v) indeg[v] = g->pred_ptr[v + 1] - g->pred_ptr[v];
  for (int v = 0; v < n; ++v)
    if (!indeg[v]) topo.push_back(v);
  for (size_t h = 0; h < topo.size(); ++h) {
    const int u = topo[h];
    for (int k = g->succ_ptr[u]; k < g->succ_ptr[u + 1]; ++k)
      if (--indeg[g->succ_idx[k]] == 0) topo.push_back(g->succ_idx[k]);
  }
  if ((int)topo.size() != n) return fail(RM_ERR_INVALID_ARG, "graph contains a cycle");
  std::memset(rows, 0, sizeof(uint64_t) * words * size_t(n));
  for (const int v : topo) {
    uint64_t* rv = rows + size_t(v) * words;
    for (int k = g->pred_ptr[v]; k < g->pred_ptr[v + 1]; ++k) {
      const int p = g->pred_idx[k];
      const uint64_t* rp = rows + size_t(p) * words;
      for (size_t i = 0; i < words; ++i) rv[i] |= rp[i];
      rv[p >> 6] |= 1ull << (p & 63);
    }
  }
  return RM_OK;
}

int rm_graph_asap_alap(const RmGraph* g, int32_t* asap, int32_t* alap) {
  // graph.py:365-372: asap(v) = |transitive predecessors|, alap(v) = n-1 -
  // |transitive successors|; transitive closure as bitsets in topological
  // order (descendants) and reverse topological order (ancestors), popcounts
  if (!g || (g->n > 0 && (!asap || !alap))) return fail(RM_ERR_INVALID_ARG, "NULL argument");
  const int n = g->n;
  if (n == 0) return RM_OK;
  if (n > 60000) return fail(RM_ERR_CAPACITY, "asap_alap: closure bitsets above 60k ops");
  std::vector<uint64_t> desc;
  size_t words = 0;
  if (!descendants(*g, desc, words)) return fail(RM_ERR_INVALID_ARG, "graph contains a cycle");
  for (int v = 0; v < n; ++v) {
    int c = 0;
    for (size_t i = 0; i < words; ++i) c += __builtin_popcountll(desc[size_t(v) * words + i]);
    alap[v] = n - 1 - c;
  }
  // ancestors: the same sweep forward over direct_preds (reusing the buffer),
  // popcounts per row -- not column counts of the descendant matrix, which
  // visit every one of the O(n^2) closure bits
  std::vector<int32_t> indeg(n), topo;
  topo.reserve(n);
  for (int v = 0; v < n; ++v) indeg[v] = g->pred_ptr[v + 1] - g->pred_ptr[v];
  for (int v = 0; v < n; ++v)
    if (!indeg[v]) topo.push_back(v);
  for (size_t h = 0; h < topo.size(); ++h) {
    const int u = topo[h];
    for (int k = g->succ_ptr[u]; k < g->succ_ptr[u + 1]; ++k)
      if (--indeg[g->succ_idx[k]] == 0) topo.push_back(g->succ_idx[k]);
  }
  std::fill(desc.begin(), desc.end(), 0ull);
  for (const int v : topo) {
    uint64_t* av = &desc[size_t(v) * words];
    for (int k = g->pred_ptr[v]; k < g->pred_ptr[v + 1]; ++k) {
      const int p = g->pred_idx[k];
      const uint64_t* ap = &desc[size_t(p) * words];
      for (size_t i = 0; i < words; ++i) av[i] |= ap[i];
      av[p >> 6] |= 1ull << (p & 63);
    }
    int c = 0;
    for (size_t i = 0; i < words; ++i) c += __builtin_popcountll(av[i]);
    asap[v] = c;
  }
  return RM_OK;
}

}  // extern "C"
