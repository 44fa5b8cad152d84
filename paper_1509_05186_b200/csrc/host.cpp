// host.cpp -- C ABI of libetree: argument checks, index build (sort, leaves,
// groups, forest tuples, IVF lists, statistics), workspace planning and kernel
// launches.  The build follows Algorithm 1's semantics: codes are
// sorted lexicographically, identical codes share one leaf (A6), and the tree
// is described by its leaves in depth-first order with each leaf's LCP to its
// predecessor.  No code is shared with oracle/.
#include "../../include/etree.h"
#include "internal.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace et {

static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches += n; }

// ---------------------------------------------------------------------------
// optional per-kernel timing: CUDA events recorded on the launching stream
// around each launcher call (et_timing_enable); read back by et_timing_get.
// ---------------------------------------------------------------------------
static std::atomic<bool> g_timing{false};
static std::mutex g_tmu;
struct Pending { std::string name; cudaEvent_t a, b; };
static std::vector<Pending> g_pending;
static std::vector<cudaEvent_t> g_event_pool;
static std::map<std::string, std::pair<double, long long>> g_tacc;

static cudaEvent_t get_event() {
  std::lock_guard<std::mutex> lk(g_tmu);
  if (!g_event_pool.empty()) { cudaEvent_t e = g_event_pool.back(); g_event_pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

template <class F>
static cudaError_t timed(const char* name, cudaStream_t st, F f) {
  if (!g_timing.load(std::memory_order_relaxed)) return f();
  cudaEvent_t a = get_event(), b = get_event();
  cudaEventRecord(a, st);
  cudaError_t e = f();
  cudaEventRecord(b, st);
  std::lock_guard<std::mutex> lk(g_tmu);
  g_pending.push_back({name, a, b});
  return e;
}

static void drain_timing() {
  std::lock_guard<std::mutex> lk(g_tmu);
  for (auto& p : g_pending) {
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    auto& acc = g_tacc[p.name];
    acc.first += ms;
    acc.second += 1;
    g_event_pool.push_back(p.a);
    g_event_pool.push_back(p.b);
  }
  g_pending.clear();
}

static thread_local std::string g_err;
static thread_local bool g_dry_run = false;   // build on the host only (et_build_stats)

struct Error {
  et_status st;
  std::string msg;
};

[[noreturn]] static void fail(et_status st, const std::string& msg) { throw Error{st, msg}; }

static void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) fail(ET_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
    fail(ET_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// ---------------------------------------------------------------------------
// device buffers owned by an index
// ---------------------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { if (p) cudaFree(p); }
  template <class T>
  void upload(const std::vector<T>& v) {
    bytes = v.size() * sizeof(T);
    if (bytes == 0 || g_dry_run) return;
    cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(index)");
    cuda_check(cudaMemcpy(p, v.data(), bytes, cudaMemcpyHostToDevice), "upload(index)");
  }
  void upload_raw(const void* src, size_t n) {
    bytes = n;
    if (!n || g_dry_run) return;
    cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(index)");
    cuda_check(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice), "upload(index)");
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
  void reset() { if (p) cudaFree(p); p = nullptr; bytes = 0; }
  void adopt(void* ptr, size_t n) { reset(); p = ptr; bytes = n; }   // device memory made elsewhere
};

enum Kind { kTree = 0, kIvf = 1, kFlat = 2 };

struct HostTree {
  int MT = 0, layer0 = 0;
  std::vector<uint64_t> code;   // packed little-endian, byte l at bits 8l
  std::vector<uint8_t> lcp;
  std::vector<uint64_t> mult;   // ids per leaf (stats)
  et_tree_stats st{};
};

}  // namespace et

struct et_index {
  int kind = et::kTree;
  int64_t N = 0;
  int M = 0, K = 0, T = 1, d = 0, nlist = 0;
  int split[et::kMaxTrees + 1] = {};
  std::vector<int> layer_sub;
  int64_t n_groups = 0;
  int device = 0;
  et_tree_stats stats[et::kMaxTrees] = {};
  et::DevBuf code[et::kMaxTrees], lcp[et::kMaxTrees];
  bool fused = false;                // forest with M <= 8: one scan over masked tuple records
  et::DevBuf fused_rec;
  et::DevBuf narrow_rec;             // forest with 8 < M <= 16: narrow-scan tuple records (2 x uint4)
  et::DevBuf group_extra;            // leaf extra byte per group (et_index_set_extra)
  int64_t n_leaves[et::kMaxTrees] = {};
  et::DevBuf group_off, ids, group_mult, group_minid, slot2group;
  et::DevBuf t0_tup_off, tup_leaf[et::kMaxTrees];
  et::DevBuf layer_sub_d;
  et::DevBuf coarse, coarse_t, codebooks;   // IVF ([nlist][d], [d][nlist], [M][K][s])
  std::vector<uint32_t> list_leaf_off;
  et::DevBuf list_leaf_off_d;
  et::DevBuf cell_order_d;           // IVF cells by list length, longest first (chunk order)
  double lookups_per_query = 0;      // sum over trees (+ tuples) -- planning
};

namespace et {

// ---------------------------------------------------------------------------
// sorting: stable LSD radix sort of slots by code bytes (lexicographic order)
// ---------------------------------------------------------------------------
// Returns the permutation of [0, n) that sorts rows of `codes` (row stride M,
// using bytes [b0, b1)) lexicographically; equal rows keep slot order.
static std::vector<uint32_t> sort_slots(const uint8_t* codes, int64_t n, int M, int b0, int b1,
                                        const std::vector<uint32_t>* subset = nullptr) {
  std::vector<uint32_t> a, b;
  if (subset) a = *subset;
  else { a.resize(n); std::iota(a.begin(), a.end(), 0u); }
  b.resize(a.size());
  std::vector<uint8_t> digit(a.size());
  for (int l = b1 - 1; l >= b0; --l) {
    size_t cnt[257] = {0};
    for (size_t i = 0; i < a.size(); ++i) {
      digit[i] = codes[(size_t)a[i] * M + l];
      ++cnt[digit[i] + 1];
    }
    for (int v = 0; v < 256; ++v) cnt[v + 1] += cnt[v];
    for (size_t i = 0; i < a.size(); ++i) b[cnt[digit[i]]++] = a[i];
    a.swap(b);
  }
  return a;
}

static inline bool rows_equal(const uint8_t* codes, int M, uint32_t x, uint32_t y, int b0, int b1) {
  return std::memcmp(codes + (size_t)x * M + b0, codes + (size_t)y * M + b0, b1 - b0) == 0;
}

static inline int row_lcp(const uint8_t* codes, int M, uint32_t x, uint32_t y, int b0, int b1) {
  const uint8_t* a = codes + (size_t)x * M;
  const uint8_t* b = codes + (size_t)y * M;
  int l = 0;
  while (b0 + l < b1 && a[b0 + l] == b[b0 + l]) ++l;
  return l;
}

static inline uint64_t pack(const uint8_t* row, int b0, int b1) {
  uint64_t v = 0;
  for (int l = b0; l < b1; ++l) v |= (uint64_t)row[l] << (8 * (l - b0));
  return v;
}

// Statistics of a tree given its leaves' LCP-with-predecessor and multiplicity
// (plain definition): internal nodes at depth l = runs of
// adjacent leaves sharing l+1 bytes => L1 = sum_i max(0, lcp_i - lcp_{i-1});
// leaf depth = max(lcp_i, lcp_{i+1}); postfix = MT-1-depth.
static void tree_stats(HostTree& t, int64_t N) {
  const int64_t L2 = (int64_t)t.lcp.size();
  int64_t L1 = 0, post = 0, recs = 0, post_recs = 0, look = 0;
  for (int64_t i = 0; i < L2; ++i) {
    const int li = (i == 0) ? 0 : t.lcp[i];
    const int prev = (i <= 1) ? 0 : t.lcp[i - 1];
    if (i >= 1) L1 += std::max(0, li - prev);
    const int nxt = (i + 1 < L2) ? t.lcp[i + 1] : 0;
    const int depth = std::min(t.MT - 1, std::max(li, nxt));
    const int pf = t.MT - 1 - depth;
    post += pf;
    const int64_t r = ((int64_t)t.mult[i] + 126) / 127;
    recs += r;
    post_recs += r * pf;
    look += t.MT - li;
  }
  if (L1 + L2 + post != look) fail(ET_ERR_CORRUPT, "internal: lookup identity violated");
  t.st.N = N;
  t.st.M = t.MT;
  t.st.layer0 = t.layer0;
  t.st.L1 = L1;
  t.st.L2 = L2;
  t.st.total_postfix = post;
  t.st.lookups = look;
  t.st.L2_records = recs;
  t.st.paper_bytes = 4 * N + 2 * (L1 + recs) + post_recs;
  t.st.device_bytes = L2 * 16;   // leaf records (make_records)
}

static void check_codes(const uint8_t* codes, int64_t n, int M, int K) {
  if (K < 256) {
    for (int64_t i = 0; i < n * M; ++i)
      if (codes[i] >= K) fail(ET_ERR_INVALID_CODE, "code byte >= K");
  }
}

// groups (distinct full codes in sorted order) + ids, from a sorted slot list
struct Groups {
  std::vector<uint32_t> off;      // [G+1]
  std::vector<int32_t> ids;       // ascending within a group
  std::vector<uint32_t> first;    // representative slot of each group
};

static Groups make_groups(const uint8_t* codes, int M, const std::vector<uint32_t>& order,
                          const int32_t* ids, int b0, int b1) {
  Groups g;
  const size_t n = order.size();
  g.ids.resize(n);
  for (size_t i = 0; i < n; ++i) {
    if (i == 0 || !rows_equal(codes, M, order[i - 1], order[i], b0, b1)) {
      g.off.push_back((uint32_t)i);
      g.first.push_back(order[i]);
    }
    g.ids[i] = ids ? ids[order[i]] : (int32_t)order[i];
  }
  g.off.push_back((uint32_t)n);
  if (ids) {
    for (size_t j = 0; j + 1 < g.off.size(); ++j) std::sort(g.ids.begin() + g.off[j], g.ids.begin() + g.off[j + 1]);
  }
  return g;
}

static void upload_groups(et_index* ix, const Groups& g, const std::vector<uint32_t>& slot2group) {
  const size_t G = g.off.size() - 1;
  std::vector<uint32_t> mult(G);
  std::vector<int32_t> minid(G);
  for (size_t j = 0; j < G; ++j) {
    mult[j] = g.off[j + 1] - g.off[j];
    minid[j] = g.ids[g.off[j]];
  }
  ix->n_groups = (int64_t)G;
  ix->group_off.upload(g.off);
  ix->ids.upload(g.ids);
  ix->group_mult.upload(mult);
  ix->group_minid.upload(minid);
  if (!slot2group.empty()) ix->slot2group.upload(slot2group);
}

// Leaf records of the device layout: one uint4 = 8
// half-words; half-word l = the pre-swizzled byte offset of table entry
// (l, k = code byte l) inside that level's 32 KB shared-memory table,
// (k << 7) | ((k & 31) << 2), so a lookup is one XOR with the lane's offset.
// Levels 0 and 1 of an 8-level tree (held in TMEM) store the column k; half-
// word 0 adds the lookup mask of the levels >= the LCP with the previous leaf
// in bits 8..15 and half-word 1 floor(log2(multiplicity)) in bits 8..11;
// shorter trees keep the LCP and the bucket in half-word 7 (bits 0..3, 4..7).
static std::vector<uint4> make_records(const HostTree& h) {
  const int MT = h.MT;
  std::vector<uint4> rec(h.code.size());
  for (size_t i = 0; i < h.code.size(); ++i) {
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int l = 0; l < MT; ++l) {
      const uint32_t k = (uint32_t)((h.code[i] >> (8 * l)) & 255u);
      w[l] = (MT == 8 && l < kTmemLevels) ? k : ((k << 7) | ((k & 31u) << 2));   // TMEM levels: the column
    }
    const uint32_t lcp = (i < h.lcp.size()) ? h.lcp[i] : 0u;
    const uint64_t mu = (i < h.mult.size()) ? h.mult[i] : 1;
    uint32_t mb = 0;   // floor(log2(multiplicity)), capped at 15
    while (mb < 15 && (2ull << mb) <= mu) ++mb;
    // 8-level trees: the lookup mask (levels >= LCP) in half-word 0 bits
    // 8..15 and the bucket in half-word 1 bits 8..11 -- the fused-forest
    // record layout, so one scan loop serves both
    if (MT == 8) { w[0] |= ((0xffu << lcp) & 0xffu) << 8; w[1] |= mb << 8; }
    else w[7] = lcp | (mb << 4);
    rec[i] = make_uint4(w[0] | (w[1] << 16), w[2] | (w[3] << 16), w[4] | (w[5] << 16), w[6] | (w[7] << 16));
  }
  return rec;
}

// Fused E-Forest records (M <= 8): one record per tuple
// (distinct full code, in lexicographic order) = the single-tree record of
// its full code whose LCP field is an 8-bit lookup mask: bit l is set iff
// l - split[u] >= LCP(tuple t-1, tuple t) over tree u's bytes, u the tree of
// level l.  Each tree's Distance Context then runs along the tuple
// sequence and the per-tree partials are summed in tree order (A13).
static int64_t build_fused(et_index* ix, const uint8_t* codes, const Groups& g, int M, int T, const int32_t* split) {
  const size_t G = g.off.size() - 1;
  std::vector<uint4> rec(G);
  int64_t look = 0;
  for (size_t j = 0; j < G; ++j) {
    const uint8_t* row = codes + (size_t)g.first[j] * M;
    const uint8_t* prev = j ? codes + (size_t)g.first[j - 1] * M : nullptr;
    uint32_t mask = 0;
    for (int u = 0; u < T; ++u) {
      int l = 0;
      if (prev) while (split[u] + l < split[u + 1] && row[split[u] + l] == prev[split[u] + l]) ++l;
      for (int b = split[u] + l; b < split[u + 1]; ++b) mask |= 1u << b;
    }
    look += __builtin_popcount(mask);
    const uint64_t mu = g.off[j + 1] - g.off[j];
    uint32_t mb = 0;
    while (mb < 15 && (2ull << mb) <= mu) ++mb;
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int l = 0; l < M; ++l) {
      const uint32_t k = row[l];
      w[l] = (M == 8 && l < kTmemLevels) ? k : ((k << 7) | ((k & 31u) << 2));
    }
    if (M == 8) { w[0] |= mask << 8; w[1] |= mb << 8; }
    else w[7] = mask | (mb << 8);
    rec[j] = make_uint4(w[0] | (w[1] << 16), w[2] | (w[3] << 16), w[4] | (w[5] << 16), w[6] | (w[7] << 16));
  }
  ix->fused = true;
  ix->fused_rec.upload(rec);
  return look;
}

// Narrow-scan records (narrow.cuh; forests with 8 < M <= 16): two uint4 per
// tuple (distinct full code, lexicographic order) = 16 half-words, half-word
// l = (code byte l) << 5 | lookup-mask bit l (the mask of build_fused: level l
// is looked up iff l - split[u] >= LCP(tuple t-1, tuple t) over tree u's
// bytes), half-word 0 adds floor(log2(multiplicity)) in bits 1..4; levels >= M
// are 0.
static void build_narrow(et_index* ix, const uint8_t* codes, const Groups& g, int M, int T, const int32_t* split) {
  const size_t G = g.off.size() - 1;
  std::vector<uint4> rec(2 * G);
  for (size_t j = 0; j < G; ++j) {
    const uint8_t* row = codes + (size_t)g.first[j] * M;
    const uint8_t* prev = j ? codes + (size_t)g.first[j - 1] * M : nullptr;
    uint32_t mask = 0;
    for (int u = 0; u < T; ++u) {
      int l = 0;
      if (prev) while (split[u] + l < split[u + 1] && row[split[u] + l] == prev[split[u] + l]) ++l;
      for (int b = split[u] + l; b < split[u + 1]; ++b) mask |= 1u << b;
    }
    const uint64_t mu = g.off[j + 1] - g.off[j];
    uint32_t mb = 0;
    while (mb < 15 && (2ull << mb) <= mu) ++mb;
    uint32_t hw[16] = {};
    for (int l = 0; l < M; ++l) hw[l] = ((uint32_t)row[l] << 5) | ((mask >> l) & 1u);
    hw[0] |= mb << 1;
    uint32_t w[8];
    for (int i = 0; i < 8; ++i) w[i] = hw[2 * i] | (hw[2 * i + 1] << 16);
    rec[2 * j] = make_uint4(w[0], w[1], w[2], w[3]);
    rec[2 * j + 1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
  ix->narrow_rec.upload(rec);
}

static void finish_tree(et_index* ix, int t, HostTree& h) {
  ix->n_leaves[t] = (int64_t)h.code.size();
  ix->code[t].upload(make_records(h));
  ix->lcp[t].upload(h.lcp);
  ix->stats[t] = h.st;
}

static void set_layers(et_index* ix, const int32_t* byte_perm) {
  ix->layer_sub.resize(ix->M);
  for (int l = 0; l < ix->M; ++l) ix->layer_sub[l] = byte_perm ? byte_perm[l] : l;
  if (byte_perm) {
    std::vector<int> seen(ix->M, 0);
    for (int l = 0; l < ix->M; ++l) {
      if (byte_perm[l] < 0 || byte_perm[l] >= ix->M || seen[byte_perm[l]]++) fail(ET_ERR_CONFIG, "invalid byte permutation");
    }
  }
  ix->layer_sub_d.upload(ix->layer_sub);
}

// codes permuted so that byte l of the stored code is original byte perm[l]
static std::vector<uint8_t> permute_codes(const uint8_t* codes, int64_t n, int M, const int32_t* perm) {
  std::vector<uint8_t> out((size_t)n * M);
  for (int64_t i = 0; i < n; ++i)
    for (int l = 0; l < M; ++l) out[(size_t)i * M + l] = codes[(size_t)i * M + (perm ? perm[l] : l)];
  return out;
}

static void check_ids(const int32_t* ids, int64_t n) {
  if (!ids) return;
  for (int64_t i = 0; i < n; ++i)
    if (ids[i] < 0) fail(ET_ERR_CONFIG, "ids must be non-negative");
}

// E-Forest / E-Tree build (T = 1 is the E-Tree).
static et_index* build_forest(const uint8_t* codes_in, const int32_t* ids, int64_t n, int M, int K,
                              const int32_t* byte_perm, int T, const int32_t* split) {
  if (n <= 0) fail(ET_ERR_EMPTY, "empty dataset");
  if (n > INT32_MAX) fail(ET_ERR_CONFIG, "n exceeds int32 ids");
  if (M <= 0 || K <= 0 || K > 256) fail(ET_ERR_CONFIG, "need 1 <= K <= 256 and M >= 1");
  if (T < 1 || T > kMaxTrees) fail(ET_ERR_CONFIG, "T must be 1..4");
  if (split[0] != 0 || split[T] != M) fail(ET_ERR_CONFIG, "split must start at 0 and end at M");
  for (int t = 0; t < T; ++t) {
    const int w = split[t + 1] - split[t];
    if (w < 1 || w > kMaxMT) fail(ET_ERR_CONFIG, "each tree must cover 1..8 code bytes (use a forest for M > 8)");
  }
  check_codes(codes_in, n, M, K);
  check_ids(ids, n);
  std::unique_ptr<et_index> ix(new et_index);
  ix->kind = kTree;
  ix->N = n; ix->M = M; ix->K = K; ix->T = T;
  for (int t = 0; t <= T; ++t) ix->split[t] = split[t];
  if (!g_dry_run) cudaGetDevice(&ix->device);
  set_layers(ix.get(), byte_perm);

  // full-code sort -> groups (distinct full codes, in lexicographic order):
  // on the GPU when there is one (build_gpu.cu: radix sort + flag scan; the
  // per-id arrays stay on the device), else on the host (et_build_stats).
  // The trees are then built from one (permuted) code row per group.
  Groups g;
  std::vector<uint8_t> reps;
  if (!g_dry_run) {
    GpuGroups gg;
    cuda_check(gpu_group_codes(codes_in, ids, n, M, byte_perm, nullptr, &gg), "GPU index build (sort + group)");
    const size_t G0 = (size_t)gg.G;
    ix->n_groups = (int64_t)G0;
    ix->ids.adopt(gg.ids, (size_t)n * 4);
    ix->group_off.adopt(gg.group_off, (G0 + 1) * 4);
    ix->group_mult.adopt(gg.mult, G0 * 4);
    ix->group_minid.adopt(gg.minid, G0 * 4);
    ix->slot2group.adopt(gg.slot2group, (size_t)n * 4);
    g.off = std::move(gg.off);
    reps.resize(G0 * M);
    for (size_t j = 0; j < G0; ++j)
      for (int l = 0; l < M; ++l) reps[j * M + l] = codes_in[(size_t)gg.first[j] * M + (byte_perm ? byte_perm[l] : l)];
  } else {
    std::vector<uint8_t> pc = permute_codes(codes_in, n, M, byte_perm);
    std::vector<uint32_t> order = sort_slots(pc.data(), n, M, 0, M);
    Groups hg = make_groups(pc.data(), M, order, ids, 0, M);
    const size_t G0 = hg.off.size() - 1;
    std::vector<uint32_t> slot2group(n);
    for (size_t j = 0; j < G0; ++j)
      for (uint32_t i = hg.off[j]; i < hg.off[j + 1]; ++i) slot2group[order[i]] = (uint32_t)j;
    upload_groups(ix.get(), hg, slot2group);
    reps.resize(G0 * M);
    for (size_t j = 0; j < G0; ++j) std::memcpy(&reps[j * M], &pc[(size_t)hg.first[j] * M], M);
    g.off = std::move(hg.off);
  }
  const size_t G = g.off.size() - 1;
  g.first.resize(G);
  std::iota(g.first.begin(), g.first.end(), 0u);   // row j of `reps` is group j's code
  const uint8_t* codes = reps.data();

  double look = 0;
  // tree 0: groups sorted by full code are sorted by the tree-0 projection too
  {
    HostTree h;
    h.MT = split[1]; h.layer0 = 0;
    std::vector<uint32_t> tup_off;
    for (size_t j = 0; j < G; ++j) {
      const uint32_t r = g.first[j];
      const bool newleaf = (j == 0) || !rows_equal(codes, M, g.first[j - 1], r, 0, split[1]);
      if (newleaf) {
        h.code.push_back(pack(codes + (size_t)r * M, 0, split[1]));
        h.lcp.push_back(j == 0 ? 0 : (uint8_t)row_lcp(codes, M, g.first[j - 1], r, 0, split[1]));
        h.mult.push_back(0);
        tup_off.push_back((uint32_t)j);
      }
      h.mult.back() += g.off[j + 1] - g.off[j];
    }
    tup_off.push_back((uint32_t)G);
    tree_stats(h, n);
    look += (double)h.st.lookups;
    finish_tree(ix.get(), 0, h);
    if (T > 1) {
      ix->t0_tup_off.upload(tup_off);
      std::vector<uint32_t> tl0(G);   // tree-0 leaf of each tuple
      for (size_t i = 0; i + 1 < tup_off.size(); ++i)
        for (uint32_t g2 = tup_off[i]; g2 < tup_off[i + 1]; ++g2) tl0[g2] = (uint32_t)i;
      ix->tup_leaf[0].upload(tl0);
      look += (double)G;   // one join per tuple
    }
  }
  // trees 1..T-1: distinct projections, sorted; tuple -> leaf
  for (int t = 1; t < T; ++t) {
    const int b0 = split[t], b1 = split[t + 1];
    std::vector<uint32_t> rows(g.first.begin(), g.first.end());
    std::vector<uint32_t> so = sort_slots(codes, (int64_t)G, M, b0, b1, &rows);
    // group id of each rep (rep -> position in g.first): use slot2group
    HostTree h;
    h.MT = b1 - b0; h.layer0 = b0;
    std::vector<uint32_t> tup_leaf(G);
    for (size_t i = 0; i < so.size(); ++i) {
      const uint32_t r = so[i];
      const bool newleaf = (i == 0) || !rows_equal(codes, M, so[i - 1], r, b0, b1);
      if (newleaf) {
        h.code.push_back(pack(codes + (size_t)r * M, b0, b1));
        h.lcp.push_back(i == 0 ? 0 : (uint8_t)row_lcp(codes, M, so[i - 1], r, b0, b1));
        h.mult.push_back(0);
      }
      const uint32_t grp = r;   // row r of `reps` is group r
      tup_leaf[grp] = (uint32_t)(h.code.size() - 1);
      h.mult.back() += g.off[grp + 1] - g.off[grp];
    }
    tree_stats(h, n);
    look += (double)h.st.lookups;
    finish_tree(ix.get(), t, h);
    ix->tup_leaf[t].upload(tup_leaf);
  }
  int64_t scan_look = (int64_t)look;
  if (T > 1 && M <= kMaxMT) {   // fused forest: one masked scan over the tuples
    scan_look = build_fused(ix.get(), codes, g, M, T, split);
    look = (double)scan_look;
  }
  if (T > 1 && M > kMaxMT && M <= 16) build_narrow(ix.get(), codes, g, M, T, split);   // few-query scan
  for (int t = 0; t < T; ++t) { ix->stats[t].groups = (int64_t)G; ix->stats[t].scan_lookups = scan_look; }
  ix->lookups_per_query = look;
  return ix.release();
}

static et_index* build_flat(const uint8_t* codes, const int32_t* ids, int64_t n, int M, int K) {
  if (n <= 0) fail(ET_ERR_EMPTY, "empty dataset");
  if (M < 1 || M > kMaxMT) fail(ET_ERR_CONFIG, "flat index: 1 <= M <= 8");
  if (K <= 0 || K > 256) fail(ET_ERR_CONFIG, "K must be 1..256");
  check_codes(codes, n, M, K);
  check_ids(ids, n);
  std::unique_ptr<et_index> ix(new et_index);
  ix->kind = kFlat;
  ix->N = n; ix->M = M; ix->K = K; ix->T = 1;
  ix->split[0] = 0; ix->split[1] = M;
  cudaGetDevice(&ix->device);
  set_layers(ix.get(), nullptr);
  HostTree h;
  h.MT = M;
  h.code.resize(n);
  h.lcp.assign(n, 0);
  h.mult.assign(n, 1);
  for (int64_t i = 0; i < n; ++i) h.code[i] = pack(codes + (size_t)i * M, 0, M);
  h.st.N = n; h.st.M = M; h.st.L2 = n; h.st.lookups = n * M; h.st.device_bytes = n * 16;
  h.st.L2_records = n; h.st.total_postfix = n * (M - 1); h.st.paper_bytes = 4 * n + n * M;
  finish_tree(ix.get(), 0, h);
  ix->stats[0].scan_lookups = n * M;
  Groups g;
  g.off.resize(n + 1);
  g.ids.resize(n);
  for (int64_t i = 0; i <= n; ++i) g.off[i] = (uint32_t)i;
  for (int64_t i = 0; i < n; ++i) g.ids[i] = ids ? ids[i] : (int32_t)i;
  std::vector<uint32_t> s2g(n);
  std::iota(s2g.begin(), s2g.end(), 0u);
  upload_groups(ix.get(), g, s2g);
  ix->stats[0].groups = n;
  ix->lookups_per_query = (double)n * M;
  return ix.release();
}

static et_index* build_ivf(const uint8_t* codes_in, const int32_t* ids, int64_t n, int M, int K,
                           const int32_t* list_of, int nlist, const float* coarse, int d,
                           const float* codebooks) {
  if (n <= 0) fail(ET_ERR_EMPTY, "empty dataset");
  if (M < 1 || M > kMaxMT) fail(ET_ERR_CONFIG, "IVF lists: 1 <= M <= 8");
  if (K <= 0 || K > 256) fail(ET_ERR_CONFIG, "K must be 1..256");
  if (nlist < 1) fail(ET_ERR_CONFIG, "nlist >= 1");
  if (d <= 0 || d % M) fail(ET_ERR_SUBSPACE_SPLIT, "d % M != 0");
  check_codes(codes_in, n, M, K);
  check_ids(ids, n);
  for (int64_t i = 0; i < n; ++i)
    if (list_of[i] < 0 || list_of[i] >= nlist) fail(ET_ERR_CONFIG, "list_of out of range");
  for (int64_t i = 0; i < (int64_t)nlist * d; ++i)
    if (!std::isfinite(coarse[i])) fail(ET_ERR_INVALID_VECTOR, "non-finite coarse centroid");
  for (int64_t i = 0; i < (int64_t)M * K * (d / M); ++i)
    if (!std::isfinite(codebooks[i])) fail(ET_ERR_INVALID_VECTOR, "non-finite residual codebook");
  std::unique_ptr<et_index> ix(new et_index);
  ix->kind = kIvf;
  ix->N = n; ix->M = M; ix->K = K; ix->T = 1; ix->d = d; ix->nlist = nlist;
  ix->split[0] = 0; ix->split[1] = M;
  cudaGetDevice(&ix->device);
  set_layers(ix.get(), nullptr);
  // (list, code) groups in (list, code) order on the GPU (build_gpu.cu); one
  // tree per list over its distinct codes, LCPs restart at every list
  GpuGroups gg;
  cuda_check(gpu_group_codes(codes_in, ids, n, M, nullptr, list_of, &gg), "GPU index build (sort + group)");
  const size_t G = (size_t)gg.G;
  ix->n_groups = (int64_t)G;
  ix->ids.adopt(gg.ids, (size_t)n * 4);
  ix->group_off.adopt(gg.group_off, (G + 1) * 4);
  ix->group_mult.adopt(gg.mult, G * 4);
  ix->group_minid.adopt(gg.minid, G * 4);
  ix->slot2group.adopt(gg.slot2group, (size_t)n * 4);
  HostTree h;
  h.MT = M;
  ix->list_leaf_off.assign(nlist + 1, 0);
  et_tree_stats tot{};
  size_t j = 0;
  for (int c = 0; c < nlist; ++c) {
    ix->list_leaf_off[c] = (uint32_t)h.code.size();
    HostTree lt;
    lt.MT = M;
    int64_t nc = 0;
    for (; j < G && list_of[gg.first[j]] == c; ++j) {
      const uint32_t r = gg.first[j];
      const uint64_t pk = pack(codes_in + (size_t)r * M, 0, M);
      const uint8_t lp = lt.code.empty() ? 0 : (uint8_t)row_lcp(codes_in, M, gg.first[j - 1], r, 0, M);
      const uint64_t mu = gg.off[j + 1] - gg.off[j];
      lt.code.push_back(pk); lt.lcp.push_back(lp); lt.mult.push_back(mu);
      h.code.push_back(pk); h.lcp.push_back(lp); h.mult.push_back(mu);
      nc += (int64_t)mu;
    }
    if (lt.code.empty()) continue;
    tree_stats(lt, nc);
    tot.L1 += lt.st.L1; tot.L2 += lt.st.L2; tot.total_postfix += lt.st.total_postfix;
    tot.lookups += lt.st.lookups; tot.L2_records += lt.st.L2_records; tot.paper_bytes += lt.st.paper_bytes;
  }
  if (j != G) fail(ET_ERR_CORRUPT, "internal: IVF groups out of list order");
  ix->list_leaf_off[nlist] = (uint32_t)h.code.size();
  tot.N = n; tot.M = M; tot.device_bytes = (int64_t)h.code.size() * 16;
  tot.groups = (int64_t)G;
  ix->n_leaves[0] = (int64_t)h.code.size();
  ix->code[0].upload(make_records(h));
  ix->lcp[0].upload(h.lcp);
  tot.scan_lookups = tot.lookups;
  ix->stats[0] = tot;
  ix->list_leaf_off_d.upload(ix->list_leaf_off);
  {   // chunk order of the scan: longest lists first within each region (their
      // chunks take longest; started last they would set the kernel's tail)
    std::vector<int> order(nlist);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return ix->list_leaf_off[a + 1] - ix->list_leaf_off[a] > ix->list_leaf_off[b + 1] - ix->list_leaf_off[b];
    });
    ix->cell_order_d.upload(order);
  }
  ix->coarse.upload_raw(coarse, (size_t)nlist * d * 4);
  {
    std::vector<float> ct((size_t)nlist * d);
    for (int c = 0; c < nlist; ++c)
      for (int j = 0; j < d; ++j) ct[(size_t)j * nlist + c] = coarse[(size_t)c * d + j];
    ix->coarse_t.upload(ct);
  }
  ix->codebooks.upload_raw(codebooks, (size_t)M * K * (d / M) * 4);
  ix->lookups_per_query = (double)tot.lookups / std::max(1, nlist);
  return ix.release();
}

// ---------------------------------------------------------------------------
// query planning
// ---------------------------------------------------------------------------
static int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev < 64) cached[dev] = n;
  return n;
}

struct Plan {
  int n_chunks = 0, S = 1, n_units = 0, MTmax = 0, B = 0;
  bool lut0 = false;
  bool mat_luts = false;   // tables materialised by lut_kernel, copied into each scan CTA
  bool long_ranges = false;   // top-k scans of 8-level trees with >= kLongRange leaves per warp: kStreamsLong
  int64_t part_stride = 0;
  int64_t part_base[kMaxTrees] = {};
};

// candidate buffer per (unit, warp, lane): k survivors of a refresh + ties, plus
// one batch of emissions (kBatchEmit) before the next buffer check
// (ns: lockstep streams per scan warp, 32 candidates per stream per batch)
static int topk_B(int k, int ns = kStreams) { return ((2 * k + 32 * ns + 31) / 32) * 32; }

// Tables built once by lut_kernel ([Q][M][K] in the workspace) and copied
// into each scan CTA, instead of built inside the CTA: ET_TABLES=materialised
// (experiments; the default is the fused build -- on c3, whose CTAs hold ~7
// queries, fused 136 us vs materialised 185 us of which lut_kernel 98 us).
static bool materialise_tables(const et_index* ix, int64_t Q) {
  static int mode = [] {
    const char* e = std::getenv("ET_TABLES");
    return !e ? 0 : (std::strcmp(e, "fused") == 0 ? 1 : (std::strcmp(e, "materialised") == 0 ? 2 : 0));
  }();
  if (mode == 1) return false;
  const bool big = (double)Q * ix->M * ix->K * 4 > 512.0 * (1 << 20);
  if (mode == 2) return !big;
  return false;   // auto: fused (measured: c3 fused 136 us vs materialised 185 us, lut_kernel 98 us of it)
}

static Plan make_plan(const et_index* ix, int64_t Q, int k, int nsm) {
  Plan pl;
  pl.mat_luts = materialise_tables(ix, Q);
  for (int t = 0; t < ix->T; ++t) pl.MTmax = std::max(pl.MTmax, ix->stats[t].M);
  if (ix->fused) pl.MTmax = ix->M;   // one scan over all M levels
  pl.lut0 = (pl.MTmax == 8);
  const int64_t base = (Q + 31) / 32;
  // Cost model per unit (cycles of one SM): tables ~ nq * K * d * 2 / 128 * 1.25
  // (fp32 lanes), scan ~ 1.5 * lookups per query / S (one warp-wide smem lookup
  // per lookup for 32 queries).  Pick the (chunks, S) with the least makespan.
  // (A leaf-step term -- c5 313 chunks x S = 4 instead of 444 x 1 -- measured
  // 0.863 vs 0.846 ms: not taken.)
  const double K = ix->K;
  const double d = std::max(1, ix->kind == kIvf ? ix->d : ix->M * 16);
  // scan cycles of one unit: a leaf (tuple) step costs ~37 warp instructions
  // per 32 queries on 4 schedulers at ~50% issue efficiency (~18 cycles per
  // leaf), a lookup ~1.5 -- whichever dominates (fused forests: many tuple
  // steps with ~1.7 lookups each)
  const double look = std::max(1.0, 1.5 * ix->lookups_per_query);
  double best = 1e300;
  const int64_t cand_chunks[2] = {base, std::min<int64_t>(Q, ((base + nsm - 1) / nsm) * nsm)};
  const int smax = (ix->T > 1 && !ix->fused) ? 1 : 64;
  for (int ci = 0; ci < 2; ++ci) {
    const int64_t nc = std::max<int64_t>(1, cand_chunks[ci]);
    const double nq = std::min<double>(32.0, std::ceil((double)Q / nc));
    for (int S = 1; S <= smax; S *= 2) {
      const int64_t units = nc * S;
      if (units > (1 << 30)) break;
      const double per = nq * K * d * 2.0 / 128.0 * 1.25 + look / S + 2000.0;
      const double waves = std::ceil((double)units / nsm);
      const double cost = waves * per;
      if (cost < best * 0.98) { best = cost; pl.n_chunks = (int)nc; pl.S = S; }
    }
  }
  pl.n_units = pl.n_chunks * pl.S;
  const int64_t leaves = ix->fused ? ix->n_groups : ix->n_leaves[0];
  pl.long_ranges = pl.MTmax == 8 && leaves / pl.S / kWarps >= kLongRange;
  pl.B = topk_B(std::max(1, k), pl.long_ranges ? kStreamsLong : kStreams);
  int64_t off = 0;
  if (ix->T > 1 && !ix->fused)   // joined forests: per-leaf partials of every tree (the join reads them)
    for (int t = 0; t < ix->T; ++t) { pl.part_base[t] = off; off += ix->n_leaves[t] * 32; }
  pl.part_stride = off;
  return pl;
}

// IVF: chunks are (tier, cell, <= 32 probing queries) -- tier 0 = each
// query's nearest probe, scanned first (kernels.cu, ivf_entry); their number
// is data dependent, bounded by ceil(Q*w/32) + 2*nlist (one partial chunk per
// (tier, cell)).
static Plan make_ivf_plan(const et_index* ix, int64_t Q, int w, int k) {
  Plan pl;
  pl.MTmax = ix->M;
  pl.lut0 = (pl.MTmax == 8);
  pl.n_chunks = (int)((Q * w + 31) / 32 + 2 * ix->nlist);   // one partial chunk per (tier, cell)
  pl.S = 1;
  pl.n_units = pl.n_chunks;
  pl.long_ranges = pl.MTmax == 8 && ix->n_groups / std::max(1, ix->nlist) / kWarps >= kLongRange;   // mean list
  pl.B = topk_B(std::max(1, k), pl.long_ranges ? kStreamsLong : kStreams);
  return pl;
}

struct Carve {
  char* base;
  size_t off = 0, cap;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~(size_t)255;
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += n * sizeof(T);
    return p;
  }
};

struct Work {
  float4* cbt;   // chunk-major codebook copy for the wide table build (s > 16)
  float* luts;
  int* chunk_q; int* qslot_off; int* qslot;
  float* lut0; float* partials; float* leafdist;
  uint2* cand; int* cand_cnt; float* unit_thr;
  unsigned* qthr;
};

static Work carve(Carve& c, const et_index* ix, const Plan& pl, int64_t Q, bool full, int slots_per_q) {
  Work w{};
  // (s is a per-call argument: room for s <= 64, i.e. K * M * 16 float4)
  w.cbt = (pl.MTmax == 8) ? c.take<float4>((size_t)ix->K * ix->M * 16) : nullptr;
  w.luts = pl.mat_luts ? c.take<float>((size_t)Q * ix->M * ix->K) : nullptr;
  w.chunk_q = c.take<int>((size_t)pl.n_chunks * 32);
  w.qslot_off = c.take<int>(Q + 1);
  w.qslot = c.take<int>((size_t)Q * slots_per_q);
  w.lut0 = pl.lut0 ? c.take<float>((size_t)pl.n_units * kTmemLevels * 256 * 32) : nullptr;
  w.partials = pl.part_stride ? c.take<float>((size_t)pl.n_units * pl.part_stride) : nullptr;
  if (full) {
    w.leafdist = c.take<float>((size_t)pl.n_chunks * ix->n_groups * 32);
  } else {
    w.cand = c.take<uint2>((size_t)pl.n_units * kWarps * 32 * pl.B);
    w.cand_cnt = c.take<int>((size_t)pl.n_units * 32 * kWarps);
    w.unit_thr = c.take<float>((size_t)pl.n_units * 32);
    w.qthr = c.take<unsigned>((size_t)Q);
  }
  return w;
}

static size_t ws_bytes(const et_index* ix, const Plan& pl, int64_t Q, bool full, int slots_per_q) {
  Carve c{nullptr, 0, 0};
  carve(c, ix, pl, Q, full, slots_per_q);
  return c.off + 256;
}

struct IvfWork {
  int32_t* probes; int* cell_cnt; int* pair_pos; int* chunk_off; int* n_chunks;
  int* chunk_cell; uint32_t* chunk_lo; uint32_t* chunk_hi;
};

static IvfWork carve_ivf(Carve& c, const et_index* ix, const Plan& pl, int64_t Q, int w) {
  IvfWork v{};
  v.probes = c.take<int32_t>((size_t)Q * w);
  v.cell_cnt = c.take<int>(2 * ix->nlist);
  v.pair_pos = c.take<int>((size_t)Q * w);
  v.chunk_off = c.take<int>(2 * ix->nlist + 1);
  v.n_chunks = c.take<int>(1);
  v.chunk_cell = c.take<int>(pl.n_chunks);
  v.chunk_lo = c.take<uint32_t>(pl.n_chunks);
  v.chunk_hi = c.take<uint32_t>(pl.n_chunks);
  return v;
}

static size_t ivf_ws_bytes(const et_index* ix, const Plan& pl, int64_t Q, int w) {
  Carve c{nullptr, 0, 0};
  carve_ivf(c, ix, pl, Q, w);
  carve(c, ix, pl, Q, false, w);
  return c.off + 256;
}

static void fill_scan_common(ScanParams& sp, const et_index* ix, const Plan& pl) {
  sp.M = ix->M; sp.K = ix->K;
  static const int wide_old = [] { const char* e = std::getenv("ET_WIDE_OLD"); return e && e[0] == '1'; }();
  sp.wide_old = wide_old;
  sp.layer_sub = ix->layer_sub_d.as<int>();
  for (int l = 0; l < ix->M && l < kMaxTrees * kMaxMT; ++l) sp.lsub[l] = ix->layer_sub[l];
  if (ix->fused) {   // the forest's tuples scanned as one masked tree over all M levels
    sp.T = 1;
    sp.masked = 1;
    sp.fsplit = 0;
    for (int t = 1; t < ix->T; ++t) sp.fsplit |= 1u << ix->split[t];
    sp.tree[0].MT = ix->M;
    sp.tree[0].layer0 = 0;
    sp.tree[0].n_leaves = ix->n_groups;
    sp.tree[0].rec = ix->fused_rec.as<uint4>();
  } else {
    sp.T = ix->T;
  }
  for (int t = 0; t < ix->T && !ix->fused; ++t) {
    sp.tree[t].MT = ix->stats[t].M;
    sp.tree[t].layer0 = ix->split[t];
    sp.tree[t].n_leaves = ix->n_leaves[t];
    sp.tree[t].rec = ix->code[t].as<uint4>();
    sp.tree[t].lcp = ix->lcp[t].as<uint8_t>();
    sp.tup_leaf[t] = ix->tup_leaf[t].as<uint32_t>();
    sp.part_base[t] = pl.part_base[t];
  }
  sp.t0_tup_off = ix->t0_tup_off.as<uint32_t>();
  sp.group_mult = ix->group_mult.as<uint32_t>();
  sp.group_minid = ix->group_minid.as<int32_t>();
  sp.n_groups = ix->n_groups;
  sp.part_stride = pl.part_stride;
  sp.n_units = pl.n_units;
  sp.S = pl.S;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// tables source check shared by distances/topk
static void table_source(ScanParams& sp, const et_index* ix, const float* codebooks, int d,
                         const float* luts, const float* queries) {
  if (luts) {
    sp.luts = luts;
  } else {
    if (!queries || !codebooks) fail(ET_ERR_CONFIG, "need either luts or (queries and codebooks)");
    if (d <= 0 || d % ix->M) fail(ET_ERR_SUBSPACE_SPLIT, "d % M != 0");
    sp.queries = queries;
    sp.codebooks = codebooks;
    sp.d = d;
    sp.s = d / ix->M;
    sp.vec4 = aligned16(queries) && aligned16(codebooks) && (d % 4 == 0) ? 1 : 0;
  }
}

// experiments: ET_NARROW=0 keeps joined forests on the per-tree scan + join
static bool narrow_off() {
  static const bool off = [] { const char* e = std::getenv("ET_NARROW"); return e && e[0] == '0'; }();
  return off;
}

// Fused tables with 16 < s <= 64 (c3): the chunk-major codebook copy the wide
// build reads (layout only; one small kernel per call).
static void chunk_codebook(ScanParams& sp, const et_index* ix, const Work& w, cudaStream_t st) {
  if (sp.luts || !w.cbt || !sp.vec4 || sp.s <= 16 || sp.s > 64 || sp.s % 4) return;
  cuda_check(timed("cb_chunks", st, [&] { return launch_cb_chunks(sp.codebooks, ix->M, ix->K, sp.s, w.cbt, st); }),
             "cb_chunks");
  sp.cbt = w.cbt;
}

// Materialised-tables plan: lut_kernel writes [Q][M][K] into the workspace
// and the scan CTAs copy their queries' rows (same arithmetic).
static void materialise(ScanParams& sp, const et_index* ix, const Plan& pl, const Work& w, int64_t Q, cudaStream_t st) {
  if (!pl.mat_luts || sp.luts) return;
  const bool v4 = aligned16(sp.codebooks) && aligned16(sp.queries);
  cuda_check(timed("luts", st, [&] { return launch_luts(sp.codebooks, sp.d, ix->M, ix->K, sp.queries, Q, w.luts, v4, st); }),
             "luts");
  sp.luts = w.luts;
}

}  // namespace et

using namespace et;

#define ET_API_BEGIN try {
#define ET_API_END                                              \
  }                                                             \
  catch (const Error& e) {                                      \
    g_err = e.msg;                                              \
    return e.st;                                                \
  }                                                             \
  catch (const std::bad_alloc&) {                               \
    g_err = "host allocation failed";                           \
    return ET_ERR_OOM;                                          \
  }                                                             \
  catch (const std::exception& e) {                             \
    g_err = e.what();                                           \
    return ET_ERR_CONFIG;                                       \
  }                                                             \
  g_err.clear();                                                \
  return ET_OK;

static void host_graphs_forget(const et_index* ix);   // et_etree_topk_host's graph cache

extern "C" {

const char* et_last_error(void) { return g_err.c_str(); }

void et_timing_enable(int on) {
  if (!on) drain_timing();
  g_timing.store(on != 0);
}

void et_timing_reset(void) {
  drain_timing();
  std::lock_guard<std::mutex> lk(g_tmu);
  g_tacc.clear();
}

int et_timing_get(const char* name, double* total_ms, int64_t* count) {
  drain_timing();
  std::lock_guard<std::mutex> lk(g_tmu);
  auto it = g_tacc.find(name);
  if (it == g_tacc.end()) { if (total_ms) *total_ms = 0; if (count) *count = 0; return 0; }
  if (total_ms) *total_ms = it->second.first;
  if (count) *count = it->second.second;
  return 1;
}
const char* et_version(void) { return "etree-b200 0.1 (sm_100a)"; }
int64_t et_launch_count(void) { return (int64_t)g_launches.load(); }

et_status et_build_etree(const uint8_t* codes, const int32_t* ids, int64_t n, int32_t M, int32_t K,
                         const int32_t* byte_perm, et_index** out) {
  ET_API_BEGIN
  if (!codes || !out) fail(ET_ERR_CONFIG, "null argument");
  if (M > kMaxMT) fail(ET_ERR_CONFIG, "a single E-Tree supports M <= 8 on the GPU; build a forest");
  int32_t split[2] = {0, M};
  *out = build_forest(codes, ids, n, M, K, byte_perm, 1, split);
  ET_API_END
}

et_status et_build_eforest(const uint8_t* codes, const int32_t* ids, int64_t n, int32_t M, int32_t K,
                           const int32_t* byte_perm, int32_t T, const int32_t* split, et_index** out) {
  ET_API_BEGIN
  if (!codes || !out || !split) fail(ET_ERR_CONFIG, "null argument");
  *out = build_forest(codes, ids, n, M, K, byte_perm, T, split);
  ET_API_END
}

et_status et_build_flat(const uint8_t* codes, const int32_t* ids, int64_t n, int32_t M, int32_t K,
                        et_index** out) {
  ET_API_BEGIN
  if (!codes || !out) fail(ET_ERR_CONFIG, "null argument");
  *out = build_flat(codes, ids, n, M, K);
  ET_API_END
}

et_status et_build_ivf(const uint8_t* codes, const int32_t* ids, int64_t n, int32_t M, int32_t K,
                       const int32_t* list_of, int32_t nlist, const float* coarse, int32_t d,
                       const float* codebooks, et_index** out) {
  ET_API_BEGIN
  if (!codes || !out || !list_of || !coarse || !codebooks) fail(ET_ERR_CONFIG, "null argument");
  *out = build_ivf(codes, ids, n, M, K, list_of, nlist, coarse, d, codebooks);
  ET_API_END
}

et_status et_build_stats(const uint8_t* codes, const int32_t* ids, int64_t n, int32_t M, int32_t K,
                         const int32_t* byte_perm, int32_t T, const int32_t* split, et_tree_stats* out) {
  ET_API_BEGIN
  if (!codes || !out || !split) fail(ET_ERR_CONFIG, "null argument");
  struct Dry { Dry() { g_dry_run = true; } ~Dry() { g_dry_run = false; } } dry;
  std::unique_ptr<et_index> ix(build_forest(codes, ids, n, M, K, byte_perm, T, split));
  for (int t = 0; t < T; ++t) out[t] = ix->stats[t];
  ET_API_END
}

et_status et_index_stats(const et_index* ix, int32_t tree, et_tree_stats* out) {
  ET_API_BEGIN
  if (!ix || !out) fail(ET_ERR_CONFIG, "null argument");
  if (tree < 0 || tree >= ix->T) fail(ET_ERR_CONFIG, "tree index out of range");
  *out = ix->stats[tree];
  ET_API_END
}

et_status et_index_info(const et_index* ix, int32_t* T, int64_t* n, int32_t* M, int32_t* K, int64_t* groups,
                        int32_t* nlist) {
  ET_API_BEGIN
  if (!ix) fail(ET_ERR_CONFIG, "null index");
  if (T) *T = ix->T;
  if (n) *n = ix->N;
  if (M) *M = ix->M;
  if (K) *K = ix->K;
  if (groups) *groups = ix->n_groups;
  if (nlist) *nlist = ix->nlist;
  ET_API_END
}

void et_index_free(et_index* ix) {
  host_graphs_forget(ix);
  delete ix;
}

et_status et_compute_luts(const float* codebooks, int32_t d, int32_t M, int32_t K, const float* queries,
                          int64_t Q, float* luts, void* stream) {
  ET_API_BEGIN
  if (M <= 0 || K <= 0 || K > 256) fail(ET_ERR_CONFIG, "bad M/K");
  if (d <= 0 || d % M) fail(ET_ERR_SUBSPACE_SPLIT, "d % M != 0");
  if (Q < 0) fail(ET_ERR_CONFIG, "Q < 0");
  if (Q == 0) { g_err.clear(); return ET_OK; }
  if (!codebooks || !queries || !luts) fail(ET_ERR_CONFIG, "null argument");
  const bool v4 = aligned16(codebooks) && aligned16(queries);
  cudaStream_t st = (cudaStream_t)stream;
  cuda_check(timed("luts", st, [&] { return launch_luts(codebooks, d, M, K, queries, Q, luts, v4, st); }), "compute_luts");
  ET_API_END
}

et_status et_compute_ip_luts(const float* codebooks, int32_t d, int32_t M, int32_t K, const float* queries,
                             int64_t Q, float* luts, float* offsets, void* stream) {
  ET_API_BEGIN
  if (M <= 0 || K <= 0 || K > 256) fail(ET_ERR_CONFIG, "bad M/K");
  if (d <= 0 || d % M) fail(ET_ERR_SUBSPACE_SPLIT, "d % M != 0");
  if (Q < 0) fail(ET_ERR_CONFIG, "Q < 0");
  if (Q == 0) { g_err.clear(); return ET_OK; }
  if (!codebooks || !queries || !luts || !offsets) fail(ET_ERR_CONFIG, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  cuda_check(timed("luts", st, [&] { return launch_ip_luts(codebooks, d, M, K, queries, Q, luts, offsets, st); }),
             "compute_ip_luts");
  ET_API_END
}

et_status et_workspace_size(const et_index* ix, int64_t Q, int32_t k, int32_t nprobe, size_t* bytes) {
  ET_API_BEGIN
  if (!ix || !bytes) fail(ET_ERR_CONFIG, "null argument");
  if (Q < 0) fail(ET_ERR_CONFIG, "Q < 0");
  const int nsm = num_sms();
  if (ix->kind == kIvf) {
    if (nprobe < 1 || nprobe > ix->nlist) fail(ET_ERR_CONFIG, "nprobe must be 1..nlist");
    Plan pl = make_ivf_plan(ix, std::max<int64_t>(Q, 1), nprobe, k);
    *bytes = ivf_ws_bytes(ix, pl, std::max<int64_t>(Q, 1), nprobe);
    g_err.clear();
    return ET_OK;
  }
  const bool full = (k <= 0);
  Plan pl = make_plan(ix, std::max<int64_t>(Q, 1), full ? 1 : k, nsm);
  *bytes = ws_bytes(ix, pl, std::max<int64_t>(Q, 1), full, 1);
  (void)nprobe;
  ET_API_END
}

et_status et_plan_info(const et_index* ix, int64_t Q, int32_t k, int32_t* n_chunks, int32_t* S, int32_t* streams) {
  ET_API_BEGIN
  if (!ix || !n_chunks || !S || !streams) fail(ET_ERR_CONFIG, "null argument");
  if (ix->kind == kIvf) fail(ET_ERR_CONFIG, "IVF plans depend on the probes (device data)");
  if (Q < 1) fail(ET_ERR_CONFIG, "Q < 1");
  const Plan pl = make_plan(ix, Q, k <= 0 ? 1 : k, num_sms());
  *n_chunks = pl.n_chunks;
  *S = k <= 0 ? 1 : pl.S;
  *streams = (k > 0 && pl.long_ranges) ? kStreamsLong : kStreams;
  ET_API_END
}

et_status et_etree_distances(const et_index* ix, const float* codebooks, int32_t d, const float* luts,
                             const float* queries, int64_t Q, float* out, void* workspace, size_t ws,
                             void* stream) {
  ET_API_BEGIN
  if (!ix || !out) fail(ET_ERR_CONFIG, "null argument");
  if (ix->kind == kIvf) fail(ET_ERR_CONFIG, "full output is not defined for IVF indexes");
  if (Q < 0) fail(ET_ERR_CONFIG, "Q < 0");
  if (Q == 0) { g_err.clear(); return ET_OK; }
  ScanParams sp;
  table_source(sp, ix, codebooks, d, luts, queries);
  const int nsm = num_sms();
  Plan pl = make_plan(ix, Q, 1, nsm);
  pl.S = 1;   // full output: one unit per chunk writes every group
  pl.n_units = pl.n_chunks;
  const size_t need = ws_bytes(ix, pl, Q, true, 1);
  if (!workspace || ws < need) fail(ET_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  Carve c{reinterpret_cast<char*>(workspace), 0, ws};
  Work w = carve(c, ix, pl, Q, true, 1);
  cudaStream_t st = (cudaStream_t)stream;
  cuda_check(timed("fill", st, [&] { return launch_fill_flat(Q, pl.n_chunks, w.chunk_q, w.qslot_off, w.qslot, st); }), "fill");
  materialise(sp, ix, pl, w, Q, st);
  chunk_codebook(sp, ix, w, st);
  fill_scan_common(sp, ix, pl);
  sp.chunk_q = w.chunk_q;
  sp.lut0 = w.lut0;
  sp.partials = w.partials;
  sp.mode = kModeFull;
  sp.leafdist = w.leafdist;
  cuda_check(timed("scan", st, [&] { return launch_scan(sp, pl.MTmax, st); }), "scan(full)");
  cuda_check(timed("gather", st, [&] {
               return launch_gather_full(w.leafdist, ix->slot2group.as<uint32_t>(), ix->n_groups, ix->N, w.qslot, Q, out, st);
             }), "gather");
  ET_API_END
}

}  // extern "C"

// et_etree_topk / et_etree_topk_extra (etab: the leaf extra byte's decode
// table, device [256], or null).
static void etree_topk_impl(const et_index* ix, const float* codebooks, int32_t d, const float* luts,
                            const float* queries, int64_t Q, int32_t k, const float* etab, float* dist, int32_t* ids,
                            void* workspace, size_t ws, void* stream) {
  if (!ix || !dist || !ids) fail(ET_ERR_CONFIG, "null argument");
  if (ix->kind == kIvf) fail(ET_ERR_CONFIG, "use et_ivf_topk for IVF indexes");
  if (k < 1 || k > kTopkMax) fail(ET_ERR_CONFIG, "k must be 1..256");
  if (Q < 0) fail(ET_ERR_CONFIG, "Q < 0");
  if (Q == 0) return;
  if (etab && (!ix->group_extra.p || ix->T != 1)) fail(ET_ERR_CONFIG, "no leaf extra bytes (et_index_set_extra)");
  ScanParams sp;
  table_source(sp, ix, codebooks, d, luts, queries);
  const int nsm = num_sms();
  Plan pl = make_plan(ix, Q, k, nsm);
  if (etab && pl.MTmax != 8) fail(ET_ERR_CONFIG, "leaf extra bytes: 8-level trees (M = 8)");
  const size_t need = ws_bytes(ix, pl, Q, false, 1);
  if (!workspace || ws < need) fail(ET_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  Carve c{reinterpret_cast<char*>(workspace), 0, ws};
  Work w = carve(c, ix, pl, Q, false, 1);
  cudaStream_t st = (cudaStream_t)stream;
  materialise(sp, ix, pl, w, Q, st);
  chunk_codebook(sp, ix, w, st);
  fill_scan_common(sp, ix, pl);
  sp.flatQ = Q;   // arithmetic chunking: no fill launch
  sp.lut0 = w.lut0;
  sp.partials = w.partials;
  sp.mode = kModeTopk;
  sp.k = k;
  sp.B = pl.B;
  sp.cand = w.cand;
  sp.cand_cnt = w.cand_cnt;
  sp.unit_thr = w.unit_thr;
  sp.qthr = w.qthr;
  sp.qthr_shared = pl.S > 1;
  sp.long_ranges = pl.long_ranges;
  cuda_check(cudaMemsetAsync(w.qthr, 0x7f, (size_t)Q * 4, (cudaStream_t)stream), "qthr init");
  FinParams fp;
  fp.Q = Q; fp.k = k; fp.B = pl.B; fp.S = pl.S;
  fp.flat_nchunks = pl.n_chunks;
  fp.cand = w.cand; fp.cand_cnt = w.cand_cnt;
  fp.group_off = ix->group_off.as<uint32_t>();
  fp.ids = ix->ids.as<int32_t>();
  fp.group_mult = ix->group_mult.as<uint32_t>();
  fp.group_minid = ix->group_minid.as<int32_t>();
  fp.unit_thr = w.unit_thr;
  fp.qthr = w.qthr;
  fp.out_dist = dist; fp.out_ids = ids;
  // register fast path when groups are large (few candidates per query)
  fp.fast = (double)ix->N >= (double)ix->n_groups * std::max(1.0, k / 8.0);
  // small groups (many candidates): the scan kernel merges each query's
  // per-warp lists into one and cuts it to its exact unit top-k, so the
  // finalize reads one list per unit; large groups (few candidates) keep the
  // per-warp lists (the in-CTA merge costs ~5 us per CTA on c2)
  sp.compact = !fp.fast;
  fp.lpu = sp.compact ? 1 : kWarps;
  // Narrow forest scan (narrow.cuh): forests of 8 < M <= 16 bytes when every
  // chunk holds <= 8 queries (few queries per SM, c3) -- all 16 levels' tables
  // in shared memory, the tuples scanned once, no per-tree partials or join;
  // same plan, same workspace.  Lists of query slot q: lanes q + 8 g, g < 4.
  if (etab) {   // leaf extra byte: the 4-stream top-k scan with + E[e] (buffers sized for 4 streams)
    sp.gextra = ix->group_extra.as<uint8_t>();
    sp.etab = etab;
    sp.long_ranges = 0;
    cuda_check(timed("scan", st, [&] { return launch_scan(sp, pl.MTmax, st); }), "scan(topk, extra)");
    cuda_check(timed("finalize", st, [&] { return launch_finalize(fp, st); }), "finalize");
    return;
  }
  const bool narrow = ix->narrow_rec.p && !sp.luts && sp.vec4 && narrow_supported(sp.s) && fp.fast &&
                      pl.S == 1 && (Q + pl.n_chunks - 1) / pl.n_chunks <= 8 && !narrow_off();
  if (narrow) {
    sp.nrec = ix->narrow_rec.as<uint4>();
    sp.fsplit = 0;   // the trees' first levels: per-tree partials summed in tree order (A13)
    for (int t = 1; t < ix->T; ++t) sp.fsplit |= 1u << ix->split[t];
    fp.lgroups = 4;
    cuda_check(timed("scan", st, [&] { return launch_narrow(sp, st); }), "scan(narrow)");
    cuda_check(timed("finalize", st, [&] { return launch_finalize(fp, st); }), "finalize");
    return;
  }
  // (a finalize fused into the scan kernel was measured +30 us on c2: its
  // latency-bound tail runs with the SM otherwise idle)
  cuda_check(timed("scan", st, [&] { return launch_scan(sp, pl.MTmax, st); }), "scan(topk)");
  cuda_check(timed("finalize", st, [&] { return launch_finalize(fp, st); }), "finalize");
}

extern "C" {

et_status et_etree_topk(const et_index* ix, const float* codebooks, int32_t d, const float* luts,
                        const float* queries, int64_t Q, int32_t k, float* dist, int32_t* ids, void* workspace,
                        size_t ws, void* stream) {
  ET_API_BEGIN
  etree_topk_impl(ix, codebooks, d, luts, queries, Q, k, nullptr, dist, ids, workspace, ws, stream);
  ET_API_END
}

et_status et_etree_topk_extra(const et_index* ix, const float* codebooks, int32_t d, const float* luts,
                              const float* queries, int64_t Q, int32_t k, const float* extra_table, float* dist,
                              int32_t* ids, void* workspace, size_t ws, void* stream) {
  ET_API_BEGIN
  if (!extra_table) fail(ET_ERR_CONFIG, "null extra_table");
  etree_topk_impl(ix, codebooks, d, luts, queries, Q, k, extra_table, dist, ids, workspace, ws, stream);
  ET_API_END
}

}  // extern "C"

// et_etree_topk_host: the host->device copy of batch b + 1 and the
// device->host copy of batch b - 1 run on two copy streams (one per copy
// engine) while batch b is searched on the compute stream.  Per host thread
// and device: the two copy streams, a capture stream and an event pool,
// created on first use.  With page-locked host buffers the whole sequence is
// captured once into a CUDA graph per argument set (every pointer and size)
// and replayed by later calls: one cudaGraphLaunch instead of ~10 host
// launches per batch (the host enqueue otherwise exceeds the GPU time of a
// batch).
namespace {
struct HostPipe {
  cudaStream_t h2d = nullptr, d2h = nullptr, cap = nullptr;
  std::vector<cudaEvent_t> ev;
};
thread_local std::map<int, HostPipe> t_pipes;

HostPipe& host_pipe(size_t nev) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  HostPipe& hp = t_pipes[dev];
  if (!hp.h2d) {
    cuda_check(cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking), "copy stream");
    cuda_check(cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking), "copy stream");
    cuda_check(cudaStreamCreateWithFlags(&hp.cap, cudaStreamNonBlocking), "capture stream");
  }
  while (hp.ev.size() < nev) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    hp.ev.push_back(e);
  }
  return hp;
}

struct HostArgs {
  const et_index* ix;
  const float* codebooks;
  int32_t d;
  const float* qh;
  int64_t Q;
  int32_t k;
  float* dh;
  int32_t* ih;
  int32_t nb;
  float* qd;
  float* dd;
  int32_t* idd;
  void* ws;
  size_t wsb;
};

// the pipelined sequence on compute stream st (eager, or into a capture)
void enqueue_host_pipeline(const HostArgs& a, cudaStream_t st) {
  HostPipe& hp = host_pipe((size_t)2 * a.nb + 2);
  cudaEvent_t ev_start = hp.ev[2 * a.nb], ev_done = hp.ev[2 * a.nb + 1];
  // the copies start after the earlier work on st (previous users of the
  // staging buffers)
  cuda_check(cudaEventRecord(ev_start, st), "event record");
  cuda_check(cudaStreamWaitEvent(hp.h2d, ev_start, 0), "stream wait");
  cuda_check(cudaStreamWaitEvent(hp.d2h, ev_start, 0), "stream wait");
  const size_t qrow = (size_t)a.d * 4, krow = (size_t)a.k * 4;
  for (int32_t b = 0; b < a.nb; ++b) {
    const int64_t q0 = a.Q * b / a.nb, q1 = a.Q * (b + 1) / a.nb, Qb = q1 - q0;
    cudaEvent_t ev_in = hp.ev[2 * b], ev_out = hp.ev[2 * b + 1];
    cuda_check(cudaMemcpyAsync(a.qd + (size_t)q0 * a.d, a.qh + (size_t)q0 * a.d, (size_t)Qb * qrow,
                               cudaMemcpyHostToDevice, hp.h2d), "copy queries");
    cuda_check(cudaEventRecord(ev_in, hp.h2d), "event record");
    cuda_check(cudaStreamWaitEvent(st, ev_in, 0), "stream wait");
    etree_topk_impl(a.ix, a.codebooks, a.d, nullptr, a.qd + (size_t)q0 * a.d, Qb, a.k, nullptr,
                    a.dd + (size_t)q0 * a.k, a.idd + (size_t)q0 * a.k, a.ws, a.wsb, st);
    cuda_check(cudaEventRecord(ev_out, st), "event record");
    cuda_check(cudaStreamWaitEvent(hp.d2h, ev_out, 0), "stream wait");
    cuda_check(cudaMemcpyAsync(a.dh + (size_t)q0 * a.k, a.dd + (size_t)q0 * a.k, (size_t)Qb * krow,
                               cudaMemcpyDeviceToHost, hp.d2h), "copy distances");
    cuda_check(cudaMemcpyAsync(a.ih + (size_t)q0 * a.k, a.idd + (size_t)q0 * a.k, (size_t)Qb * krow,
                               cudaMemcpyDeviceToHost, hp.d2h), "copy ids");
  }
  // st completes only after the last result reached the host
  cuda_check(cudaEventRecord(ev_done, hp.d2h), "event record");
  cuda_check(cudaStreamWaitEvent(st, ev_done, 0), "stream wait");
}

bool page_locked(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeHost;
}

std::mutex g_hgmu;
std::map<std::vector<uint64_t>, cudaGraphExec_t> g_host_graphs;   // key[0] = the index
}  // namespace

// et_index_free: drop the graphs that reference the index
static void host_graphs_forget(const et_index* ix) {
  std::lock_guard<std::mutex> lk(g_hgmu);
  for (auto it = g_host_graphs.begin(); it != g_host_graphs.end();) {
    if (it->first[0] == (uint64_t)(uintptr_t)ix) { cudaGraphExecDestroy(it->second); it = g_host_graphs.erase(it); }
    else ++it;
  }
}

constexpr int kHostBatchesMax = 64;
constexpr size_t kHostGraphsMax = 32;

static int32_t host_batches(int64_t Q, int32_t n_batches) {
  // default: batches of >= 16 queries per SM (one full wave of chunks each),
  // at most 8
  int64_t nb = n_batches > 0 ? n_batches : std::min<int64_t>(8, std::max<int64_t>(1, Q / ((int64_t)num_sms() * 16)));
  nb = std::min<int64_t>(nb, std::min<int64_t>(Q, kHostBatchesMax));
  return (int32_t)std::max<int64_t>(nb, 1);
}

extern "C" {

et_status et_host_batches(int64_t Q, int32_t n_batches, int32_t* out) {
  ET_API_BEGIN
  if (!out) fail(ET_ERR_CONFIG, "null argument");
  if (Q < 0) fail(ET_ERR_CONFIG, "Q < 0");
  *out = host_batches(Q, n_batches);
  ET_API_END
}

et_status et_etree_topk_host(const et_index* ix, const float* codebooks, int32_t d, const float* queries_host,
                             int64_t Q, int32_t k, float* dist_host, int32_t* ids_host, int32_t n_batches,
                             float* queries_dev, float* dist_dev, int32_t* ids_dev, void* workspace, size_t ws,
                             void* stream) {
  ET_API_BEGIN
  if (!ix || !codebooks || !queries_host || !dist_host || !ids_host || !queries_dev || !dist_dev || !ids_dev)
    fail(ET_ERR_CONFIG, "null argument");
  if (ix->kind == kIvf) fail(ET_ERR_CONFIG, "use et_ivf_topk for IVF indexes");
  if (k < 1 || k > kTopkMax) fail(ET_ERR_CONFIG, "k must be 1..256");
  if (Q < 0) fail(ET_ERR_CONFIG, "Q < 0");
  if (d <= 0) fail(ET_ERR_DIMENSION, "d <= 0");
  if (Q == 0) { g_err.clear(); return ET_OK; }
  const int32_t nb = host_batches(Q, n_batches);
  {  // the largest batch's workspace, checked before anything is enqueued
    const int64_t qmax = (Q + nb - 1) / nb;
    const Plan pl = make_plan(ix, qmax, k, num_sms());
    const size_t need = ws_bytes(ix, pl, qmax, false, 1);
    if (!workspace || ws < need) fail(ET_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  }
  const HostArgs a{ix, codebooks, d, queries_host, Q, k, dist_host, ids_host, nb,
                   queries_dev, dist_dev, ids_dev, workspace, ws};
  cudaStream_t st = (cudaStream_t)stream;
  const bool graph = !g_timing.load() && page_locked(queries_host) && page_locked(dist_host) &&
                     page_locked(ids_host) && !getenv("ET_HOST_EAGER");
  if (!graph) {
    enqueue_host_pipeline(a, st);
    g_err.clear();
    return ET_OK;
  }
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  const std::vector<uint64_t> key{(uint64_t)(uintptr_t)ix, (uint64_t)(uintptr_t)codebooks, (uint64_t)d,
                                  (uint64_t)(uintptr_t)queries_host, (uint64_t)Q, (uint64_t)k,
                                  (uint64_t)(uintptr_t)dist_host, (uint64_t)(uintptr_t)ids_host, (uint64_t)nb,
                                  (uint64_t)(uintptr_t)queries_dev, (uint64_t)(uintptr_t)dist_dev,
                                  (uint64_t)(uintptr_t)ids_dev, (uint64_t)(uintptr_t)workspace, (uint64_t)ws,
                                  (uint64_t)dev};
  cudaGraphExec_t exec = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_hgmu);
    auto it = g_host_graphs.find(key);
    if (it != g_host_graphs.end()) exec = it->second;
  }
  if (!exec) {
    HostPipe& hp = host_pipe((size_t)2 * nb + 2);
    cuda_check(cudaStreamBeginCapture(hp.cap, cudaStreamCaptureModeRelaxed), "begin capture");
    cudaGraph_t g = nullptr;
    try {
      enqueue_host_pipeline(a, hp.cap);
    } catch (...) {
      cudaStreamEndCapture(hp.cap, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cuda_check(cudaStreamEndCapture(hp.cap, &g), "end capture");
    const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    cuda_check(e, "graph instantiate");
    std::lock_guard<std::mutex> lk(g_hgmu);
    if (g_host_graphs.size() >= kHostGraphsMax) {
      for (auto& kv : g_host_graphs) cudaGraphExecDestroy(kv.second);
      g_host_graphs.clear();
    }
    g_host_graphs[key] = exec;
  }
  cuda_check(cudaGraphLaunch(exec, st), "graph launch");
  ET_API_END
}

et_status et_index_set_extra(et_index* ix, const uint8_t* extra, int64_t n) {
  ET_API_BEGIN
  if (!ix || !extra) fail(ET_ERR_CONFIG, "null argument");
  if (ix->kind != kTree || ix->T != 1) fail(ET_ERR_CONFIG, "leaf extra bytes: single E-Tree indexes only");
  if (n != ix->N) fail(ET_ERR_DIMENSION, "n != the index's N");
  if (!ix->slot2group.p) fail(ET_ERR_CONFIG, "index without slot map");
  std::vector<uint32_t> s2g((size_t)n);
  cuda_check(cudaMemcpy(s2g.data(), ix->slot2group.p, (size_t)n * 4, cudaMemcpyDeviceToHost), "slot map");
  std::vector<int> ge((size_t)ix->n_groups, -1);
  for (int64_t i = 0; i < n; ++i) {   // the byte lives on the leaf: one per distinct code
    int& g = ge[s2g[(size_t)i]];
    if (g < 0) g = extra[i];
    else if (g != extra[i]) fail(ET_ERR_INVALID_CODE, "extra byte differs among vectors with the same code");
  }
  std::vector<uint8_t> gb(ge.size());
  for (size_t j = 0; j < ge.size(); ++j) gb[j] = (uint8_t)std::max(0, ge[j]);
  ix->group_extra.reset();
  ix->group_extra.upload(gb);
  ET_API_END
}

et_status et_ivf_topk(const et_index* ix, const float* queries, int64_t Q, int32_t nprobe, int32_t k,
                      float* dist, int32_t* ids, int32_t* probes, void* workspace, size_t ws, void* stream) {
  ET_API_BEGIN
  if (!ix || !queries || !dist || !ids) fail(ET_ERR_CONFIG, "null argument");
  if (ix->kind != kIvf) fail(ET_ERR_CONFIG, "not an IVF index");
  if (k < 1 || k > kTopkMax) fail(ET_ERR_CONFIG, "k must be 1..256");
  if (nprobe < 1 || nprobe > ix->nlist) fail(ET_ERR_CONFIG, "nprobe must be 1..nlist");
  if (Q < 0) fail(ET_ERR_CONFIG, "Q < 0");
  if (Q == 0) { g_err.clear(); return ET_OK; }
  if ((size_t)Q * nprobe >= (size_t)INT32_MAX / 2) fail(ET_ERR_CONFIG, "Q * nprobe too large");
  Plan pl = make_ivf_plan(ix, Q, nprobe, k);
  const size_t need = ivf_ws_bytes(ix, pl, Q, nprobe);
  if (!workspace || ws < need) fail(ET_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  Carve c{reinterpret_cast<char*>(workspace), 0, ws};
  IvfWork v = carve_ivf(c, ix, pl, Q, nprobe);
  Work w = carve(c, ix, pl, Q, false, nprobe);
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* pr = probes ? probes : v.probes;
  cuda_check(timed("probe", st, [&] {
               return launch_probe(ix->coarse_t.as<float>(), ix->nlist, ix->d, queries, Q, nprobe, pr, st);
             }), "probe");
  cuda_check(timed("bucket", st, [&] {
               return launch_ivf_bucket(pr, Q, nprobe, ix->nlist, ix->list_leaf_off_d.as<uint32_t>(),
                                        ix->cell_order_d.as<int>(), v.cell_cnt,
                                        v.pair_pos, v.chunk_off, v.n_chunks, v.chunk_cell, v.chunk_lo, v.chunk_hi,
                                        w.chunk_q, pl.n_chunks, w.qslot_off, w.qslot, st);
             }), "bucket");
  ScanParams sp;
  sp.queries = queries;
  sp.codebooks = ix->codebooks.as<float>();
  sp.coarse = ix->coarse.as<float>();
  sp.d = ix->d;
  sp.s = ix->d / ix->M;
  sp.vec4 = aligned16(queries) && (ix->d % 4 == 0) ? 1 : 0;
  fill_scan_common(sp, ix, pl);
  sp.chunk_q = w.chunk_q;
  sp.chunk_cell = v.chunk_cell;
  sp.chunk_lo = v.chunk_lo;
  sp.chunk_hi = v.chunk_hi;
  sp.n_chunks_dev = v.n_chunks;
  sp.lut0 = w.lut0;
  sp.mode = kModeTopk;
  sp.k = k;
  sp.B = pl.B;
  sp.cand = w.cand;
  sp.cand_cnt = w.cand_cnt;
  sp.unit_thr = w.unit_thr;
  sp.qthr = w.qthr;
  sp.qthr_shared = 1;
  sp.long_ranges = pl.long_ranges;
  cuda_check(cudaMemsetAsync(w.qthr, 0x7f, (size_t)Q * 4, st), "qthr init");
  const bool ivf_fast = (double)ix->N >= (double)ix->n_groups * std::max(1.0, k / 8.0);
  sp.compact = !ivf_fast;
  cuda_check(timed("scan", st, [&] { return launch_scan(sp, pl.MTmax, st); }), "scan(ivf)");
  FinParams fp;
  fp.Q = Q; fp.k = k; fp.B = pl.B; fp.S = pl.S;
  fp.qslot_off = w.qslot_off; fp.qslot = w.qslot;
  fp.cand = w.cand; fp.cand_cnt = w.cand_cnt;
  fp.group_off = ix->group_off.as<uint32_t>();
  fp.ids = ix->ids.as<int32_t>();
  fp.group_mult = ix->group_mult.as<uint32_t>();
  fp.group_minid = ix->group_minid.as<int32_t>();
  fp.unit_thr = w.unit_thr;
  fp.qthr = w.qthr;
  fp.out_dist = dist; fp.out_ids = ids;
  fp.fast = ivf_fast;
  fp.lpu = sp.compact ? 1 : kWarps;
  cuda_check(timed("finalize", st, [&] { return launch_finalize(fp, st); }), "finalize");
  ET_API_END
}

et_status et_merge_topk(const float* in_dist, const int32_t* in_ids, int32_t G, int64_t Q, int32_t k,
                        float* out_dist, int32_t* out_ids, void* stream) {
  ET_API_BEGIN
  if (G < 1 || k < 1 || k > kTopkMax) fail(ET_ERR_CONFIG, "bad G or k");
  if (Q <= 0) { g_err.clear(); return ET_OK; }
  if (!in_dist || !in_ids || !out_dist || !out_ids) fail(ET_ERR_CONFIG, "null argument");
  cuda_check(launch_merge(in_dist, in_ids, G, Q, k, out_dist, out_ids, (cudaStream_t)stream), "merge");
  ET_API_END
}

// The cut rule of et_shard_bounds on a first-byte histogram (shared by both entry points).
static void shard_cut(const int64_t* hist, int K, int G, int32_t* bounds) {
  std::vector<int64_t> below(K + 1, 0);   // below[v] = #codes with byte 0 < v
  for (int v = 0; v < K; ++v) {
    if (hist[v] < 0) fail(ET_ERR_CONFIG, "negative histogram count");
    below[v + 1] = below[v] + hist[v];
  }
  const int64_t n = below[K];
  bounds[0] = 0;
  int v = 0;
  for (int r = 1; r < G; ++r) {   // below[] is non-decreasing: the cut only moves right
    while (v < K && (__int128)below[v] * G < (__int128)r * n) ++v;
    bounds[r] = std::max(bounds[r - 1], v);
  }
  bounds[G] = K;
}

et_status et_shard_bounds(const uint8_t* codes, int64_t n, int32_t M, int32_t G, int32_t K, int32_t* bounds) {
  ET_API_BEGIN
  if (!bounds || (n > 0 && !codes)) fail(ET_ERR_CONFIG, "null argument");
  if (G < 1 || K < 1 || K > 256 || M < 1 || n < 0) fail(ET_ERR_CONFIG, "bad G/K/M/n");
  std::vector<int64_t> hist(K, 0);
  for (int64_t i = 0; i < n; ++i) {
    const int b = codes[(size_t)i * M];
    if (b >= K) fail(ET_ERR_INVALID_CODE, "code byte >= K");
    ++hist[b];
  }
  shard_cut(hist.data(), K, G, bounds);
  ET_API_END
}

et_status et_shard_bounds_hist(const int64_t* hist, int32_t K, int32_t G, int32_t* bounds) {
  ET_API_BEGIN
  if (!hist || !bounds) fail(ET_ERR_CONFIG, "null argument");
  if (G < 1 || K < 1 || K > 256) fail(ET_ERR_CONFIG, "bad G/K");
  shard_cut(hist, K, G, bounds);
  ET_API_END
}

et_status et_shard_lists(const int64_t* list_sizes, int32_t nlist, int32_t G, int32_t* owner) {
  ET_API_BEGIN
  if (!list_sizes || !owner) fail(ET_ERR_CONFIG, "null argument");
  if (G < 1 || nlist < 1) fail(ET_ERR_CONFIG, "bad G/nlist");
  std::vector<int32_t> order(nlist);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return list_sizes[a] > list_sizes[b]; });
  std::vector<int64_t> load(G, 0);
  for (int32_t c : order) {
    const int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());   // first minimum
    owner[c] = r;
    load[r] += list_sizes[c];
  }
  ET_API_END
}

et_status et_flat_adc(const float* luts, int64_t Q, int32_t M, int32_t K, const uint8_t* codes, int64_t n,
                      float* out, void* stream) {
  ET_API_BEGIN
  if (M <= 0 || K <= 0 || K > 256) fail(ET_ERR_CONFIG, "bad M/K");
  if (Q <= 0 || n <= 0) { g_err.clear(); return ET_OK; }
  if (!luts || !codes || !out) fail(ET_ERR_CONFIG, "null argument");
  cuda_check(launch_flat_adc(luts, Q, M, K, codes, n, out, (cudaStream_t)stream), "flat_adc");
  ET_API_END
}

et_status et_encode(const float* codebooks, int32_t d, int32_t M, int32_t K, const float* x, int64_t n,
                    const float* centroids, const int32_t* assign, uint8_t* codes, void* stream) {
  ET_API_BEGIN
  if (M <= 0 || K <= 0 || K > 256) fail(ET_ERR_CONFIG, "bad M/K");
  if (d <= 0 || d % M) fail(ET_ERR_SUBSPACE_SPLIT, "d % M != 0");
  if ((centroids == nullptr) != (assign == nullptr)) fail(ET_ERR_CONFIG, "centroids and assign go together");
  if (n <= 0) { g_err.clear(); return ET_OK; }
  if (!codebooks || !x || !codes) fail(ET_ERR_CONFIG, "null argument");
  if ((size_t)K * (d / M) * 4 > 200 * 1024) fail(ET_ERR_CONFIG, "codebook of one subspace exceeds shared memory");
  cuda_check(launch_encode(codebooks, d, M, K, x, n, centroids, assign, codes, (cudaStream_t)stream), "encode");
  ET_API_END
}

et_status et_assign(const float* centroids, int32_t nlist, int32_t d, const float* x, int64_t n, int32_t* assign,
                    void* stream) {
  ET_API_BEGIN
  if (nlist < 1 || d < 1) fail(ET_ERR_CONFIG, "bad nlist/d");
  if (n <= 0) { g_err.clear(); return ET_OK; }
  if (!centroids || !x || !assign) fail(ET_ERR_CONFIG, "null argument");
  if ((size_t)32 * d * 4 > 200 * 1024) fail(ET_ERR_CONFIG, "d too large");
  cuda_check(launch_assign(centroids, nlist, d, x, n, assign, nullptr, (cudaStream_t)stream), "assign");
  ET_API_END
}

}  // extern "C"

// ---------------------------------------------------------------------------
// k-means (et_build_codebooks): k-means++ on the host (fp64, splitmix64 RNG),
// Lloyd with the GPU encode kernel as the assignment step, fp64 updates.
// ---------------------------------------------------------------------------
namespace et {

static inline uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline double u01(uint64_t& s) { return (splitmix64(s) >> 11) * (1.0 / 9007199254740992.0); }

static void kmeanspp_sub(const float* train, int64_t n, int d, int off, int s, int K, uint64_t seed,
                         double* C /* K*s */) {
  uint64_t rs = seed;
  std::vector<double> D(n);
  auto dist = [&](int64_t i, const double* c) {
    const float* x = train + (size_t)i * d + off;
    double a = 0;
    for (int j = 0; j < s; ++j) { const double t = (double)x[j] - c[j]; a += t * t; }
    return a;
  };
  int64_t i0 = (int64_t)(splitmix64(rs) % (uint64_t)n);
  for (int j = 0; j < s; ++j) C[j] = train[(size_t)i0 * d + off + j];
  double tot = 0;
  for (int64_t i = 0; i < n; ++i) { D[i] = dist(i, C); tot += D[i]; }
  for (int k = 1; k < K; ++k) {
    int64_t pick;
    if (tot <= 0) pick = (int64_t)(splitmix64(rs) % (uint64_t)n);
    else {
      const double u = u01(rs) * tot;
      double acc = 0;
      pick = n - 1;
      for (int64_t i = 0; i < n; ++i) { acc += D[i]; if (acc > u) { pick = i; break; } }
    }
    double* ck = C + (size_t)k * s;
    for (int j = 0; j < s; ++j) ck[j] = train[(size_t)pick * d + off + j];
    tot = 0;
    for (int64_t i = 0; i < n; ++i) { D[i] = std::min(D[i], dist(i, ck)); tot += D[i]; }
  }
}

}  // namespace et

extern "C" et_status et_build_codebooks(const float* train, int64_t n, int32_t d, int32_t M, int32_t K,
                                        int32_t lloyd_iters, uint64_t seed, float* codebooks,
                                        double* objective_hist) {
  ET_API_BEGIN
  if (!train || !codebooks) fail(ET_ERR_CONFIG, "null argument");
  if (M <= 0 || d <= 0 || d % M) fail(ET_ERR_SUBSPACE_SPLIT, "d % M != 0");
  if (K <= 0 || K > 256) fail(ET_ERR_CONFIG, "K must be 1..256");
  if (n < K) fail(ET_ERR_INSUFFICIENT_DATA, "n < K");
  if (lloyd_iters < 1) fail(ET_ERR_CONFIG, "lloyd_iters >= 1");
  for (int64_t i = 0; i < n * d; ++i)
    if (!std::isfinite(train[i])) fail(ET_ERR_INVALID_VECTOR, "non-finite training value");
  const int s = d / M;
  std::vector<double> C((size_t)M * K * s);
  {
    std::vector<std::thread> th;
    for (int m = 0; m < M; ++m)
      th.emplace_back(kmeanspp_sub, train, n, d, m * s, s, K, seed * 1000003ull + (uint64_t)m, C.data() + (size_t)m * K * s);
    for (auto& t : th) t.join();
  }
  float* dx = nullptr; float* dc = nullptr; uint8_t* dcodes = nullptr;
  auto cleanup = [&]() { if (dx) cudaFree(dx); if (dc) cudaFree(dc); if (dcodes) cudaFree(dcodes); };
  try {
    cuda_check(cudaMalloc(&dx, (size_t)n * d * 4), "cudaMalloc(train)");
    cuda_check(cudaMalloc(&dc, (size_t)M * K * s * 4), "cudaMalloc(cb)");
    cuda_check(cudaMalloc(&dcodes, (size_t)n * M), "cudaMalloc(codes)");
    cuda_check(cudaMemcpy(dx, train, (size_t)n * d * 4, cudaMemcpyHostToDevice), "upload train");
    std::vector<float> Cf((size_t)M * K * s);
    std::vector<uint8_t> codes((size_t)n * M);
    for (int it = 0; it < lloyd_iters; ++it) {
      for (size_t i = 0; i < Cf.size(); ++i) Cf[i] = (float)C[i];
      cuda_check(cudaMemcpy(dc, Cf.data(), Cf.size() * 4, cudaMemcpyHostToDevice), "upload cb");
      cuda_check(launch_encode(dc, d, M, K, dx, n, nullptr, nullptr, dcodes, 0), "assign");
      cuda_check(cudaMemcpy(codes.data(), dcodes, codes.size(), cudaMemcpyDeviceToHost), "download codes");
      for (int m = 0; m < M; ++m) {
        std::vector<double> sum((size_t)K * s, 0.0), far(n);
        std::vector<int64_t> cnt(K, 0);
        double obj = 0;
        const float* cm = Cf.data() + (size_t)m * K * s;
        for (int64_t i = 0; i < n; ++i) {
          const int k = codes[(size_t)i * M + m];
          const float* x = train + (size_t)i * d + m * s;
          double a = 0;
          for (int j = 0; j < s; ++j) {
            const double t = (double)x[j] - (double)cm[(size_t)k * s + j];
            a += t * t;
            sum[(size_t)k * s + j] += x[j];
          }
          far[i] = a;
          obj += a;
          ++cnt[k];
        }
        if (objective_hist) objective_hist[(size_t)m * lloyd_iters + it] = obj;
        std::vector<int64_t> order;
        for (int k = 0; k < K; ++k) {
          double* ck = C.data() + ((size_t)m * K + k) * s;
          if (cnt[k] > 0) {
            for (int j = 0; j < s; ++j) ck[j] = sum[(size_t)k * s + j] / (double)cnt[k];
          } else {   // empty cluster -> farthest point from its assigned centroid
            if (order.empty()) {
              order.resize(n);
              std::iota(order.begin(), order.end(), 0);
              std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return far[a] > far[b]; });
            }
            int64_t pick = order.front();
            order.erase(order.begin());
            for (int j = 0; j < s; ++j) ck[j] = train[(size_t)pick * d + m * s + j];
          }
        }
      }
    }
    for (size_t i = 0; i < C.size(); ++i) codebooks[i] = (float)C[i];
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  ET_API_END
}

// ---------------------------------------------------------------------------
// coarse quantizer for IVF (K' up to 65536 centroids of full dimension d):
// k-means++ on the host (fp64; distance updates split over threads), Lloyd
// with the GPU assign kernel, fp64 centroid updates, empty -> farthest point.
// ---------------------------------------------------------------------------
extern "C" et_status et_build_coarse(const float* train, int64_t n, int32_t d, int32_t nlist, int32_t lloyd_iters,
                                     uint64_t seed, float* centroids, double* objective_hist) {
  ET_API_BEGIN
  if (!train || !centroids) fail(ET_ERR_CONFIG, "null argument");
  if (d <= 0 || nlist <= 0 || nlist > 65536) fail(ET_ERR_CONFIG, "bad d / nlist");
  if (n < nlist) fail(ET_ERR_INSUFFICIENT_DATA, "n < nlist");
  if (lloyd_iters < 1) fail(ET_ERR_CONFIG, "lloyd_iters >= 1");
  if ((size_t)32 * d * 4 > 200 * 1024) fail(ET_ERR_CONFIG, "d too large");
  for (int64_t i = 0; i < n * d; ++i)
    if (!std::isfinite(train[i])) fail(ET_ERR_INVALID_VECTOR, "non-finite training value");
  std::vector<double> C((size_t)nlist * d);
  {
    uint64_t rs = seed * 1000003ull + 77;
    std::vector<double> D(n);
    const int nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    auto update = [&](const double* c, bool first) {
      std::vector<std::thread> th;
      std::vector<double> part(nth, 0.0);
      for (int w = 0; w < nth; ++w)
        th.emplace_back([&, w]() {
          const int64_t a = n * w / nth, b = n * (w + 1) / nth;
          double acc = 0;
          for (int64_t i = a; i < b; ++i) {
            const float* x = train + (size_t)i * d;
            double s2 = 0;
            for (int j = 0; j < d; ++j) { const double t = (double)x[j] - c[j]; s2 += t * t; }
            D[i] = first ? s2 : std::min(D[i], s2);
            acc += D[i];
          }
          part[w] = acc;
        });
      for (auto& t : th) t.join();
      double tot = 0;
      for (double v : part) tot += v;
      return tot;
    };
    int64_t i0 = (int64_t)(splitmix64(rs) % (uint64_t)n);
    for (int j = 0; j < d; ++j) C[j] = train[(size_t)i0 * d + j];
    double tot = update(C.data(), true);
    for (int k = 1; k < nlist; ++k) {
      int64_t pick = n - 1;
      if (tot <= 0) pick = (int64_t)(splitmix64(rs) % (uint64_t)n);
      else {
        const double u = u01(rs) * tot;
        double acc = 0;
        for (int64_t i = 0; i < n; ++i) { acc += D[i]; if (acc > u) { pick = i; break; } }
      }
      double* ck = C.data() + (size_t)k * d;
      for (int j = 0; j < d; ++j) ck[j] = train[(size_t)pick * d + j];
      tot = update(ck, false);
    }
  }
  float* dx = nullptr; float* dc = nullptr; int32_t* da = nullptr; float* dd = nullptr;
  auto cleanup = [&]() { if (dx) cudaFree(dx); if (dc) cudaFree(dc); if (da) cudaFree(da); if (dd) cudaFree(dd); };
  try {
    cuda_check(cudaMalloc(&dx, (size_t)n * d * 4), "cudaMalloc(train)");
    cuda_check(cudaMalloc(&dc, (size_t)nlist * d * 4), "cudaMalloc(centroids)");
    cuda_check(cudaMalloc(&da, (size_t)n * 4), "cudaMalloc(assign)");
    cuda_check(cudaMalloc(&dd, (size_t)n * 4), "cudaMalloc(dist)");
    cuda_check(cudaMemcpy(dx, train, (size_t)n * d * 4, cudaMemcpyHostToDevice), "upload train");
    std::vector<float> Cf((size_t)nlist * d);
    std::vector<int32_t> a(n);
    for (int it = 0; it < lloyd_iters; ++it) {
      for (size_t i = 0; i < Cf.size(); ++i) Cf[i] = (float)C[i];
      cuda_check(cudaMemcpy(dc, Cf.data(), Cf.size() * 4, cudaMemcpyHostToDevice), "upload centroids");
      cuda_check(launch_assign(dc, nlist, d, dx, n, da, dd, 0), "assign");
      cuda_check(cudaMemcpy(a.data(), da, (size_t)n * 4, cudaMemcpyDeviceToHost), "download assign");
      std::vector<double> sum((size_t)nlist * d, 0.0), far(n);
      std::vector<int64_t> cnt(nlist, 0);
      double obj = 0;
      for (int64_t i = 0; i < n; ++i) {
        const int k = a[i];
        const float* x = train + (size_t)i * d;
        double s2 = 0;
        for (int j = 0; j < d; ++j) {
          const double t = (double)x[j] - (double)Cf[(size_t)k * d + j];
          s2 += t * t;
          sum[(size_t)k * d + j] += x[j];
        }
        far[i] = s2;
        obj += s2;
        ++cnt[k];
      }
      if (objective_hist) objective_hist[it] = obj;
      std::vector<int64_t> order;
      size_t next_far = 0;
      for (int k = 0; k < nlist; ++k) {
        double* ck = C.data() + (size_t)k * d;
        if (cnt[k] > 0) {
          for (int j = 0; j < d; ++j) ck[j] = sum[(size_t)k * d + j] / (double)cnt[k];
        } else {
          if (order.empty()) {
            order.resize(n);
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return far[x] > far[y]; });
          }
          const int64_t pick = order[std::min(next_far++, order.size() - 1)];
          for (int j = 0; j < d; ++j) ck[j] = train[(size_t)pick * d + j];
        }
      }
    }
    for (size_t i = 0; i < C.size(); ++i) centroids[i] = (float)C[i];
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  ET_API_END
}
