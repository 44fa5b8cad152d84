// internal.h -- structures shared by the host build (host.cpp) and the sm_100a
// kernels (kernels.cu) of libetree.  Not part of the C ABI (see include/etree.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include <vector>

namespace et {

constexpr int kWarps = 8;                  // warps per scan CTA (1 CTA / SM: the tables fill smem; 255 registers)
constexpr int kThreads = kWarps * 32;
constexpr int kMaxTrees = 4;               // E-Forest trees supported by one index
constexpr int kMaxMT = 8;                  // levels (code bytes) per tree on the GPU
constexpr int kKMax = 256;                 // codewords per subspace (one byte)
constexpr int kTopkMax = 256;              // largest k of the fused top-k
constexpr int kFinWarps = 8;               // warps per finalize CTA
constexpr int kStreams = 4;                // lockstep leaf streams per scan warp (8 warps: 32 chains per SM)
#ifndef ET_STREAMS_LONG
#define ET_STREAMS_LONG 6
#endif
constexpr int kStreamsLong = ET_STREAMS_LONG;   // ... for long leaf ranges (>= kLongRange leaves per warp, host plan)
constexpr int kLongRange = 384;
constexpr int kBatchEmit = 32 * kStreams;  // candidates a lane can append between two buffer checks
constexpr int kBatchEmitLong = 32 * kStreamsLong;   // ... with kStreamsLong streams (buffers 64 entries longer)

// One tree of the device layout ("leaf-major HMS"): the leaves in
// depth-first (= lexicographic) order, each with its full projected code and
// the length of its common prefix with the previous leaf.  The internal nodes
// of the paper's Hierarchical Memory Structure are implicit: a leaf whose LCP
// with its predecessor is p enters the new internal nodes at depths p..depth-1,
// whose K fields are the leaf's own code bytes.  The code is stored
// "compiled": 16 bits per level = the pre-swizzled shared-memory byte offset of
// table entry (l, code byte l) -- (k << 7) | ((k & 31) << 2) -- or, for level 0
// of an 8-level tree (TMEM), the raw byte k.
struct TreeDev {
  int MT = 0;                  // levels of this tree
  int layer0 = 0;              // first code byte it covers
  int64_t n_leaves = 0;
  const uint4* rec = nullptr;       // 8 x u16 per leaf (level l in half-word l)
  const uint8_t* lcp = nullptr;     // LCP with the previous leaf (0 for leaf 0)
};

struct FinParams {
  int64_t Q = 0;
  int k = 0, B = 0, S = 1;
  int lpu = kWarps;                   // candidate lists per unit (1: compacted by the scan kernel)
  int lgroups = 1;                    // lane groups per query slot (narrow scan: 4, lanes q + 8 g)
  const int* qslot_off = nullptr;     // [Q+1]
  const int* qslot = nullptr;         // chunk*32 + lane for each (query, probe)
  int flat_nchunks = 0;               // > 0: one slot per query, computed from the flat chunking
  const uint2* cand = nullptr;
  const int* cand_cnt = nullptr;
  const uint32_t* group_off = nullptr;  // [n_groups+1]
  const int32_t* ids = nullptr;         // [N] grouped, ascending within a group
  const uint32_t* group_mult = nullptr;
  const int32_t* group_minid = nullptr;
  const float* unit_thr = nullptr;      // [n_units][32] or null
  const unsigned* qthr = nullptr;       // [Q] final per-query thresholds (float bits) or null
  float* out_dist = nullptr;
  int32_t* out_ids = nullptr;
  // two-tier finalize: a register fast path for few candidates per query; the
  // shared-memory path (finalize_query) for the rest (kernels.cu)
  int fast = 0;
};


enum ScanMode : int { kModeFull = 0, kModeTopk = 1 };

struct ScanParams {
  // ---- distance-table source ----
  const float* codebooks = nullptr;   // [M][K][s]        (fused tables)
  const float* queries = nullptr;     // [Q][d]           (fused tables)
  const float* luts = nullptr;        // [Q][M][K]        (materialised tables) or null
  const float4* cbt = nullptr;        // [M][s/4][K] chunk-major codebook copy (16 < s <= 64) or null
  const uint4* nrec = nullptr;        // narrow forest records, 2 per tuple (narrow.cuh) or null
  const uint8_t* gextra = nullptr;    // leaf extra byte per group or null
  const float* etab = nullptr;        // its decode table [256] (device, per call)
  const float* coarse = nullptr;      // [nlist][d]       (IVF residual tables) or null
  const int* layer_sub = nullptr;     // [M] subspace of each code byte (chunk order), device copy
  int lsub[kMaxTrees * kMaxMT] = {};  // the same, by value (kernel parameters: no dependent load)
  int d = 0, M = 0, K = 0, s = 0;
  // ---- work decomposition ----
  int n_units = 0;                    // CTAs = n_chunks * S
  int S = 1;                          // leaf segments per chunk
  const int* chunk_q = nullptr;       // [n_chunks][32] query of each lane, -1 = idle (active lanes first)
  int64_t flatQ = 0;                  // > 0: chunk c holds queries [c*Q/n, (c+1)*Q/n) (chunk_q unused)
  const int* chunk_cell = nullptr;    // [n_chunks] coarse cell (IVF) or null
  const uint32_t* chunk_lo = nullptr; // [n_chunks] tree-0 leaf range (IVF lists) or null
  const uint32_t* chunk_hi = nullptr;
  const int* n_chunks_dev = nullptr;  // IVF: actual chunk count (device), units beyond it exit
  // ---- trees / groups ----
  int T = 1;
  TreeDev tree[kMaxTrees];
  const uint32_t* t0_tup_off = nullptr;            // forest: [L2_0+1] tuples of each tree-0 leaf
  const uint32_t* tup_leaf[kMaxTrees] = {};        // forest: [n_groups] leaf of tuple in tree t>=1
  const uint32_t* group_mult = nullptr;            // [n_groups] ids per group
  const int32_t* group_minid = nullptr;            // [n_groups] smallest id of the group
  int64_t n_groups = 0;
  // ---- scratch ----
  float* lut0 = nullptr;              // [n_units][256][32] level-0 tables when MT == 8
  float* partials = nullptr;          // forest: per unit, trees 1..T-1: [L2_t][32]
  int64_t part_base[kMaxTrees] = {};  // offset of tree t's block inside a unit's partials
  int64_t part_stride = 0;            // floats per unit
  // ---- outputs ----
  int mode = kModeTopk;
  float* leafdist = nullptr;          // FULL: [n_chunks][n_groups][32]
  int k = 0;                          // TOPK
  int B = 0;                          // candidate buffer capacity per (unit, warp, lane)
  uint2* cand = nullptr;              // [n_units][kWarps][32][B] (dist bits, group)
  int* cand_cnt = nullptr;            // [n_units][kWarps][32]
  float* unit_thr = nullptr;          // [n_units][32] final CTA threshold per lane
  unsigned* qthr = nullptr;           // [Q] per-query threshold (float bits), shared by all units
  int qthr_shared = 0;                // several units per query (S > 1, IVF): share during the scan
  int vec4 = 1;                       // query/codebook rows 16-byte aligned
  int compact = 0;                    // merge each lane's 16 per-warp lists at the end (long lists)
  int wide_old = 0;                   // experiments (ET_WIDE_OLD=1): s > 16 8-level trees use build_tables_wide
  int long_ranges = 0;                // >= kLongRange leaves per scan warp: kStreamsLong streams (top-k)
  // ---- fused E-Forest (M <= 8) ----
  int masked = 0;                     // records carry a per-level lookup mask (fused forest tuple records)
  uint32_t fsplit = 0;                // bit l set: level l starts a forest tree (partials summed in tree order)
};

// Shared-memory layout of the scan kernel (byte offsets from the dynamic
// shared-memory base).  8-level trees keep levels 0 and 1 in TMEM and levels
// 2..7 in six 32 KB regions, and stage the chunk's query sub-vectors of all 8
// levels in their own area; shorter trees keep every level in shared memory.
constexpr int kTmemLevels = 2;             // levels of an 8-level tree held in TMEM
#ifndef ET_REC_SMEM
#define ET_REC_SMEM 1                      // 1: leaf records broadcast through shared memory (scan_tree3 RS)
#endif
// RS: kWarps x kStreamsLong x 32 records x 16 B = 24 KB, the 16 KB staging area + this extension
constexpr uint32_t kRecExtra = ET_REC_SMEM ? (uint32_t)(kWarps * kStreamsLong * 512 - 8 * 16 * 128) : 0u;
struct ScanSmem { uint32_t levels, big_stage, thr, qidx, stage, tmem_slot, total; };
__host__ __device__ inline ScanSmem scan_smem(int MTmax) {
  ScanSmem L{};
  L.levels = (MTmax == 8) ? 8 - kTmemLevels : (uint32_t)MTmax;
  uint32_t off = L.levels * 32768u;
  L.big_stage = off;
  if (MTmax == 8) off += 8u * 16u * 128u + kRecExtra;   // [level][query pair][dim][2] fp32 (+ the RS records)
  L.thr = off; off += 128u;
  L.qidx = off; off += 128u;
  L.stage = off; off += 32u * 16u * 4u;
  L.tmem_slot = off; off += 16u;
  L.total = off;
  return L;
}

// ---- launchers (kernels.cu); each returns cudaGetLastError() ----
cudaError_t launch_scan(const ScanParams& p, int MTmax, cudaStream_t st);
// narrow forest scan (<= 8 queries per CTA, 8 < M <= 16, s in {16, 60}); false if no instantiation
bool narrow_supported(int s);
cudaError_t launch_narrow(const ScanParams& p, cudaStream_t st);
cudaError_t launch_finalize(const FinParams& p, cudaStream_t st);
cudaError_t launch_fill_flat(int64_t Q, int n_chunks, int* chunk_q, int* qslot_off, int* qslot,
                             cudaStream_t st);
cudaError_t launch_gather_full(const float* leafdist, const uint32_t* slot2group,
                               int64_t n_groups, int64_t n, const int* qslot, int64_t Q,
                               float* out, cudaStream_t st);
cudaError_t launch_ip_luts(const float* codebooks, int d, int M, int K, const float* queries, int64_t Q,
                           float* luts, float* off, cudaStream_t st);
cudaError_t launch_cb_chunks(const float* codebooks, int M, int K, int s, float4* out, cudaStream_t st);
cudaError_t launch_luts(const float* codebooks, int d, int M, int K, const float* queries,
                        int64_t Q, float* luts, bool vec4, cudaStream_t st);
cudaError_t launch_flat_adc(const float* luts, int64_t Q, int M, int K, const uint8_t* codes,
                            int64_t n, float* out, cudaStream_t st);
cudaError_t launch_encode(const float* codebooks, int d, int M, int K, const float* x, int64_t n,
                          const float* centroids, const int32_t* assign, uint8_t* codes,
                          cudaStream_t st);
cudaError_t launch_assign(const float* centroids, int nlist, int d, const float* x, int64_t n,
                          int32_t* assign, float* best_dist, cudaStream_t st);
cudaError_t launch_probe(const float* centroids_t, int nlist, int d, const float* queries, int64_t Q,
                         int w, int32_t* probes, cudaStream_t st);
cudaError_t launch_ivf_bucket(const int32_t* probes, int64_t Q, int w, int nlist, const uint32_t* list_leaf_off,
                              const int* cell_order, int* cell_cnt, int* pair_pos, int* chunk_off, int* n_chunks, int* chunk_cell,
                              uint32_t* chunk_lo, uint32_t* chunk_hi, int* chunk_q, int max_chunks,
                              int* qslot_off, int* qslot, cudaStream_t st);
cudaError_t launch_merge(const float* in_dist, const int32_t* in_ids, int G, int64_t Q, int k,
                         float* out_dist, int32_t* out_ids, cudaStream_t st);
void count_launch(int n = 1);

// GPU grouping step of the index build (build_gpu.cu): codes sorted
// lexicographically (byte order `perm`), ids ascending within equal codes;
// G groups of identical codes (IVF: of identical (list, code) pairs).  Device arrays (owned by the caller after the
// call): ids [n] grouped, group_off [G+1], mult [G], minid [G], slot2group [n].
// Host: off [G+1], first [G] = one slot of each group.
struct GpuGroups {
  int64_t G = 0;
  std::vector<uint32_t> off, first;
  int32_t* ids = nullptr;
  uint32_t* group_off = nullptr;
  uint32_t* mult = nullptr;
  int32_t* minid = nullptr;
  uint32_t* slot2group = nullptr;
};
cudaError_t gpu_group_codes(const uint8_t* codes_h, const int32_t* ids_h, int64_t n, int M, const int32_t* perm_h,
                            const int32_t* list_h, GpuGroups* out);   // list_h: IVF (list, code) order

}  // namespace et
