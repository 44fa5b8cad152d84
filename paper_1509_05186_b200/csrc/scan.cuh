// scan.cuh -- K2 scan kernel (fused distance tables + Distance-Context scan
// + emit, E-Forest join).  Included by the per-s
// translation units scan_s*.cu, which are compiled in parallel.
#pragma once
#include "common.cuh"

#include <type_traits>

namespace et {
namespace {   // internal linkage: every scan_s*.cu has its own copy

// ---------------------------------------------------------------------------
// table build helpers
// ---------------------------------------------------------------------------

// Swizzled shared-memory table: entry (level, k, lane) of the CTA's 32 queries.
// A lookup by warp-uniform (level, k) with lane = query touches 32 consecutive
// words (conflict-free); a build store with lanes = 32 consecutive codewords and
// a uniform query slot i lands on bank (i ^ lane): also conflict-free.
__device__ __forceinline__ int tab_index(int lvl, int k, int i) {
  return ((lvl << 8) + k) * 32 + (i ^ (k & 31));
}

// Dynamic shared memory of the scan kernel, addressed by byte offset through
// this extern array so the compiler emits LDS/STS (and may reorder loads).
extern __shared__ __align__(16) unsigned char et_dsm[];
__device__ __forceinline__ float4 lds4_off(uint32_t off) {
  return *reinterpret_cast<const float4*>(et_dsm + off);
}
__device__ __forceinline__ void sts_off(uint32_t off, float v) {
  *reinterpret_cast<float*>(et_dsm + off) = v;
}

// Explicit shared-memory accesses (32-bit shared addresses; avoids generic
// addressing in the hot loops).
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float lds(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
// predicated load: v is returned unchanged when !pred (no shared-memory traffic)
// leaf-record staging (ET_REC_SMEM): a warp's batch of 32 records per stream in
// shared memory, read back by every lane at a warp-uniform address (one
// broadcast LDS.128 per leaf instead of four shuffles)
__device__ __forceinline__ uint4 lds_u4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u4(uint32_t a, const uint4& v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" :: "r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ float lds_if(uint32_t a, bool pred, float v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.f32 %0, [%1];\n\t}"
               : "+f"(v) : "r"(a), "r"((int)pred));
  return v;
}
// predicated load; the result is undefined when !pred (callers never use it then)
__device__ __forceinline__ float lds_if_w(uint32_t a, bool pred) {
  float v;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.f32 %0, [%1];\n\t}"
               : "=f"(v) : "r"(a), "r"((int)pred));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" :: "r"(a), "f"(v) : "memory");
}
// byte address of table entry (level, k, lane): see tab_index
__device__ __forceinline__ uint32_t tab_addr(uint32_t tab_s, int lvl, uint32_t k, uint32_t lane4) {
  return tab_s + ((uint32_t)lvl << 15) + (k << 7) + ((lane4 ^ (k << 2)) & 0x7cu);
}


// ---------------------------------------------------------------------------
// K2: the scan kernel
// ---------------------------------------------------------------------------

struct SmemScan {
  float* tab;          // [(levels)][256][32] swizzled
  unsigned* thr;       // [32] CTA-shared top-k thresholds (float bits)
  int* qidx;           // [32] query of each lane
  float* stage;        // [32 queries][kDC dims] query sub-vector chunk (table build)
  float* bigstage;     // 8-level trees: [8 levels][16 pairs][16 dims][2] staged queries
  uint32_t* tmem_slot; // TMEM base address written by tcgen05.alloc
  uint32_t tmem;       // TMEM base (level-0 tables of 8-level trees), 0 if unused
};

// ---------------------------------------------------------------------------
// Tensor Memory (TMEM) as a lookup-table store.  An 8-level tree needs 8
// tables of 32 KB for the CTA's 32 queries; levels 0 and 1 live in TMEM --
// 2 x 256 columns x 32 lanes (lane = query, column = 256 * level + codeword),
// one copy per warp quadrant (a warp may only address its own 32 TMEM lanes),
// read with tcgen05.ld.32x32b.x1 at a warp-uniform column -- so shared memory
// holds levels 2..7 plus a staging area for all 8 levels' query sub-vectors.
// ---------------------------------------------------------------------------
constexpr int kTmemCols = 256 * kTmemLevels;

// levels of a tree of MT levels held in TMEM
__host__ __device__ constexpr int lv0_of(int MT) { return MT == 8 ? kTmemLevels : 0; }

__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(slot);
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(a), "r"(kTmemCols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(base), "r"(kTmemCols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ uint32_t tmem_lane_base(uint32_t base) {
  return base + ((uint32_t)((threadIdx.x >> 5) & 3) * 32u << 16);   // this warp's 32-lane quadrant
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               :: "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                  "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                  "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])) : "memory");
}
__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
  uint32_t x;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(x) : "r"(taddr));
  return x;
}
__device__ __forceinline__ void tmem_wait_ld(uint32_t& x) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(x));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Copy the TMEM levels (global scratch [kTmemLevels][256][32], just built by
// this CTA) into each warp quadrant's TMEM lanes: warp w copies a quarter of
// the columns for quadrant w & 3.
__device__ void tmem_load_level0(const SmemScan& sm, const float* lut0) {
  const int lane = lane_id(), warp = warp_id();
  const int sub = warp >> 2;               // kWarps / 4 warps per quadrant
  const uint32_t tb = tmem_lane_base(sm.tmem);
  constexpr int per = kTmemCols / (kWarps / 4);
  for (int c0 = sub * per; c0 < sub * per + per; c0 += 8) {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = lut0[(c0 + j) * 32 + lane];
    tmem_st8(tb + (uint32_t)c0, v);
  }
  tmem_wait_st();
}

constexpr int kDC = 16;   // query dimensions staged per table-build pass

// Table entry (level l, codeword k, query slot i): the TMEM levels of an
// 8-level tree are built into the global scratch lut0 [kTmemLevels][256][32]
// and copied to TMEM (tmem_load_level0).
__device__ __forceinline__ float* tab_slot(const SmemScan& sm, float* lut0, int l, int lv0, int k, int i) {
  return (l < lv0) ? lut0 + ((size_t)l * 256 + k) * 32 + i : sm.tab + tab_index(l - lv0, k, i);
}

// Inner loop of one build pass: codeword chunk c[0..NJ) (registers) against
// query slots i = g, g+G, ... read from the staged chunk (broadcast loads).
template <int NJ, int DC = kDC>
__device__ __forceinline__ void build_pass_fixed(const SmemScan& sm, float* lut0, int l, int lv0, int k,
                                                 bool kvalid, const float* c, int nq, int g, int G,
                                                 bool first) {
  int i = g;
  for (; i + G < nq; i += 2 * G) {   // two independent FMA chains
    const float* x0 = sm.stage + i * DC;
    const float* x1 = sm.stage + (i + G) * DC;
    float* o0 = tab_slot(sm, lut0, l, lv0, k, i);
    float* o1 = tab_slot(sm, lut0, l, lv0, k, i + G);
    float a0 = 0.f, a1 = 0.f;
    if (!first && kvalid) { a0 = *o0; a1 = *o1; }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const float t0 = x0[j] - c[j];
      const float t1 = x1[j] - c[j];
      a0 = fmaf(t0, t0, a0);
      a1 = fmaf(t1, t1, a1);
    }
    if (kvalid) { *o0 = a0; *o1 = a1; }
  }
  if (i < nq) {
    const float* x0 = sm.stage + i * DC;
    float* o0 = tab_slot(sm, lut0, l, lv0, k, i);
    float a0 = (!first && kvalid) ? *o0 : 0.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const float t0 = x0[j] - c[j];
      a0 = fmaf(t0, t0, a0);
    }
    if (kvalid) *o0 = a0;
  }
}

__device__ __forceinline__ void build_pass_generic(const SmemScan& sm, float* lut0, int l, int lv0, int k,
                                                   bool kvalid, const float* c, int nj, int nq, int g, int G,
                                                   bool first) {
  for (int i = g; i < nq; i += G) {
    const float* x0 = sm.stage + i * kDC;
    float* o0 = tab_slot(sm, lut0, l, lv0, k, i);
    float a0 = (!first && kvalid) ? *o0 : 0.f;
    for (int j = 0; j < nj; ++j) {
      const float t0 = x0[j] - c[j];
      a0 = fmaf(t0, t0, a0);
    }
    if (kvalid) *o0 = a0;
  }
}

// Packed fp32x2 arithmetic (sm_100a FADD2 / FFMA2): two independent IEEE fp32
// operations per instruction, each rounded exactly like the scalar op, so an
// entry computed two-queries-at-a-time equals the scalar j-ascending chain.
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long f2sub(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2sqacc(unsigned long long t, unsigned long long acc) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(t), "l"(acc));
  return r;
}

// Copy the two TMEM levels' tables (smem regions r0_s, r1_s, swizzled
// [k][lane ^ (k & 31)]) into every warp quadrant's TMEM lanes: warp w copies
// its share of the 512 columns for quadrant w & 3.
__device__ __forceinline__ void tmem_load_from_smem(const SmemScan& sm, uint32_t r0_s, uint32_t r1_s) {
  const int lane = lane_id(), warp = warp_id();
  const int sub = warp >> 2;
  const uint32_t tb = tmem_lane_base(sm.tmem);
  const uint32_t lane4 = (uint32_t)lane << 2;
  constexpr int per = kTmemCols / (kWarps / 4);
  for (int c0 = sub * per; c0 < sub * per + per; c0 += 32) {   // 32 columns in flight per warp
    const uint32_t rs = (c0 < 256) ? r0_s : r1_s;
    float v[4][8];
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int j = 0; j < 8; ++j) v[g][j] = lds(tab_addr(rs, 0, (uint32_t)((c0 + 8 * g + j) & 255), lane4));
#pragma unroll
    for (int g = 0; g < 4; ++g) tmem_st8(tb + (uint32_t)(c0 + 8 * g), v[g]);
  }
  tmem_wait_st();
}

// Staging layout of the resident build: level l's query pairs at
// region + l * kStageLevelBytes (16 pairs x 16 dims x 2 queries), the last
// level's in the small stage.  Element (slot i, dim j) of a level lives at
// (i / 2) * 128 + j * 8 + (i % 2) * 4.
constexpr uint32_t kStageLevelBytes = 16 * 16 * 2 * 4;

// Issued at kernel entry (plain E-Tree tables, no coarse residual): the
// chunk's query sub-vectors are copied straight into the staging layout with
// cp.async (no registers held), overlapping the CTA's setup (TMEM allocation,
// first barrier); the build waits with cp.async.wait_all.  Slots without a
// query are left unwritten (their entries are never looked up).
template <int SS, int MT>
__device__ __forceinline__ void stage_async(const ScanParams& p, int t, int chunk, int nch, uint32_t region_s,
                                            uint32_t stage_s) {
  const TreeDev& tr = p.tree[t];
  const int j = threadIdx.x & (SS - 1);
  // arithmetic chunking: the chunk's queries are rows [s0, s1) (bounds once,
  // not per slot: two 64-bit divisions)
  int64_t s0 = 0, s1 = 0;
  if (p.flatQ > 0) {
    s0 = (int64_t)chunk * p.flatQ / nch;
    s1 = (int64_t)(chunk + 1) * p.flatQ / nch;
  }
#pragma unroll
  for (int i = threadIdx.x >> 4; i < 32; i += kThreads / SS) {   // query slot i, dimension j
    int q = -1;
    if (p.flatQ > 0) {
      q = (s0 + i < s1) ? (int)(s0 + i) : -1;
    } else {
      q = __ldg(p.chunk_q + (size_t)chunk * 32 + i);
    }
    if (q < 0) continue;
    const float* xr = p.queries + (size_t)q * p.d + j;
    const uint32_t o = (uint32_t)(i >> 1) * 128u + (uint32_t)j * 8u + (uint32_t)(i & 1) * 4u;
#pragma unroll
    for (int l = 0; l < MT; ++l) {
      // 8 levels: every level in the staging area (region_s); else levels
      // 0..MT-2 in the last level's region and MT-1 in the small stage
      const uint32_t dst = (MT == 8 || l < MT - 1) ? region_s + (uint32_t)l * kStageLevelBytes + o : stage_s + o;
      const float* src = xr + (size_t)p.lsub[tr.layer0 + l] * SS;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src) : "memory");
    }
  }
}

// Packed f32x2 subtract of a broadcast scalar: (a.lo - c, a.hi - c).  ptxas
// encodes the duplicated 32-bit operand as FADD2's scalar form (R.F32).
__device__ __forceinline__ unsigned long long f2subs(unsigned long long a, float c) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(((unsigned long long)__float_as_uint(c) << 32) | __float_as_uint(c)));
  return r;
}

// Table build of an 8-level tree, s == 16 (every d = 128 configuration).
// Levels 0 and 1 end up in TMEM, levels 2..7 in shared-memory regions 0..5;
// the active queries' sub-vectors of all 8 levels are staged once, as query
// pairs [level][pair][dim][2] in their own area (cp.async at kernel entry,
// or synchronously with the coarse centroid subtracted for IVF residuals).
// Four levels are built at a time by kWarps / 4 warps each; a warp owns
// kR = 8 / (kWarps / 4) codeword rows per lane (rows kRow0 + 32 r + lane), so
// every broadcast LDS.128 of a staged query pair (2 queries x 2 dims) feeds
// 4 kR packed instructions (FADD2 with the codeword as the scalar operand,
// then FFMA2) -- the shared-memory pipe stays well below the FP32 pipe.
// Each entry is the j-ascending fp32 FMA chain sum_j (x_j - c_j)^2.
// Round 0 builds levels 0..3 (levels 0 and 1 into regions 2 and 3, which
// levels 4 and 5 only need in round 1; both are then copied to TMEM), round 1
// levels 4..7.  Codewords of round 1 are loaded before the copy.
constexpr int kWPL = kWarps / 4;          // warps per level
constexpr int kR = 8 / kWPL;              // codeword rows per lane

template <int SS>
__device__ __forceinline__ void build_tables_resident8(const ScanParams& p, const SmemScan& sm, int t, int unit, int nq,
                                                       int cell, bool staged) {
  static_assert(SS == kDC, "resident staging handles s == 16");
  static_assert(kWPL * kR * 32 == 256, "four levels x 256 codewords per round");
  const TreeDev& tr = p.tree[t];
  const int K = p.K, d = p.d;
  const int lane = lane_id(), warp = warp_id();
  const uint32_t dsm_s = smem_u32(et_dsm);
  const uint32_t tab_s = smem_u32(sm.tab);
  const uint32_t stg_s = smem_u32(sm.bigstage);
  const int np = (nq + 1) >> 1;                                          // query pairs
  constexpr uint32_t pair_bytes = SS * 2 * 4;                            // 128 B per (level, pair)
  const int lw = warp / kWPL;                         // level within the round
  const int row0 = (warp % kWPL) * 32 * kR;           // first codeword row of this warp
  const bool active = row0 < K;                       // K < 256: idle codeword blocks
  auto load_cw = [&](int l, float (&c)[kR][SS]) {
    const int m = p.lsub[tr.layer0 + l];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int k = row0 + 32 * r + lane;
      const float* row = p.codebooks + ((size_t)m * K + (k < K ? k : 0)) * SS;
#pragma unroll
      for (int j = 0; j < SS; j += 4) {
        const float4 u = __ldg(reinterpret_cast<const float4*>(row + j));
        c[r][j] = u.x; c[r][j + 1] = u.y; c[r][j + 2] = u.z; c[r][j + 3] = u.w;
      }
    }
  };
  float c[kR][SS];
  if (active) load_cw(lw, c);                         // round 0's rows: in flight during the staging wait
  if (staged) {
    asm volatile("cp.async.wait_all;" ::: "memory");   // this thread's stage_async copies landed
  } else {
    __syncthreads();                                 // previous users of the tables / stage are done
    const int j = threadIdx.x & (SS - 1);
    for (int i = threadIdx.x >> 4; i < nq; i += kThreads / SS) {
      float v[8];
      const int q = sm.qidx[i];
      const float* xr = p.queries + (size_t)q * d + j;
      const float* cr = (cell >= 0 && p.coarse) ? p.coarse + (size_t)cell * d + j : nullptr;
#pragma unroll
      for (int l = 0; l < 8; ++l) v[l] = __ldg(xr + (size_t)p.lsub[tr.layer0 + l] * SS);
      if (cr) {
#pragma unroll
        for (int l = 0; l < 8; ++l) v[l] -= __ldg(cr + (size_t)p.lsub[tr.layer0 + l] * SS);
      }
      const uint32_t o = (uint32_t)(i >> 1) * pair_bytes + (uint32_t)j * 8u + (uint32_t)(i & 1) * 4u;
#pragma unroll
      for (int l = 0; l < 8; ++l) sts(stg_s + (uint32_t)l * kStageLevelBytes + o, v[l]);
    }
  }
  // Entries of one table (region dst_s) for this lane's kR rows and every
  // staged query pair of xs_s, two pairs per iteration.  Query slots >= nq and
  // rows >= K are written but never looked up.
  auto item = [&](uint32_t dst_s, uint32_t xs_s, const float (&c)[kR][SS]) {
    const uint32_t rows = dst_s - dsm_s + ((uint32_t)(row0 + lane) << 7);   // row of r = 0 (byte offset)
    const uint32_t sw = (uint32_t)(row0 + lane) << 2;   // swizzle (k & 31) << 2 -- the same for every r
    uint32_t xo = xs_s - dsm_s;
    uint32_t i4 = 0;                                 // 4 * (first query of the pair)
    int pi = 0;
    for (; pi + 1 < np; pi += 2, xo += 2 * pair_bytes, i4 += 16) {
      unsigned long long a[2][kR];                   // (pair, row)
#pragma unroll
      for (int r = 0; r < kR; ++r) { a[0][r] = 0ull; a[1][r] = 0ull; }
#pragma unroll
      for (int j = 0; j < SS; j += 2) {
        const float4 u0 = lds4_off(xo + (uint32_t)j * 8u), u1 = lds4_off(xo + pair_bytes + (uint32_t)j * 8u);
        const unsigned long long p0 = f2pack(u0.x, u0.y), p1 = f2pack(u1.x, u1.y);
        const unsigned long long q0 = f2pack(u0.z, u0.w), q1 = f2pack(u1.z, u1.w);
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          a[0][r] = f2sqacc(f2subs(p0, c[r][j]), a[0][r]);
          a[1][r] = f2sqacc(f2subs(p1, c[r][j]), a[1][r]);
        }
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          a[0][r] = f2sqacc(f2subs(q0, c[r][j + 1]), a[0][r]);
          a[1][r] = f2sqacc(f2subs(q1, c[r][j + 1]), a[1][r]);
        }
      }
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        float e0, o0, e1, o1;
        f2unpack(a[0][r], e0, o0);
        f2unpack(a[1][r], e1, o1);
        const uint32_t row = rows + ((uint32_t)r << 12);   // row + 32 r
        ET_CHECK(row + 128u <= (dst_s - dsm_s) + 32768u && i4 + 12u < 128u);
        sts_off(row + ((i4 ^ sw) & 0x7cu), e0);
        sts_off(row + (((i4 + 4) ^ sw) & 0x7cu), o0);
        sts_off(row + (((i4 + 8) ^ sw) & 0x7cu), e1);
        sts_off(row + (((i4 + 12) ^ sw) & 0x7cu), o1);
      }
    }
    if (pi < np) {
      unsigned long long a[kR];
#pragma unroll
      for (int r = 0; r < kR; ++r) a[r] = 0ull;
#pragma unroll
      for (int j = 0; j < SS; j += 2) {
        const float4 u0 = lds4_off(xo + (uint32_t)j * 8u);
        const unsigned long long p0 = f2pack(u0.x, u0.y), q0 = f2pack(u0.z, u0.w);
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          a[r] = f2sqacc(f2subs(p0, c[r][j]), a[r]);
          a[r] = f2sqacc(f2subs(q0, c[r][j + 1]), a[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        float e0, o0;
        f2unpack(a[r], e0, o0);
        const uint32_t row = rows + ((uint32_t)r << 12);
        sts_off(row + ((i4 ^ sw) & 0x7cu), e0);
        sts_off(row + (((i4 + 4) ^ sw) & 0x7cu), o0);
      }
    }
  };
  __syncthreads();                                   // stage complete
  phase_mark(unit, 5);
  // round 0: level lw -> region (levels 0, 1: regions 2, 3 until the TMEM copy)
  const uint32_t r0 = (lw < 2) ? (uint32_t)(lw + 2) : (uint32_t)(lw - 2);
  if (active) item(tab_s + (r0 << 15), stg_s + (uint32_t)lw * kStageLevelBytes, c);
  if (active) load_cw(lw + 4, c);                    // round 1's rows, in flight during the copy
  __syncthreads();
  tmem_fence_after();
  phase_mark(unit, 6);
  tmem_load_from_smem(sm, tab_s + (2u << 15), tab_s + (3u << 15));
  tmem_fence_before();
  __syncthreads();                                   // regions 2, 3 free again
  phase_mark(unit, 7);
  // round 1: level lw + 4 -> region lw + 2
  if (active) item(tab_s + ((uint32_t)(lw + 2) << 15), stg_s + (uint32_t)(lw + 4) * kStageLevelBytes, c);
  __syncthreads();
  tmem_fence_after();                                // TMEM levels visible to the scan's tcgen05.ld
}

// Resident-staging table build for s == 16 and trees of fewer than 8 levels
// (8-level trees: build_tables_resident8).  The active queries' sub-vectors
// are staged ONCE, as query pairs
// [level][pair][dim][2], levels 0..MT-2 into the shared-memory region of the
// tree's last level (built last) and level MT-1 into the small stage.  Warp w
// owns codeword block kb = (w >> 1) & 7 (lane = codeword) and query-pair half
// g = w & 1; for each level it keeps its codeword in registers and runs two
// packed FADD2/FFMA2 chains (two query pairs, four entries) at a time against
// broadcast LDS.128 loads of the staged pairs.
template <int SS, int MT>
__device__ __forceinline__ void build_tables_resident(const ScanParams& p, const SmemScan& sm, int t, int unit,
                                                      int nq, int cell, bool staged) {
  static_assert(SS == kDC, "resident staging handles s == 16");
  if constexpr (MT == 8) {
    build_tables_resident8<SS>(p, sm, t, unit, nq, cell, staged);
    return;
  }
  const TreeDev& tr = p.tree[t];
  constexpr int lv0 = 0;
  const int K = p.K, d = p.d;
  const int lane = lane_id(), warp = warp_id();
  const uint32_t tab_s = smem_u32(sm.tab);
  const uint32_t region_s = tab_s + ((uint32_t)(MT - 1 - lv0) << 15);   // last level's table region
  const uint32_t stage_s = smem_u32(sm.stage);
  const int np = (nq + 1) >> 1;                                          // query pairs
  const uint32_t pair_bytes = SS * 2 * 4;                                // 128 B per (level, pair)
  if (staged) {
    asm volatile("cp.async.wait_all;" ::: "memory");   // this thread's stage_async copies landed
  } else {
    __syncthreads();                                 // previous tree's scan is done with the tables
    // thread -> (query slot i, dim j); all loads first, then the stores
    const int j = threadIdx.x & (SS - 1);
    for (int i = threadIdx.x >> 4; i < nq; i += kThreads / SS) {
      float v[MT];
      const int q = sm.qidx[i];
      const float* xr = p.queries + (size_t)q * d + j;
      const float* cr = (cell >= 0 && p.coarse) ? p.coarse + (size_t)cell * d + j : nullptr;
#pragma unroll
      for (int l = 0; l < MT; ++l) v[l] = __ldg(xr + (size_t)p.lsub[tr.layer0 + l] * SS);
      if (cr) {
#pragma unroll
        for (int l = 0; l < MT; ++l) v[l] -= __ldg(cr + (size_t)p.lsub[tr.layer0 + l] * SS);
      }
      const uint32_t o = (uint32_t)(i >> 1) * pair_bytes + (uint32_t)j * 8u + (uint32_t)(i & 1) * 4u;
#pragma unroll
      for (int l = 0; l < MT - 1; ++l) sts(region_s + (uint32_t)l * kStageLevelBytes + o, v[l]);
      sts(stage_s + o, v[MT - 1]);
    }
  }
  constexpr int WG = kWarps / 8;                     // warps per codeword block (query-pair groups)
  const int kb = (warp / WG) & 7, g = warp % WG;
  const int k = kb * 32 + lane;
  const bool kvalid = k < K;
  const int p0 = g ? (np + 1) >> 1 : 0, p1 = (g || WG == 1) ? np : (np + 1) >> 1;
  const bool active = kb * 32 < K;                   // K < 256: idle codeword blocks
  const uint32_t dsm_s = smem_u32(et_dsm);
  auto load_cw = [&](int l, float (&c)[SS]) {
    const int m = p.lsub[tr.layer0 + l];
    const float* crow = p.codebooks + ((size_t)m * K + (kvalid ? k : 0)) * SS;
#pragma unroll
    for (int j = 0; j < SS; j += 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(crow + j));
      c[j] = v.x; c[j + 1] = v.y; c[j + 2] = v.z; c[j + 3] = v.w;
    }
  };
  // Entries of one table (region dst_s) for this warp's query pairs [p0, p1)
  // of stage xs_s, two pairs (four entries) per iteration.  Every lane writes
  // all query slots of its codeword's row: slots >= nq are never looked up
  // (and rows k >= K never addressed), so no store is predicated.
  auto item = [&](uint32_t dst_s, uint32_t xs_s, const float (&c)[SS]) {
    const uint32_t drow = dst_s - dsm_s + ((uint32_t)k << 7);   // this lane's row (byte offset)
    const uint32_t kk = (uint32_t)k << 2;
    uint32_t xo = xs_s - dsm_s + (uint32_t)p0 * pair_bytes;
    uint32_t i4 = (uint32_t)p0 << 3;                             // 4 * (first query of the pair)
    int pi = p0;
    for (; pi + 1 < p1; pi += 2, xo += 2 * pair_bytes, i4 += 16) {
      unsigned long long a0 = 0ull, a1 = 0ull;
#pragma unroll
      for (int j = 0; j < SS; j += 2) {
        const float4 u0 = lds4_off(xo + (uint32_t)j * 8u), u1 = lds4_off(xo + pair_bytes + (uint32_t)j * 8u);
        const unsigned long long cj = f2pack(c[j], c[j]), cj1 = f2pack(c[j + 1], c[j + 1]);
        unsigned long long t0 = f2sub(f2pack(u0.x, u0.y), cj), t1 = f2sub(f2pack(u1.x, u1.y), cj);
        a0 = f2sqacc(t0, a0); a1 = f2sqacc(t1, a1);
        t0 = f2sub(f2pack(u0.z, u0.w), cj1); t1 = f2sub(f2pack(u1.z, u1.w), cj1);
        a0 = f2sqacc(t0, a0); a1 = f2sqacc(t1, a1);
      }
      float e0, o0, e1, o1;
      f2unpack(a0, e0, o0);
      f2unpack(a1, e1, o1);
      sts_off(drow + ((i4 ^ kk) & 0x7cu), e0);
      sts_off(drow + (((i4 + 4) ^ kk) & 0x7cu), o0);
      sts_off(drow + (((i4 + 8) ^ kk) & 0x7cu), e1);
      sts_off(drow + (((i4 + 12) ^ kk) & 0x7cu), o1);
    }
    if (pi < p1) {
      unsigned long long a0 = 0ull;
#pragma unroll
      for (int j = 0; j < SS; j += 2) {
        const float4 u0 = lds4_off(xo + (uint32_t)j * 8u);
        a0 = f2sqacc(f2sub(f2pack(u0.x, u0.y), f2pack(c[j], c[j])), a0);
        a0 = f2sqacc(f2sub(f2pack(u0.z, u0.w), f2pack(c[j + 1], c[j + 1])), a0);
      }
      float e0, o0;
      f2unpack(a0, e0, o0);
      sts_off(drow + ((i4 ^ kk) & 0x7cu), e0);
      sts_off(drow + (((i4 + 4) ^ kk) & 0x7cu), o0);
    }
  };
  float cw[SS], cwn[SS];
  if (active) load_cw(0, cw);
  __syncthreads();                                   // stage complete
  phase_mark(unit, 5);
  // levels lv0 .. MT-2 (their queries staged in the last level's region)
  for (int l = lv0; l < MT - 1; ++l) {
    if (active) {
      load_cw(l + 1, cwn);                           // prefetch the next level's codeword
      item(tab_s + ((uint32_t)(l - lv0) << 15), region_s + (uint32_t)l * kStageLevelBytes, cw);
#pragma unroll
      for (int j = 0; j < SS; ++j) cw[j] = cwn[j];
    }
  }
  __syncthreads();                                   // region free: build the last level into it
  phase_mark(unit, 7);
  if (active) item(region_s, stage_s, cw);
  __syncthreads();
}

// Few queries with long sub-vectors (c3: s = 60, <= 8 queries per CTA): one
// staging pass per level (the small stage holds 8 queries x 64 dims), each
// warp owns codeword block kb = w & 7 and the queries g, g+2, g+4, g+6
// (g = w >> 3) and runs the whole j-ascending FMA chain of each entry in
// registers over 16-dimension codeword chunks (next chunk prefetched) -- two
// barriers per level instead of two per 16-dimension pass.
template <int SS>
__device__ void build_tables_wide(const ScanParams& p, const SmemScan& sm, int t, int unit, int nq, int cell) {
  static_assert(SS > kDC && SS <= 64 && SS % 4 == 0, "wide staging: 16 < s <= 64, s % 4 == 0");
  constexpr int NCH = (SS + kDC - 1) / kDC;
  const TreeDev& tr = p.tree[t];
  const int MT = tr.MT;
  const int lv0 = lv0_of(MT);
  const int K = p.K, d = p.d;
  const int lane = lane_id(), warp = warp_id();
  float* lut0 = p.lut0 ? p.lut0 + (size_t)unit * kTmemLevels * 256 * 32 : nullptr;
  constexpr int WG = kWarps / 8;                // query groups (warps per codeword block)
  constexpr int NQW = 8 / WG;                   // query slots per warp: g, g + WG, ...
  constexpr int SPT = 512 / kThreads;           // staging elements (8 x 64) per thread
  const int kb = warp & 7, g = warp >> 3;
  const int k = kb * 32 + lane;
  const bool kvalid = k < K;
  auto fetch = [&](int l, int e) -> float {     // staging element e = (slot e >> 6, dim e & 63)
    const int si = e >> 6, sj = e & 63;
    const int sq = (si < nq) ? sm.qidx[si] : -1;
    if (sq < 0 || sj >= SS) return 0.f;
    const int m = p.lsub[tr.layer0 + l];
    float v = __ldg(p.queries + (size_t)sq * d + (size_t)m * SS + sj);
    if (cell >= 0 && p.coarse) v -= __ldg(p.coarse + (size_t)cell * d + (size_t)m * SS + sj);
    return v;
  };
  float nxt[SPT];
#pragma unroll
  for (int u = 0; u < SPT; ++u) nxt[u] = fetch(0, threadIdx.x + u * kThreads);
  __syncthreads();                              // previous users of the stage are done
#pragma unroll
  for (int u = 0; u < SPT; ++u) sm.stage[threadIdx.x + u * kThreads] = nxt[u];
  __syncthreads();
  for (int l = 0; l < MT; ++l) {
    if (l + 1 < MT) {                           // next level's stage values
#pragma unroll
      for (int u = 0; u < SPT; ++u) nxt[u] = fetch(l + 1, threadIdx.x + u * kThreads);
    }
    const int m = p.lsub[tr.layer0 + l];
    const float* crow = p.codebooks + ((size_t)m * K + (kvalid ? k : 0)) * SS;
    float acc[NQW];
#pragma unroll
    for (int qq = 0; qq < NQW; ++qq) acc[qq] = 0.f;
    float c[kDC], cn[kDC];
#pragma unroll
    for (int j = 0; j < kDC; j += 4) {
      const float4 v = (j < SS) ? __ldg(reinterpret_cast<const float4*>(crow + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
      c[j] = v.x; c[j + 1] = v.y; c[j + 2] = v.z; c[j + 3] = v.w;
    }
#pragma unroll
    for (int jc = 0; jc < NCH; ++jc) {
      if (jc + 1 < NCH) {
#pragma unroll
        for (int j = 0; j < kDC; j += 4) {
          const int jj = (jc + 1) * kDC + j;
          const float4 v = (jj < SS) ? __ldg(reinterpret_cast<const float4*>(crow + jj)) : make_float4(0.f, 0.f, 0.f, 0.f);
          cn[j] = v.x; cn[j + 1] = v.y; cn[j + 2] = v.z; cn[j + 3] = v.w;
        }
      }
      constexpr int NJ0 = SS - (NCH - 1) * kDC;   // size of the last chunk
#pragma unroll
      for (int qq = 0; qq < NQW; ++qq) {
        const int i = g + WG * qq;
        if (i < nq) {
          const float* x = sm.stage + i * 64 + jc * kDC;
#pragma unroll
          for (int j = 0; j < kDC; ++j) {
            if (jc < NCH - 1 || j < NJ0) {
              const float tt = x[j] - c[j];
              acc[qq] = fmaf(tt, tt, acc[qq]);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kDC; ++j) c[j] = cn[j];
    }
#pragma unroll
    for (int qq = 0; qq < NQW; ++qq) {
      const int i = g + WG * qq;
      if (i < nq && kvalid) *tab_slot(sm, lut0, l, lv0, k, i) = acc[qq];
    }
    __syncthreads();
    if (l + 1 < MT) {
#pragma unroll
      for (int u = 0; u < SPT; ++u) sm.stage[threadIdx.x + u * kThreads] = nxt[u];
    }
    __syncthreads();
  }
}

// Table build of an 8-level tree with long sub-vectors (16 < s <= 64, s % 4 ==
// 0; c3: s = 60) for at most 8 queries, organised like build_tables_resident8:
// the queries' sub-vectors of all 8 levels are staged once as query pairs
// [level][pair][dim][2] in the staging area (8 x 4 x s x 8 B <= 16 KB), four
// levels are built at a time by kWPL warps each, a lane owns kR codeword rows
// and keeps its 4 x kR x pairs packed accumulators in registers over the whole
// j-ascending chain while the codeword rows stream through registers 4
// dimensions at a time (next chunk in flight).  Every broadcast LDS.128 of a
// staged pair (2 queries x 2 dims) feeds 4 kR packed FADD2/FFMA2.  Levels 0/1
// are built into regions 2/3 and copied to TMEM before round 1, exactly as in
// the resident build, so the scan sees the same layout.
template <int SS>
struct Wide8 {
  static_assert(SS > kDC && SS <= 64 && SS % 4 == 0, "wide resident build: 16 < s <= 64, s % 4 == 0");
  static constexpr int NP = 4;                            // query pairs (nq <= 8)
  static constexpr uint32_t pair_bytes = SS * 8u;         // [dim][2] fp32
  static constexpr uint32_t lvl_bytes = NP * pair_bytes;
  static constexpr int NCH = SS / 4;                      // 4-dimension codeword chunks
  static_assert(8 * lvl_bytes <= 8u * 16u * 128u, "staging area");
};

// Stage tree t's query sub-vectors for build_tables_wide8: plain E-Tree
// tables are copied with cp.async (issued early -- at kernel entry, or while
// the previous tree is scanned -- and awaited by the build); IVF residuals
// (x - cc) synchronously.
template <int SS>
__device__ __forceinline__ void stage_wide8(const ScanParams& p, const SmemScan& sm, int t, int nq, int cell) {
  using W = Wide8<SS>;
  const TreeDev& tr = p.tree[t];
  const uint32_t stg_s = smem_u32(sm.bigstage);
  for (int e = threadIdx.x; e < 8 * 8 * SS; e += kThreads) {   // (level, slot, dim)
    const int l = e / (8 * SS), r = e - l * (8 * SS);
    const int i = r / SS, j = r - i * SS;
    if (i >= nq) continue;                                // slots >= nq: never looked up
    const int m = p.lsub[tr.layer0 + l];
    const float* src = p.queries + (size_t)sm.qidx[i] * p.d + (size_t)m * SS + j;
    const uint32_t dst = stg_s + (uint32_t)l * W::lvl_bytes + (uint32_t)(i >> 1) * W::pair_bytes + (uint32_t)j * 8u +
                         (uint32_t)(i & 1) * 4u;
    if (cell >= 0 && p.coarse) sts(dst, __ldg(src) - __ldg(p.coarse + (size_t)cell * p.d + (size_t)m * SS + j));
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src) : "memory");
  }
}

// Table build of an 8-level tree with long sub-vectors (16 < s <= 64, s % 4 ==
// 0; c3: s = 60) for at most 8 queries, organised like build_tables_resident8:
// the queries' sub-vectors of all 8 levels are staged once as query pairs
// [level][pair][dim][2] in the staging area (stage_wide8), four levels are
// built at a time by kWPL warps each, a lane owns kR codeword rows and keeps
// its kR x pairs packed accumulators in registers over the whole j-ascending
// chain while the codeword rows stream through registers 4 dimensions at a
// time (two chunks in flight).  Codeword chunks come from the chunk-major copy
// p.cbt [m][s/4][K] float4 (one coalesced 512 B load per warp and row block;
// the row-major codebook would touch 32 rows per load instruction), else from
// the rows.  Every broadcast LDS.128 of a staged pair (2 queries x 2 dims)
// feeds 2 kR packed FADD2/FFMA2.  Levels 0/1 are built into regions 2/3 and
// copied to TMEM before round 1, exactly as in the resident build.
template <int SS>
__device__ void build_tables_wide8(const ScanParams& p, const SmemScan& sm, int t, int nq) {
  using W = Wide8<SS>;
  constexpr int NP = W::NP, NCH = W::NCH;
  const TreeDev& tr = p.tree[t];
  const int K = p.K;
  const int lane = lane_id(), warp = warp_id();
  const uint32_t dsm_s = smem_u32(et_dsm);
  const uint32_t tab_s = smem_u32(sm.tab);
  const uint32_t stg_s = smem_u32(sm.bigstage);
  (void)nq;
  const int lw = warp / kWPL;                             // level within the round
  const int row0 = (warp % kWPL) * 32 * kR;               // first codeword row of this warp
  const bool active = row0 < K;
  // codeword chunks of level l stream through a register ring, kRing - 1
  // chunks ahead (the L2 latency is longer than one chunk's arithmetic); the
  // ring of the next level is filled before each barrier / copy
  constexpr int kRing = 5;
  float4 c[kRing][kR];
  auto chunk = [&](int l, int r, int jc) -> float4 {
    const int m = p.lsub[tr.layer0 + l];
    const int k = min(row0 + 32 * r + lane, K - 1);
    if (p.cbt) return __ldg(p.cbt + ((size_t)m * NCH + jc) * K + k);
    return __ldg(reinterpret_cast<const float4*>(p.codebooks + ((size_t)m * K + k) * SS) + jc);
  };
  auto prefill = [&](int l) {
#pragma unroll
    for (int d = 0; d < kRing - 1; ++d)
#pragma unroll
      for (int r = 0; r < kR; ++r)
        if (d < NCH) c[d][r] = chunk(l, r, d);
  };
  if (active) prefill(lw);
  asm volatile("cp.async.wait_all;" ::: "memory");         // this thread's staged copies landed
  __syncthreads();                                        // everyone's; previous users of the tables done
  auto item = [&](uint32_t dst_s, int l) {
    const uint32_t xs = stg_s - dsm_s + (uint32_t)l * W::lvl_bytes;
    unsigned long long a[NP][kR];
#pragma unroll
    for (int pi = 0; pi < NP; ++pi)
#pragma unroll
      for (int r = 0; r < kR; ++r) a[pi][r] = 0ull;
#pragma unroll
    for (int jc = 0; jc < NCH; ++jc) {
      if (jc + kRing - 1 < NCH) {
#pragma unroll
        for (int r = 0; r < kR; ++r) c[(jc + kRing - 1) % kRing][r] = chunk(l, r, jc + kRing - 1);
      }
      const int cs = jc % kRing;
#pragma unroll
      for (int h = 0; h < 2; ++h) {                       // dims 4 jc + 2 h, 4 jc + 2 h + 1
        // every pair, branch-free (slots >= nq hold stale stage data: their
        // entries are computed and stored but never looked up)
#pragma unroll
        for (int pi = 0; pi < NP; ++pi) {
          const float4 u = lds4_off(xs + (uint32_t)pi * W::pair_bytes + (uint32_t)(4 * jc + 2 * h) * 8u);
          const unsigned long long p0 = f2pack(u.x, u.y), p1 = f2pack(u.z, u.w);
#pragma unroll
          for (int r = 0; r < kR; ++r) {
            const float c0 = h ? c[cs][r].z : c[cs][r].x, c1 = h ? c[cs][r].w : c[cs][r].y;
            a[pi][r] = f2sqacc(f2subs(p0, c0), a[pi][r]);
            a[pi][r] = f2sqacc(f2subs(p1, c1), a[pi][r]);
          }
        }
      }
    }
    const uint32_t rows = dst_s - dsm_s + ((uint32_t)(row0 + lane) << 7);
    const uint32_t sw = (uint32_t)(row0 + lane) << 2;
#pragma unroll
    for (int pi = 0; pi < NP; ++pi) {
      const uint32_t i4 = (uint32_t)pi * 8u;
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        float e0, e1;
        f2unpack(a[pi][r], e0, e1);
        const uint32_t row = rows + ((uint32_t)r << 12);
        sts_off(row + ((i4 ^ sw) & 0x7cu), e0);
        sts_off(row + (((i4 + 4) ^ sw) & 0x7cu), e1);
      }
    }
  };
  // round 0: level lw -> region (levels 0, 1: regions 2, 3 until the TMEM copy)
  const uint32_t r0 = (lw < 2) ? (uint32_t)(lw + 2) : (uint32_t)(lw - 2);
  if (active) item(tab_s + (r0 << 15), lw);
  if (active) prefill(lw + 4);                            // round 1's first chunks, in flight during the copy
  __syncthreads();
  tmem_fence_after();
  tmem_load_from_smem(sm, tab_s + (2u << 15), tab_s + (3u << 15));
  tmem_fence_before();
  __syncthreads();                                        // regions 2, 3 free again
  // round 1: level lw + 4 -> region lw + 2
  if (active) item(tab_s + ((uint32_t)(lw + 2) << 15), lw + 4);
  __syncthreads();                                        // tables complete; the stage is free
  tmem_fence_after();
}

// Build the tables of tree t for this CTA's queries (fused).
// Passes over (level, 16-dimension chunk): the chunk of the active queries'
// sub-vectors (minus the coarse centroid for IVF residuals) is staged in shared
// memory -- the next pass's values are prefetched into registers while the
// current pass computes -- and each warp computes 32 codewords (one per lane,
// codeword chunk in registers) against a share of the queries.  Entries are
// accumulated across chunks in place, so every entry is the j-ascending fp32
// FMA chain sum_j (x_j - c_j)^2 regardless of the chunking.
template <int SS, int DC = kDC>
__device__ void build_tables(const ScanParams& p, const SmemScan& sm, int t, int unit, int nq, int cell) {
  const TreeDev& tr = p.tree[t];
  const int MT = tr.MT;
  const int lv0 = lv0_of(MT);
  const int K = p.K, d = p.d;
  const int s = (SS > 0) ? SS : p.s;
  const int nb = (K + 31) >> 5;
  const int lane = lane_id(), warp = warp_id();
  float* lut0 = p.lut0 ? p.lut0 + (size_t)unit * kTmemLevels * 256 * 32 : nullptr;
  if (p.luts) {   // materialised tables: copy
    for (int item = warp; item < MT * nb; item += kWarps) {
      const int l = item / nb, kb = item - l * nb;
      const int k = kb * 32 + lane;
      const int m = p.lsub[tr.layer0 + l];
      for (int i = 0; i < nq; ++i) {
        const float v = (k < K) ? __ldg(p.luts + ((size_t)sm.qidx[i] * p.M + m) * K + k) : 0.f;
        if (k < K) *tab_slot(sm, lut0, l, lv0, k, i) = v;
      }
    }
    return;
  }
  const int npl = (s + DC - 1) / DC;            // passes per level
  const int P = MT * npl;
  const int G = max(1, kWarps / nb);            // query groups
  const int kb = warp % nb, g = warp / nb;
  const bool computes = g < G;
  // staging elements of this thread: e = threadIdx.x + u * kThreads -> query
  // slot e / DC, dimension e % DC of the chunk
  constexpr int SPG = (32 * DC + kThreads - 1) / kThreads;
  auto fetch = [&](int pass, int e) -> float {
    const int si = e / DC, sj = e % DC;
    const int sq = (si < nq && si < 32) ? sm.qidx[si] : -1;
    const int l = pass / npl, jc = pass - l * npl;
    const int j = jc * DC + sj;
    if (sq < 0 || j >= s) return 0.f;
    const int m = p.lsub[tr.layer0 + l];
    float v = __ldg(p.queries + (size_t)sq * d + (size_t)m * s + j);
    if (cell >= 0 && p.coarse) v -= __ldg(p.coarse + (size_t)cell * d + (size_t)m * s + j);
    return v;
  };
  // codeword chunk of pass `pass` for this lane's codeword (registers)
  const int k = kb * 32 + lane;
  const bool kvalid = computes && k < K;
  auto fetch_cw = [&](int pass, float (&c)[DC]) {
    const int l = pass / npl, jc = pass - l * npl;
    const int j0 = jc * DC;
    const int nj = min(DC, s - j0);
    const int m = p.lsub[tr.layer0 + l];
    const float* crow = p.codebooks + ((size_t)m * K + (kvalid ? k : 0)) * s + j0;
    if (p.vec4 && (s & 3) == 0) {   // 16-byte aligned rows: float4 loads
#pragma unroll
      for (int j = 0; j < DC; j += 4) {
        const float4 v = (j < nj) ? __ldg(reinterpret_cast<const float4*>(crow + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
        c[j] = v.x; c[j + 1] = v.y; c[j + 2] = v.z; c[j + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < DC; ++j) c[j] = (j < nj) ? __ldg(crow + j) : 0.f;
    }
  };
  // DC == kDC: the next pass's codeword chunk is prefetched into registers;
  // wide passes (DC > kDC, few queries) load it at the pass start instead
  constexpr bool kPrefetchCw = (DC == kDC);
  float cw[DC], cwn[kPrefetchCw ? DC : 1];
  fetch_cw(0, cw);
  float nxt[SPG];
#pragma unroll
  for (int u = 0; u < SPG; ++u) nxt[u] = fetch(0, threadIdx.x + u * kThreads);
  __syncthreads();                              // previous users of the stage are done
#pragma unroll
  for (int u = 0; u < SPG; ++u)
    if (threadIdx.x + u * kThreads < 32 * kDC) sm.stage[threadIdx.x + u * kThreads] = nxt[u];
  __syncthreads();
  for (int pass = 0; pass < P; ++pass) {
    if (pass + 1 < P) {                         // prefetch the next pass: stage values (+ codeword chunk)
#pragma unroll
      for (int u = 0; u < SPG; ++u) nxt[u] = fetch(pass + 1, threadIdx.x + u * kThreads);
      if constexpr (kPrefetchCw) fetch_cw(pass + 1, cwn);
    }
    const int l = pass / npl, jc = pass - l * npl;
    const int nj = min(DC, s - jc * DC);
    if (computes) {
      if constexpr (SS > 0 && SS % DC == 0) {
        build_pass_fixed<DC, DC>(sm, lut0, l, lv0, k, kvalid, cw, nq, g, G, jc == 0);
      } else if constexpr (SS > 0) {
        if (nj == DC) build_pass_fixed<DC, DC>(sm, lut0, l, lv0, k, kvalid, cw, nq, g, G, jc == 0);
        else build_pass_fixed<(SS % DC) ? (SS % DC) : DC, DC>(sm, lut0, l, lv0, k, kvalid, cw, nq, g, G, jc == 0);
      } else {
        build_pass_generic(sm, lut0, l, lv0, k, kvalid, cw, nj, nq, g, G, jc == 0);
      }
    }
    __syncthreads();
    if (pass + 1 < P) {
#pragma unroll
      for (int u = 0; u < SPG; ++u)
        if (threadIdx.x + u * kThreads < 32 * kDC) sm.stage[threadIdx.x + u * kThreads] = nxt[u];
      if constexpr (kPrefetchCw) {
#pragma unroll
        for (int j = 0; j < DC; ++j) cw[j] = cwn[j];
      } else {
        fetch_cw(pass + 1, cw);
      }
    }
    __syncthreads();
  }
}

// Warp-cooperative pruning of one lane's candidate buffer (rare; see DESIGN.md
// §4.3).  Keeps every candidate that can still be among the query's k smallest
// (distance, id) pairs: t = smallest distance whose cumulative multiplicity
// reaches k; all candidates < t; of the candidates == t, those whose smallest
// id ranks below k - (multiplicity < t).  Returns the new count and threshold.
constexpr int kRefreshPer = (2 * kTopkMax + kBatchEmitLong) / 32;   // entries per lane held in registers (>= B)

__device__ __noinline__ void refresh_buffer(uint2* buf, int n, int k, const uint32_t* gmult,
                                            const int32_t* gminid, int* new_cnt, float* new_thr) {
  const int lane = lane_id();
  uint32_t key[kRefreshPer], grp[kRefreshPer], mul[kRefreshPer];
#pragma unroll
  for (int r = 0; r < kRefreshPer; ++r) {
    const int i = r * 32 + lane;
    if (i < n) {
      uint2 e = buf[i];
      key[r] = e.x; grp[r] = e.y; mul[r] = __ldg(gmult + e.y);
    } else {
      key[r] = 0xffffffffu; grp[r] = 0; mul[r] = 0;
    }
  }
  // total multiplicity
  uint32_t tot = 0;
#pragma unroll
  for (int r = 0; r < kRefreshPer; ++r) tot += mul[r];
  tot = __reduce_add_sync(FULLMASK, tot);
  if (tot < (uint32_t)k) {  // cannot prune (only possible with a tiny k vs B; keep all)
    *new_cnt = n; *new_thr = __int_as_float(0x7f800000); return;
  }
  uint32_t v = 0;
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t cand = v | ((1u << bit) - 1u);
    uint32_t c = 0;
#pragma unroll
    for (int r = 0; r < kRefreshPer; ++r) c += (key[r] <= cand) ? mul[r] : 0u;
    c = __reduce_add_sync(FULLMASK, c);
    if (c < (uint32_t)k) v |= (1u << bit);
  }
  const uint32_t t = v;
  uint32_t slt = 0, ntied = 0;
#pragma unroll
  for (int r = 0; r < kRefreshPer; ++r) {
    slt += (key[r] < t) ? mul[r] : 0u;
    ntied += (key[r] == t) ? 1u : 0u;
  }
  slt = __reduce_add_sync(FULLMASK, slt);
  ntied = __reduce_add_sync(FULLMASK, ntied);
  const uint32_t R = (uint32_t)k - slt;
  uint32_t tau = 0xffffffffu;
  uint32_t mid[kRefreshPer];
#pragma unroll
  for (int r = 0; r < kRefreshPer; ++r) mid[r] = 0xffffffffu;
  if (ntied > R) {
#pragma unroll
    for (int r = 0; r < kRefreshPer; ++r)
      if (key[r] == t) mid[r] = (uint32_t)__ldg(gminid + grp[r]);
    uint32_t w = 0;
    for (int bit = 31; bit >= 0; --bit) {
      const uint32_t cand = w | ((1u << bit) - 1u);
      uint32_t c = 0;
#pragma unroll
      for (int r = 0; r < kRefreshPer; ++r) c += (key[r] == t && mid[r] <= cand) ? 1u : 0u;
      c = __reduce_add_sync(FULLMASK, c);
      if (c < R) w |= (1u << bit);
    }
    tau = w;
  }
  __syncwarp();
  int base = 0;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kRefreshPer; ++r) {
    const bool keep = (r * 32 + lane < n) && (key[r] < t || (key[r] == t && (ntied <= R || mid[r] <= tau)));
    const unsigned m = __ballot_sync(FULLMASK, keep);
    if (keep) buf[base + __popc(m & lt)] = make_uint2(key[r], grp[r]);
    base += __popc(m);
  }
  __syncwarp();
  *new_cnt = base;
  *new_thr = __uint_as_float(t);
}

// Per-lane top-k candidate state.
struct TopkState {
  float thr;
  int cnt;
  uint32_t msum;      // sum of 2^bucket (<= multiplicity) of the candidates emitted so far
  uint2* buf;         // this lane's buffer
  uint2* warp_buf;    // lane 0's buffer of this warp (lane L's = warp_buf + L*kWarps*B)
  bool active;
};

struct EmitCtx {
  const ScanParams* p;
  int role;           // 0: forest per-leaf partials (every tree), 1: single tree, leaves are the groups
  int t;              // tree index for role 0
  int unit, chunk;
  int q;              // query of this lane (-1: idle lane)
  float* part;        // this unit's partials base
  TopkState ts;
};

// Append one group's distance to this lane's candidates if it can still be in
// the top-k (hot path: no calls, no syncs).  Buffers are pruned at batch
// boundaries by maybe_refresh, which keeps >= kBatchEmit free slots per lane
// (a batch of 32 leaves of each of a warp's kStreams streams).
__device__ __forceinline__ void emit_group(EmitCtx& e, float dist, uint32_t g, uint32_t mult) {
  const ScanParams& p = *e.p;
  if (p.mode == kModeFull) {
    p.leafdist[((size_t)e.chunk * 32 + lane_id()) * p.n_groups + g] = dist;   // query-major rows
    return;
  }
  TopkState& ts = e.ts;
  if (ts.active && dist <= ts.thr) {
    ET_CHECK(ts.cnt < p.B && g < (uint32_t)p.n_groups);
    ts.buf[ts.cnt] = make_uint2(__float_as_uint(dist), g);
    ++ts.cnt;
    if (mult >= (uint32_t)p.k) ts.thr = dist;   // one group alone bounds the k-th distance
  }
}

struct CntThr { int cnt; float thr; };

// Per-query thresholds shared by every unit (CTA) that scans the query --
// leaf segments, IVF probes -- through global atomicMin on the float bits
// (distances are >= 0, so the bit order is the value order).  Initialised to
// 0x7f7f7f7f (~3.4e38) by a memset; kThrNone marks "no bound yet".
constexpr float kThrNone = 1e38f;

__device__ __noinline__ CntThr maybe_refresh(uint2* warp_buf, int cnt, float thr, uint32_t msum, int B, int k,
                                             const uint32_t* gmult, const int32_t* gminid, int batch) {
  const int lane = lane_id();
  // full buffers, and (once) buffers that first reach k candidates while the
  // lane has no threshold yet: an early exact bound stops the flood of
  // candidates that every fresh warp would otherwise emit
  unsigned full = __ballot_sync(FULLMASK, cnt > B - batch || ((cnt >= k || msum >= (uint32_t)k) && !(thr < kThrNone)));
  while (full) {
    const int L = __ffs(full) - 1;
    full &= full - 1;
    int nc; float nt;
    const int n = __shfl_sync(FULLMASK, cnt, L);
    refresh_buffer(warp_buf + (size_t)L * kWarps * B, n, k, gmult, gminid, &nc, &nt);
    if (lane == L) { cnt = nc; thr = fminf(thr, nt); }
  }
  return CntThr{cnt, thr};
}

// batch: the most candidates a lane can append before the next check (32 per
// stream); B = 2k + batch rounded up (the plan's topk_B).
__device__ __forceinline__ void refresh_if_needed(EmitCtx& e, int batch = kBatchEmit) {
  const ScanParams& p = *e.p;
  if (__any_sync(FULLMASK, e.ts.cnt > p.B - batch ||
                             ((e.ts.cnt >= p.k || e.ts.msum >= (uint32_t)p.k) && !(e.ts.thr < kThrNone)))) {
    const CntThr r = maybe_refresh(e.ts.warp_buf, e.ts.cnt, e.ts.thr, e.ts.msum, p.B, p.k, p.group_mult,
                                   p.group_minid, batch);
    e.ts.cnt = r.cnt;
    e.ts.thr = r.thr;
  }
}

// Leaf record: one uint4 = 8 half-words; half-word l is the
// pre-swizzled byte offset of table entry (level l, k = code byte l) inside
// that level's 32 KB shared-memory region, (k << 7) | ((k & 31) << 2), so a
// lookup is one extract/XOR with the lane's offset and one LDS whose immediate
// carries the level's region base.  Levels 0 and 1 of an 8-level tree live in
// TMEM: their half-words are the columns k0, k1 (bits 0..7); half-word 0
// carries the LCP with the previous leaf in bits 8..11 and
// floor(log2(multiplicity)) in bits 12..15; trees with MT < 8 keep both in
// half-word 7 (bits 0..3, 4..7).

// The scan kernel has no static shared memory, so its dynamic shared memory
// (the tables, at offset 0) starts at the fixed shared-window address
// kDsmBase (after the 1 KB the system reserves); scan_kernel traps if not.
constexpr uint32_t kDsmBase = 0x400;

// A shared-memory word by its 32-bit shared address, through cvta: the
// compiler emits a plain LDS (no generic-window arithmetic) and can predicate it.
__device__ __forceinline__ const float* smem_f32(uint32_t a) {
  return reinterpret_cast<const float*>(__cvta_shared_to_generic(a));
}


// Levels a leaf looks up (bit l: l >= its LCP with the previous leaf): 8-level
// records store the mask (half-word 0 bits 8..15, one byte extract), shorter
// trees the LCP (half-word 7 bits 0..3).
template <int MT>
__device__ __forceinline__ uint32_t rec_look(const uint4& r) {
  if constexpr (MT == 8) return __byte_perm(r.x, 0u, 0x4441);
  else return (0xffu << ((r.w >> 16) & 15u)) & ((1u << MT) - 1u);
}
// floor(log2(multiplicity)) of the leaf's group (single trees), capped at 15:
// 2^bucket >= k proves the group alone holds k ids (a conservative test)
template <int MT>
__device__ __forceinline__ uint32_t rec_mbucket(const uint4& r) {
  if constexpr (MT == 8) return (r.x >> 24) & 15u;
  else return (r.w >> 20) & 15u;
}

// Distance-Context update of one leaf, branch-free.  v[l] holds the table
// entry T[l][k_l] of the path's node at depth l.  A leaf whose LCP with its
// predecessor is p shares the nodes at depths < p, whose entries are still in
// v[0..p-1]; it looks up levels p..MT-1 only (predicated LDS: the internal
// nodes entered at depths p..depth-1, its own K, and its
// postfix).  The distance is then the left-to-right sum
// ((v0 + v1) + v2) + ... -- the Distance Context ctx[l] = ctx[l-1] + T[l][k_l]
// of P:238-252 recomputed in registers, bit-identical to naive ADC.
// `valid` = false makes the call a no-op on v (the padding leaf of a stream).
// The TMEM levels' entries of a record (levels 0 and 1 of an 8-level tree:
// columns k0 and 256 + k1): issued without waiting; the caller waits once
// for every stream's reads (tmem_wait_all) before dc_leaf uses them.
// The address is one byte permute: the column byte of the record under the
// quadrant's lane base (tq's column bits are 0: the CTA allocates all 512
// columns), level 1 at column offset 256.
__device__ __forceinline__ void tmem_rec_ld(uint32_t tq, const uint4& r, uint32_t& t0, uint32_t& t1) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(t0) : "r"(__byte_perm(r.x, tq, 0x7650)));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(t1) : "r"(__byte_perm(r.x, tq, 0x7652) + 256u));
}
template <int NS>
__device__ __forceinline__ void tmem_wait_all(uint32_t (&t0)[NS], uint32_t (&t1)[NS]) {
  static_assert(NS == 1 || NS == 2 || NS == 4 || NS == 6 || NS == 8, "streams");
  if constexpr (NS == 1) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(t0[0]), "+r"(t1[0]));
  } else if constexpr (NS == 2) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(t0[0]), "+r"(t1[0]), "+r"(t0[1]), "+r"(t1[1]));
  } else if constexpr (NS == 4) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(t0[0]), "+r"(t1[0]), "+r"(t0[1]), "+r"(t1[1]), "+r"(t0[2]), "+r"(t1[2]), "+r"(t0[3]),
                   "+r"(t1[3]));
  } else if constexpr (NS == 6) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(t0[0]), "+r"(t1[0]), "+r"(t0[1]), "+r"(t1[1]), "+r"(t0[2]), "+r"(t1[2]), "+r"(t0[3]),
                   "+r"(t1[3]), "+r"(t0[4]), "+r"(t1[4]), "+r"(t0[5]), "+r"(t1[5]));
  } else {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(t0[0]), "+r"(t1[0]), "+r"(t0[1]), "+r"(t1[1]), "+r"(t0[2]), "+r"(t1[2]), "+r"(t0[3]),
                   "+r"(t1[3]), "+r"(t0[4]), "+r"(t1[4]), "+r"(t0[5]), "+r"(t1[5]), "+r"(t0[6]), "+r"(t1[6]),
                   "+r"(t0[7]), "+r"(t1[7]));
  }
}

// Forest distance with the tree boundaries at run time (bit l of fsplit:
// level l starts tree u >= 1): per-tree partials left to right, summed in
// tree order (A13).
template <int MT>
__device__ __forceinline__ float dc_sum_forest(const float (&v)[MT], uint32_t fsplit) {
  float tot = 0.f, s = v[0];
  bool have = false;
#pragma unroll
  for (int l = 1; l < MT; ++l) {
    if ((fsplit >> l) & 1u) { tot = have ? tot + s : s; have = true; s = v[l]; }
    else s = s + v[l];
  }
  return have ? tot + s : s;
}

// The lookups of one leaf: level l's entry is (re)loaded iff bit l of
// `look` (warp-uniform) -- the levels after the leaf's LCP (P:249, P:239,
// P:242-243), or a fused-forest tuple's mask; the TMEM levels' entries were
// read by the caller (t0, t1).
template <int MT>
__device__ __forceinline__ void dc_look(float (&v)[MT], const uint4& r, uint32_t look, uint32_t lane4, uint32_t t0,
                                        uint32_t t1) {
  constexpr int lv0 = lv0_of(MT);
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
  if constexpr (lv0 == 2) {
    // the TMEM levels are read for every leaf: a level outside `look` holds
    // the byte of the previous leaf (shared prefix / unchanged tree bytes), so
    // the read returned the very entry v already holds -- no select needed
    (void)look;
    v[0] = __uint_as_float(t0);
    v[1] = __uint_as_float(t1);
  }
#pragma unroll
  for (int l = lv0; l < MT; ++l) {
    // shared-memory half-words are pure offsets (< 32768; the LCP / mask /
    // bucket fields live in the TMEM half-words or in unused level 7)
    const uint32_t off = ((l & 1) ? (w[l >> 1] >> 16) : (w[l >> 1] & 0xffffu)) ^ lane4;
    ET_CHECK(off < 32768u);
    if (look & (1u << l)) v[l] = *smem_f32(off + (kDsmBase + ((uint32_t)(l - lv0) << 15)));
  }
}

template <int MT>
__device__ __forceinline__ float dc_leaf(float (&v)[MT], const uint4& r, uint32_t look,
                                         uint32_t lane4, uint32_t t0, uint32_t t1) {
  constexpr int lv0 = lv0_of(MT);
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
  // look: levels looked up (l >= LCP) as a bit mask (the compiler turns the
  // tests below into one R2P instead of a compare per level)
  if constexpr (lv0 == 2) {
    // levels 0 and 1 (TMEM, columns k0 and 256 + k1, read by the caller: t0,
    // t1): outside `look` the read returned the very entry the path holds
    v[0] = __uint_as_float(t0);
    v[1] = __uint_as_float(t1);
  }
#pragma unroll
  for (int l = lv0; l < MT; ++l) {
    const uint32_t off = (l & 1) ? ((w[l >> 1] >> 16) ^ lane4) : ((w[l >> 1] & 0xffffu) ^ lane4);
    // predicated LDS at a 32-bit shared address (no shared-memory access when off)
    if (look & (1u << l)) v[l] = *smem_f32(off + (kDsmBase + ((uint32_t)(l - lv0) << 15)));
  }
  float s = v[0];
#pragma unroll
  for (int l = 1; l < MT; ++l) s = s + v[l];
  return s;
}

// ---- masked records: fused E-Forest tuples ----
// Tuple t's record is the single-tree record of its full code with the LCP
// field replaced by an 8-bit lookup mask: bit l is set iff level l's entry
// must be (re)looked up, i.e. l - split[u] >= the LCP of tuples t-1 and t over
// the bytes of the tree u that holds level l -- each tree's own Distance
// Context carried along the tuple sequence.  M == 8: mask in
// half-word 0 bits 8..15 (next to the TMEM column k0), multiplicity bucket
// in half-word 1 bits 8..11 (next to the TMEM column k1); M < 8: half-word 7
// = mask | bucket << 8.
template <int MT>
__device__ __forceinline__ uint32_t rec_mask(const uint4& r) {
  if constexpr (MT == 8) return __byte_perm(r.x, 0u, 0x4441);
  else return (r.w >> 16) & 255u;
}
template <int MT>
__device__ __forceinline__ uint32_t rec_mbucket_m(const uint4& r) {
  if constexpr (MT == 8) return (r.x >> 24) & 15u;
  else return (r.w >> 24) & 15u;
}


// Scan of leaves [a, b) of one tree by one warp, lane = query.  The range is
// split into two halves scanned in lockstep (two independent dependency
// chains per warp); records come with one coalesced load per 32 leaves per
// half (the next batch in flight) and four shuffles per leaf.  A leaf costs
// (MT - LCP) shared-memory lookups, MT - 1 FADDs and no branches.
template <int MT, int ROLE>
__device__ void scan_tree(EmitCtx& e, const SmemScan& sm, const TreeDev& tr, uint32_t a, uint32_t b,
                          const float* lut0g) {
  (void)lut0g;
  const ScanParams& p = *e.p;
  const int lane = lane_id();
  const uint32_t lane4 = (uint32_t)lane << 2;
  const uint32_t tq = tmem_lane_base(sm.tmem);
  const bool topk = p.mode == kModeTopk;
  const uint4* rec = tr.rec;
  auto shfl_rec = [&](const uint4& mine, int j) {
    uint4 r;
    r.x = __shfl_sync(FULLMASK, mine.x, j);
    r.y = (MT > 2) ? __shfl_sync(FULLMASK, mine.y, j) : 0u;
    r.z = (MT > 4) ? __shfl_sync(FULLMASK, mine.z, j) : 0u;
    r.w = __shfl_sync(FULLMASK, mine.w, j);   // levels 6-7, or the LCP when MT < 8
    return r;
  };
  auto load_batch = [&](uint32_t base, uint32_t end) {
    return (base + lane < end) ? __ldg(rec + base + lane) : make_uint4(0u, 0u, 0u, 0u);
  };
  auto batch_end = [&]() {
    if (topk && ROLE != 0) {   // prune full buffers; share the threshold with the CTA's other warps
      refresh_if_needed(e);    // and with every other unit scanning the same query
      if (e.ts.active) {
        const unsigned mine = __float_as_uint(e.ts.thr);
        atomicMin(&sm.thr[lane], mine);
        unsigned t = *((volatile unsigned*)&sm.thr[lane]);
        if (p.qthr_shared) t = min(t, atomicMin(p.qthr + e.q, t));
        e.ts.thr = __uint_as_float(t);
      }
    }
  };
  {
    const uint32_t m = a + (b - a + 1) / 2;   // halves [a, m) and [m, b); |[m, b)| <= |[a, m)|
    float v0[MT], v1[MT];
#pragma unroll
    for (int l = 0; l < MT; ++l) { v0[l] = 0.f; v1[l] = 0.f; }
    uint4 nx0 = load_batch(a, m), nx1 = load_batch(m, b);
    auto emit = [&](uint32_t leaf, float dist, const uint4& r, bool valid) {
      if constexpr (ROLE == 0) {
        if (valid) e.part[(size_t)p.part_base[e.t] + (size_t)leaf * 32 + lane] = dist;
      } else {
        if (p.mode == kModeFull) {
          if (valid) p.leafdist[((size_t)e.chunk * 32 + lane) * p.n_groups + leaf] = dist;   // query-major rows
        } else {
          TopkState& ts = e.ts;
          const bool em = valid && ts.active && dist <= ts.thr;
          if (em) ts.buf[ts.cnt] = make_uint2(__float_as_uint(dist), leaf);
          ts.cnt += em ? 1 : 0;
          // one group alone (2^bucket <= multiplicity ids) bounds the k-th distance
          if (em && (1u << rec_mbucket<MT>(r)) >= (uint32_t)p.k) ts.thr = dist;
        }
      }
    };
    for (uint32_t off = 0; a + off < m; off += 32) {
      const uint4 mine0 = nx0, mine1 = nx1;
      nx0 = load_batch(a + off + 32, m);
      nx1 = load_batch(m + off + 32, b);
      const int n0 = (int)min(32u, m - (a + off));
      const int n1 = (m + off < b) ? (int)min(32u, b - (m + off)) : 0;
      for (int j = 0; j < n0; ++j) {
        const uint4 r0 = shfl_rec(mine0, j), r1 = shfl_rec(mine1, j);
        const uint32_t leaf0 = a + off + j, leaf1 = m + off + j;
        const bool ok1 = j < n1;
        constexpr uint32_t kAll = (1u << MT) - 1u;
        const uint32_t lk0 = (off + j == 0) ? kAll : rec_look<MT>(r0);   // range starts: rebuild the path
        const uint32_t lk1 = ok1 ? ((off + j == 0) ? kAll : rec_look<MT>(r1)) : 0u;
        uint32_t t0[2] = {0u, 0u}, t1[2] = {0u, 0u};
        if constexpr (lv0_of(MT) == 2) {
          tmem_rec_ld(tq, r0, t0[0], t1[0]);
          tmem_rec_ld(tq, r1, t0[1], t1[1]);
          tmem_wait_all<2>(t0, t1);
        }
        const float d0 = dc_leaf<MT>(v0, r0, lk0, lane4, t0[0], t1[0]);
        const float d1 = dc_leaf<MT>(v1, r1, lk1, lane4, t0[1], t1[1]);
        emit(leaf0, d0, r0, true);
        emit(leaf1, d1, r1, ok1);
      }
      batch_end();
    }
  }
}

// Top-k / full-output scan of leaves [a, b) of one tree (or of the fused
// forest's tuples) by one warp, lane = query.  The range is split into NS
// contiguous streams scanned in lockstep -- NS independent dependency chains
// per warp, one branch-free block per step (lengths differ by at most one
// leaf: the shorter streams' last step is predicated off).  Records come with
// one coalesced load per 32 leaves per stream (the next batch in flight) and
// four shuffles per leaf; a leaf costs (MT - LCP) shared-memory / TMEM
// lookups (masked records: the levels of its mask), MT - 1 FADDs and a
// predicated emit.
// EX: leaf extra byte: the leaf's byte (p.gextra, one per group,
// loaded with the record batch) indexes the decode table staged in shared
// memory (sm.bigstage, free after the table build) and its entry is added
// after the M lookups: dist = (((v0 + v1) + ...) + E[e]) (oracle/leafextra.py).
// RS (ET_REC_SMEM builds, 8-level trees of the fused-build kernel): the batch's
// records go through the warp's slice of the staging area (sm.bigstage, free
// after the table build) instead of shuffles.
template <int MT, bool MASKED, bool TOPK, int NS, int FS, bool EX = false, bool RS = false>
__device__ void scan_tree3(EmitCtx& e, const SmemScan& sm, const TreeDev& tr, uint32_t a, uint32_t b) {
  const ScanParams& p = *e.p;
  const int lane = lane_id();
  const uint32_t lane4 = (uint32_t)lane << 2;
  const uint32_t tq = tmem_lane_base(sm.tmem);
  const uint4* rec = tr.rec;
  constexpr uint32_t kAll = (1u << MT) - 1u;
  auto shfl_rec = [&](const uint4& mine, int j) {
    uint4 r;
    r.x = __shfl_sync(FULLMASK, mine.x, j);
    r.y = (MT > 2 || MASKED) ? __shfl_sync(FULLMASK, mine.y, j) : 0u;
    r.z = (MT > 4) ? __shfl_sync(FULLMASK, mine.z, j) : 0u;
    r.w = __shfl_sync(FULLMASK, mine.w, j);
    return r;
  };
  const uint32_t len = b - a;
  uint32_t s0[NS], sl[NS];                           // stream start, length
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    s0[k] = a + (uint32_t)(((uint64_t)len * k) / NS);
    sl[k] = a + (uint32_t)(((uint64_t)len * (k + 1)) / NS) - s0[k];
  }
  uint32_t steps = 0;                                // the longest stream (lengths differ by <= 1)
#pragma unroll
  for (int k = 0; k < NS; ++k) steps = max(steps, sl[k]);
  auto load_batch = [&](int k, uint32_t off) {
    ET_CHECK(off + lane >= sl[k] || s0[k] + off + lane < (uint32_t)tr.n_leaves);
    return (off + lane < sl[k]) ? __ldg(rec + s0[k] + off + lane) : make_uint4(0u, 0u, 0u, 0u);
  };
  uint4 nx[NS];
  float v[NS][MT];
  uint32_t nxe[NS], cure[NS];                        // EX: the leaves' extra bytes (next / current batch)
  auto load_extra = [&](int k, uint32_t off) -> uint32_t {
    return (EX && off + lane < sl[k]) ? (uint32_t)__ldg(p.gextra + s0[k] + off + lane) : 0u;
  };
  const uint32_t etab_s = smem_u32(sm.bigstage);
  const uint32_t rs_s = smem_u32(sm.bigstage) + (uint32_t)warp_id() * (uint32_t)(NS * 512);
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    nx[k] = load_batch(k, 0);
    nxe[k] = load_extra(k, 0);
    cure[k] = 0u;
#pragma unroll
    for (int l = 0; l < MT; ++l) v[k][l] = 0.f;
  }
  for (uint32_t off = 0; off < steps; off += 32) {
    uint4 cur[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      cur[k] = nx[k];
      nx[k] = load_batch(k, off + 32);
      if constexpr (EX) { cure[k] = nxe[k]; nxe[k] = load_extra(k, off + 32); }
    }
    if constexpr (RS) {
      ET_CHECK(rs_s + (uint32_t)(NS * 512) <= smem_u32(sm.bigstage) + 8u * 16u * 128u + kRecExtra);
      __syncwarp();                                  // the previous batch's reads are done
#pragma unroll
      for (int k = 0; k < NS; ++k) sts_u4(rs_s + (uint32_t)(k * 512) + ((uint32_t)lane << 4), cur[k]);
      __syncwarp();
    }
    const int n = (int)min(32u, steps - off);
    // Generic steps (the range's first leaf: every level looked up; the last
    // step: the shorter streams are done) test per stream; all other steps
    // run a copy of the body with those tests compiled out.
    auto step = [&](int j, auto gen_tag) {
      constexpr bool GEN = decltype(gen_tag)::value;
      // range start: rebuild the path (generic steps only)
      const uint32_t fm = GEN ? ((off + j == 0) ? kAll : 0u) : 0u;
      uint4 rr[NS];
      uint32_t t0[NS], t1[NS];                       // TMEM levels: every stream's reads, one wait
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        if constexpr (RS) rr[k] = lds_u4(rs_s + (uint32_t)(k * 512) + ((uint32_t)j << 4));
        else rr[k] = shfl_rec(cur[k], j);
        t0[k] = t1[k] = 0u;
        if constexpr (lv0_of(MT) == 2) tmem_rec_ld(tq, rr[k], t0[k], t1[k]);
      }
      if constexpr (lv0_of(MT) == 2) tmem_wait_all<NS>(t0, t1);
      // lookups of every stream, then the streams' sums interleaved level by
      // level (independent FADD chains side by side), then the emits
      bool ok[NS];
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        ok[k] = GEN ? (off + j < sl[k]) : true;   // fast steps: every stream has this leaf
        uint32_t look;
        if constexpr (MASKED) look = ok[k] ? (rec_mask<MT>(rr[k]) | fm) : 0u;
        else look = ok[k] ? (rec_look<MT>(rr[k]) | fm) : 0u;
        dc_look<MT>(v[k], rr[k], look, lane4, t0[k], t1[k]);
      }
      float dist[NS];
      if constexpr (MASKED && FS > 0 && FS < MT) {   // two trees: (p_0 + p_1), each left to right (A13)
        float s1[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) { dist[k] = v[k][0]; s1[k] = v[k][FS]; }
#pragma unroll
        for (int l = 1; l < MT; ++l) {
          if (l == FS) continue;
#pragma unroll
          for (int k = 0; k < NS; ++k) {
            if (l < FS) dist[k] = dist[k] + v[k][l];
            else s1[k] = s1[k] + v[k][l];
          }
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) dist[k] = dist[k] + s1[k];
      } else if constexpr (MASKED) {
#pragma unroll
        for (int k = 0; k < NS; ++k) dist[k] = dc_sum_forest<MT>(v[k], p.fsplit);
      } else {   // ((v0 + v1) + v2) + ...: the Distance Context, bit-identical to naive ADC
#pragma unroll
        for (int k = 0; k < NS; ++k) dist[k] = v[k][0];
#pragma unroll
        for (int l = 1; l < MT; ++l)
#pragma unroll
          for (int k = 0; k < NS; ++k) dist[k] = dist[k] + v[k][l];
      }
      if constexpr (EX) {   // + E[e] of the leaf's extra byte (one broadcast LDS per stream)
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const uint32_t ek = __shfl_sync(FULLMASK, cure[k], j);
          dist[k] = dist[k] + lds(etab_s + (ek << 2));
        }
      }
      if constexpr (!TOPK) {
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if (ok[k]) p.leafdist[((size_t)e.chunk * 32 + lane) * p.n_groups + s0[k] + off + j] = dist[k];
      } else {
        TopkState& ts = e.ts;
        bool any = false;
#pragma unroll
        for (int k = 0; k < NS; ++k) any |= ok[k] && dist[k] <= ts.thr;
        if (__any_sync(FULLMASK, any && ts.active)) {   // warp-uniform: once thresholds are tight, rare
#pragma unroll
          for (int k = 0; k < NS; ++k) {
            const uint4 r = rr[k];
            const uint32_t bucket = MASKED ? rec_mbucket_m<MT>(r) : rec_mbucket<MT>(r);
            const bool em = ok[k] && ts.active && dist[k] <= ts.thr;
            ET_CHECK(!em || ts.cnt < p.B);
            if (em) ts.buf[ts.cnt] = make_uint2(__float_as_uint(dist[k]), s0[k] + off + j);
            ts.cnt += em ? 1 : 0;
            ts.msum += em ? (1u << bucket) : 0u;
            // one group alone (2^bucket <= multiplicity ids) bounds the k-th distance
            if (em && (1u << bucket) >= (uint32_t)p.k) ts.thr = dist[k];
          }
        }
      }
    };
    for (int j = 0; j < n; ++j) {
      // (fast copies for the top-k scans of single trees and two-tree fused
      // forests; ptxas 12.9 runs out of predicate registers on the others)
      constexpr bool kFast = TOPK && (!MASKED || (FS > 0 && FS < MT));
      if (!kFast || off + j == 0 || off + j + 1 >= steps) step(j, std::true_type{});
      else step(j, std::false_type{});
    }
    if constexpr (TOPK) {   // prune full buffers; share the threshold with the CTA's other warps
      refresh_if_needed(e, 32 * NS);  // and with every other unit scanning the same query
      if (e.ts.active) {
        const unsigned mine = __float_as_uint(e.ts.thr);
        atomicMin(&sm.thr[lane], mine);
        unsigned t = *((volatile unsigned*)&sm.thr[lane]);
        if (p.qthr_shared) t = min(t, atomicMin(p.qthr + e.q, t));
        e.ts.thr = __uint_as_float(t);
      }
    }
  }
}


template <int MT, bool MASKED, int NS = kStreams, bool EX = false, bool RS = false>
__device__ __forceinline__ void scan_tree3_mode(EmitCtx& e, const SmemScan& sm, const TreeDev& tr, uint32_t a,
                                                uint32_t b) {
  if constexpr (EX) {   // leaf extra byte: single trees, top-k (host: et_etree_topk_extra)
    if constexpr (!MASKED) scan_tree3<MT, false, true, NS, 0, true>(e, sm, tr, a, b);
    return;
  }
  // fused forests of two 4-level trees (the c5 split 0-3 | 4-7): the tree
  // boundary at compile time
  if (MASKED && MT == 8 && e.p->fsplit == (1u << 4)) {
    if (e.p->mode == kModeTopk) scan_tree3<MT, MASKED, true, NS, 4, false, RS>(e, sm, tr, a, b);
    else scan_tree3<MT, MASKED, false, kStreams, 4, false, RS>(e, sm, tr, a, b);
    return;
  }
  if (e.p->mode == kModeTopk) scan_tree3<MT, MASKED, true, NS, 0, false, RS>(e, sm, tr, a, b);
  else scan_tree3<MT, MASKED, false, kStreams, 0, false, RS>(e, sm, tr, a, b);
}

template <bool MASKED>
__device__ __forceinline__ void scan2_dispatch(EmitCtx& e, const SmemScan& sm, const TreeDev& tr,
                                               uint32_t a, uint32_t b) {
  switch (tr.MT) {
    case 1: scan_tree3_mode<1, MASKED>(e, sm, tr, a, b); break;
    case 2: scan_tree3_mode<2, MASKED>(e, sm, tr, a, b); break;
    case 3: scan_tree3_mode<3, MASKED>(e, sm, tr, a, b); break;
    case 4: scan_tree3_mode<4, MASKED>(e, sm, tr, a, b); break;
    case 5: scan_tree3_mode<5, MASKED>(e, sm, tr, a, b); break;
    case 6: scan_tree3_mode<6, MASKED>(e, sm, tr, a, b); break;
    case 7: scan_tree3_mode<7, MASKED>(e, sm, tr, a, b); break;
    case 8: scan_tree3_mode<8, MASKED>(e, sm, tr, a, b); break;
    default: break;
  }
}

// Prune full candidate buffers and share the lanes' thresholds with the CTA's
// other warps (shared memory) and, when a query spans several units, with
// every unit scanning it (global per-query atomicMin).
__device__ __forceinline__ void share_threshold(EmitCtx& e, const SmemScan& sm) {
  const ScanParams& p = *e.p;
  const int lane = lane_id();
  refresh_if_needed(e);
  if (e.ts.active) {
    atomicMin(&sm.thr[lane], __float_as_uint(e.ts.thr));
    unsigned t = *((volatile unsigned*)&sm.thr[lane]);
    if (p.qthr_shared) t = min(t, atomicMin(p.qthr + e.q, t));
    e.ts.thr = __uint_as_float(t);
  }
}

// E-Forest join (reading A13): every tuple -- one distinct full
// code, i.e. one group -- gets dist = ((p_0 + p_1) + ...) summed in tree order
// from the per-tree partials of its leaves (written by the trees' scans).
// Tuples [ga, gb) of this warp, 32 at a time: their leaves and multiplicities
// in one coalesced load each, then the per-query partials (coalesced across
// lanes) kJoinBatch tuples at a time.
constexpr int kJoinBatch = 16;   // tuples whose partials are in flight at once

__device__ void join_tuples(EmitCtx& e, const SmemScan& sm, uint32_t ga, uint32_t gb) {
  const ScanParams& p = *e.p;
  const int lane = lane_id();
  const bool topk = p.mode == kModeTopk;
  for (uint32_t g0 = ga; g0 < gb; g0 += 32) {
    const int n = (int)min(32u, gb - g0);
    uint32_t my_l[kMaxTrees];
#pragma unroll
    for (int t = 0; t < kMaxTrees; ++t) my_l[t] = (t < p.T && lane < n) ? __ldg(p.tup_leaf[t] + g0 + lane) : 0u;
    const uint32_t my_mu = (topk && lane < n) ? __ldg(p.group_mult + g0 + lane) : 0u;
    for (int u0 = 0; u0 < n; u0 += kJoinBatch) {
      float acc[kJoinBatch];
#pragma unroll
      for (int u = 0; u < kJoinBatch; ++u) {
        const uint32_t l0 = __shfl_sync(FULLMASK, my_l[0], u0 + u);
        acc[u] = (u0 + u < n) ? e.part[(size_t)p.part_base[0] + (size_t)l0 * 32 + lane] : 0.f;
      }
#pragma unroll
      for (int t = 1; t < kMaxTrees; ++t) {
        if (t < p.T) {
          float pv[kJoinBatch];
#pragma unroll
          for (int u = 0; u < kJoinBatch; ++u) {
            const uint32_t lt = __shfl_sync(FULLMASK, my_l[t], u0 + u);
            pv[u] = (u0 + u < n) ? e.part[(size_t)p.part_base[t] + (size_t)lt * 32 + lane] : 0.f;
          }
#pragma unroll
          for (int u = 0; u < kJoinBatch; ++u) acc[u] = acc[u] + pv[u];
        }
      }
#pragma unroll
      for (int u = 0; u < kJoinBatch; ++u) {
        const uint32_t mult = __shfl_sync(FULLMASK, my_mu, u0 + u);
        if (u0 + u < n) emit_group(e, acc[u], g0 + u0 + u, mult);
      }
    }
    if (topk) share_threshold(e, sm);
  }
}

template <int ROLE>
__device__ __forceinline__ void scan_dispatch(EmitCtx& e, const SmemScan& sm, const TreeDev& tr,
                                              uint32_t a, uint32_t b, const float* lut0g) {
  switch (tr.MT) {
    case 1: scan_tree<1, ROLE>(e, sm, tr, a, b, lut0g); break;
    case 2: scan_tree<2, ROLE>(e, sm, tr, a, b, lut0g); break;
    case 3: scan_tree<3, ROLE>(e, sm, tr, a, b, lut0g); break;
    case 4: scan_tree<4, ROLE>(e, sm, tr, a, b, lut0g); break;
    case 5: scan_tree<5, ROLE>(e, sm, tr, a, b, lut0g); break;
    case 6: scan_tree<6, ROLE>(e, sm, tr, a, b, lut0g); break;
    case 7: scan_tree<7, ROLE>(e, sm, tr, a, b, lut0g); break;
    case 8: scan_tree<8, ROLE>(e, sm, tr, a, b, lut0g); break;
    default: break;
  }
}

// MTC > 0: every tree has MTC levels (compile time); 0: runtime switch.
template <int MTC, int ROLE>
__device__ __forceinline__ void scan_any(EmitCtx& e, const SmemScan& sm, const TreeDev& tr,
                                         uint32_t a, uint32_t b, const float* lut0g) {
  if constexpr (MTC > 0) scan_tree<MTC, ROLE>(e, sm, tr, a, b, lut0g);
  else scan_dispatch<ROLE>(e, sm, tr, a, b, lut0g);
}


// MODE 0: one E-Tree (or IVF lists); 1: E-Forest with per-tree partials and
// the tuple join (M > 8, e.g. c3); 2: fused E-Forest over masked tuple
// records (M <= 8, e.g. c5).
// NS: lockstep streams per warp of the 8-level top-k scans (kStreamsLong for
// long leaf ranges, p.long_ranges: more independent chains per warp; short
// ranges keep kStreams -- a separate instantiation, so neither pays the other's
// registers or code).
template <int SS, int MTC, int MODE, int NS = kStreams, bool EX = false>
__global__ void __launch_bounds__(kThreads, 1) scan_kernel(const __grid_constant__ ScanParams p) {
  constexpr bool FOREST = (MODE == 1);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // Segment-major launch order: every chunk's first segment runs in the first
  // waves, so later segments start from the per-query bound they left in
  // qthr.  The unit (candidate buffers, scratch) stays chunk * S + seg.
  const int n_ch = p.n_units / p.S;
  const int seg = (int)blockIdx.x / n_ch;
  const int chunk = (int)blockIdx.x - seg * n_ch;
  const int unit = chunk * p.S + seg;
  const int lane = lane_id(), warp = warp_id();
  if (threadIdx.x == 0 && smem_u32(smem_raw) != kDsmBase) __trap();   // tab_ld's fixed base
  phase_mark(unit, 0);
  if (p.n_chunks_dev && chunk >= *p.n_chunks_dev) return;   // IVF: fewer chunks than the bound
  int MTmax = 0;
  for (int t = 0; t < p.T; ++t) MTmax = max(MTmax, p.tree[t].MT);
  const ScanSmem L = scan_smem(MTmax);
  // resident build of the first tree: stage the queries asynchronously now
  constexpr bool kResident = (SS == kDC && MTC > 0);
  const bool staged = kResident && !p.luts && !p.chunk_cell;
  if constexpr (kResident) {
    if (staged) {
      const int MTf = p.tree[p.T - 1].MT;
      const uint32_t base = smem_u32(smem_raw);
      // 8 levels: the staging area; else the last level's region + the small stage
      const uint32_t region_s = (MTf == 8) ? base + L.big_stage : base + ((uint32_t)(MTf - 1) << 15);
      stage_async<SS, MTC>(p, p.T - 1, chunk, p.n_units / p.S, region_s, base + L.stage);
    }
  }
  SmemScan sm;
  sm.tab = reinterpret_cast<float*>(smem_raw);
  sm.bigstage = reinterpret_cast<float*>(smem_raw + L.big_stage);
  sm.thr = reinterpret_cast<unsigned*>(smem_raw + L.thr);
  sm.qidx = reinterpret_cast<int*>(smem_raw + L.qidx);
  sm.stage = reinterpret_cast<float*>(smem_raw + L.stage);
  sm.tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + L.tmem_slot);
  sm.tmem = 0;
  const bool use_tmem = (MTmax == 8);
  if (use_tmem) {
    if (warp == 0) tmem_alloc(sm.tmem_slot);
    tmem_fence_before();
  }

  if (threadIdx.x < 32) {
    if (p.flatQ > 0) {
      const int nch = p.n_units / p.S;
      const int64_t s0 = (int64_t)chunk * p.flatQ / nch, s1 = (int64_t)(chunk + 1) * p.flatQ / nch;
      sm.qidx[lane] = (s0 + lane < s1) ? (int)(s0 + lane) : -1;
    } else {
      sm.qidx[lane] = __ldg(p.chunk_q + (size_t)chunk * 32 + lane);
    }
    // the query's bound from the units that finished before this one started
    // (qthr: the min of proven k-th distance bounds; 0x7f7f7f7f = none yet)
    const int q = sm.qidx[lane];
    // (only queries spanning several units: S > 1, IVF probes)
    sm.thr[lane] = (p.qthr_shared && p.mode == kModeTopk && q >= 0) ? min(0x7f800000u, __ldcg(p.qthr + q))
                                                                     : 0x7f800000u;
  }
  __syncthreads();
  if (use_tmem) {
    tmem_fence_after();
    sm.tmem = *sm.tmem_slot;
  }
  int nq = 0;
  {
    const int q = sm.qidx[lane];
    nq = __popc(__ballot_sync(FULLMASK, q >= 0));   // active lanes are a prefix
  }
  const int cell = p.chunk_cell ? __ldg(p.chunk_cell + chunk) : -1;
  const float* lut0g = p.lut0 ? p.lut0 + (size_t)unit * kTmemLevels * 256 * 32 : nullptr;

  EmitCtx e;
  e.p = &p;
  e.unit = unit;
  e.chunk = chunk;
  e.q = sm.qidx[lane];
  e.part = p.partials ? p.partials + (size_t)unit * p.part_stride : nullptr;
  e.ts.active = lane < nq;
  e.ts.thr = e.ts.active ? __uint_as_float(sm.thr[lane]) : -1.0f;
  e.ts.cnt = 0;
  e.ts.msum = 0;
  e.ts.warp_buf = nullptr;
  e.ts.buf = nullptr;
  if (p.mode == kModeTopk) {
    // candidates of (unit, lane): kWarps consecutive per-warp buffers of B entries
    e.ts.warp_buf = p.cand + ((size_t)unit * 32 * kWarps + warp) * p.B;
    e.ts.buf = e.ts.warp_buf + (size_t)lane * kWarps * p.B;
  }

  if constexpr (!(SS == kDC && MTC > 0)) phase_mark(unit, 1);
  // s > 16 trees of 8 levels for <= 8 queries: the wide resident build
  auto wide8 = [&](int tt) {
    if constexpr (SS > kDC && SS <= 64 && SS % 4 == 0)
      return nq <= 8 && !p.luts && p.vec4 && p.tree[tt].MT == 8 && use_tmem && !p.wide_old;
    else
      return false;
  };
  // Forest: trees T-1..1 first (per-leaf partials for this CTA's queries),
  // then tree 0, whose leaves walk their tuples and sum in tree order.
  for (int t = p.T - 1; t >= 0; --t) {
    const TreeDev& tr = p.tree[t];
    bool level0_done = false;   // resident build copies level 0 to TMEM itself
    if constexpr (SS == kDC && MTC > 0) {
      if (p.luts) { build_tables<SS>(p, sm, t, unit, nq, cell); __syncthreads(); }
      else {
        phase_mark(unit, 1);
        build_tables_resident<SS, MTC>(p, sm, t, unit, nq, cell, staged && t == p.T - 1);
        level0_done = true;
        phase_mark(unit, 2);
      }
    } else {
      if constexpr (SS > kDC && SS <= 64 && SS % 4 == 0) {
        if (wide8(t)) {
          if (t == p.T - 1) stage_wide8<SS>(p, sm, t, nq, cell);   // (later trees: staged during the previous scan)
          build_tables_wide8<SS>(p, sm, t, nq);
          level0_done = true;
          if (t > 0 && wide8(t - 1)) stage_wide8<SS>(p, sm, t - 1, nq, cell);   // lands while tree t is scanned
        } else if (nq <= 8 && !p.luts && p.vec4) build_tables_wide<SS>(p, sm, t, unit, nq, cell);
        else build_tables<SS>(p, sm, t, unit, nq, cell);
      } else {
        build_tables<SS>(p, sm, t, unit, nq, cell);
      }
      __syncthreads();
    }
    if (tr.MT == 8 && !level0_done) {   // level 0 -> TMEM (every warp copies a quarter of its quadrant's columns)
      tmem_fence_after();
      tmem_load_level0(sm, lut0g);
      tmem_fence_before();
      __syncthreads();
      tmem_fence_after();
    }
    if constexpr (!(SS == kDC && MTC > 0)) phase_mark(unit, t == 0 ? 7 : 5);   // tables of tree t ready
    if constexpr (EX) {   // the extra byte's decode table -> the (now free) staging area
      for (int i = threadIdx.x; i < 256; i += kThreads) sm.bigstage[i] = __ldg(p.etab + i);
      __syncthreads();
    }
    uint32_t lo = 0, hi = (uint32_t)tr.n_leaves;
    if (t == 0) {
      if (p.chunk_lo) { lo = __ldg(p.chunk_lo + chunk); hi = __ldg(p.chunk_hi + chunk); }
      const uint32_t len = hi - lo;
      const uint32_t a = lo + (uint32_t)(((uint64_t)len * seg) / p.S);
      const uint32_t b = lo + (uint32_t)(((uint64_t)len * (seg + 1)) / p.S);
      lo = a; hi = b;
    }
    const uint32_t len = hi - lo;
    const uint32_t wa = lo + (uint32_t)(((uint64_t)len * warp) / kWarps);
    const uint32_t wb = lo + (uint32_t)(((uint64_t)len * (warp + 1)) / kWarps);
    e.t = t;
    if (wa < wb) {
      if constexpr (FOREST) {
        scan_any<MTC, 0>(e, sm, tr, wa, wb, lut0g);   // per-leaf partials of every tree
      } else if constexpr (MTC > 0) {
        // (ET_REC_SMEM: 16-dim fused build only -- its staging area is free during the scan)
        constexpr bool kRS = (ET_REC_SMEM != 0) && SS == kDC && MTC == 8 && !EX;
        scan_tree3_mode<MTC, MODE == 2, NS, EX, kRS>(e, sm, tr, wa, wb);
      } else {
        scan2_dispatch<MODE == 2>(e, sm, tr, wa, wb);
      }
    }
    tmem_fence_before();
    __syncthreads();   // partials visible / tables free for the next tree
    tmem_fence_after();
    if constexpr (!(SS == kDC && MTC > 0)) phase_mark(unit, t == 0 ? 2 : 6);   // tree t scanned
  }
  if constexpr (FOREST) {   // the CTA's warps split the tuples evenly
    const uint64_t G = (uint64_t)p.n_groups;
    join_tuples(e, sm, (uint32_t)((G * warp) / kWarps), (uint32_t)((G * (warp + 1)) / kWarps));
  }
  phase_mark(unit, 3);
  if (use_tmem && warp == 0) tmem_dealloc(sm.tmem);

  if (p.mode == kModeTopk && p.qthr && !p.qthr_shared && warp == 0 && sm.qidx[lane] >= 0)
    p.qthr[sm.qidx[lane]] = sm.thr[lane];   // the query's only unit: its final threshold
  if (p.mode == kModeTopk && !p.compact) {
    // per-warp candidate lists stay where the scan wrote them: lane L's 16
    // buffers are contiguous, counts at cand_cnt[(unit*32 + L)*kWarps + warp]
    p.cand_cnt[((size_t)unit * 32 + lane) * kWarps + warp] = e.ts.cnt;
    if (warp == 0 && p.unit_thr) p.unit_thr[(size_t)unit * 32 + lane] = __uint_as_float(sm.thr[lane]);
  } else if (p.mode == kModeTopk) {
    // Long lists (small groups): merge the 16 warps' candidates of each lane
    // into its first buffer under the final threshold, in place -- lane L's
    // buffers are contiguous, so write position <= read position.
    int* cnt_s = reinterpret_cast<int*>(smem_raw);   // tables are dead now
    cnt_s[warp * 32 + lane] = e.ts.cnt;
    __syncthreads();
    for (int L = warp; L < 32; L += kWarps) {
      const int myc = (lane < kWarps) ? cnt_s[lane * 32 + L] : 0;
      int inc = myc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULLMASK, inc, o);
        if (lane >= o) inc += y;
      }
      const int total = __shfl_sync(FULLMASK, inc, 31);
      const int excl = inc - myc;
      uint32_t tb = sm.thr[L];
      if (p.qthr && sm.qidx[L] >= 0) tb = min(tb, *((volatile unsigned*)(p.qthr + sm.qidx[L])));
      uint2* base = p.cand + ((size_t)unit * 32 + L) * kWarps * p.B;
      int n = 0;
      for (int i0 = 0; i0 < total; i0 += 32) {
        const int idx = i0 + lane;
        int w = 0;
#pragma unroll
        for (int st = 8; st >= 1; st >>= 1) {
          const int o = __shfl_sync(FULLMASK, excl, (w + st) & 31);
          if (w + st < kWarps && o <= idx) w += st;
        }
        const int wo = __shfl_sync(FULLMASK, excl, w & 31);
        uint2 v = make_uint2(0xffffffffu, 0);
        if (idx < total) v = base[(size_t)w * p.B + (idx - wo)];
        const bool keep = (idx < total) && v.x <= tb;
        const unsigned m = __ballot_sync(FULLMASK, keep);
        __syncwarp();
        if (keep) base[n + __popc(m & ((1u << lane) - 1u))] = v;
        n += __popc(m);
      }
      // exact unit-level top-k of the merged list (it fits the warp's registers):
      // at most ~k survivors per unit and a tight per-query bound for the
      // other units and the finalize prefilter
      constexpr int kCap = kRefreshPer * 32;
      bool tightened = false;
      while (n > kCap) {
        // longer lists: the exact k-th of the first kCap entries bounds the
        // query's k-th distance; filter the rest by it (in place) and repeat
        __syncwarp();
        int nc;
        float nt;
        refresh_buffer(base, kCap, p.k, p.group_mult, p.group_minid, &nc, &nt);
        const uint32_t ntb = __float_as_uint(nt);
        int m = nc;
        for (int i0 = kCap; i0 < n; i0 += 32) {
          const int idx = i0 + lane;
          uint2 v = make_uint2(0xffffffffu, 0);
          if (idx < n) v = base[idx];
          const bool keep = (idx < n) && v.x <= ntb;
          const unsigned mk = __ballot_sync(FULLMASK, keep);
          __syncwarp();
          if (keep) base[m + __popc(mk & ((1u << lane) - 1u))] = v;
          m += __popc(mk);
        }
        __syncwarp();
        tb = min(tb, ntb);
        tightened = true;
        if (m >= n) break;   // no progress (ties): leave the list as it is
        n = m;
      }
      if (n > p.k && n <= kCap) {
        __syncwarp();
        int nc;
        float nt;
        refresh_buffer(base, n, p.k, p.group_mult, p.group_minid, &nc, &nt);
        n = nc;
        tb = min(tb, __float_as_uint(nt));
        tightened = true;
      }
      if (tightened && p.qthr && lane == 0 && sm.qidx[L] >= 0) atomicMin(p.qthr + sm.qidx[L], tb);
      if (lane < kWarps) p.cand_cnt[((size_t)unit * 32 + L) * kWarps + lane] = (lane == 0) ? n : 0;
      if (lane == 0 && p.unit_thr) p.unit_thr[(size_t)unit * 32 + L] = __uint_as_float(tb);
    }
  }
  phase_mark(unit, 4);
}


template <int SS, int MTC, int MODE, int NS = kStreams, bool EX = false>
static cudaError_t launch_scan_t(const ScanParams& p, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(scan_kernel<SS, MTC, MODE, NS, EX>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  scan_kernel<SS, MTC, MODE, NS, EX><<<p.n_units, kThreads, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <int SS>
cudaError_t launch_scan_s(const ScanParams& p, size_t smem, cudaStream_t st) {
  bool uni = true;
  for (int t = 1; t < p.T; ++t) uni = uni && (p.tree[t].MT == p.tree[0].MT);
  const int mt = uni ? p.tree[0].MT : 0;
  if (p.T > 1) {   // per-tree partials + join
    if constexpr (SS != 16) {   // (s = 16 forests have M <= 8 levels of 16 dims: fused)
      if (mt == 8) return launch_scan_t<SS, 8, 1>(p, smem, st);
    }
    return launch_scan_t<SS, 0, 1>(p, smem, st);
  }
  if (p.masked) {  // fused forest
    if constexpr (SS != 60) {
      if (mt == 8) return p.long_ranges ? launch_scan_t<SS, 8, 2, kStreamsLong>(p, smem, st)
                                        : launch_scan_t<SS, 8, 2>(p, smem, st);
    }
    return launch_scan_t<SS, 0, 2>(p, smem, st);
  }
  if (p.gextra) {   // leaf extra byte: 8-level single trees, top-k
    if constexpr (SS == 16 || SS == 0) {
      if (mt == 8 && p.mode == kModeTopk) return launch_scan_t<SS, 8, 0, kStreams, true>(p, smem, st);
    }
    return cudaErrorNotSupported;
  }
  if (mt == 8) return p.long_ranges ? launch_scan_t<SS, 8, 0, kStreamsLong>(p, smem, st)
                                    : launch_scan_t<SS, 8, 0>(p, smem, st);
  if (mt == 4) return launch_scan_t<SS, 4, 0>(p, smem, st);
  return launch_scan_t<SS, 0, 0>(p, smem, st);
}

}  // namespace
}  // namespace et
