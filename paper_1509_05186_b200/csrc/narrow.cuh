// narrow.cuh -- the E-Forest scan for few queries per CTA and codes of 8 < M
// <= 16 bytes (c3: d = 960, M = 16, T = 2 over bytes 0-7 | 8-15, ~7 queries
// per SM).  Included by the scan translation units (one instantiation per s).
//
// With at most 8 queries per CTA the tables of all 16 levels fit shared
// memory when a table row holds 8 queries instead of 32 lanes ([level][k][8]
// fp32 = 8 KB per level, 128 KB in all), so the forest's trees need neither
// per-tree partials nor a join: the distinct full codes (tuples) are scanned
// once in lexicographic order with a per-level lookup mask -- bit l set iff
// l - split[u] >= LCP(tuple t-1, tuple t) over the bytes of the tree u holding
// level l, i.e. each tree's Distance Context carried along the tuple
// sequence, the same reading (A23) as the fused forest of M <= 8 -- and the
// distance is the per-tree partials summed in tree order, ((p_0 + p_1) + ...)
// (reading A13).  A warp's 32 lanes are 4 groups x 8 query
// slots: each group walks its own contiguous stream of tuples, so one warp
// step serves 4 tuples x 8 queries.
#pragma once
#include "scan.cuh"

namespace et {
namespace {

constexpr int kNarrowQ = 8;                              // query slots per CTA (lane & 7)
constexpr int kNarrowG = 32 / kNarrowQ;                  // tuple streams per warp (lane >> 3)
constexpr int kNarrowLevels = 16;
constexpr uint32_t kNarrowLvlBytes = 256u * kNarrowQ * 4u;   // one level's table, [k][8] fp32

// Shared-memory layout of the narrow kernel (byte offsets).
template <int SS>
struct NarrowSmem {
  static constexpr uint32_t pair_bytes = SS * 8u;        // staged query pair [dim][2]
  static constexpr uint32_t lvl_bytes = (kNarrowQ / 2) * pair_bytes;
  static constexpr uint32_t stage = kNarrowLevels * kNarrowLvlBytes;
  static constexpr uint32_t thr = stage + kNarrowLevels * lvl_bytes;
  static constexpr uint32_t recs = thr + 32u * 4u;        // the tuple records, when they fit
  static constexpr uint32_t total = recs;                // + 32 B per tuple (kNarrowSmemRecs)
};
constexpr int kNarrowSmemRecs = 2048;                    // tuples whose records are staged in smem

// Tables of every level for the CTA's <= 8 queries: rounds of 4 levels, kWPL
// warps per level, kR codeword rows per lane; the j-ascending packed FADD2 /
// FFMA2 chains of build_tables_wide8 (same entries bit for bit), codeword
// chunks from the chunk-major copy p.cbt through a register ring; a row's 8
// entries are stored as two 16-byte words.
template <int SS>
__device__ __forceinline__ void narrow_build(const ScanParams& p, uint32_t base) {
  using L = NarrowSmem<SS>;
  static_assert(SS % 4 == 0 && SS <= 64, "narrow build: s % 4 == 0, s <= 64");
  constexpr int NCH = SS / 4, NP = kNarrowQ / 2, kRing = 5;
  const int K = p.K;
  const int lane = lane_id(), warp = warp_id();
  const int lw = warp / kWPL;
  const int row0 = (warp % kWPL) * 32 * kR;
  const bool active = row0 < K;
  float4 c[kRing][kR];
  auto chunk = [&](int l, int r, int jc) -> float4 {
    const int m = p.lsub[l];
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
  const int rounds = (p.M + 3) / 4;
  if (active && lw < p.M) prefill(lw);                    // in flight during the staging wait
  asm volatile("cp.async.wait_all;" ::: "memory");         // this thread's staged copies landed
  __syncthreads();                                        // everyone's
  phase_mark((int)blockIdx.x, 1);
  for (int rd = 0; rd < rounds; ++rd) {
    const int l = rd * 4 + lw;
    if (active && l < p.M) {
      const uint32_t xs = base + L::stage + (uint32_t)l * L::lvl_bytes;
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
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int pi = 0; pi < NP; ++pi) {   // every pair (slots >= nq: stale stage data, never looked up)
            const float4 u = lds4(xs + (uint32_t)pi * L::pair_bytes + (uint32_t)(4 * jc + 2 * h) * 8u);
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
      if (l + 4 < p.M) prefill(l + 4);                    // next round's first chunks in flight
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        const uint32_t row = base + (uint32_t)l * kNarrowLvlBytes + (uint32_t)(row0 + 32 * r + lane) * 32u;
        float q[8];
#pragma unroll
        for (int pi = 0; pi < NP; ++pi) f2unpack(a[pi][r], q[2 * pi], q[2 * pi + 1]);
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" :: "r"(row), "f"(q[0]), "f"(q[1]), "f"(q[2]), "f"(q[3]) : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" :: "r"(row + 16u), "f"(q[4]), "f"(q[5]), "f"(q[6]), "f"(q[7]) : "memory");
      }
    }
  }
}

// Narrow tuple record (host: build_narrow): two uint4 = 16 half-words, half-
// word l = (code byte l) << 5 | lookup-mask bit l, half-word 0 adds
// floor(log2(multiplicity)) (capped at 15) in bits 1..4; levels >= M are 0.
__device__ __forceinline__ uint32_t nrec_hw(const uint4 (&r)[2], int l) {
  const uint4& u = r[l >> 3];
  const uint32_t w = ((l >> 1) & 3) == 0 ? u.x : ((l >> 1) & 3) == 1 ? u.y : ((l >> 1) & 3) == 2 ? u.z : u.w;
  return (l & 1) ? (w >> 16) : (w & 0xffffu);
}

// The tuples [wa, wb) of this warp: lane group g walks [ga, gb), lane slot ql
// is query slot ql.  FS = the level where tree 1 starts (compile time) or 0
// (tree boundaries from p.fsplit at run time).
// recs_s: the records in shared memory (staged at kernel entry) or 0 (global).
template <int FS>
__device__ void narrow_scan(EmitCtx& e, uint32_t base, uint32_t thr_s, uint32_t recs_s, uint32_t wa, uint32_t wb) {
  const ScanParams& p = *e.p;
  const int lane = lane_id();
  const int ql = lane & (kNarrowQ - 1), g = lane / kNarrowQ;
  const uint32_t len = wb - wa;
  const uint32_t ga = wa + (uint32_t)(((uint64_t)len * g) / kNarrowG);
  const uint32_t gb = wa + (uint32_t)(((uint64_t)len * (g + 1)) / kNarrowG);
  const uint32_t steps = (len + kNarrowG - 1) / kNarrowG;   // the longest stream
  const uint4* rec = p.nrec;
  const uint32_t q4 = (uint32_t)ql << 2;
  float v[kNarrowLevels];
#pragma unroll
  for (int l = 0; l < kNarrowLevels; ++l) v[l] = 0.f;
  auto load = [&](uint32_t t, uint4 (&r)[2]) {
    if (t >= gb) { r[0] = make_uint4(0u, 0u, 0u, 0u); r[1] = r[0]; return; }
    if (recs_s) {   // broadcast 16-byte shared loads (8 lanes share one tuple)
      const float4 a = lds4(recs_s + 32u * t), b = lds4(recs_s + 32u * t + 16u);
      r[0] = make_uint4(__float_as_uint(a.x), __float_as_uint(a.y), __float_as_uint(a.z), __float_as_uint(a.w));
      r[1] = make_uint4(__float_as_uint(b.x), __float_as_uint(b.y), __float_as_uint(b.z), __float_as_uint(b.w));
    } else {
      r[0] = __ldg(rec + 2 * (size_t)t); r[1] = __ldg(rec + 2 * (size_t)t + 1);
    }
  };
  uint4 cur[2], nx[2];
  load(ga, nx);
  TopkState& ts = e.ts;
  for (uint32_t s = 0; s < steps; ++s) {
    cur[0] = nx[0]; cur[1] = nx[1];
    load(ga + s + 1, nx);                                  // next record in flight
    const bool ok = ga + s < gb;
    const bool first = (s == 0);
#pragma unroll
    for (int l = 0; l < kNarrowLevels; ++l) {
      const uint32_t hw = nrec_hw(cur, l);
      // levels >= M have half-word 0: never looked up, v stays 0
      if (ok && ((hw & 1u) || (first && l < p.M)))
        v[l] = lds(base + (uint32_t)l * kNarrowLvlBytes + ((hw & 0x1fe0u) | q4));
    }
    float dist;
    if constexpr (FS > 0) {   // two trees split at level FS: p_0 + p_1, each left to right (A13)
      float s0 = v[0], s1 = v[FS];
#pragma unroll
      for (int l = 1; l < FS; ++l) s0 = s0 + v[l];
#pragma unroll
      for (int l = FS + 1; l < kNarrowLevels; ++l) s1 = s1 + v[l];
      dist = s0 + s1;
    } else {
      dist = dc_sum_forest<kNarrowLevels>(v, p.fsplit);
    }
    if (__any_sync(FULLMASK, ok && ts.active && dist <= ts.thr)) {
      const uint32_t bucket = (nrec_hw(cur, 0) >> 1) & 15u;
      const bool em = ok && ts.active && dist <= ts.thr;
      ET_CHECK(!em || ts.cnt < p.B);
      if (em) ts.buf[ts.cnt] = make_uint2(__float_as_uint(dist), ga + s);
      ts.cnt += em ? 1 : 0;
      ts.msum += em ? (1u << bucket) : 0u;
      if (em && (1u << bucket) >= (uint32_t)p.k) ts.thr = dist;   // one group alone bounds the k-th distance
    }
    // every 4 steps: prune full buffers and pool the query's bound in the CTA
    // (a warp walks only ~G / 32 steps, so a lane would otherwise keep its own
    // first bound and leave ~3 candidates per list for the finalize)
    if ((s & 3u) == 3u || s + 1 == steps) {
      refresh_if_needed(e);
      if (ts.active) {
        const unsigned mine = __float_as_uint(ts.thr);
        unsigned old;
        asm volatile("atom.shared.min.u32 %0, [%1], %2;" : "=r"(old) : "r"(thr_s + 4u * (uint32_t)ql), "r"(mine) : "memory");
        ts.thr = __uint_as_float(min(old, mine));
      }
    }
  }
}

// One CTA per chunk of <= 8 queries (S = 1, arithmetic chunking of flatQ):
// stage the queries (cp.async), build the 16 levels' tables, scan the tuples
// (the CTA's 8 warps split them evenly), leave per-(lane, warp) candidate
// lists for the finalize (lists of query slot q: lanes q + 8 g, g < 4).
template <int SS>
__global__ void __launch_bounds__(kThreads, 1) narrow_kernel(const __grid_constant__ ScanParams p) {
  using L = NarrowSmem<SS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  const int chunk = (int)blockIdx.x, unit = chunk;
  const int lane = lane_id(), warp = warp_id();
  const int ql = lane & (kNarrowQ - 1);
  phase_mark(unit, 0);
  const int64_t s0 = (int64_t)chunk * p.flatQ / p.n_units, s1 = (int64_t)(chunk + 1) * p.flatQ / p.n_units;
  const int nq = (int)(s1 - s0);
  ET_CHECK(nq <= kNarrowQ);
  for (int e = threadIdx.x; e < p.M * kNarrowQ * SS; e += kThreads) {   // (level, slot, dim)
    const int l = e / (kNarrowQ * SS), r = e - l * (kNarrowQ * SS);
    const int i = r / SS, j = r - i * SS;
    if (i >= nq) continue;
    const float* src = p.queries + (size_t)(s0 + i) * p.d + (size_t)p.lsub[l] * SS + j;
    const uint32_t dst = base + L::stage + (uint32_t)l * L::lvl_bytes + (uint32_t)(i >> 1) * L::pair_bytes +
                         (uint32_t)j * 8u + (uint32_t)(i & 1) * 4u;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src) : "memory");
  }
  // few tuples (c3: 541): every record into shared memory now, in flight
  // during the table build (the scan then reads them with broadcast LDS)
  const bool srec = p.n_groups <= kNarrowSmemRecs;
  if (srec) {
    const char* src = reinterpret_cast<const char*>(p.nrec);
    for (int i = threadIdx.x; i < 2 * p.n_groups; i += kThreads)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(base + L::recs + 16u * (uint32_t)i),
                   "l"(src + 16 * (size_t)i) : "memory");
  }
  unsigned* thr = reinterpret_cast<unsigned*>(smem_raw + L::thr);
  if (threadIdx.x < 32) thr[lane] = 0x7f800000u;
  narrow_build<SS>(p, base);   // (waits for the staged queries after its first codeword loads)
  __syncthreads();
  phase_mark(unit, 5);

  EmitCtx e;
  e.p = &p;
  e.unit = unit;
  e.chunk = chunk;
  e.q = (ql < nq) ? (int)(s0 + ql) : -1;
  e.part = nullptr;
  e.ts.active = ql < nq;
  e.ts.thr = e.ts.active ? __int_as_float(0x7f800000) : -1.0f;
  e.ts.cnt = 0;
  e.ts.msum = 0;
  e.ts.warp_buf = p.cand + ((size_t)unit * 32 * kWarps + warp) * p.B;
  e.ts.buf = e.ts.warp_buf + (size_t)lane * kWarps * p.B;
  const uint64_t G = (uint64_t)p.n_groups;
  const uint32_t wa = (uint32_t)((G * warp) / kWarps), wb = (uint32_t)((G * (warp + 1)) / kWarps);
  const uint32_t recs_s = srec ? base + L::recs : 0u;
  if (wa < wb) {
    if (p.fsplit == (1u << 8)) narrow_scan<8>(e, base, base + L::thr, recs_s, wa, wb);
    else narrow_scan<0>(e, base, base + L::thr, recs_s, wa, wb);
  }
  __syncthreads();
  phase_mark(unit, 3);
  if (warp == 0 && lane < nq && p.qthr) p.qthr[s0 + lane] = thr[lane];   // the query's only unit
  p.cand_cnt[((size_t)unit * 32 + lane) * kWarps + warp] = e.ts.cnt;
  if (warp == 0 && p.unit_thr) p.unit_thr[(size_t)unit * 32 + lane] = __uint_as_float(thr[ql]);
  phase_mark(unit, 4);
}

template <int SS>
cudaError_t launch_narrow_s(const ScanParams& p, cudaStream_t st) {
  const size_t smem = NarrowSmem<SS>::total + (p.n_groups <= kNarrowSmemRecs ? 32u * (size_t)p.n_groups : 0u);
  cudaError_t e = cudaFuncSetAttribute(narrow_kernel<SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  narrow_kernel<SS><<<p.n_units, kThreads, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace
}  // namespace et
