// kernels.cu -- sm_100a kernels of libetree (E-Tree / E-Forest ADC, arXiv 1509.05186).
//
// K1  lut_kernel            distance tables, materialised [Q][M][K]
// K2  scan_kernel           fused tables + Distance-Context scan + emit
//                           (full output P:244/P:257, or top-k candidates), E-Forest
//                           join for T >= 2
// K4  finalize_kernel       exact top-k by (distance, id) with leaf multiplicities
//     gather_full_kernel    out[q][slot] = leaf distance of slot's leaf (full output)
// K5  flat_adc_kernel       naive ADC comparison
// K7  merge_kernel          merge G shard top-k lists
// K8  encode_kernel         PQ encode argmin, residual variant for IVF
//     assign_kernel         nearest coarse centroid
//
// Design notes are in DESIGN.md §4-5; every floating-point table entry is the
// direct difference sum_j (x_j - c_j)^2 accumulated in fp32 with j ascending.
#include "common.cuh"

namespace et {

cudaError_t launch_scan_16(const ScanParams& p, size_t smem, cudaStream_t st);
cudaError_t launch_scan_60(const ScanParams& p, size_t smem, cudaStream_t st);
cudaError_t launch_scan_0(const ScanParams& p, size_t smem, cudaStream_t st);

// K2 dispatch by sub-vector length (template instantiations live in scan_s*.cu)
cudaError_t launch_narrow_16(const ScanParams& p, cudaStream_t st);
cudaError_t launch_narrow_60(const ScanParams& p, cudaStream_t st);
bool narrow_supported(int s) { return s == 16 || s == 60; }
cudaError_t launch_narrow(const ScanParams& p, cudaStream_t st) {
  if (p.n_units <= 0) return cudaSuccess;
  return p.s == 60 ? launch_narrow_60(p, st) : launch_narrow_16(p, st);
}

cudaError_t launch_scan(const ScanParams& p, int MTmax, cudaStream_t st) {
  if (p.n_units <= 0) return cudaSuccess;
  const size_t smem = scan_smem(MTmax).total;
  const bool v4 = (p.luts == nullptr) && (p.d % 4 == 0) && p.vec4;
  switch (v4 ? p.s : 0) {
    case 16: return launch_scan_16(p, smem, st);
    case 60: return launch_scan_60(p, smem, st);
    default: return launch_scan_0(p, smem, st);
  }
}


// ---------------------------------------------------------------------------
// warp bitonic sort of n (power of two, <= 512) u64 keys in shared memory
// ---------------------------------------------------------------------------
__device__ void warp_bitonic_sort(unsigned long long* a, int n) {
  const int lane = lane_id();
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncwarp();
      for (int i = lane; i < n / 2; i += 32) {
        const int lo = ((i & ~(stride - 1)) << 1) | (i & (stride - 1));   // stride is a power of two
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const unsigned long long x = a[lo], y = a[hi];
        if ((x > y) == up) { a[lo] = y; a[hi] = x; }
      }
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// K4: finalize -- exact top-k per query over the candidates of all its units
// ---------------------------------------------------------------------------
constexpr int kFinCap = 512;   // candidates staged in shared memory per warp

struct FinWarp {                // one warp's finalize scratch (shared memory)
  unsigned long long stage[kTopkMax];
  unsigned long long xs[kTopkMax];   // slow-path (distance, id) keys
  uint32_t key[kFinCap];
  uint32_t grp[kFinCap];
  uint32_t mul[kFinCap];
  uint32_t hist[256];
  int nstage;
  uint32_t tied_g;
  uint32_t pad[2];
};

// Slots (chunk*32 + lane) of query q: explicit (IVF: one per probe) or, for the
// flat plan, the query's position in the arithmetic chunking.
__device__ __forceinline__ int fin_s0(const FinParams& p, int64_t q) { return p.flat_nchunks ? 0 : p.qslot_off[q]; }
__device__ __forceinline__ int fin_s1(const FinParams& p, int64_t q) { return p.flat_nchunks ? 1 : p.qslot_off[q + 1]; }
__device__ __forceinline__ int fin_slot(const FinParams& p, int64_t q, int j) {
  if (p.flat_nchunks) {   // chunk c holds queries [floor(cQ/n), floor((c+1)Q/n))
    // q's chunk is the smallest c with floor((c+1)Q/n) > q, i.e.
    // c = ceil((q+1) n / Q) - 1 = floor(((q+1) n - 1) / Q)
    const uint64_t n = (uint64_t)p.flat_nchunks, Q = (uint64_t)p.Q, qu = (uint64_t)q;
    const uint64_t c = ((qu + 1) * n - 1) / Q;
    return (int)(c * 32 + (qu - c * Q / n));
  }
  return __ldg(p.qslot + j);
}

// Candidate list li of query q, 0 <= li < (s1 - s0) * S * lpu: one per
// (slot, leaf segment, scan warp).  Its count is cand_cnt[list], its entries
// cand[list * B ...] (the scan kernel's per-warp, per-lane buffers).
__device__ __forceinline__ size_t fin_list(const FinParams& p, int64_t q, int s0, int li) {
  const int lpg = p.lpu * p.lgroups;          // lists per (unit, slot)
  const int per = p.S * lpg;
  const int j = li / per, r = li - j * per;
  const int sg = r / lpg, r2 = r - sg * lpg;
  const int g = r2 / p.lpu, w = r2 - g * p.lpu;
  const int slot = fin_slot(p, q, s0 + j);
  return ((size_t)((slot >> 5) * p.S + sg) * 32 + (slot & 31) + 8 * g) * kWarps + w;
}

// Enumerates the candidates of query q: smem copy when they fit, else global.
// f(key, group, multiplicity) is called once per candidate by the owning lane.
// Each (slot, segment) unit list holds cand_cnt[unit*32+lane] entries at
// cand + (unit*32 + lane) * kWarps * B (compacted by the scan kernel).
struct CandSrc {
  const FinParams* p;
  int64_t q;
  int s0, s1;
  bool in_smem;
  int n;               // staged count (smem)
  const uint32_t* key;
  const uint32_t* grp;
  const uint32_t* mul;
  float thr;           // prefilter: candidates above every unit's final threshold are dead
  template <class F>
  __device__ void each(F f) const {
    const int lane = lane_id();
    if (in_smem) {
      for (int i = lane; i < n; i += 32) f(key[i], grp[i], mul[i]);
      return;
    }
    // 32 lists per round: counts loaded in parallel (lane = list), then the
    // round's entries spread over the lanes (binary search on the prefix)
    const uint32_t tb = __float_as_uint(thr);
    const int nl = (s1 - s0) * p->S * p->lpu * p->lgroups;
    for (int l0 = 0; l0 < nl; l0 += 32) {
      const int li = l0 + lane;
      size_t ul = 0;
      int myc = 0;
      if (li < nl) {
        ul = fin_list(*p, q, s0, li);
        myc = __ldcg(p->cand_cnt + ul);
      }
      int inc = myc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULLMASK, inc, o);
        if (lane >= o) inc += y;
      }
      const int total = __shfl_sync(FULLMASK, inc, 31);
      const int excl = inc - myc;
      for (int i0 = 0; i0 < total; i0 += 32) {
        const int idx = i0 + lane;
        int w = 0;
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1) {
          const int o = __shfl_sync(FULLMASK, excl, (w + st) & 31);
          if (w + st < 32 && o <= idx) w += st;
        }
        const int wo = __shfl_sync(FULLMASK, excl, w);
        const unsigned long long ulw = __shfl_sync(FULLMASK, (unsigned long long)ul, w);
        if (idx < total) {
          const uint2 v = p->cand[ulw * p->B + (idx - wo)];
          if (v.x <= tb) f(v.x, v.y, __ldg(p->group_mult + v.y));
        }
      }
    }
  }
};

// Exact top-k of query q from the candidates of all its units (one warp).
__device__ void finalize_query(const FinParams& p, FinWarp& fw, int64_t q) {
  const float* unit_thr = p.unit_thr;
  const int lane = lane_id();
  const int k = p.k;
  const int s0 = fin_s0(p, q), s1 = fin_s1(p, q);

  // 1. threshold prefilter: min over the query's units of their final thresholds
  float thr = __int_as_float(0x7f800000);
  if (p.qthr) {   // every unit of the query folded its final threshold into qthr
    thr = __uint_as_float(__ldcg(p.qthr + q));
  } else if (unit_thr) {
    for (int j = s0; j < s1; ++j) {
      const int slot = fin_slot(p, q, j);
      const int chunk = slot >> 5, ln = slot & 31;
      for (int sg = lane; sg < p.S; sg += 32)
        thr = fminf(thr, __ldcg(unit_thr + (size_t)(chunk * p.S + sg) * 32 + ln));
    }
    for (int o = 16; o > 0; o >>= 1) thr = fminf(thr, __shfl_xor_sync(FULLMASK, thr, o));
  }
  const uint32_t tb = __float_as_uint(thr);

  // 2. stage candidates (<= thr) into shared memory, with their multiplicities:
  //    the query's unit lists, up to 32 lists per round loaded in parallel
  int n = 0;
  bool overflow = false;
  {
    uint32_t* K_ = fw.key;
    uint32_t* G_ = fw.grp;
    uint32_t* U_ = fw.mul;
    const int nl = (s1 - s0) * p.S * p.lpu * p.lgroups;
    for (int l0 = 0; l0 < nl && !overflow; l0 += 32) {
      const int li = l0 + lane;
      size_t ul = 0;
      int myc = 0;
      if (li < nl) {
        ul = fin_list(p, q, s0, li);
        myc = __ldcg(p.cand_cnt + ul);
      }
      int inc = myc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULLMASK, inc, o);
        if (lane >= o) inc += y;
      }
      const int total = __shfl_sync(FULLMASK, inc, 31);
      const int excl = inc - myc;
      for (int i0 = 0; i0 < total; i0 += 32) {
        const int idx = i0 + lane;
        int w = 0;
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1) {
          const int o = __shfl_sync(FULLMASK, excl, (w + st) & 31);
          if (w + st < 32 && o <= idx) w += st;
        }
        const int wo = __shfl_sync(FULLMASK, excl, w);
        const unsigned long long ulw = __shfl_sync(FULLMASK, (unsigned long long)ul, w);
        uint2 v = make_uint2(0xffffffffu, 0);
        ET_CHECK(idx >= total || idx - wo < p.B);
        if (idx < total) v = p.cand[ulw * p.B + (idx - wo)];
        const bool keep = (idx < total) && v.x <= tb;
        const unsigned m = __ballot_sync(FULLMASK, keep);
        const int pos = n + __popc(m & ((1u << lane) - 1u));
        if (keep && pos < kFinCap) { K_[pos] = v.x; G_[pos] = v.y; U_[pos] = __ldg(p.group_mult + v.y); }
        n += __popc(m);
      }
      if (n > kFinCap) overflow = true;
    }
  }
  __syncwarp();
  CandSrc src;
  src.p = &p; src.q = q; src.s0 = s0; src.s1 = s1; src.in_smem = !overflow; src.n = n;
  src.key = fw.key; src.grp = fw.grp; src.mul = fw.mul; src.thr = thr;

  // 3. weighted radix select: t = smallest distance with cumulative multiplicity >= k
  uint32_t* hist = fw.hist;
  uint32_t prefix = 0, pmask = 0, need = (uint32_t)k;
  bool all = false;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = lane; i < 256; i += 32) hist[i] = 0;
    __syncwarp();
    src.each([&](uint32_t key, uint32_t g, uint32_t mu) {
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], mu);
    });
    __syncwarp();
    uint32_t h[8], loc = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) { h[r] = hist[lane * 8 + r]; loc += h[r]; }
    uint32_t inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULLMASK, inc, o);
      if (lane >= o) inc += y;
    }
    const uint32_t tot = __shfl_sync(FULLMASK, inc, 31);
    if (tot < need) { all = true; break; }   // fewer than k ids in total (only possible in pass 0)
    const uint32_t excl = inc - loc;
    const bool mine = excl < need && need <= inc;
    const unsigned who = __ballot_sync(FULLMASK, mine);
    const int L = __ffs(who) - 1;
    uint32_t digit = 0, before = 0;
    if (lane == L) {
      uint32_t c = excl;
      for (int r = 0; r < 8; ++r) {
        if (c + h[r] >= need) { digit = lane * 8 + r; before = c; break; }
        c += h[r];
      }
    }
    digit = __shfl_sync(FULLMASK, digit, L);
    before = __shfl_sync(FULLMASK, before, L);
    need -= before;
    prefix |= digit << shift;
    pmask |= 255u << shift;
  }
  const uint32_t t = all ? 0xffffffffu : prefix;

  // 4. output.  Groups with distance < t contribute all their ids (< k in
  //    total); among groups tied at t the R = k - mult(< t) smallest ids.
  //    Fast path: sort only the (few) groups < t by distance; when no two of
  //    them share a distance, each group's ids (ascending) are already in
  //    (distance, id) order and are written out directly.
  unsigned long long* stage = fw.stage;
  if (lane == 0) fw.nstage = 0;
  __syncwarp();
  uint32_t slt = 0, ntied = 0;
  src.each([&](uint32_t key, uint32_t g, uint32_t mu) {
    if (key < t || all) {
      slt += mu;
      const int pos = atomicAdd(&fw.nstage, 1);
      if (pos < kTopkMax) stage[pos] = ((unsigned long long)key << 32) | g;
    } else if (key == t) {
      ntied += 1;
      fw.tied_g = g;
    }
  });
  slt = __reduce_add_sync(FULLMASK, slt);
  ntied = __reduce_add_sync(FULLMASK, ntied);
  __syncwarp();
  const int ng = min(fw.nstage, kTopkMax);   // groups < t (< k of them)
  {
    int np2 = 32;
    while (np2 < ng) np2 <<= 1;
    for (int i = ng + lane; i < np2; i += 32) stage[i] = ~0ull;
    __syncwarp();
    if (ng > 1) warp_bitonic_sort(stage, np2);
  }
  // exact distance ties between different groups < t need an id merge (slow path)
  bool dup = false;
  for (int i = lane; i + 1 < ng; i += 32) dup |= (stage[i] >> 32) == (stage[i + 1] >> 32);
  dup = __any_sync(FULLMASK, dup);
  float* od = p.out_dist + (size_t)q * k;
  int32_t* oi = p.out_ids + (size_t)q * k;
  int written = 0;
  if (!dup) {
    // prefix offsets of the sorted groups' multiplicities, 32 groups at a time
    for (int g0 = 0; g0 < ng; g0 += 32) {
      const int gi = g0 + lane;
      uint32_t key = 0, g = 0, mu = 0, o0 = 0;
      if (gi < ng) {
        key = (uint32_t)(stage[gi] >> 32);
        g = (uint32_t)(stage[gi] & 0xffffffffu);
        o0 = __ldg(p.group_off + g);
        mu = __ldg(p.group_off + g + 1) - o0;
      }
      uint32_t inc = mu;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULLMASK, inc, o);
        if (lane >= o) inc += y;
      }
      const uint32_t base = (uint32_t)written + inc - mu;
      const int cnt = min(32, ng - g0);
      for (int j = 0; j < cnt; ++j) {   // lanes copy group j's ids
        const uint32_t bj = __shfl_sync(FULLMASK, base, j);
        const uint32_t mj = __shfl_sync(FULLMASK, mu, j);
        const uint32_t oj = __shfl_sync(FULLMASK, o0, j);
        const float dj = __uint_as_float(__shfl_sync(FULLMASK, key, j));
        for (uint32_t r = lane; r < mj; r += 32)
          if (bj + r < (uint32_t)k) { od[bj + r] = dj; oi[bj + r] = __ldg(p.ids + oj + r); }
      }
      written += (int)__shfl_sync(FULLMASK, inc, 31);
    }
  } else {
    // slow path: expand every group < t into (distance, id) keys and sort them
    __syncwarp();
    int n_ids = 0;
    for (int gi = 0; gi < ng; ++gi) {
      const uint32_t key = (uint32_t)(stage[gi] >> 32), g = (uint32_t)(stage[gi] & 0xffffffffu);
      const uint32_t o0 = __ldg(p.group_off + g), mu = __ldg(p.group_off + g + 1) - o0;
      unsigned long long* xs = fw.xs;
      for (uint32_t r = lane; r < mu; r += 32)
        if (n_ids + (int)r < kTopkMax)
          xs[n_ids + r] = ((unsigned long long)key << 32) | (uint32_t)__ldg(p.ids + o0 + r);
      n_ids += (int)mu;
    }
    __syncwarp();
    n_ids = min(n_ids, kTopkMax);
    int np2 = 32;
    while (np2 < n_ids) np2 <<= 1;
    unsigned long long* xs = fw.xs;
    for (int i = n_ids + lane; i < np2; i += 32) xs[i] = ~0ull;
    __syncwarp();
    warp_bitonic_sort(xs, np2);
    for (int i = lane; i < n_ids && i < k; i += 32) {
      od[i] = __uint_as_float((uint32_t)(xs[i] >> 32));
      oi[i] = (int32_t)(uint32_t)(xs[i] & 0xffffffffu);
    }
    written = n_ids;
  }
  written = min(written, k);
  __syncwarp();
  if (!all && ntied == 1) {
    // common case: one group holds the k-th distance -> its R smallest ids
    const uint32_t R = (uint32_t)k - slt;
    const uint32_t g = fw.tied_g;
    const uint32_t o0 = __ldg(p.group_off + g), o1 = __ldg(p.group_off + g + 1);
    const uint32_t take = min(R, o1 - o0);
    for (uint32_t i = lane; i < take; i += 32) {
      od[written + i] = __uint_as_float(t);
      oi[written + i] = __ldg(p.ids + o0 + i);
    }
    written += (int)take;
  } else if (!all && ntied > 1) {
    const uint32_t R = (uint32_t)k - slt;
    // tau: R-th smallest minid among tied groups (only groups with minid <= tau matter)
    uint32_t tau = 0xffffffffu;
    if (ntied > R) {
      uint32_t w = 0;
      for (int bit = 31; bit >= 0; --bit) {
        const uint32_t cand = w | ((1u << bit) - 1u);
        uint32_t c = 0;
        src.each([&](uint32_t key, uint32_t g, uint32_t mu) {
          if (key == t && (uint32_t)__ldg(p.group_minid + g) <= cand) ++c;
        });
        c = __reduce_add_sync(FULLMASK, c);
        if (c < R) w |= (1u << bit);
      }
      tau = w;
    }
    // sigma: R-th smallest id of the union of those groups' ids
    auto count_le = [&](uint32_t v) {
      uint32_t c = 0;
      src.each([&](uint32_t key, uint32_t g, uint32_t mu) {
        if (key != t || (uint32_t)__ldg(p.group_minid + g) > tau) return;
        uint32_t lo = __ldg(p.group_off + g), hi = lo + mu;
        const uint32_t o0 = lo;
        while (lo < hi) {   // ids ascending within a group
          const uint32_t mid = (lo + hi) >> 1;
          if ((uint32_t)__ldg(p.ids + mid) <= v) lo = mid + 1; else hi = mid;
        }
        c += lo - o0;
      });
      return __reduce_add_sync(FULLMASK, c);
    };
    uint32_t sigma = 0xffffffffu;
    if (count_le(0xfffffffeu) > R) {
      uint32_t w = 0;
      for (int bit = 31; bit >= 0; --bit) {
        const uint32_t cand = w | ((1u << bit) - 1u);
        if (count_le(cand) < R) w |= (1u << bit);
      }
      sigma = w;
    }
    if (lane == 0) fw.nstage = 0;
    __syncwarp();
    src.each([&](uint32_t key, uint32_t g, uint32_t mu) {
      if (key != t || (uint32_t)__ldg(p.group_minid + g) > tau) return;
      const uint32_t o0 = __ldg(p.group_off + g);
      for (uint32_t o = 0; o < mu; ++o) {
        const uint32_t id = (uint32_t)__ldg(p.ids + o0 + o);
        if (id > sigma) break;
        const int pos = atomicAdd(&fw.nstage, 1);
        if (pos < kTopkMax) stage[pos] = id;
      }
    });
    __syncwarp();
    const int nt = min(fw.nstage, (int)R);
    int np2 = 32;
    while (np2 < fw.nstage && np2 < kTopkMax) np2 <<= 1;
    for (int i = fw.nstage + lane; i < np2; i += 32) stage[i] = ~0ull;
    __syncwarp();
    warp_bitonic_sort(stage, np2);
    for (int i = lane; i < nt && written + i < k; i += 32) {
      od[written + i] = __uint_as_float(t);
      oi[written + i] = (int32_t)(uint32_t)stage[i];
    }
    written += nt;
  }
  written = min(written, k);
  for (int i = written + lane; i < k; i += 32) {
    od[i] = __int_as_float(0x7f800000);
    oi[i] = -1;
  }
}


__global__ void __launch_bounds__(kFinWarps * 32) finalize_kernel(const __grid_constant__ FinParams p) {
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  FinWarp* fw = reinterpret_cast<FinWarp*>(fsm_raw);
  const int64_t q = (int64_t)blockIdx.x * kFinWarps + warp_id();
  if (q >= p.Q) return;
  finalize_query(p, fw[warp_id()], q);
}

// ---------------------------------------------------------------------------
// K4 fast path: the same exact top-k, with the query's surviving candidates
// (<= kFastCap) held in registers -- no shared memory, so many warps per SM
// hide the few dependent global loads.  It decides the query only when every
// selected group has a distinct distance (then each group's ascending ids are
// already in (distance, id) order); otherwise -- or with more candidates --
// the warp runs the shared-memory slow path (finalize_query) under a CTA lock.
// ---------------------------------------------------------------------------
constexpr int kFastCap = 64;       // 2 candidates per lane
constexpr int kFastWarps = 8;

// Ascending bitonic sort of 64 keys held as element e = r * 32 + lane in register r.
__device__ __forceinline__ void bitonic64(unsigned long long& a0, unsigned long long& a1) {
  const int lane = lane_id();
#pragma unroll
  for (int size = 2; size <= 64; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride == 32) {   // size == 64: partner is the other register of this lane
        const unsigned long long x = a0, y = a1;
        if (x > y) { a0 = y; a1 = x; }
      } else {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          unsigned long long& a = r ? a1 : a0;
          const int e = r * 32 + lane;
          const unsigned long long o = __shfl_xor_sync(FULLMASK, a, stride);
          const bool up = (e & size) == 0;
          const bool lower = (e & stride) == 0;
          a = (lower == up) ? (a < o ? a : o) : (a > o ? a : o);
        }
      }
    }
  }
}

// Slow path inside the fast kernel: the CTA's one FinWarp scratch, taken under
// a CTA lock (rare: more than kFastCap candidates or exact distance ties).
__device__ __noinline__ void finalize_locked(const FinParams& p, int64_t q) {
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  FinWarp* fw = reinterpret_cast<FinWarp*>(fsm_raw + 16);
  int* lock = reinterpret_cast<int*>(fsm_raw);
  if (lane_id() == 0) while (atomicCAS(lock, 0, 1) != 0) __nanosleep(64);
  __syncwarp();
  __threadfence_block();
  finalize_query(p, *fw, q);
  __threadfence_block();
  __syncwarp();
  if (lane_id() == 0) atomicExch(lock, 0);
}

// Ascending bitonic sort of 32 keys, one per lane.
__device__ __forceinline__ void bitonic32(unsigned long long& a) {
  const int lane = lane_id();
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const unsigned long long o = __shfl_xor_sync(FULLMASK, a, stride);
      const bool up = (lane & size) == 0 || size == 32;
      const bool lower = (lane & stride) == 0;
      a = (lower == up) ? (a < o ? a : o) : (a > o ? a : o);
    }
  }
}

// One query, one warp.  own_fw: a private slow-path scratch, or null (the
// CTA's shared one, taken under a lock).
__device__ __forceinline__ void finalize_fast_query(const FinParams& p, int64_t q, FinWarp* own_fw) {
  const int lane = lane_id();
  const int k = p.k;
  const int s0 = fin_s0(p, q), s1 = fin_s1(p, q);

  // 1. threshold prefilter (as the slow path)
  float thr = __int_as_float(0x7f800000);
  if (p.qthr) {
    thr = __uint_as_float(__ldcg(p.qthr + q));
  } else if (p.unit_thr) {
    for (int j = s0; j < s1; ++j) {
      const int slot = fin_slot(p, q, j);
      const int chunk = slot >> 5, ln = slot & 31;
      for (int sg = lane; sg < p.S; sg += 32)
        thr = fminf(thr, __ldcg(p.unit_thr + (size_t)(chunk * p.S + sg) * 32 + ln));
    }
    for (int o = 16; o > 0; o >>= 1) thr = fminf(thr, __shfl_xor_sync(FULLMASK, thr, o));
  }
  const uint32_t tb = __float_as_uint(thr);

  // 2. gather the candidates <= thr into registers: position i -> lane i & 31, register i >> 5
  uint2 r0 = make_uint2(0xffffffffu, 0), r1 = make_uint2(0xffffffffu, 0);
  int n = 0;
  bool overflow = false;
  const int nl = (s1 - s0) * p.S * p.lpu * p.lgroups;
  for (int l0 = 0; l0 < nl && !overflow; l0 += 32) {
    const int li = l0 + lane;
    size_t ul = 0;
    int myc = 0;
    if (li < nl) {
      ul = fin_list(p, q, s0, li);
      myc = __ldcg(p.cand_cnt + ul);
    }
    int inc = myc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULLMASK, inc, o);
      if (lane >= o) inc += y;
    }
    const int total = __shfl_sync(FULLMASK, inc, 31);
    const int excl = inc - myc;
    constexpr int kRounds = 4;   // candidate loads of four rounds in flight at once
    for (int i00 = 0; i00 < total && !overflow; i00 += 32 * kRounds) {
      uint2 vv[kRounds];
      const int live = (total - i00 + 31) >> 5;   // rounds with candidates (warp-uniform)
#pragma unroll
      for (int rr = 0; rr < kRounds; ++rr) {
        vv[rr] = make_uint2(0xffffffffu, 0);
        if (rr >= live) continue;                  // (few candidates: one round, not four)
        const int idx = i00 + rr * 32 + lane;
        int w = 0;
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1) {
          const int o = __shfl_sync(FULLMASK, excl, (w + st) & 31);
          if (w + st < 32 && o <= idx) w += st;
        }
        const int wo = __shfl_sync(FULLMASK, excl, w);
        const unsigned long long ulw = __shfl_sync(FULLMASK, (unsigned long long)ul, w);
        ET_CHECK(idx >= total || idx - wo < p.B);
        vv[rr] = (idx < total) ? p.cand[ulw * p.B + (idx - wo)] : make_uint2(0xffffffffu, 0);
      }
#pragma unroll
      for (int rr = 0; rr < kRounds; ++rr) {
        if (rr >= live) break;
        const int idx = i00 + rr * 32 + lane;
        const uint2 v = vv[rr];
        const bool keep = (idx < total) && v.x <= tb;
        const unsigned m = __ballot_sync(FULLMASK, keep);
        const int c = __popc(m);
        if (n + c > kFastCap) { overflow = true; break; }
        // lane L receives the r-th kept entry, r = (L - n) mod 32, at position n + r
        const int r = (lane - n) & 31;
        const int src = (r < c) ? (int)__fns(m, 0, r + 1) : 0;
        const uint32_t vx = __shfl_sync(FULLMASK, v.x, src);
        const uint32_t vy = __shfl_sync(FULLMASK, v.y, src);
        if (r < c) {
          if (((n + r) >> 5) == 0) r0 = make_uint2(vx, vy); else r1 = make_uint2(vx, vy);
        }
        n += c;
      }
    }
  }
  if (overflow) {
    if (own_fw) finalize_query(p, *own_fw, q); else finalize_locked(p, q);
    return;
  }

  // 3. offsets / multiplicities of the held groups (one dependent load)
  uint32_t o0a = 0, mua = 0, o0b = 0, mub = 0;
  if (lane < n) { o0a = __ldg(p.group_off + r0.y); mua = __ldg(p.group_off + r0.y + 1) - o0a; }
  if (32 + lane < n) { o0b = __ldg(p.group_off + r1.y); mub = __ldg(p.group_off + r1.y + 1) - o0b; }

  // 4. sort by (distance, position); unused positions sort last
  unsigned long long a0 = ((unsigned long long)r0.x << 32) | (uint32_t)lane;
  unsigned long long a1 = ((unsigned long long)r1.x << 32) | (uint32_t)(32 + lane);
  if (lane >= n) a0 = ~0ull;
  if (32 + lane >= n) a1 = ~0ull;
  if (n > 32) bitonic64(a0, a1);
  else if (n > 1) bitonic32(a0);
  auto payload = [&](unsigned long long a, uint32_t& off, uint32_t& mu) {
    const uint32_t pos = (uint32_t)(a & 63u);
    const uint32_t hl = pos & 31u;
    const uint32_t oa = __shfl_sync(FULLMASK, o0a, hl), ob = __shfl_sync(FULLMASK, o0b, hl);
    const uint32_t ma = __shfl_sync(FULLMASK, mua, hl), mb = __shfl_sync(FULLMASK, mub, hl);
    off = (pos >> 5) ? ob : oa;
    mu = (a == ~0ull) ? 0u : ((pos >> 5) ? mb : ma);
  };
  uint32_t offA, muA, offB, muB;
  payload(a0, offA, muA);
  payload(a1, offB, muB);
  uint32_t cA = muA, cB = muB;   // inclusive prefix of multiplicities, sorted order
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t ya = __shfl_up_sync(FULLMASK, cA, o), yb = __shfl_up_sync(FULLMASK, cB, o);
    if (lane >= o) { cA += ya; cB += yb; }
  }
  cB += __shfl_sync(FULLMASK, cA, 31);
  // last selected element: the first with cumulative multiplicity >= k (else all n)
  const unsigned hitA = __ballot_sync(FULLMASK, lane < n && cA >= (uint32_t)k);
  const unsigned hitB = __ballot_sync(FULLMASK, 32 + lane < n && cB >= (uint32_t)k);
  const int last = hitA ? (__ffs(hitA) - 1) : (hitB ? 32 + __ffs(hitB) - 1 : n - 1);
  // an exact distance tie among the selected elements, or between the last one
  // and the next, needs the id-level merge of the slow path
  const uint32_t dA = (uint32_t)(a0 >> 32), dB = (uint32_t)(a1 >> 32);
  const uint32_t dA_next = __shfl_down_sync(FULLMASK, dA, 1);
  const uint32_t dB_first = __shfl_sync(FULLMASK, dB, 0);
  const uint32_t dB_next = __shfl_down_sync(FULLMASK, dB, 1);
  const uint32_t nA = (lane == 31) ? dB_first : dA_next;
  const bool tieA = (lane <= last) && (lane + 1 < n) && nA == dA;
  const bool tieB = (32 + lane <= last) && (32 + lane + 1 < n) && lane < 31 && dB_next == dB;
  if (__any_sync(FULLMASK, tieA || tieB)) {
    if (own_fw) finalize_query(p, *own_fw, q); else finalize_locked(p, q);
    return;
  }

  // 5. output: the selected groups in distance order, ids ascending within each
  float* od = p.out_dist + (size_t)q * k;
  int32_t* oi = p.out_ids + (size_t)q * k;
  for (int e = 0; e <= last; ++e) {
    const int r = e >> 5, L = e & 31;
    const uint32_t d = __shfl_sync(FULLMASK, r ? dB : dA, L);
    const uint32_t off = __shfl_sync(FULLMASK, r ? offB : offA, L);
    const uint32_t mu = __shfl_sync(FULLMASK, r ? muB : muA, L);
    const uint32_t cum = __shfl_sync(FULLMASK, r ? cB : cA, L);
    const uint32_t base = cum - mu;
    const uint32_t take = min(mu, (uint32_t)k - base);
    for (uint32_t i = lane; i < take; i += 32) {
      od[base + i] = __uint_as_float(d);
      oi[base + i] = __ldg(p.ids + off + i);
    }
  }
  uint32_t written = 0;
  if (last >= 0) written = __shfl_sync(FULLMASK, (last >> 5) ? cB : cA, last & 31);
  written = min(written, (uint32_t)k);
  for (uint32_t i = written + lane; i < (uint32_t)k; i += 32) {
    od[i] = __int_as_float(0x7f800000);
    oi[i] = -1;
  }
}

__global__ void __launch_bounds__(kFastWarps * 32, 6) finalize_fast_kernel(const __grid_constant__ FinParams p) {
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  if (threadIdx.x == 0) *reinterpret_cast<int*>(fsm_raw) = 0;
  __syncthreads();
  const int64_t q = (int64_t)blockIdx.x * kFastWarps + warp_id();
  if (q >= p.Q) return;
  finalize_fast_query(p, q, nullptr);
}

cudaError_t launch_finalize(const FinParams& p, cudaStream_t st) {
  if (p.Q <= 0) return cudaSuccess;
  if (p.fast) {
    const size_t smem = sizeof(FinWarp) + 16;
    cudaError_t e = cudaFuncSetAttribute(finalize_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    finalize_fast_kernel<<<(unsigned)((p.Q + kFastWarps - 1) / kFastWarps), kFastWarps * 32, smem, st>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  const size_t smem = sizeof(FinWarp) * kFinWarps;
  cudaError_t e = cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)((p.Q + kFinWarps - 1) / kFinWarps);
  finalize_kernel<<<grid, kFinWarps * 32, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// full output gather: out[q][slot] = leafdist[chunk(q)][group(slot)][lane(q)]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) gather_full_kernel(const float* __restrict__ leafdist,
                                                           const uint32_t* __restrict__ slot2group, int64_t n_groups,
                                                           int64_t n, const int* __restrict__ qslot,
                                                           float* __restrict__ out, int use_smem) {
  extern __shared__ float col[];
  const int64_t q = blockIdx.y;
  const int slot = qslot[q];
  const float* src = leafdist + (size_t)slot * n_groups;   // row of (chunk, lane) = slot
  if (use_smem) {
    for (int64_t g = threadIdx.x; g < n_groups; g += blockDim.x) col[g] = __ldg(src + g);
    __syncthreads();
  }
  float* o = out + (size_t)q * n;
  const int64_t per = (((n + gridDim.x - 1) / gridDim.x) + 3) & ~(int64_t)3;
  const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(n, i0 + per);
  if ((n & 3) == 0 && (per & 3) == 0) {   // 16-byte stores
    for (int64_t i = i0 + 4 * threadIdx.x; i < i1; i += 4 * blockDim.x) {
      const uint4 g4 = __ldg(reinterpret_cast<const uint4*>(slot2group + i));
      float4 v;
      v.x = use_smem ? col[g4.x] : __ldg(src + g4.x);
      v.y = use_smem ? col[g4.y] : __ldg(src + g4.y);
      v.z = use_smem ? col[g4.z] : __ldg(src + g4.z);
      v.w = use_smem ? col[g4.w] : __ldg(src + g4.w);
      __stcs(reinterpret_cast<float4*>(o + i), v);
    }
  } else {
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      const uint32_t g = __ldg(slot2group + i);
      o[i] = use_smem ? col[g] : __ldg(src + g);
    }
  }
}

cudaError_t launch_gather_full(const float* leafdist, const uint32_t* slot2group, int64_t n_groups, int64_t n,
                               const int* qslot, int64_t Q, float* out, cudaStream_t st) {
  if (Q <= 0 || n <= 0) return cudaSuccess;
  const size_t smem = (size_t)n_groups * 4;
  const int use_smem = smem <= 96 * 1024;
  if (use_smem) {
    cudaError_t e = cudaFuncSetAttribute(gather_full_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  // ~2 CTAs per SM in total, each query's row split into bx slices
  int64_t bx = std::max<int64_t>(1, std::min<int64_t>((296 + Q - 1) / Q, (n + 4095) / 4096));
  for (int64_t q0 = 0; q0 < Q; q0 += 65535) {
    dim3 grid((unsigned)bx, (unsigned)std::min<int64_t>(65535, Q - q0));
    gather_full_kernel<<<grid, 1024, use_smem ? smem : 0, st>>>(leafdist, slot2group, n_groups, n, qslot + q0,
                                                                 out + (size_t)q0 * n, use_smem);
    count_launch();
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Chunk-major codebook copy for the wide table build (s > 16): out[m][jc][k] =
// codebook row (m, k) dimensions 4 jc .. 4 jc + 3, so a warp's 32 rows of one
// chunk are one contiguous 512 B load.  Layout only, no arithmetic.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) cb_chunks_kernel(const float* __restrict__ cb, int K, int s,
                                                        float4* __restrict__ out) {
  const int nch = s / 4;
  const int m = blockIdx.y, jc = blockIdx.x;       // block = (subspace, chunk); thread = codeword
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    out[((size_t)m * nch + jc) * K + k] = __ldg(reinterpret_cast<const float4*>(cb + ((size_t)m * K + k) * s) + jc);
}

cudaError_t launch_cb_chunks(const float* codebooks, int M, int K, int s, float4* out, cudaStream_t st) {
  cb_chunks_kernel<<<dim3((unsigned)(s / 4), (unsigned)M), 256, 0, st>>>(codebooks, K, s, out);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K1: materialised distance tables [Q][M][K]
// ---------------------------------------------------------------------------
template <int SS>
__global__ void __launch_bounds__(256) lut_kernel(const float* __restrict__ codebooks, int d, int M, int K,
                                                  const float* __restrict__ queries, int64_t Q,
                                                  float* __restrict__ luts) {
  const int m = blockIdx.y;
  const int s = d / M;
  const int64_t q0 = (int64_t)blockIdx.x * 32;
  const int nq = (int)(Q - q0 < 32 ? Q - q0 : 32);
  for (int k = threadIdx.x; k < ((K + 31) & ~31); k += blockDim.x) {
    const bool kvalid = k < K;
    const float* crow = codebooks + ((size_t)m * K + (kvalid ? k : 0)) * s;
    auto xq = [&](int i) { return queries + (size_t)(q0 + i) * d + (size_t)m * s; };
    auto store = [&](int i, float v) { if (kvalid) luts[((size_t)(q0 + i) * M + m) * K + k] = v; };
    entries<SS>(crow, kvalid, s, nq, xq, nullptr, store);
  }
}

cudaError_t launch_luts(const float* codebooks, int d, int M, int K, const float* queries, int64_t Q,
                        float* luts, bool vec4, cudaStream_t st) {
  if (Q <= 0) return cudaSuccess;
  dim3 grid((unsigned)((Q + 31) / 32), (unsigned)M);
  const int s = d / M;
  switch ((vec4 && d % 4 == 0) ? s : 0) {
    case 4: lut_kernel<4><<<grid, 256, 0, st>>>(codebooks, d, M, K, queries, Q, luts); break;
    case 8: lut_kernel<8><<<grid, 256, 0, st>>>(codebooks, d, M, K, queries, Q, luts); break;
    case 16: lut_kernel<16><<<grid, 256, 0, st>>>(codebooks, d, M, K, queries, Q, luts); break;
    case 32: lut_kernel<32><<<grid, 256, 0, st>>>(codebooks, d, M, K, queries, Q, luts); break;
    case 60: lut_kernel<60><<<grid, 256, 0, st>>>(codebooks, d, M, K, queries, Q, luts); break;
    default: lut_kernel<0><<<grid, 256, 0, st>>>(codebooks, d, M, K, queries, Q, luts); break;
  }
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K1': inner-product tables for maximum inner product search (P:107-108,
// P:135, reading A26; oracle/ip.py): T[q][m][k] = B[q][m] - <q_m, c_m(k)>,
// B[q][m] = max_k <q_m, c_m(k)>, off[q] = sum_m B[q][m] (m ascending).  Every
// entry is >= 0 (B - ip in fp32 with B >= ip), so the E-Tree's smallest table
// sums -- off[q] - <q, x_hat> -- are the largest inner products.  Block = 8
// queries, thread = codeword; the dot product is the j-ascending FMA chain.
// ---------------------------------------------------------------------------
constexpr int kIpQ = 8;

__global__ void __launch_bounds__(256) ip_lut_kernel(const float* __restrict__ codebooks, int d, int M, int K,
                                                     const float* __restrict__ queries, int64_t Q,
                                                     float* __restrict__ luts, float* __restrict__ off) {
  __shared__ float red[8][kIpQ];
  __shared__ float bq[kIpQ];
  const int s = d / M;
  const int64_t q0 = (int64_t)blockIdx.x * kIpQ;
  const int nq = (Q - q0 < (int64_t)kIpQ) ? (int)(Q - q0) : kIpQ;
  const int k = threadIdx.x, lane = k & 31, warp = k >> 5;
  const bool kv = k < K;
  float osum = 0.f;                                  // thread i < nq: off of query q0 + i
  for (int m = 0; m < M; ++m) {
    const float* c = codebooks + ((size_t)m * K + (kv ? k : 0)) * s;
    float ip[kIpQ];
#pragma unroll
    for (int i = 0; i < kIpQ; ++i) ip[i] = 0.f;
    for (int j = 0; j < s; ++j) {
      const float cj = __ldg(c + j);
#pragma unroll
      for (int i = 0; i < kIpQ; ++i)
        if (i < nq) ip[i] = fmaf(__ldg(queries + (size_t)(q0 + i) * d + (size_t)m * s + j), cj, ip[i]);
    }
#pragma unroll
    for (int i = 0; i < kIpQ; ++i) {                 // max over the codewords
      float v = kv ? ip[i] : -FLT_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULLMASK, v, o));
      if (lane == 0) red[warp][i] = v;
    }
    __syncthreads();
    if (k < kIpQ) {
      float b = red[0][k];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) b = fmaxf(b, red[w][k]);
      bq[k] = b;
      osum = (m == 0) ? b : osum + b;
    }
    __syncthreads();
    if (kv) {
#pragma unroll
      for (int i = 0; i < kIpQ; ++i)
        if (i < nq) luts[((size_t)(q0 + i) * M + m) * K + k] = bq[i] - ip[i];
    }
    __syncthreads();
  }
  if (k < nq) off[q0 + k] = osum;
}

cudaError_t launch_ip_luts(const float* codebooks, int d, int M, int K, const float* queries, int64_t Q,
                           float* luts, float* off, cudaStream_t st) {
  if (Q <= 0) return cudaSuccess;
  ip_lut_kernel<<<(unsigned)((Q + kIpQ - 1) / kIpQ), 256, 0, st>>>(codebooks, d, M, K, queries, Q, luts, off);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K5: naive ADC (comparison): out[q][i] = sum_m T[q][m][code_i[m]], m ascending
// ---------------------------------------------------------------------------
__global__ void flat_adc_kernel(const float* __restrict__ luts, int64_t Q, int M, int K,
                                const uint8_t* __restrict__ codes, int64_t n, float* __restrict__ out) {
  const int64_t q = blockIdx.y;
  const float* T = luts + (size_t)q * M * K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* c = codes + (size_t)i * M;
    float acc = __ldg(T + c[0]);
    for (int m = 1; m < M; ++m) acc = acc + __ldg(T + (size_t)m * K + c[m]);
    out[(size_t)q * n + i] = acc;
  }
}

cudaError_t launch_flat_adc(const float* luts, int64_t Q, int M, int K, const uint8_t* codes, int64_t n,
                            float* out, cudaStream_t st) {
  if (Q <= 0 || n <= 0) return cudaSuccess;
  dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 1024), (unsigned)Q);
  flat_adc_kernel<<<grid, 256, 0, st>>>(luts, Q, M, K, codes, n, out);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K8: encode (argmin per subspace, ties -> lowest k), optional residual
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) encode_kernel(const float* __restrict__ codebooks, int d, int M, int K,
                                                     const float* __restrict__ x, int64_t n,
                                                     const float* __restrict__ centroids,
                                                     const int32_t* __restrict__ assign, uint8_t* __restrict__ codes) {
  extern __shared__ float cb[];   // [K][s] of subspace m
  const int m = blockIdx.y;
  const int s = d / M;
  for (int i = threadIdx.x; i < K * s; i += blockDim.x) cb[i] = __ldg(codebooks + (size_t)m * K * s + i);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float xs[128];
  const float* xr = x + (size_t)i * d + (size_t)m * s;
  const float* cr = centroids ? centroids + (size_t)assign[i] * d + (size_t)m * s : nullptr;
  float best = __int_as_float(0x7f800000);
  int bk = 0;
  if (s <= 128) {
    for (int j = 0; j < s; ++j) xs[j] = cr ? (__ldg(xr + j) - __ldg(cr + j)) : __ldg(xr + j);
    for (int k = 0; k < K; ++k) {
      const float* c = cb + k * s;
      float a = 0.f;
      for (int j = 0; j < s; ++j) { const float t = xs[j] - c[j]; a = fmaf(t, t, a); }
      if (a < best) { best = a; bk = k; }
    }
  } else {
    for (int k = 0; k < K; ++k) {
      const float* c = cb + k * s;
      float a = 0.f;
      for (int j = 0; j < s; ++j) {
        const float xv = cr ? (__ldg(xr + j) - __ldg(cr + j)) : __ldg(xr + j);
        const float t = xv - c[j];
        a = fmaf(t, t, a);
      }
      if (a < best) { best = a; bk = k; }
    }
  }
  codes[(size_t)i * M + m] = (uint8_t)bk;
}

cudaError_t launch_encode(const float* codebooks, int d, int M, int K, const float* x, int64_t n,
                          const float* centroids, const int32_t* assign, uint8_t* codes, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int s = d / M;
  const size_t smem = (size_t)K * s * 4;
  cudaError_t e = cudaFuncSetAttribute(encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)M);
  encode_kernel<<<grid, 256, smem, st>>>(codebooks, d, M, K, x, n, centroids, assign, codes);
  count_launch();
  return cudaGetLastError();
}

// nearest centroid (ties -> lower index); centroids staged through smem in tiles
__global__ void __launch_bounds__(256) assign_kernel(const float* __restrict__ C, int nlist, int d,
                                                     const float* __restrict__ x, int64_t n,
                                                     int32_t* __restrict__ assign, float* __restrict__ best_dist) {
  extern __shared__ float tile[];  // [TC][d]
  const int TC = 32;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float* xr = x + (size_t)(i < n ? i : n - 1) * d;
  float best = __int_as_float(0x7f800000);
  int bi = 0;
  for (int c0 = 0; c0 < nlist; c0 += TC) {
    const int nc = min(TC, nlist - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < nc * d; e += blockDim.x) tile[e] = __ldg(C + (size_t)c0 * d + e);
    __syncthreads();
    for (int c = 0; c < nc; ++c) {
      const float* cr = tile + c * d;
      float a = 0.f;
      for (int j = 0; j < d; ++j) { const float t = __ldg(xr + j) - cr[j]; a = fmaf(t, t, a); }
      if (a < best) { best = a; bi = c0 + c; }
    }
  }
  if (i < n) {
    assign[i] = bi;
    if (best_dist) best_dist[i] = best;
  }
}

cudaError_t launch_assign(const float* centroids, int nlist, int d, const float* x, int64_t n,
                          int32_t* assign, float* best_dist, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = (size_t)32 * d * 4;
  cudaError_t e = cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  assign_kernel<<<(unsigned)((n + 255) / 256), 256, smem, st>>>(centroids, nlist, d, x, n, assign, best_dist);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K7: merge G shard lists per query (warp per query)
// ---------------------------------------------------------------------------
__global__ void merge_kernel(const float* __restrict__ in_dist, const int32_t* __restrict__ in_ids, int G,
                             int64_t Q, int k, float* __restrict__ out_dist, int32_t* __restrict__ out_ids) {
  __shared__ unsigned long long buf[4][2 * kTopkMax];
  const int lane = lane_id(), warp = warp_id();
  const int64_t q = (int64_t)blockIdx.x * 4 + warp;
  if (q >= Q) return;
  unsigned long long* a = buf[warp];
  int np2 = 32;
  while (np2 < k) np2 <<= 1;
  auto load = [&](int g, unsigned long long* dst) {
    for (int i = lane; i < np2; i += 32) {
      unsigned long long v = ~0ull;
      if (i < k) {
        const size_t o = ((size_t)g * Q + q) * k + i;
        const int32_t id = in_ids[o];
        if (id >= 0) v = ((unsigned long long)__float_as_uint(in_dist[o]) << 32) | (uint32_t)id;
      }
      dst[i] = v;
    }
  };
  load(0, a);
  __syncwarp();
  warp_bitonic_sort(a, np2);
  for (int g = 1; g < G; ++g) {
    load(g, a + np2);
    __syncwarp();
    warp_bitonic_sort(a, 2 * np2);
  }
  for (int i = lane; i < k; i += 32) {
    const unsigned long long v = a[i];
    out_dist[(size_t)q * k + i] = (v == ~0ull) ? __int_as_float(0x7f800000) : __uint_as_float((uint32_t)(v >> 32));
    out_ids[(size_t)q * k + i] = (v == ~0ull) ? -1 : (int32_t)(uint32_t)(v & 0xffffffffu);
  }
}

cudaError_t launch_merge(const float* in_dist, const int32_t* in_ids, int G, int64_t Q, int k,
                         float* out_dist, int32_t* out_ids, cudaStream_t st) {
  if (Q <= 0) return cudaSuccess;
  merge_kernel<<<(unsigned)((Q + 3) / 4), 128, 0, st>>>(in_dist, in_ids, G, Q, k, out_dist, out_ids);
  count_launch();
  return cudaGetLastError();
}

// chunk_q / qslot for the flat plan: chunk c holds queries [c*Q/n, (c+1)*Q/n)
__global__ void fill_flat_kernel(int64_t Q, int n_chunks, int* chunk_q, int* qslot_off, int* qslot) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < (int64_t)n_chunks * 32) {
    const int c = (int)(t >> 5), i = (int)(t & 31);
    const int64_t s = (int64_t)c * Q / n_chunks, e = (int64_t)(c + 1) * Q / n_chunks;
    const bool act = s + i < e;
    chunk_q[t] = act ? (int)(s + i) : -1;
    if (act) qslot[s + i] = c * 32 + i;
  }
  if (t <= Q) qslot_off[t] = (int)t;
}

cudaError_t launch_fill_flat(int64_t Q, int n_chunks, int* chunk_q, int* qslot_off, int* qslot, cudaStream_t st) {
  const int64_t n = std::max<int64_t>((int64_t)n_chunks * 32, Q + 1);
  fill_flat_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Q, n_chunks, chunk_q, qslot_off, qslot);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K6: IVF probe -- coarse distances (fp32 direct difference) and the w nearest
// cells per query by (distance, cell) (Table 1 "w")
// ---------------------------------------------------------------------------
template <int QB>
__global__ void __launch_bounds__(256) probe_kernel(const float* __restrict__ cT, int nlist, int d,
                                                    const float* __restrict__ queries, int64_t Q, int w,
                                                    int32_t* __restrict__ probes) {
  extern __shared__ float psm[];
  float* qv = psm;                 // [QB][d]
  float* ds = psm + QB * d;        // [QB][nlist]
  const int64_t q0 = (int64_t)blockIdx.x * QB;
  const int nq = (int)((Q - q0) < QB ? (Q - q0) : QB);
  for (int i = threadIdx.x; i < QB * d; i += blockDim.x) {
    const int qq = i / d;
    qv[i] = qq < nq ? __ldg(queries + (size_t)(q0 + qq) * d + (i - qq * d)) : 0.f;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nlist; c += blockDim.x) {
    float acc[QB];
#pragma unroll
    for (int qq = 0; qq < QB; ++qq) acc[qq] = 0.f;
#pragma unroll 4
    for (int j = 0; j < d; ++j) {
      const float cv = __ldg(cT + (size_t)j * nlist + c);
#pragma unroll
      for (int qq = 0; qq < QB; ++qq) {
        const float t = qv[qq * d + j] - cv;
        acc[qq] = fmaf(t, t, acc[qq]);
      }
    }
#pragma unroll
    for (int qq = 0; qq < QB; ++qq) ds[qq * nlist + c] = (acc[qq] != acc[qq]) ? __int_as_float(0x7f800000) : acc[qq];   // NaN -> +inf
  }
  __syncthreads();
  const int lane = lane_id(), warp = warp_id();
  for (int qq = warp; qq < nq; qq += blockDim.x / 32) {
    float* row = ds + qq * nlist;
    for (int r = 0; r < w; ++r) {
      float bd = __int_as_float(0x7f800000);
      int bc = INT_MAX;
      for (int c = lane; c < nlist; c += 32) {
        const float v = row[c];
        if (v != v) continue;   // NaN marks a cell already taken (distances are never NaN: see above)
        if (v < bd || (v == bd && c < bc)) { bd = v; bc = c; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const float od = __shfl_xor_sync(FULLMASK, bd, o);
        const int oc = __shfl_xor_sync(FULLMASK, bc, o);
        if (od < bd || (od == bd && oc < bc)) { bd = od; bc = oc; }
      }
      if (lane == 0) {   // w <= nlist, so a cell is always left (bc < nlist); guard anyway
        probes[(size_t)(q0 + qq) * w + r] = (bc < nlist) ? bc : 0;
        if (bc < nlist) row[bc] = __int_as_float(0x7fc00000);   // NaN: never selected again
      }
      __syncwarp();
    }
  }
}

cudaError_t launch_probe(const float* cT, int nlist, int d, const float* queries, int64_t Q, int w,
                         int32_t* probes, cudaStream_t st) {
  if (Q <= 0) return cudaSuccess;
  const size_t budget = 200 * 1024;
  int qb = 8;
  while (qb > 1 && (size_t)qb * (nlist + d) * 4 > budget) qb >>= 1;
  const size_t smem = (size_t)qb * (nlist + d) * 4;
  if (smem > budget) return cudaErrorInvalidValue;
  const unsigned grid = (unsigned)((Q + qb - 1) / qb);
  cudaError_t e;
#define ET_PROBE(QB_)                                                                               \
  case QB_:                                                                                         \
    e = cudaFuncSetAttribute(probe_kernel<QB_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                 \
    probe_kernel<QB_><<<grid, 256, smem, st>>>(cT, nlist, d, queries, Q, w, probes);                \
    break;
  switch (qb) { ET_PROBE(8) ET_PROBE(4) ET_PROBE(2) ET_PROBE(1) default: return cudaErrorInvalidValue; }
#undef ET_PROBE
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// IVF pair bucketing: (query, probe) pairs grouped by cell into chunks of 32
// lanes so a warp scans one list's tree for 32 residual tables at once.
// ---------------------------------------------------------------------------
// Pairs are counted by (tier, cell): tier 0 holds every query's nearest
// probe (rank 0), tier 1 the other probes.  A cell's pairs then form one list
// -- its tier-0 pairs first -- cut into chunks of 32; every cell's FIRST chunk
// comes first in the chunk order (region A), the cells' remaining chunks after
// (region B), each region's cells longest list first.  So the scan of a
// query's nearest list -- where its nearest codes
// most likely are -- runs in the first waves and leaves a tight k-th distance
// bound in qthr for the query's other probes, and a cell costs ceil(n / 32)
// chunk scans rather than one per tier (c4: ~4 -> ~3 per cell).
__device__ __forceinline__ int ivf_entry(const int32_t* probes, int64_t i, int w, int nlist) {
  return ((i % w) == 0 ? 0 : nlist) + probes[i];
}

__global__ void ivf_count_kernel(const int32_t* __restrict__ probes, int64_t P, int w, int nlist, int* cell_cnt,
                                 int* pair_pos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) pair_pos[i] = atomicAdd(&cell_cnt[ivf_entry(probes, i, w, nlist)], 1);
}

// chunk_off[c] = the cell's first chunk (region A), chunk_off[nlist + c] = the
// first of its remaining chunks (region B); chunk_off[2 nlist] = total.
__global__ void __launch_bounds__(1024) ivf_chunks_kernel(const int* __restrict__ cell_cnt, int nlist,
                                                          const uint32_t* __restrict__ list_leaf_off,
                                                          const int* __restrict__ cell_order,
                                                          int* chunk_off, int* n_chunks, int* chunk_cell,
                                                          uint32_t* chunk_lo, uint32_t* chunk_hi) {
  __shared__ int pa[1024], pb[1024];
  const int t = threadIdx.x;
  const int per = (nlist + blockDim.x - 1) / blockDim.x;
  const int c0 = min(nlist, t * per), c1 = min(nlist, c0 + per);
  int la = 0, lb = 0;
  for (int ci = c0; ci < c1; ++ci) {   // cells in list-length order (longest first)
    const int c = cell_order[ci];
    const int n = cell_cnt[c] + cell_cnt[nlist + c];
    la += n > 0 ? 1 : 0;
    lb += n > 0 ? ((n + 31) >> 5) - 1 : 0;
  }
  pa[t] = la;
  pb[t] = lb;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {   // Hillis-Steele inclusive scans
    const int va = (t >= o) ? pa[t - o] : 0, vb = (t >= o) ? pb[t - o] : 0;
    __syncthreads();
    pa[t] += va;
    pb[t] += vb;
    __syncthreads();
  }
  const int total_a = pa[blockDim.x - 1];
  int ra = pa[t] - la, rb = total_a + pb[t] - lb;
  for (int ci = c0; ci < c1; ++ci) {
    const int c = cell_order[ci];
    const int n = cell_cnt[c] + cell_cnt[nlist + c];
    const int nb = n > 0 ? ((n + 31) >> 5) - 1 : 0;
    chunk_off[c] = n > 0 ? ra : -1;
    chunk_off[nlist + c] = rb;
    if (n > 0) {
      chunk_cell[ra] = c; chunk_lo[ra] = list_leaf_off[c]; chunk_hi[ra] = list_leaf_off[c + 1];
      ++ra;
    }
    for (int j = 0; j < nb; ++j) {
      chunk_cell[rb + j] = c; chunk_lo[rb + j] = list_leaf_off[c]; chunk_hi[rb + j] = list_leaf_off[c + 1];
    }
    rb += nb;
  }
  if (t == blockDim.x - 1) { chunk_off[2 * nlist] = total_a + pb[t]; *n_chunks = total_a + pb[t]; }
}

__global__ void ivf_scatter_kernel(const int32_t* __restrict__ probes, int64_t Q, int w, int nlist,
                                   const int* __restrict__ cell_cnt, const int* __restrict__ pair_pos,
                                   const int* __restrict__ chunk_off, int* chunk_q, int* qslot_off, int* qslot) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < Q * w) {
    const int cell = probes[i];
    const int p = ((i % w) == 0) ? pair_pos[i] : cell_cnt[cell] + pair_pos[i];   // tier-0 pairs first
    const int ch = (p < 32) ? chunk_off[cell] : chunk_off[nlist + cell] + (p >> 5) - 1;
    const int ln = p & 31;
    chunk_q[(size_t)ch * 32 + ln] = (int)(i / w);
    qslot[i] = ch * 32 + ln;
  }
  if (i <= Q) qslot_off[i] = (int)(i * w);
}

cudaError_t launch_ivf_bucket(const int32_t* probes, int64_t Q, int w, int nlist, const uint32_t* list_leaf_off,
                              const int* cell_order, int* cell_cnt, int* pair_pos, int* chunk_off, int* n_chunks, int* chunk_cell,
                              uint32_t* chunk_lo, uint32_t* chunk_hi, int* chunk_q, int max_chunks,
                              int* qslot_off, int* qslot, cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(cell_cnt, 0, (size_t)2 * nlist * 4, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(chunk_q, 0xff, (size_t)max_chunks * 32 * 4, st)) != cudaSuccess) return e;
  const int64_t P = Q * w;
  ivf_count_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(probes, P, w, nlist, cell_cnt, pair_pos);
  ivf_chunks_kernel<<<1, 1024, 0, st>>>(cell_cnt, nlist, list_leaf_off, cell_order, chunk_off, n_chunks, chunk_cell,
                                        chunk_lo, chunk_hi);
  const int64_t n = (P > Q + 1) ? P : Q + 1;
  ivf_scatter_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(probes, Q, w, nlist, cell_cnt, pair_pos, chunk_off,
                                                                   chunk_q, qslot_off, qslot);
  count_launch(3);
  return cudaGetLastError();
}

}  // namespace et
