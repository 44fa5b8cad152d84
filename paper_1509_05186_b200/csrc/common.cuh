// common.cuh -- device helpers shared by the kernel translation units of libetree.
#pragma once
#include "internal.h"

#include <cfloat>
#include <climits>
#include <cstdint>
#include <algorithm>

namespace et {

// Device-side bounds checks of a checked build (-DET_CHECKS, tools/
// sanitize_cases.py): a violated check traps (the launch fails with an error
// the host reports).  compute-sanitizer is unavailable on this pool.
#ifdef ET_CHECKS
#define ET_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define ET_CHECK(cond) do { } while (0)
#endif

#define FULLMASK 0xffffffffu

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

// Optional per-CTA phase timestamps (experiment builds: -DET_PHASE_TIMING).
#ifdef ET_PHASE_TIMING
__device__ unsigned long long g_phase[1 << 16][8];
__device__ __forceinline__ void phase_mark(int unit, int i) {
  if (threadIdx.x == 0 && unit < (1 << 16)) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_phase[unit][i] = t;
  }
}
#else
__device__ __forceinline__ void phase_mark(int, int) {}
#endif


// Squared distance between the query sub-vector x[0..s) (optionally minus the
// coarse centroid cc) and codeword c (registers), fp32, j ascending, FMA.
template <int SS>
struct Codeword {
  float c[SS];
  __device__ __forceinline__ void load(const float* row) {
#pragma unroll
    for (int j = 0; j < SS; j += 4) {
      float4 v = __ldg(reinterpret_cast<const float4*>(row + j));
      c[j] = v.x; c[j + 1] = v.y; c[j + 2] = v.z; c[j + 3] = v.w;
    }
  }
};

// Computes table entries for queries slots [0, nq) and codeword `crow` (one per
// lane).  `xq(i)` returns the pointer to slot i's sub-vector; `cc` is the coarse
// centroid sub-vector (IVF) or null.  `store(i, v)` writes the entry.
template <int SS, class XQ, class ST>
__device__ __forceinline__ void entries_fixed(const float* crow, bool kvalid, int nq,
                                              XQ xq, const float* cc, ST store) {
  Codeword<SS> cw;
  if (kvalid) cw.load(crow);
  else {
#pragma unroll
    for (int j = 0; j < SS; ++j) cw.c[j] = 0.f;
  }
  int i = 0;
  for (; i + 4 <= nq; i += 4) {
    const float4* x0 = reinterpret_cast<const float4*>(xq(i));
    const float4* x1 = reinterpret_cast<const float4*>(xq(i + 1));
    const float4* x2 = reinterpret_cast<const float4*>(xq(i + 2));
    const float4* x3 = reinterpret_cast<const float4*>(xq(i + 3));
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int jb = 0; jb < SS / 4; ++jb) {
      float4 v0 = __ldg(x0 + jb), v1 = __ldg(x1 + jb), v2 = __ldg(x2 + jb), v3 = __ldg(x3 + jb);
      if (cc) {
        float4 cv = __ldg(reinterpret_cast<const float4*>(cc) + jb);
        v0.x -= cv.x; v0.y -= cv.y; v0.z -= cv.z; v0.w -= cv.w;
        v1.x -= cv.x; v1.y -= cv.y; v1.z -= cv.z; v1.w -= cv.w;
        v2.x -= cv.x; v2.y -= cv.y; v2.z -= cv.z; v2.w -= cv.w;
        v3.x -= cv.x; v3.y -= cv.y; v3.z -= cv.z; v3.w -= cv.w;
      }
      const float* c = cw.c + 4 * jb;
      float t;
      t = v0.x - c[0]; a0 = fmaf(t, t, a0); t = v0.y - c[1]; a0 = fmaf(t, t, a0);
      t = v0.z - c[2]; a0 = fmaf(t, t, a0); t = v0.w - c[3]; a0 = fmaf(t, t, a0);
      t = v1.x - c[0]; a1 = fmaf(t, t, a1); t = v1.y - c[1]; a1 = fmaf(t, t, a1);
      t = v1.z - c[2]; a1 = fmaf(t, t, a1); t = v1.w - c[3]; a1 = fmaf(t, t, a1);
      t = v2.x - c[0]; a2 = fmaf(t, t, a2); t = v2.y - c[1]; a2 = fmaf(t, t, a2);
      t = v2.z - c[2]; a2 = fmaf(t, t, a2); t = v2.w - c[3]; a2 = fmaf(t, t, a2);
      t = v3.x - c[0]; a3 = fmaf(t, t, a3); t = v3.y - c[1]; a3 = fmaf(t, t, a3);
      t = v3.z - c[2]; a3 = fmaf(t, t, a3); t = v3.w - c[3]; a3 = fmaf(t, t, a3);
    }
    store(i, a0); store(i + 1, a1); store(i + 2, a2); store(i + 3, a3);
  }
  for (; i < nq; ++i) {
    const float4* x0 = reinterpret_cast<const float4*>(xq(i));
    float a0 = 0.f;
#pragma unroll
    for (int jb = 0; jb < SS / 4; ++jb) {
      float4 v0 = __ldg(x0 + jb);
      if (cc) {
        float4 cv = __ldg(reinterpret_cast<const float4*>(cc) + jb);
        v0.x -= cv.x; v0.y -= cv.y; v0.z -= cv.z; v0.w -= cv.w;
      }
      const float* c = cw.c + 4 * jb;
      float t;
      t = v0.x - c[0]; a0 = fmaf(t, t, a0); t = v0.y - c[1]; a0 = fmaf(t, t, a0);
      t = v0.z - c[2]; a0 = fmaf(t, t, a0); t = v0.w - c[3]; a0 = fmaf(t, t, a0);
    }
    store(i, a0);
  }
}

// Generic sub-vector length (any s): scalar loads.
template <class XQ, class ST>
__device__ __forceinline__ void entries_generic(const float* crow, bool kvalid, int s, int nq,
                                                XQ xq, const float* cc, ST store) {
  for (int i = 0; i < nq; ++i) {
    const float* x = xq(i);
    float a = 0.f;
    for (int j = 0; j < s; ++j) {
      float xv = __ldg(x + j);
      if (cc) xv -= __ldg(cc + j);
      float t = xv - (kvalid ? __ldg(crow + j) : 0.f);
      a = fmaf(t, t, a);
    }
    store(i, a);
  }
}

template <int SS, class XQ, class ST>
__device__ __forceinline__ void entries(const float* crow, bool kvalid, int s, int nq, XQ xq,
                                        const float* cc, ST store) {
  if constexpr (SS > 0) entries_fixed<SS>(crow, kvalid, nq, xq, cc, store);
  else entries_generic(crow, kvalid, s, nq, xq, cc, store);
}

}  // namespace et
