// microbench_alu.cu -- measured fp32 ceiling for the distance-table inner loop
// (t = x - c; a = fma(t, t, a)), scalar FADD/FFMA vs packed FADD2/FFMA2.
// Used to derive the "alu" roofline peak in DESIGN.md §5.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_alu tools/microbench_alu.cu && /tmp/mb_alu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void __launch_bounds__(512) scalar_kernel(float* out, float x0, float c0) {
  float a[kChains], x[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { a[i] = 0.f; x[i] = x0 + i + threadIdx.x; }
  float c = c0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      const float t = x[i] - c;
      a[i] = fmaf(t, t, a[i]);
    }
    c += 1e-7f;   // one extra FADD per kChains pairs (keeps the loop honest)
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}

__global__ void __launch_bounds__(512) packed_kernel(float* out, float x0, float c0) {
  unsigned long long a[kChains / 2], x[kChains / 2];
#pragma unroll
  for (int i = 0; i < kChains / 2; ++i) { a[i] = 0ull; x[i] = pk(x0 + 2 * i + threadIdx.x, x0 + 2 * i + 1 + threadIdx.x); }
  float cs = c0;
  for (int it = 0; it < kIters; ++it) {
    const unsigned long long c = pk(cs, cs);
#pragma unroll
    for (int i = 0; i < kChains / 2; ++i) {
      unsigned long long t;
      asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(x[i]), "l"(c));
      asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(a[i]) : "l"(t));
    }
    cs += 1e-7f;
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains / 2; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

void bench_build_loop();

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 4, threads = 512;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double ops = 2.0 * kChains * kIters * (double)blocks * threads;   // FADD + FFMA lane ops
  for (int v = 0; v < 2; ++v) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (v == 0) scalar_kernel<<<blocks, threads>>>(out, 1.f, 0.5f);
      else packed_kernel<<<blocks, threads>>>(out, 1.f, 0.5f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("{\"variant\": \"%s\", \"lane_ops_per_s\": %.4e, \"ms\": %.4f, \"sms\": %d, \"clock_khz\": %d}\n",
           v == 0 ? "scalar FADD+FFMA" : "packed FADD2+FFMA2", ops / (best * 1e-3), best, sms, clk);
  }
  bench_build_loop();
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}

// ---------------------------------------------------------------------------
// The table-build inner loop as the scan kernel runs it: query pairs staged in
// shared memory (broadcast LDS.128 = 2 dims x 2 queries), codeword rows in
// registers, packed FADD2/FFMA2 chains; run with 16 and 64 warps per SM.
__device__ __forceinline__ unsigned long long f2sub_(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2sq_(unsigned long long t, unsigned long long acc) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(t), "l"(acc));
  return r;
}

template <int ROWS>
__global__ void __launch_bounds__(512) build_loop_kernel(float* out, int iters) {
  __shared__ __align__(16) float stage[16 * 32 * 2];   // 16 pairs x 16 dims x 2
  for (int i = threadIdx.x; i < 16 * 32 * 2; i += blockDim.x) stage[i] = 0.001f * i;
  __syncthreads();
  float c[ROWS][16];
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int j = 0; j < 16; ++j) c[r][j] = 0.5f * j + r + threadIdx.x * 1e-3f;
  float sink = 0.f;
  for (int it = 0; it < iters; ++it) {
    const int pi = (it + (threadIdx.x >> 5)) & 15;
    unsigned long long a[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) a[r] = 0ull;
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const float4 u = *reinterpret_cast<const float4*>(stage + pi * 32 + j * 2);
      unsigned long long x0, x1;
      asm("mov.b64 %0, {%1, %2};" : "=l"(x0) : "f"(u.x), "f"(u.y));
      asm("mov.b64 %0, {%1, %2};" : "=l"(x1) : "f"(u.z), "f"(u.w));
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        unsigned long long c0, c1;
        asm("mov.b64 %0, {%1, %1};" : "=l"(c0) : "f"(c[r][j]));
        asm("mov.b64 %0, {%1, %1};" : "=l"(c1) : "f"(c[r][j + 1]));
        a[r] = f2sq_(f2sub_(x0, c0), a[r]);
        a[r] = f2sq_(f2sub_(x1, c1), a[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[r]));
      sink += lo + hi;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink;
}

void bench_build_loop() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 4 * 512);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048;
  for (int rows = 1; rows <= 2; ++rows) {
    for (int per_sm = 1; per_sm <= 4; per_sm *= 4) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        if (rows == 1) build_loop_kernel<1><<<sms * per_sm, 512>>>(out, iters);
        else build_loop_kernel<2><<<sms * per_sm, 512>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double ops = 64.0 * rows * iters * (double)sms * per_sm * 512;   // FADD+FFMA lane ops (16 dims x 2 queries x 2 per row)
      printf("{\"variant\": \"build loop rows=%d warps/SM=%d\", \"lane_ops_per_s\": %.4e, \"ms\": %.4f}\n",
             rows, 16 * per_sm, ops / (best * 1e-3) / 1.0, best);
    }
  }
}
