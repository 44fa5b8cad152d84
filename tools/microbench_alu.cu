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
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
