// microbench_tmem.cu -- latency of a dependent tcgen05.ld.32x32b.x1 + wait::ld
// chain vs a dependent ld.shared chain (the scan's level-0 lookup vs the
// other levels).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_tmem tools/microbench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_tmem(unsigned long long* out, int iters) {
  __shared__ uint32_t slot;
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(&slot);
  if (threadIdx.x < 32)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(a) : "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = slot;
  if (threadIdx.x < 32) {
    uint32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int c = 0; c < 256; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                   :: "r"(base + c), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t x = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t y;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(y) : "r"(base + (x & 7)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(y));
      x += y + 1;
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[2] = x; }
    // smem chain
    __shared__ uint32_t buf[256];
    buf[threadIdx.x] = 0; buf[threadIdx.x + 32] = 0;
    __syncwarp();
    x = 0;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t y;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(y) : "r"((uint32_t)__cvta_generic_to_shared(buf) + ((x & 7) << 2)));
      x += y + 1;
    }
    t1 = clock64();
    if (threadIdx.x == 0) { out[1] = (t1 - t0) / iters; out[3] = x; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(base) : "memory");
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  k_tmem<<<1, 128>>>(d, 1000);
  unsigned long long h[4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("{\"tmem_ld_wait_cycles\": %llu, \"lds_cycles\": %llu, \"err\": \"%s\"}\n", h[0], h[1], cudaGetErrorString(e));
  return 0;
}
