// build_gpu.cu -- GPU-native grouping step of the index build (SURVEY.md
// §8f-f1; "sort + linear build"): the codes are sorted
// lexicographically on the device (radix sort of big-endian byte keys, stable,
// ids ascending within equal codes, A6) and split into groups of identical
// codes (one leaf per distinct code) by a flag + prefix-sum pass.  The
// per-id arrays (grouped ids, slot -> group) and per-group arrays (offsets,
// multiplicities, minimum ids) are produced on the device; only the G group
// offsets and one representative slot per group come back to the host, where
// the trees are built over the G distinct codes (host.cpp).
#include "internal.h"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdint>

namespace et {

namespace {

struct Perm { int l[16]; };

__global__ void iota_kernel(uint32_t* a, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = (uint32_t)i;
}

// Big-endian key of a row's (permuted) code bytes b0..b{nb-1}, starting at
// byte `from`: byte `from` is the most significant.
__global__ void pack_keys_kernel(const uint8_t* __restrict__ codes, int64_t n, int M, Perm perm, int from, int nb,
                                 const uint32_t* __restrict__ slots, uint64_t* __restrict__ key) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t* row = codes + (size_t)slots[i] * M;
  uint64_t k = 0;
  for (int b = 0; b < nb; ++b) k |= (uint64_t)row[perm.l[from + b]] << (8 * (7 - b));
  key[i] = k;
}

__global__ void gather_i32_kernel(const int32_t* __restrict__ src, const uint32_t* __restrict__ slots, int64_t n,
                                  int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = src[slots[i]];
}

__global__ void flag_kernel(const uint64_t* __restrict__ khi, const uint64_t* __restrict__ klo,
                            const int32_t* __restrict__ lk, int64_t n, uint32_t* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (i == 0 || khi[i] != khi[i - 1] || (klo && klo[i] != klo[i - 1]) || (lk && lk[i] != lk[i - 1])) ? 1u
                                                                                                              : 0u;
}

// Sorted position i: group gid[i] - 1 (inclusive scan of the flags).
__global__ void group_out_kernel(const uint32_t* __restrict__ gid, const uint32_t* __restrict__ slots,
                                 const int32_t* __restrict__ ids, int64_t n, uint32_t* __restrict__ off,
                                 uint32_t* __restrict__ first, int32_t* __restrict__ ids_out,
                                 uint32_t* __restrict__ slot2group) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t g = gid[i] - 1u;
  const uint32_t s = slots[i];
  if (i == 0 || gid[i] != gid[i - 1]) { off[g] = (uint32_t)i; first[g] = s; }
  if (i == n - 1) off[g + 1] = (uint32_t)n;
  ids_out[i] = ids ? ids[s] : (int32_t)s;
  slot2group[s] = g;
}

__global__ void group_stats_kernel(const uint32_t* __restrict__ off, int64_t G, const int32_t* __restrict__ ids_out,
                                   uint32_t* __restrict__ mult, int32_t* __restrict__ minid) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  mult[g] = off[g + 1] - off[g];
  minid[g] = ids_out[off[g]];   // ids ascending within a group
}

template <class T>
cudaError_t dalloc(T** p, size_t n) { return cudaMalloc(reinterpret_cast<void**>(p), (n ? n : 1) * sizeof(T)); }

}  // namespace

#define ET_CU(x)                                  \
  do {                                            \
    cudaError_t e_ = (x);                         \
    if (e_ != cudaSuccess) { cleanup(); return e_; } \
  } while (0)

cudaError_t gpu_group_codes(const uint8_t* codes_h, const int32_t* ids_h, int64_t n, int M, const int32_t* perm_h,
                            const int32_t* list_h, GpuGroups* out) {
  *out = GpuGroups{};
  if (M > 16) return cudaErrorInvalidValue;
  Perm perm{};
  for (int l = 0; l < M; ++l) perm.l[l] = perm_h ? perm_h[l] : l;
  cudaStream_t st = 0;
  uint8_t* d_codes = nullptr;
  int32_t* d_ids = nullptr;
  int32_t* d_idk = nullptr;
  int32_t *d_list = nullptr, *d_lk = nullptr, *d_lk2 = nullptr;
  uint32_t *d_slots = nullptr, *d_slots2 = nullptr, *d_flag = nullptr, *d_gid = nullptr;
  uint64_t *d_key = nullptr, *d_key2 = nullptr, *d_klo = nullptr;
  void* d_tmp = nullptr;
  uint32_t *d_off = nullptr, *d_first = nullptr, *d_s2g = nullptr, *d_mult = nullptr;
  int32_t *d_idout = nullptr, *d_minid = nullptr;
  auto cleanup = [&]() {
    for (void* p : {(void*)d_codes, (void*)d_ids, (void*)d_idk, (void*)d_list, (void*)d_lk, (void*)d_lk2, (void*)d_slots, (void*)d_slots2, (void*)d_flag,
                    (void*)d_gid, (void*)d_key, (void*)d_key2, (void*)d_klo, d_tmp, (void*)d_off, (void*)d_first,
                    (void*)d_s2g, (void*)d_mult, (void*)d_idout, (void*)d_minid})
      if (p) cudaFree(p);
  };
  const unsigned blk = 256;
  const unsigned grd = (unsigned)((n + blk - 1) / blk);
  ET_CU(dalloc(&d_codes, (size_t)n * M));
  ET_CU(cudaMemcpy(d_codes, codes_h, (size_t)n * M, cudaMemcpyHostToDevice));
  ET_CU(dalloc(&d_slots, n));
  ET_CU(dalloc(&d_slots2, n));
  iota_kernel<<<grd, blk, 0, st>>>(d_slots, n);
  // temp storage: the largest of the sorts (64-bit keys + 32-bit values)
  size_t tmp_bytes = 0, t2 = 0;
  ET_CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                        (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)n, 0, 64, st));
  ET_CU(cub::DeviceRadixSort::SortPairs(nullptr, t2, (const int32_t*)nullptr, (int32_t*)nullptr,
                                        (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)n, 0, 32, st));
  tmp_bytes = tmp_bytes > t2 ? tmp_bytes : t2;
  ET_CU(cub::DeviceScan::InclusiveSum(nullptr, t2, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)n, st));
  tmp_bytes = tmp_bytes > t2 ? tmp_bytes : t2;
  ET_CU(cudaMalloc(&d_tmp, tmp_bytes));
  if (ids_h) {   // ids ascending within equal codes: sort by id first, then stably by code
    ET_CU(dalloc(&d_ids, n));
    ET_CU(dalloc(&d_idk, n));
    ET_CU(cudaMemcpy(d_ids, ids_h, (size_t)n * 4, cudaMemcpyHostToDevice));
    size_t tb = tmp_bytes;
    ET_CU(cub::DeviceRadixSort::SortPairs(d_tmp, tb, d_ids, d_idk, d_slots, d_slots2, (int64_t)n, 0, 32, st));
    std::swap(d_slots, d_slots2);
    cudaFree(d_idk);
    d_idk = nullptr;
  }
  ET_CU(dalloc(&d_key, n));
  ET_CU(dalloc(&d_key2, n));
  const int nb_hi = M < 8 ? M : 8, nb_lo = M - nb_hi;
  if (nb_lo > 0) {   // least significant bytes first (LSD over two 64-bit keys)
    pack_keys_kernel<<<grd, blk, 0, st>>>(d_codes, n, M, perm, 8, nb_lo, d_slots, d_key);
    size_t tb = tmp_bytes;
    ET_CU(cub::DeviceRadixSort::SortPairs(d_tmp, tb, d_key, d_key2, d_slots, d_slots2, (int64_t)n, 64 - 8 * nb_lo, 64,
                                          st));
    std::swap(d_slots, d_slots2);
  }
  pack_keys_kernel<<<grd, blk, 0, st>>>(d_codes, n, M, perm, 0, nb_hi, d_slots, d_key);
  {
    size_t tb = tmp_bytes;
    ET_CU(cub::DeviceRadixSort::SortPairs(d_tmp, tb, d_key, d_key2, d_slots, d_slots2, (int64_t)n, 64 - 8 * nb_hi, 64,
                                          st));
    std::swap(d_slots, d_slots2);
    std::swap(d_key, d_key2);   // d_key: sorted high keys
  }
  if (list_h) {   // IVF: (list, code) order -- a last stable pass by list
    ET_CU(dalloc(&d_list, n));
    ET_CU(dalloc(&d_lk, n));
    ET_CU(dalloc(&d_lk2, n));
    ET_CU(cudaMemcpy(d_list, list_h, (size_t)n * 4, cudaMemcpyHostToDevice));
    gather_i32_kernel<<<grd, blk, 0, st>>>(d_list, d_slots, n, d_lk);
    size_t tb = tmp_bytes;
    ET_CU(cub::DeviceRadixSort::SortPairs(d_tmp, tb, d_lk, d_lk2, d_slots, d_slots2, (int64_t)n, 0, 32, st));
    std::swap(d_slots, d_slots2);
    std::swap(d_lk, d_lk2);   // d_lk: sorted lists
    pack_keys_kernel<<<grd, blk, 0, st>>>(d_codes, n, M, perm, 0, nb_hi, d_slots, d_key);
  }
  if (nb_lo > 0) {
    ET_CU(dalloc(&d_klo, n));
    pack_keys_kernel<<<grd, blk, 0, st>>>(d_codes, n, M, perm, 8, nb_lo, d_slots, d_klo);
  }
  cudaFree(d_codes);
  d_codes = nullptr;
  ET_CU(dalloc(&d_flag, n));
  ET_CU(dalloc(&d_gid, n));
  flag_kernel<<<grd, blk, 0, st>>>(d_key, d_klo, list_h ? d_lk : nullptr, n, d_flag);
  {
    size_t tb = tmp_bytes;
    ET_CU(cub::DeviceScan::InclusiveSum(d_tmp, tb, d_flag, d_gid, (int64_t)n, st));
  }
  uint32_t G = 0;
  ET_CU(cudaMemcpy(&G, d_gid + (n - 1), 4, cudaMemcpyDeviceToHost));
  ET_CU(dalloc(&d_off, (size_t)G + 1));
  ET_CU(dalloc(&d_first, G));
  ET_CU(dalloc(&d_idout, n));
  ET_CU(dalloc(&d_s2g, n));
  group_out_kernel<<<grd, blk, 0, st>>>(d_gid, d_slots, d_ids, n, d_off, d_first, d_idout, d_s2g);
  ET_CU(dalloc(&d_mult, G));
  ET_CU(dalloc(&d_minid, G));
  group_stats_kernel<<<(unsigned)((G + blk - 1) / blk), blk, 0, st>>>(d_off, G, d_idout, d_mult, d_minid);
  ET_CU(cudaGetLastError());
  out->G = G;
  out->off.resize((size_t)G + 1);
  out->first.resize(G);
  ET_CU(cudaMemcpy(out->off.data(), d_off, ((size_t)G + 1) * 4, cudaMemcpyDeviceToHost));
  ET_CU(cudaMemcpy(out->first.data(), d_first, (size_t)G * 4, cudaMemcpyDeviceToHost));
  // hand the device arrays over to the index; free the scratch
  out->ids = d_idout; d_idout = nullptr;
  out->group_off = d_off; d_off = nullptr;
  out->mult = d_mult; d_mult = nullptr;
  out->minid = d_minid; d_minid = nullptr;
  out->slot2group = d_s2g; d_s2g = nullptr;
  cleanup();
  return cudaSuccess;
}

#undef ET_CU

}  // namespace et
