// scan_s60.cu -- scan kernel instantiations for sub-vector length s = 60
// (one translation unit per s so the kernel variants compile in parallel).
#include "scan.cuh"
#include "narrow.cuh"

namespace et {
cudaError_t launch_scan_60(const ScanParams& p, size_t smem, cudaStream_t st) { return launch_scan_s<60>(p, smem, st); }
cudaError_t launch_narrow_60(const ScanParams& p, cudaStream_t st) { return launch_narrow_s<60>(p, st); }
}  // namespace et

#ifdef ET_PHASE_TIMING
extern "C" int et_debug_phases_s60(unsigned long long* out, int n_units) {
  if (n_units > (1 << 16)) n_units = 1 << 16;
  return (int)cudaMemcpyFromSymbol(out, et::g_phase, (size_t)n_units * 8 * sizeof(unsigned long long));
}
#endif
