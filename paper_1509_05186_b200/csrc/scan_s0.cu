// scan_s0.cu -- scan kernel instantiations for sub-vector length s = any (generic)
// (one translation unit per s so the kernel variants compile in parallel).
#include "scan.cuh"

namespace et {
cudaError_t launch_scan_0(const ScanParams& p, size_t smem, cudaStream_t st) { return launch_scan_s<0>(p, smem, st); }
}  // namespace et
