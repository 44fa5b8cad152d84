// scan_s60.cu -- scan kernel instantiations for sub-vector length s = 60
// (one translation unit per s so the kernel variants compile in parallel).
#include "scan.cuh"

namespace et {
cudaError_t launch_scan_60(const ScanParams& p, size_t smem, cudaStream_t st) { return launch_scan_s<60>(p, smem, st); }
}  // namespace et
