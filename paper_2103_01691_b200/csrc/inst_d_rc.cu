// Instantiation unit: precision=double, U complex=false, L complex=true.
#include "kmb200_launch.cuh"
namespace kmb {
int launch_tma_f64(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl, const OpDev& op,
                   const Split& sp, cudaStream_t st, bool complex_tensor, bool complex_factor);
int launch_d_rc(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl,
                  const OpDev& op, const Split& sp, cudaStream_t st) {
  // the warp-specialised TMA kernel when the shape allows it, else the cp.async kernel
  const int rc = launch_tma_f64(u, L, out, M, N, K, nl, op, sp, st, false, true);
  if (rc >= 0) return rc;
  return launch_mumode<double, false, true>(u, L, out, M, N, K, nl, op, sp, st);
}
}  // namespace kmb
