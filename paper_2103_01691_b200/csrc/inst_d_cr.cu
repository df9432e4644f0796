// Instantiation unit: precision=double, U complex=true, L complex=false.
#include "kmb200_launch.cuh"
namespace kmb {
int launch_tma_c128(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl, const OpDev& op,
                    const Split& sp, cudaStream_t st, bool complex_factor);
int launch_d_cr(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl,
                  const OpDev& op, const Split& sp, cudaStream_t st) {
  // complex tensor x real factor (Hermite transforms): TMA kernel when the shape allows it
  const int rc = launch_tma_c128(u, L, out, M, N, K, nl, op, sp, st, false);
  if (rc >= 0) return rc;
  return launch_mumode<double, true, false>(u, L, out, M, N, K, nl, op, sp, st);
}
}  // namespace kmb
