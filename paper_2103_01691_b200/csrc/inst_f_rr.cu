// Instantiation unit: precision=float, U complex=false, L complex=false.
#include "kmb200_launch.cuh"
namespace kmb {
int launch_f_rr(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl,
                  const OpDev& op, const Split& sp, cudaStream_t st) {
  return launch_mumode<float, false, false>(u, L, out, M, N, K, nl, op, sp, st);
}
}  // namespace kmb
