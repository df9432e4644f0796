// Instantiation unit: precision=double, U complex=false, L complex=true.
#include "kmb200_launch.cuh"
namespace kmb {
int launch_d_rc(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl,
                  const OpDev& op, const Split& sp, cudaStream_t st) {
  return launch_mumode<double, false, true>(u, L, out, M, N, K, nl, op, sp, st);
}
}  // namespace kmb
