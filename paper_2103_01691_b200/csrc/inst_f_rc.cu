// Instantiation unit: precision=float, U complex=false, L complex=true.
#include "kmb200_launch.cuh"
namespace kmb {
int launch_f_rc(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl,
                  const OpDev& op, const Split& sp, cudaStream_t st) {
  return launch_mumode<float, false, true>(u, L, out, M, N, K, nl, op, sp, st);
}
}  // namespace kmb
