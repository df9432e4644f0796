// Host side of the fused plane kernel (kmb200_plane.cuh).
#include "kmb200_plane.cuh"

namespace kmb {

bool g_plane_disabled = false;  // KM_POLICY_NO_PLANE_FUSION

namespace {

template <int N1, int N2>
int launch_n(const void* u, const void* E1, const void* E2, void* out, int64_t n3, cudaStream_t st) {
  // rows per CTA: the most CTAs that still fit one wave and the shared memory
  const int64_t S = num_sms();
  int split = 0;
  for (int s = 4; s >= 1; --s) {
    if (N1 % (16 * s) != 0 || plane12_smem(N1 / s, N2) > 227 * 1024) continue;
    if (n3 * s <= S || split == 0) split = s;
    if (n3 * s <= S) break;
  }
  if (split == 0) return -1;
  auto kern = mumode_plane12_kernel<N1, N2>;
  const int smem = plane12_smem(N1 / split, N2);
  if (int rc = ensure_smem(reinterpret_cast<const void*>(kern), smem, "mumode_plane12_kernel")) return rc;
  if (n3 * split > 0x7fffffffLL) return -1;
  const cudaError_t e = launch_pdl(kern, dim3(static_cast<unsigned>(n3 * split)), dim3(plane::THREADS), smem, st,
                                   static_cast<const double2*>(u), static_cast<const double2*>(E1),
                                   static_cast<const double2*>(E2), static_cast<double2*>(out), split);
  if (e != cudaSuccess) return fail(KM_ECUDA, "mumode_plane12_kernel: %s", cudaGetErrorString(e));
  return check_launch("mumode_plane12_kernel");
}

template <int N1>
int launch_n1(const void* u, const void* E1, const void* E2, void* out, int64_t n2, int64_t n3, cudaStream_t st) {
  switch (n2) {
    case 32: return launch_n<N1, 32>(u, E1, E2, out, n3, st);
    case 48: return launch_n<N1, 48>(u, E1, E2, out, n3, st);
    case 64: return launch_n<N1, 64>(u, E1, E2, out, n3, st);
    default: return -1;
  }
}

}  // namespace

int launch_plane12(const void* u, const void* E1, const void* E2, void* out, int64_t n1, int64_t n2, int64_t n3,
                   cudaStream_t st) {
  if (g_plane_disabled || n3 < 1) return -1;
  if ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(E1) | reinterpret_cast<uintptr_t>(E2) |
       reinterpret_cast<uintptr_t>(out)) & 15)
    return -1;
  switch (n1) {
    case 32: return launch_n1<32>(u, E1, E2, out, n2, n3, st);
    case 48: return launch_n1<48>(u, E1, E2, out, n2, n3, st);
    case 64: return launch_n1<64>(u, E1, E2, out, n2, n3, st);
    default: return -1;
  }
}

}  // namespace kmb
