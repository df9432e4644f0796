// Host side of the fused plane kernel (kmb200_plane.cuh).
#include "kmb200_plane.cuh"

namespace kmb {

bool g_plane_disabled = false;  // KM_POLICY_NO_PLANE_FUSION

namespace {

bool extent_ok(int64_t n) { return n == 32 || n == 48 || n == 64; }

// rows per CTA: the most CTAs that still fit one wave and the shared memory (0: none fits)
int choose_split(int64_t n1, int64_t n2, int64_t n3) {
  const int64_t S = num_sms();
  int split = 0;
  for (int s = 4; s >= 1; --s) {
    if (n1 % (16 * s) != 0 || plane12_smem(static_cast<int>(n1) / s, static_cast<int>(n2)) > 227 * 1024) continue;
    if (n3 * s <= S || split == 0) split = s;
    if (n3 * s <= S) break;
  }
  return (n3 * split > 0x7fffffffLL) ? 0 : split;
}

template <int N1, int N2>
int launch_n(const void* u, const void* E1, const void* E2, void* out, int64_t n3, cudaStream_t st) {
  const int split = choose_split(N1, N2, n3);
  if (split == 0) return fail(KM_EINVAL, "mumode_plane12_kernel: no row split fits");
  auto kern = mumode_plane12_kernel<N1, N2>;
  const int smem = plane12_smem(N1 / split, N2);
  if (int rc = ensure_smem(reinterpret_cast<const void*>(kern), smem, "mumode_plane12_kernel")) return rc;
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
    default: return fail(KM_EINVAL, "mumode_plane12_kernel: n2 = %lld", static_cast<long long>(n2));
  }
}

}  // namespace

namespace {
template <int N3, int F>
int launch_p33f(const void* u, const void* Ea, const void* Eb, void* out, int64_t nfib, cudaStream_t st) {
  auto kern = mumode_pencil33_kernel<N3, F>;
  const int smem = pencil33_smem(N3, F);
  if (int rc = ensure_smem(reinterpret_cast<const void*>(kern), smem, "mumode_pencil33_kernel")) return rc;
  const cudaError_t e = launch_pdl(kern, dim3(static_cast<unsigned>(nfib / F)), dim3(plane::THREADS), smem, st,
                                   static_cast<const double2*>(u), static_cast<const double2*>(Ea),
                                   static_cast<const double2*>(Eb), static_cast<double2*>(out), nfib);
  if (e != cudaSuccess) return fail(KM_ECUDA, "mumode_pencil33_kernel: %s", cudaGetErrorString(e));
  return check_launch("mumode_pencil33_kernel");
}

// 32-fiber blocks while they give at least ~2/3 of a wave, else 16-fiber blocks
template <int N3>
int launch_p33(const void* u, const void* Ea, const void* Eb, void* out, int64_t nfib, cudaStream_t st) {
  if (3 * (nfib / 32) >= 2 * num_sms()) return launch_p33f<N3, 32>(u, Ea, Eb, out, nfib, st);
  return launch_p33f<N3, 16>(u, Ea, Eb, out, nfib, st);
}
}  // namespace

bool pencil33_supported(int64_t nfib, int64_t n3) {
  return extent_ok(n3) && nfib >= 32 && nfib % 32 == 0 && nfib / 32 <= 0x7fffffffLL;
}

int launch_pencil33(const void* u, const void* Ea, const void* Eb, void* out, int64_t nfib, int64_t n3,
                    cudaStream_t st) {
  if (!pencil33_supported(nfib, n3) ||
      ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(Ea) | reinterpret_cast<uintptr_t>(Eb) |
        reinterpret_cast<uintptr_t>(out)) & 15))
    return fail(KM_EINVAL, "mumode_pencil33_kernel: unsupported shape or alignment");
  switch (n3) {
    case 32: return launch_p33<32>(u, Ea, Eb, out, nfib, st);
    case 48: return launch_p33<48>(u, Ea, Eb, out, nfib, st);
    default: return launch_p33<64>(u, Ea, Eb, out, nfib, st);
  }
}

bool plane12_shape_ok(int64_t n1, int64_t n2, int64_t n3) {
  return n3 >= 1 && extent_ok(n1) && extent_ok(n2) && choose_split(n1, n2, n3) > 0;
}

bool plane12_supported(int64_t n1, int64_t n2, int64_t n3) { return !g_plane_disabled && plane12_shape_ok(n1, n2, n3); }

int launch_plane12(const void* u, const void* E1, const void* E2, void* out, int64_t n1, int64_t n2, int64_t n3,
                   cudaStream_t st) {
  if (!plane12_shape_ok(n1, n2, n3) ||
      ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(E1) | reinterpret_cast<uintptr_t>(E2) |
        reinterpret_cast<uintptr_t>(out)) & 15))
    return fail(KM_EINVAL, "mumode_plane12_kernel: unsupported shape or alignment");
  switch (n1) {
    case 32: return launch_n1<32>(u, E1, E2, out, n2, n3, st);
    case 48: return launch_n1<48>(u, E1, E2, out, n2, n3, st);
    case 64: return launch_n1<64>(u, E1, E2, out, n2, n3, st);
    default: return fail(KM_EINVAL, "mumode_plane12_kernel: n1 = %lld", static_cast<long long>(n1));
  }
}

}  // namespace kmb
