// Launch wrappers for mumode_kernel.  Each (precision, U complex, L complex)
// combination is instantiated in its own translation unit (inst_*.cu) so the
// build parallelises; api.cu dispatches to them.
#pragma once
#include "kmb200_kernels.cuh"

namespace kmb {

template <typename S, bool CU, bool CL, bool KC, int OPK, int WM_, int WN_, int WT_ = WT>
int launch_cfg(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl, const OpDev& op,
               const Split& sp, cudaStream_t st) {
  using TU = typename El<S, CU>::T;
  using TL = typename El<S, CL>::T;
  using TO = typename El<S, CU || CL>::T;
  constexpr int BM = WT_ * WM_, BN = WT_ * WN_;
  using Lay = SmemLayout<TU, TL, KC, BM, BN>;
  auto kern = mumode_kernel<S, CU, CL, KC, OPK, WM_, WN_, WT_>;
  if (int rc = ensure_smem(reinterpret_cast<const void*>(kern), Lay::TOTAL, "mumode_kernel")) return rc;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  if (tiles > 0x7fffffffLL) return fail(KM_EINVAL, "km_mumode: %lld tiles exceed the grid limit", (long long)tiles);
  const cudaError_t e = launch_pdl(kern, dim3(static_cast<unsigned>(tiles)), dim3(32 * WM_ * WN_), Lay::TOTAL, st,
                                   static_cast<const TU*>(u), static_cast<const TL*>(L), static_cast<TO*>(out), M, N,
                                   K, nl, op, sp);
  if (e != cudaSuccess) return fail(KM_ECUDA, "mumode_kernel: %s", cudaGetErrorString(e));
  return check_launch("mumode_kernel");
}

// 128x64 tiles (8 warps) when they fill the machine at least twice over, else
// smaller tiles so that small tensors still spread over all SMs.
template <typename S, bool CU, bool CL, bool KC, int OPK>
int launch_sized(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl, const OpDev& op,
                 const Split& sp, cudaStream_t st) {
  const int64_t big = ((M + 127) / 128) * ((N + 63) / 64);
  if (big >= 2 * num_sms()) return launch_cfg<S, CU, CL, KC, OPK, 4, 2>(u, L, out, M, N, K, nl, op, sp, st);
  // small tensors: 32x32 tiles of four 16x16 warp tiles, ~4x the warps of the 64x32 variant
  const int64_t small = ((M + 31) / 32) * ((N + 31) / 32);
  // fewer 32x32 tiles than SMs: 16x16 tiles of four 8x8 warp tiles (4x the warps again;
  // tools/small_probe.py, 10 steps in a graph: 32^3 96 -> 64 us, 48^3 127 -> 111 us, while
  // 64^3 is faster with the 32x32 tiles, 219 against 234 us)
  if (small <= num_sms()) return launch_cfg<S, CU, CL, KC, OPK, 2, 2, 8>(u, L, out, M, N, K, nl, op, sp, st);
  if (small <= 16 * num_sms()) return launch_cfg<S, CU, CL, KC, OPK, 2, 2, 16>(u, L, out, M, N, K, nl, op, sp, st);
  return launch_cfg<S, CU, CL, KC, OPK, 2, 1>(u, L, out, M, N, K, nl, op, sp, st);
}

// Returns KM_OK, or a negative value when the fused op is not instantiated for
// this combination (the caller then runs the op as a separate pass).
template <typename S, bool CU, bool CL>
int launch_mumode(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl, const OpDev& op,
                  const Split& sp, cudaStream_t st) {
  const bool kc = (nl == 1);
  if (op.kind == KM_OP_NONE) {
    if (kc) return launch_sized<S, CU, CL, true, KM_OP_NONE>(u, L, out, M, N, K, nl, op, sp, st);
    return launch_sized<S, CU, CL, false, KM_OP_NONE>(u, L, out, M, N, K, nl, op, sp, st);
  }
  // fused phase epilogues: complex x complex products in the strided layout
  // (the last direction of a d >= 2 step, where the splitting schemes need them)
  if constexpr (CU && CL) {
    if (!kc) {
      if (op.kind == KM_OP_GPE_PHASE)
        return launch_sized<S, CU, CL, false, KM_OP_GPE_PHASE>(u, L, out, M, N, K, nl, op, sp, st);
      if (op.kind == KM_OP_DIAG) return launch_sized<S, CU, CL, false, KM_OP_DIAG>(u, L, out, M, N, K, nl, op, sp, st);
    }
  }
  return -1;
}

#define KMB_DECLARE_LAUNCHER(NAME)                                                                           \
  int NAME(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl, const OpDev& op, \
           const Split& sp, cudaStream_t st);
KMB_DECLARE_LAUNCHER(launch_d_cc)
KMB_DECLARE_LAUNCHER(launch_d_cr)
KMB_DECLARE_LAUNCHER(launch_d_rc)
KMB_DECLARE_LAUNCHER(launch_d_rr)
KMB_DECLARE_LAUNCHER(launch_f_cc)
KMB_DECLARE_LAUNCHER(launch_f_cr)
KMB_DECLARE_LAUNCHER(launch_f_rc)
KMB_DECLARE_LAUNCHER(launch_f_rr)

}  // namespace kmb
