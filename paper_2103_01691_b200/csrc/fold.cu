// Direction-diagonal phase flows folded into a propagator (configuration 4,
// problems.tdpot_strang_step): out = diag(exp(-i x c_b)) E diag(exp(-i x c_a)),
// so a Strang step with a potential that is diagonal along one direction is a
// plain Tucker launch.  The phases are formed on the device from the node
// vector and two host scalars (the integrals of sin^2 over the half steps),
// so nothing is uploaded per step.  Arithmetic follows the host restatement:
// theta = -(x * c) (one rounding, as numpy's (-1j * x) * c), then
// (f_b[i] * E[i][j]) * f_a[j] with separately rounded complex products.
#include "kmb200_kernels.cuh"

namespace kmb {

__device__ __forceinline__ double2 cmul_rn(double2 a, double2 b) {
  return make_double2(__dadd_rn(__dmul_rn(a.x, b.x), -__dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

__device__ __forceinline__ double2 phase(double x, double c) {
  double s, co;
  sincos(-(x * c), &s, &co);
  return make_double2(co, s);
}

__global__ void diag_fold_kernel(const double2* __restrict__ E, double2* __restrict__ out, int m, int k,
                                 const double* __restrict__ x_rows, const double* __restrict__ x_cols, double c_a,
                                 double c_b) {
  pdl_wait();
  const int64_t total = static_cast<int64_t>(m) * k;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(p / k), j = static_cast<int>(p - static_cast<int64_t>(i) * k);
    out[p] = cmul_rn(cmul_rn(phase(__ldg(x_rows + i), c_b), E[p]), phase(__ldg(x_cols + j), c_a));
  }
}

}  // namespace kmb

using namespace kmb;

extern "C" int km_diag_phase_fold(const void* E, void* out, int64_t m, int64_t k, const double* x_rows,
                                  const double* x_cols, double c_a, double c_b, void* stream) {
  if (!E || !out || !x_rows || !x_cols) return fail(KM_EINVAL, "km_diag_phase_fold: NULL pointer");
  if (m < 1 || k < 1 || m > 0x7fffffffLL || k > 0x7fffffffLL)
    return fail(KM_EINVAL, "km_diag_phase_fold: bad extents (%lld, %lld)", (long long)m, (long long)k);
  if (E == out) return fail(KM_EINVAL, "km_diag_phase_fold: in-place fold is not supported");
  const int threads = 256;
  int64_t blocks = (m * k + threads - 1) / threads;
  if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
  const cudaError_t e = launch_pdl(diag_fold_kernel, dim3(static_cast<unsigned>(blocks)), dim3(threads), 0,
                                   static_cast<cudaStream_t>(stream), static_cast<const double2*>(E),
                                   static_cast<double2*>(out), static_cast<int>(m), static_cast<int>(k), x_rows,
                                   x_cols, c_a, c_b);
  if (e != cudaSuccess) return fail(KM_ECUDA, "diag_fold_kernel: %s", cudaGetErrorString(e));
  return check_launch("diag_fold_kernel");
}
