// Deterministic device norms: max |a-b|, ||a-b||_2 and the
// weighted two-norm sqrt(sum_i w(i) |a-b|^2) with w(i) = w_1[i_1]...w_d[i_d]
// (reference: tensor.norm, tensor.py:169-198; relative_error,
// problems.py:160-169).  b may be NULL.  One pass over the data: the
// difference is formed in registers, so relative_error needs no temporary.
// Fixed grid and fixed reduction order: the result does not depend on timing.
#include "kmb200_kernels.cuh"

namespace kmb {

constexpr int NORM_THREADS = 256;

template <typename T>
__device__ __forceinline__ double2 load_diff(const T* a, const T* b, int64_t i) {
  double2 x = widen(a[i]);
  if (b) {
    const double2 y = widen(b[i]);
    x.x -= y.x;
    x.y -= y.y;
  }
  return x;
}

template <typename T, int KIND>
__global__ void __launch_bounds__(NORM_THREADS) norm_partial_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                                    int64_t n, const OpDev w, double* partials) {
  double acc = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NORM_THREADS;
  int64_t i = blockIdx.x * static_cast<int64_t>(NORM_THREADS) + threadIdx.x;
  if constexpr (KIND == 2) {
    // (l, i_last) = (i mod inner, i / inner) advanced incrementally: one
    // division per thread instead of one per element
    const double* wl = w.w[w.d - 1];
    const int64_t qs = stride / w.inner, rs = stride - qs * w.inner;
    int64_t il = i / w.inner, l = i - il * w.inner;
    auto advance = [&](int64_t& l_, int64_t& il_) {
      l_ += rs;
      il_ += qs;
      if (l_ >= w.inner) {
        l_ -= w.inner;
        ++il_;
      }
    };
    for (; i + 3 * stride < n; i += 4 * stride) {  // four elements in flight, fixed fold order
      double2 x[4];
      double wt[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        x[j] = load_diff(a, b, i + j * stride);
        wt[j] = __ldg(w.winner + l) * __ldg(wl + il);
        advance(l, il);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) acc += (x[j].x * x[j].x + x[j].y * x[j].y) * wt[j];
    }
    for (; i < n; i += stride) {
      const double2 x = load_diff(a, b, i);
      acc += (x.x * x.x + x.y * x.y) * (__ldg(w.winner + l) * __ldg(wl + il));
      advance(l, il);
    }
  } else {
    // four independent loads in flight per thread, folded in a fixed order
    for (; i + 3 * stride < n; i += 4 * stride) {
      double2 x[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = load_diff(a, b, i + j * stride);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if constexpr (KIND == 0) acc = fmax(acc, hypot(x[j].x, x[j].y));
        else acc += x[j].x * x[j].x + x[j].y * x[j].y;
      }
    }
    for (; i < n; i += stride) {
      const double2 x = load_diff(a, b, i);
      if constexpr (KIND == 0) acc = fmax(acc, hypot(x.x, x.y));
      else acc += x.x * x.x + x.y * x.y;
    }
  }
  __shared__ double red[NORM_THREADS / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_down_sync(0xffffffffu, acc, off);
    acc = KIND == 0 ? fmax(acc, o) : acc + o;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = red[0];
    for (int k = 1; k < NORM_THREADS / 32; ++k) r = KIND == 0 ? fmax(r, red[k]) : r + red[k];
    partials[blockIdx.x] = r;
  }
}

// One warp: lane j folds partials j, j+32, ... in order, then a fixed
// shuffle tree; the order never depends on timing.
template <int KIND>
__global__ void norm_final_kernel(const double* __restrict__ partials, int np, double* out) {
  double r = 0.0;
  for (int k = threadIdx.x; k < np; k += 32) r = KIND == 0 ? fmax(r, partials[k]) : r + partials[k];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_down_sync(0xffffffffu, r, off);
    r = KIND == 0 ? fmax(r, o) : r + o;
  }
  if (threadIdx.x == 0) out[0] = KIND == 0 ? r : sqrt(r);
}

int norm_blocks() { return 4 * num_sms(); }

template <typename T, int KIND>
int norm_t(const void* a, const void* b, int64_t n, const OpDev& w, double* out, double* ws, cudaStream_t st) {
  const int nb = norm_blocks();
  norm_partial_kernel<T, KIND><<<nb, NORM_THREADS, 0, st>>>(static_cast<const T*>(a), static_cast<const T*>(b), n, w,
                                                             ws);
  norm_final_kernel<KIND><<<1, 32, 0, st>>>(ws, nb, out);
  return check_launch("norm kernels");
}

template <typename T>
int norm_kind(const void* a, const void* b, int64_t n, int kind, const OpDev& w, double* out, double* ws,
              cudaStream_t st) {
  if (kind == 0) return norm_t<T, 0>(a, b, n, w, out, ws, st);
  if (kind == 1) return norm_t<T, 1>(a, b, n, w, out, ws, st);
  return norm_t<T, 2>(a, b, n, w, out, ws, st);
}

}  // namespace kmb

using namespace kmb;

extern "C" size_t km_norm_workspace_bytes(void) { return static_cast<size_t>(norm_blocks()) * sizeof(double); }

extern "C" int km_norm(const void* a, const void* b, int dtype, int64_t n, int kind, const km_pointop* weights,
                       double* result, void* workspace, size_t workspace_bytes, void* stream) {
  if (!a || !result) return fail(KM_EINVAL, "km_norm: NULL pointer");
  if (kind < 0 || kind > 2) return fail(KM_EINVAL, "km_norm: unknown kind %d", kind);
  if (!workspace || workspace_bytes < km_norm_workspace_bytes())
    return fail(KM_EINVAL, "km_norm: workspace smaller than %zu bytes", km_norm_workspace_bytes());
  OpDev w;
  memset(&w, 0, sizeof(w));
  if (kind == 2) {
    if (!weights || weights->d < 2 || !weights->inner_weights || !weights->weights[weights->d - 1])
      return fail(KM_EINVAL, "km_norm: weighted_two needs d >= 2, inner weights and the last direction's weights");
    w = to_dev(weights);
    int64_t total = w.inner * weights->dims[weights->d - 1];
    if (total != n) return fail(KM_EINVAL, "km_norm: weight extents do not match %lld elements", (long long)n);
  }
  if (n <= 0) return fail(KM_EINVAL, "km_norm: empty tensor");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* ws = static_cast<double*>(workspace);
  switch (dtype) {
    case KM_F32: return norm_kind<float>(a, b, n, kind, w, result, ws, st);
    case KM_F64: return norm_kind<double>(a, b, n, kind, w, result, ws, st);
    case KM_C64: return norm_kind<float2>(a, b, n, kind, w, result, ws, st);
    case KM_C128: return norm_kind<double2>(a, b, n, kind, w, result, ws, st);
    default: return fail(KM_EINVAL, "km_norm: unknown dtype %d", dtype);
  }
}
