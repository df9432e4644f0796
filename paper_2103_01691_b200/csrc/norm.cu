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
    // 2-D walk (norm_grid2): x over l = the directions 1..d-1 (U coalesced
    // columns per thread, their inner weights loaded once), y over i_last (its
    // weight loaded once per row); the weight product is w_inner[l] * w_last
    // as in the reference (problems.py:528-539).  Fixed order per thread.
    constexpr int U = 4;
    const double* wl = w.w[w.d - 1];
    const int64_t nlast = n / w.inner;
    for (int64_t l0 = blockIdx.x * static_cast<int64_t>(NORM_THREADS * U) + threadIdx.x; l0 < w.inner;
         l0 += static_cast<int64_t>(gridDim.x) * NORM_THREADS * U) {
      double wf[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t l = l0 + u * NORM_THREADS;
        wf[u] = l < w.inner ? __ldg(w.winner + l) : 0.0;
      }
      for (int64_t il = blockIdx.y; il < nlast; il += gridDim.y) {
        const double wlast = __ldg(wl + il);
        const int64_t base = il * w.inner;
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t l = l0 + u * NORM_THREADS;
          x[u] = l < w.inner ? load_diff(a, b, base + l) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += (x[u].x * x[u].x + x[u].y * x[u].y) * (wf[u] * wlast);
      }
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
    partials[blockIdx.y * gridDim.x + blockIdx.x] = r;
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

// weighted_two grid: x blocks over the inner index (<= what 4 coalesced columns per
// thread need), y blocks over the last direction, x * y <= norm_blocks() partials
dim3 norm_grid2(const OpDev& w, int64_t n) {
  const int nb = norm_blocks();
  int64_t gx = (w.inner + NORM_THREADS * 4 - 1) / (NORM_THREADS * 4);
  if (gx > nb) gx = nb;
  int64_t gy = nb / gx;
  const int64_t nlast = n / w.inner;
  if (gy > nlast) gy = nlast;
  if (gy > 65535) gy = 65535;
  return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
}

template <typename T, int KIND>
int norm_t(const void* a, const void* b, int64_t n, const OpDev& w, double* out, double* ws, cudaStream_t st) {
  const dim3 grid = KIND == 2 ? norm_grid2(w, n) : dim3(norm_blocks());
  const int nb = static_cast<int>(grid.x * grid.y);
  norm_partial_kernel<T, KIND><<<grid, NORM_THREADS, 0, st>>>(static_cast<const T*>(a), static_cast<const T*>(b), n,
                                                               w, ws);
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

// the epilogue two-norm's fold: slot count in ws[0] (written by the product), slots
// ws[1..count] folded as norm_final_kernel does (fixed order: deterministic)
__global__ void norm_epilogue_final_kernel(const double* __restrict__ ws, double* out) {
  const long long np = *reinterpret_cast<const long long*>(ws);
  double r = 0.0;
  for (long long k = threadIdx.x; k < np; k += 32) r += ws[1 + k];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) r += __shfl_down_sync(0xffffffffu, r, off);
  if (threadIdx.x == 0) out[0] = sqrt(r);
}

int64_t norm_epilogue_slots(int64_t m, int64_t fibers) {
  // the finest tiling any product kernel uses: 16 x 16 tiles of four 8 x 8 warp tiles
  const int64_t fine = ((fibers + 15) / 16) * ((m + 15) / 16) * 4;
  const int64_t floor_ = norm_blocks() + 32;  // the separate-pass fallback's partials
  return 1 + (fine > floor_ ? fine : floor_);
}

// after a product whose epilogue accumulated the norm (or, when the op was not fused,
// a separate pass over `out`): *op->norm_result
int norm_epilogue_finish(const km_pointop* op, bool fused, const void* out, int out_dt, int64_t n, cudaStream_t st) {
  if (!op || !op->norm_result) return KM_OK;
  if (op->norm_ws_count < norm_epilogue_slots(1, 1))
    return fail(KM_EINVAL, "epilogue norm: workspace of %lld slots, %lld needed", (long long)op->norm_ws_count,
                (long long)norm_epilogue_slots(1, 1));
  if (fused) {
    norm_epilogue_final_kernel<<<1, 32, 0, st>>>(op->norm_ws, op->norm_result);
    return check_launch("norm_epilogue_final_kernel");
  }
  OpDev none;
  memset(&none, 0, sizeof(none));
  double* ws = op->norm_ws;
  switch (out_dt) {
    case KM_F32: return norm_t<float, 1>(out, nullptr, n, none, op->norm_result, ws, st);
    case KM_F64: return norm_t<double, 1>(out, nullptr, n, none, op->norm_result, ws, st);
    case KM_C64: return norm_t<float2, 1>(out, nullptr, n, none, op->norm_result, ws, st);
    default: return norm_t<double2, 1>(out, nullptr, n, none, op->norm_result, ws, st);
  }
}

}  // namespace kmb

using namespace kmb;

extern "C" int64_t km_norm_epilogue_slots(int64_t m, int64_t fibers) { return norm_epilogue_slots(m, fibers); }

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
