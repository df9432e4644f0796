// mumode_plane12_kernel — the first two μ-mode products of a small d = 3
// complex128 step, fused per i3-plane (SURVEY §8 north star (1): the d sweeps
// of one exponential step fused to cut round trips).
//
// For a state u (n1 x n2 x n3, column-major) and square factors E1 (n1 x n1),
// E2 (n2 x n2), both products act inside one i3-plane:
//     w(:, :, z) = E1 · u(:, :, z) · E2ᵀ          (tensor.py:143-166, μ = 1, 2)
// so a CTA that holds the plane in shared memory can apply both without the
// intermediate leaving the SM.  The plane's rows are split between `split`
// CTAs: CTA (z, h) computes rows [h·R, (h+1)·R) of w(:, :, z), R = n1 / split,
// because row block r of E1·U·E2ᵀ needs only E1's rows r (plus all of U and
// E2).  The grid is n3 · split CTAs, one wave for the small states this is
// for (64³: 64 planes x 2 = 128 CTAs on 148 SMs).
//
// Per CTA: cp.async loads of E1's R rows and the plane U (group 0) and of E2
// (group 1, in flight during the first product); T = E1[r,:] · U into shared
// memory; w = T · E2ᵀ straight to global.  Both are DMMA.8x8x4 complex
// products (4 real MMAs per complex MMA) with 16x16 warp tiles.  Every shared
// matrix is stored as rows of up to 64 complex values (1 KB) with the 16-B
// chunk swizzle chunk ^= row % 8 and read with the k permutation of the TMA
// kernel (lane t at k-step s reads k = 8(s/2) + 2t + s%2), which keeps the
// LDS.128 fragment reads and the STS.128 of T conflict free.
//
// The third product (direction 3 mixes planes) stays a separate launch.
#pragma once
#include "kmb200_kernels.cuh"

namespace kmb {
namespace plane {

constexpr int THREADS = 256;
constexpr int ROW_BYTES = 1024;  // 64 complex128 per shared row

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned off(int row, int k) {
  return static_cast<unsigned>(row * ROW_BYTES + (k >> 3) * 128 + (((k & 7) ^ (row & 7)) << 4));
}
__device__ __forceinline__ double2 lds(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(unsigned a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(a), "d"(x), "d"(y) : "memory");
}

// 16x16 complex warp tile: C[rows ra.., cols cb..] += A[ra.., :K] · B[cb.., :K]ᵀ
// (A and B both stored row = output index, k along the row)
template <int K>
__device__ __forceinline__ void warp_tile(unsigned A, unsigned B, int ra, int cb, int g, int t, double (&cr)[2][2][2],
                                          double (&ci)[2][2][2]) {
#pragma unroll 4
  for (int s = 0; s < K / 4; ++s) {
    const int k = (s >> 1) * 8 + 2 * t + (s & 1);
    double2 a[2], b[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = lds(A + off(ra + 8 * i + g, k));
#pragma unroll
    for (int j = 0; j < 2; ++j) b[j] = lds(B + off(cb + 8 * j + g, k));
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        dmma(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
        dmma(ci[i][j][0], ci[i][j][1], a[i].x, b[j].y);
      }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        dmma(cr[i][j][0], cr[i][j][1], a[i].y, -b[j].y);
        dmma(ci[i][j][0], ci[i][j][1], a[i].y, b[j].x);
      }
  }
}

}  // namespace plane

// N1 = n1, N2 = n2 (multiples of 16, <= 64); R = N1 / split rows per CTA (a multiple of 16)
template <int N1, int N2>
__global__ void __launch_bounds__(plane::THREADS, 1)
    mumode_plane12_kernel(const double2* __restrict__ u, const double2* __restrict__ E1,
                          const double2* __restrict__ E2, double2* __restrict__ out, int split) {
  using namespace plane;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int R = N1 / split;
  const int64_t z = blockIdx.x / split;
  const int r0 = static_cast<int>(blockIdx.x % split) * R;
  // shared: U (N2 rows: i2, k = i1), E1 rows (R rows: r, k = i1), E2 (N2 rows: j, k = i2), T (R rows: r, k = i2)
  unsigned char* sU = smem_raw;
  unsigned char* sA = sU + N2 * ROW_BYTES;
  unsigned char* sE2 = sA + R * ROW_BYTES;
  unsigned char* sT = sE2 + N2 * ROW_BYTES;
  const unsigned aU = su32(sU), aA = su32(sA), aE2 = su32(sE2), aT = su32(sT);

  pdl_wait();  // the previous launch's output may be this one's input
  const double2* up = u + z * (static_cast<int64_t>(N1) * N2);
  for (int e = threadIdx.x; e < R * N1; e += THREADS) {  // E1 rows r0.., row-major
    const int r = e / N1, k = e - r * N1;
    cp_async<16>(sA + off(r, k), E1 + static_cast<int64_t>(r0 + r) * N1 + k, true);
  }
  for (int e = threadIdx.x; e < N1 * N2; e += THREADS) {  // plane: i1 fastest
    const int i2 = e / N1, i1 = e - i2 * N1;
    cp_async<16>(sU + off(i2, i1), up + e, true);
  }
  cp_commit();
  for (int e = threadIdx.x; e < N2 * N2; e += THREADS) {  // E2, row-major
    const int j = e / N2, k = e - j * N2;
    cp_async<16>(sE2 + off(j, k), E2 + e, true);
  }
  cp_commit();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int tiles_c = N2 / 16;
  const int tiles = (R / 16) * tiles_c;

  cp_wait<1>();
  __syncthreads();
  // T = E1[r0.., :] · U  (rows r, cols i2, k = i1)
  for (int w = warp; w < tiles; w += THREADS / 32) {
    const int ra = (w / tiles_c) * 16, cb = (w % tiles_c) * 16;
    double cr[2][2][2] = {}, ci[2][2][2] = {};
    warp_tile<N1>(aA, aU, ra, cb, g, t, cr, ci);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) sts(aT + off(ra + 8 * i + g, cb + 8 * j + 2 * t + h), cr[i][j][h], ci[i][j][h]);
  }
  cp_wait<0>();
  __syncthreads();
  // w = T · E2ᵀ  (rows r, cols j, k = i2) -> out(r0 + r, j, z)
  double2* op = out + z * (static_cast<int64_t>(N1) * N2);
  for (int w = warp; w < tiles; w += THREADS / 32) {
    const int ra = (w / tiles_c) * 16, cb = (w % tiles_c) * 16;
    double cr[2][2][2] = {}, ci[2][2][2] = {};
    warp_tile<N2>(aT, aE2, ra, cb, g, t, cr, ci);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + ra + 8 * i + g, col = cb + 8 * j + 2 * t + h;
          KMB_ASSERT(r < N1 && col < N2);
          op[r + static_cast<int64_t>(N1) * col] = make_double2(cr[i][j][h], ci[i][j][h]);
        }
  }
}

// mumode_pencil33_kernel — two products along the trailing direction of a small
// complex128 state fused per block of fibers: w = (u ×₃ Ea) ×₃ Eb, i.e. for the
// F (32, or 16 when that leaves too few CTAs) fibers f0.. of the CTA (fibers =
// (i1, i2), contiguous in memory)
//     Y1 = X · Eaᵀ,  Y2 = Y1 · Ebᵀ     (X[f][k] = u(f0 + f, k), k = i3)
// with X, Ea, Eb and Y1 in shared memory (the layout and warp tiles of the
// plane kernel).  km_steps_paired runs the third products of two consecutive
// steps with it (tensor.py:143-166 twice along μ = 3).
template <int N3, int F>
__global__ void __launch_bounds__(plane::THREADS, 1)
    mumode_pencil33_kernel(const double2* __restrict__ u, const double2* __restrict__ Ea,
                           const double2* __restrict__ Eb, double2* __restrict__ out, int64_t nfib) {
  using namespace plane;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sX = smem_raw;              // F rows: f, k = i3
  unsigned char* sY = sX + F * ROW_BYTES;    // F rows: f, k = j (the first product)
  unsigned char* sA = sY + F * ROW_BYTES;    // N3 rows: Ea
  unsigned char* sB = sA + N3 * ROW_BYTES;   // N3 rows: Eb (aliases Ea when Eb == Ea)
  const bool same = (Ea == Eb);
  if (same) sB = sA;
  const unsigned aX = su32(sX), aY = su32(sY), aA = su32(sA), aB = su32(sB);
  const int64_t f0 = static_cast<int64_t>(blockIdx.x) * F;

  pdl_wait();
  for (int e = threadIdx.x; e < F * N3; e += THREADS) {  // X: F contiguous fibers per k
    const int k = e / F, f = e - k * F;
    cp_async<16>(sX + off(f, k), u + f0 + f + k * nfib, true);
  }
  for (int e = threadIdx.x; e < N3 * N3; e += THREADS) {  // Ea, row-major
    const int j = e / N3, k = e - j * N3;
    cp_async<16>(sA + off(j, k), Ea + e, true);
  }
  cp_commit();
  if (!same) {
    for (int e = threadIdx.x; e < N3 * N3; e += THREADS) {
      const int j = e / N3, k = e - j * N3;
      cp_async<16>(sB + off(j, k), Eb + e, true);
    }
  }
  cp_commit();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  constexpr int TC = N3 / 16, TILES = (F / 16) * TC;
  cp_wait<1>();
  __syncthreads();
  for (int w = warp; w < TILES; w += THREADS / 32) {  // Y1 = X · Eaᵀ
    const int ra = (w / TC) * 16, cb = (w % TC) * 16;
    double cr[2][2][2] = {}, ci[2][2][2] = {};
    warp_tile<N3>(aX, aA, ra, cb, g, t, cr, ci);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) sts(aY + off(ra + 8 * i + g, cb + 8 * j + 2 * t + h), cr[i][j][h], ci[i][j][h]);
  }
  cp_wait<0>();
  __syncthreads();
  for (int w = warp; w < TILES; w += THREADS / 32) {  // Y2 = Y1 · Ebᵀ -> out(f0 + f, j)
    const int ra = (w / TC) * 16, cb = (w % TC) * 16;
    double cr[2][2][2] = {}, ci[2][2][2] = {};
    warp_tile<N3>(aY, aB, ra, cb, g, t, cr, ci);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int f = ra + 8 * i + g, col = cb + 8 * j + 2 * t + h;
          KMB_ASSERT(f0 + f < nfib && col < N3);
          out[f0 + f + col * nfib] = make_double2(cr[i][j][h], ci[i][j][h]);
        }
  }
}

constexpr int pencil33_smem(int n3, int f) { return (2 * f + 2 * n3) * plane::ROW_BYTES; }

// shared bytes of one CTA computing r of the n1 rows
constexpr int plane12_smem(int r, int n2) { return (2 * n2 + 2 * r) * plane::ROW_BYTES; }

// km_tucker's fused path: plane12_supported() says whether the kernel covers the
// shape under the current policy (n1, n2 in {32, 48, 64} and a row split that fits);
// launch_plane12 needs 16-B aligned pointers and out != u
bool plane12_supported(int64_t n1, int64_t n2, int64_t n3);  // the shape, and KM_POLICY_NO_PLANE_FUSION unset
bool plane12_shape_ok(int64_t n1, int64_t n2, int64_t n3);   // the shape alone (km_steps_paired)
// two trailing-direction products on blocks of 16 or 32 fibers (nfib % 32 == 0, n3 in {32, 48, 64})
bool pencil33_supported(int64_t nfib, int64_t n3);
int launch_pencil33(const void* u, const void* Ea, const void* Eb, void* out, int64_t nfib, int64_t n3,
                    cudaStream_t st);
int launch_plane12(const void* u, const void* E1, const void* E2, void* out, int64_t n1, int64_t n2, int64_t n3,
                   cudaStream_t st);

}  // namespace kmb
