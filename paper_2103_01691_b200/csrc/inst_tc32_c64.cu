// Host side of the tcgen05 complex64 μ-mode product: factor planes, TMA maps, launch.
#include "kmb200_tc32k.cuh"

#include <cudaTypedefs.h>

namespace kmb {

#ifndef KMB_TC_HALVES_MIN
#define KMB_TC_HALVES_MIN 512  // K' above which a tile accumulates in two chains
#endif
bool g_tc_halves_disabled = false;  // A/B switch (KMB200_TC_HALVES=0): K' in (512, 1024] on the chunked kernel

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn32() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool map_f32(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
             const cuuint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn32();
  if (!fn) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Persistent launch of a CTA-pair kernel: one pair per (2*BMR) E rows x BNR
// tensor columns, the grid sized by the clusters that can be co-resident
// (not every SM can host half of a pair: TPCs with one usable SM).
template <typename Kern>
int launch_pairs(Kern kern, int smem, int threads, int64_t tiles, const char* what, const CUtensorMap& ahi,
                 const CUtensorMap& alo, const CUtensorMap& b, const CUtensorMap& mo, int64_t F, int m, int K,
                 int64_t nl, cudaStream_t st) {
  // co-resident pairs, memoised per device (key: the kernel's address + 1, distinct
  // from the shared-memory opt-in's key)
  const void* key = reinterpret_cast<const char*>(reinterpret_cast<const void*>(kern)) + 1;
  int max_pairs = 0;
  if (!memo_get(key, &max_pairs)) {
    if (int rc = ensure_smem(reinterpret_cast<const void*>(kern), smem, what)) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (num_sms() / 2));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr_c;
    attr_c.id = cudaLaunchAttributeClusterDimension;
    attr_c.val.clusterDim.x = 2;
    attr_c.val.clusterDim.y = 1;
    attr_c.val.clusterDim.z = 1;
    cfg.attrs = &attr_c;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) n = num_sms() / 2;
    max_pairs = n;
    memo_put(key, n);
  }
  const int64_t pairs = tiles < max_pairs ? tiles : max_pairs;
  const cudaError_t e = launch_pdl(kern, dim3(static_cast<unsigned>(2 * pairs)), dim3(threads), smem, st, ahi, alo,
                                   b, mo, F, m, K, nl);
  if (e != cudaSuccess) return fail(KM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return check_launch(what);
}

template <bool KC>
int launch(const CUtensorMap& ahi, const CUtensorMap& alo, const CUtensorMap& b, const CUtensorMap& mo, int64_t F,
           int m, int K, int64_t nl, bool chunked, cudaStream_t st) {
  const int64_t fib_r = KC ? F : 2 * F;
  if (chunked) {
    const int64_t tiles = ((2 * m + 2 * tc32k::BMR - 1) / (2 * tc32k::BMR)) * ((fib_r + tc32k::BNR - 1) / tc32k::BNR);
    return launch_pairs(mumode_tc32_chunk_kernel<KC>, tc32k::SMEM_BYTES, tc32k::THREADS, tiles,
                        "mumode_tc32_chunk_kernel", ahi, alo, b, mo, F, m, K, nl, st);
  }
  const int64_t tiles = ((2 * m + 2 * tc32::BMR - 1) / (2 * tc32::BMR)) * ((fib_r + tc32::BNR - 1) / tc32::BNR);
  if ((KC ? 2 * K : K) > KMB_TC_HALVES_MIN) {  // two accumulation chains per tile
    return launch_pairs(mumode_tc32_kernel<KC, true>, tc32::SMEM_BYTES, tc32::THREADS, tiles,
                        "mumode_tc32_kernel (halves)", ahi, alo, b, mo, F, m, K, nl, st);
  }
  return launch_pairs(mumode_tc32_kernel<KC>, tc32::SMEM_BYTES, tc32::THREADS, tiles, "mumode_tc32_kernel", ahi,
                      alo, b, mo, F, m, K, nl, st);
}

}  // namespace

size_t tc32_workspace_bytes(int64_t m, int64_t K) { return static_cast<size_t>(12 * m * K) * sizeof(float) + 256; }

// Returns -1 when the shape is not eligible (caller falls back to the DMMA path).
int launch_tc32_c64(const void* u, const void* L, void* out, int64_t m, int64_t nl, int64_t K, int64_t nr, void* ws,
                    size_t ws_bytes, cudaStream_t st) {
  const bool kc = (nl == 1);
  const int64_t F = nl * nr;
  if (!ws || ws_bytes < tc32_workspace_bytes(m, K)) return -1;
  if ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(ws)) & 15) return -1;
  if (K % 4 != 0 || m % 2 != 0 || m > (1 << 20) || K > (1 << 20)) return -1;
  if (reinterpret_cast<uintptr_t>(out) & 15) return -1;
  // K' <= 512: one accumulation chain per tile (kmb200_tc32.cuh); K' <= 1024: two
  // chains of <= 512 k' summed in fp32 (the same kernel, HALVES); longer
  // contractions use the chunked kernel, whose chains stay at 64 k' (kmb200_tc32k.cuh)
  const bool chunked = (kc ? 2 * K : K) > (g_tc_halves_disabled ? 512 : 1024);
  const int64_t tile_fibers = (chunked ? tc32k::BNR : tc32::BNR) / 2;
  if (!kc && nl % tile_fibers != 0) return -1;  // a pair tile's fibers lie inside one slab
  if (F >= (int64_t(1) << 31)) return -1;
  float* planes = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  {
    const int threads = 256;
    int64_t blocks = (m * K + threads - 1) / threads;
    if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
    const cudaError_t e = launch_pdl(prep_planes_kernel, dim3(static_cast<unsigned>(blocks)), dim3(threads), 0, st,
                                     static_cast<const float2*>(L), planes, static_cast<int>(m), static_cast<int>(K));
    if (e != cudaSuccess) return fail(KM_ECUDA, "prep_planes_kernel: %s", cudaGetErrorString(e));
    int rc = check_launch("prep_planes_kernel");
    if (rc) return rc;
  }
  const int64_t kc_plane = 2 * m * 2 * K, mc_plane = 2 * m * K;
  const int64_t KR = kc ? 2 * K : K;
  const float* ahi = kc ? planes : planes + 2 * kc_plane;
  const float* alo = kc ? planes + kc_plane : planes + 2 * kc_plane + mc_plane;
  CUtensorMap mahi, malo, mb;
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(KR), static_cast<cuuint64_t>(2 * m), 1};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(KR) * 4, static_cast<cuuint64_t>(KR) * 4 * 2 * m};
    cuuint32_t box[3] = {tc32::BKR, tc32::BMR, 1};
    if (!map_f32(&mahi, ahi, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B) ||
        !map_f32(&malo, alo, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B))
      return -1;
  }
  if (kc) {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(2 * K), static_cast<cuuint64_t>(F), 1};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(2 * K) * 4, static_cast<cuuint64_t>(2 * K) * 4 * F};
    const cuuint32_t bnh = chunked ? tc32k::BNH : tc32::BNH;  // each CTA of the pair stages half the columns
    cuuint32_t box[3] = {tc32::BKR, bnh, 1};
    if (!map_f32(&mb, u, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B)) return -1;
    // output (F x m complex, row-major in n): boxes of 32 fibers x 16 complex n
    CUtensorMap mo;
    cuuint64_t od[3] = {static_cast<cuuint64_t>(2 * m), static_cast<cuuint64_t>(F), 1};
    cuuint64_t os[2] = {static_cast<cuuint64_t>(2 * m) * 4, static_cast<cuuint64_t>(2 * m) * 4 * F};
    cuuint32_t ob[3] = {32, 32, 1};
    if (!map_f32(&mo, out, 3, od, os, ob)) return -1;
    return launch<true>(mahi, malo, mb, mo, F, static_cast<int>(m), static_cast<int>(K), nl, chunked, st);
  }
  cuuint64_t dims[5] = {32, static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(nl / 16), static_cast<cuuint64_t>(nr),
                        1};
  cuuint64_t strides[4] = {static_cast<cuuint64_t>(nl) * 8, 128, static_cast<cuuint64_t>(nl) * K * 8,
                           static_cast<cuuint64_t>(nl) * K * 8 * nr};
  cuuint32_t box[5] = {32, tc32::BKR, static_cast<cuuint32_t>((chunked ? tc32k::BNH : tc32::BNH) / 32), 1, 1};
  // MN-major tf32 operand: 32-B swizzle atoms (matches the BASE32B descriptor layout)
  if (!map_f32(&mb, u, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return -1;
  // output (n_left x m x n_right complex): boxes of 16 fibers x 16 rows n
  CUtensorMap mo;
  cuuint64_t od[3] = {static_cast<cuuint64_t>(2 * nl), static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(nr)};
  cuuint64_t os[2] = {static_cast<cuuint64_t>(nl) * 8, static_cast<cuuint64_t>(nl) * m * 8};
  cuuint32_t ob[3] = {32, 16, 1};
  if (!map_f32(&mo, out, 3, od, os, ob)) return -1;
  return launch<false>(mahi, malo, mb, mo, F, static_cast<int>(m), static_cast<int>(K), nl, chunked, st);
}

}  // namespace kmb
