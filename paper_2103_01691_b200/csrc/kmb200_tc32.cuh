// mumode_tc32_kernel — complex64 μ-mode product on the 5th-generation tensor
// cores: tcgen05.mma kind::tf32 with the accumulator in TMEM, operands staged
// by TMA, and a 3xTF32 split (hi*hi + lo*hi + hi*lo) that keeps the result at
// fp32 accuracy (plain TF32 misses the 1e-5 complex64 parity bar by ~80x,
// SURVEY §7.3).
//
// The factor E (m x n_mu) is the MMA's A operand (M side, 128 real rows per
// tile = 64 complex rows), the tensor is the B operand (N side):
//   * k-contiguous layout (direction 1, n_left == 1): the tensor's complex
//     interleave lies along k, so both operands are real K-major matrices with
//     K' = 2*n_mu: A = E_blk (2m x 2n_mu, rows 2n+c: [Er -Ei; Ei Er] blocks),
//     B = U (fibers x 2n_mu).  D[2n+c][f] = (cr, ci)[f][n].
//   * fiber-contiguous layout (n_left > 1): the interleave lies along the
//     fibers, so B = U viewed as a real (2*fibers x n_mu) MN-major matrix and
//     A = E' (2m x n_mu, rows 2n: Er, 2n+1: Ei).  D[2n+e][2f+c] = E_e*U_c;
//     cr = D[2n][2f] - D[2n+1][2f+1], ci = D[2n][2f+1] + D[2n+1][2f] is formed
//     in the epilogue with one lane shuffle.
// Both are exactly 4 real multiply-adds per complex multiply-add (x3 for the
// split).  Accuracy: the tensor core's fp32 accumulation loses ~7e-9 relative
// per accumulated k (measured: 1.0e-6 / 1.9e-6 / 3.7e-6 rel. l2 at K' = 128 /
// 256 / 512 against complex128), so one accumulation chain stops at K' = 512.
// HALVES (512 < K' <= 1024, e.g. direction 1 of a 512^3 state): the k-blocks of a
// tile go to two chains, the first half into TMEM columns [0, 256), the second
// into [256, 512); the epilogue folds the first into the second with fp32
// round-to-nearest adds (tcgen05.ld / tcgen05.st) and releases it at once, so
// the next tile's first half runs under the output pass.  Longer contractions
// use the chunked kernel (kmb200_tc32k.cuh).  E's hi/lo planes are prepared
// once per call (prep_planes_kernel); the tensor tile is split in shared memory
// by four transform warps.
//
// CTA pairs (cta_group::2, cluster of 2): a tile is 256 real E rows x 256
// tensor columns; each CTA stages its own 128 E rows and HALF of the tensor
// columns, the leader CTA issues M = 256 / N = 256 MMAs that read both CTAs'
// shared memory, and each CTA's TMEM receives its 128 rows x 256 columns.  The
// tensor operand's shared-memory traffic per SM (TMA writes, hi/lo split, MMA
// reads) halves; with one CTA per tile the kernel was bound by it (tensor pipe
// 75 % of elapsed, now 86 %).
//
// Warp roles (10 warps per CTA): 0 TMA producer, 1 TMEM owner + MMA issuer
// (leader CTA), 2-5 hi/lo transform of the CTA's tensor half, 6-9 epilogue
// (TMEM -> registers -> global).  Split and epilogue warps of both CTAs arrive
// on the leader's barriers; MMA completion is committed to both CTAs
// (multicast).  The grid is persistent; the two 256-column TMEM accumulators
// are double-buffered so the epilogue of tile i overlaps the MMAs of tile i+1.
#pragma once
#include "kmb200_tma.cuh"

namespace kmb {

namespace tc32 {

constexpr int BMR = 128;   // real rows of D per CTA (64 complex rows of E); a CTA pair covers 256
constexpr int BNR = 256;   // real columns of D per tile (one N=256 MMA, shared by the pair)
constexpr int BNH = BNR / 2;  // real columns of B each CTA of the pair stages (cta_group::2 splits N)
constexpr int BKR = 16;    // real k per stage (64 B of fp32: SWIZZLE_64B K-major rows)
constexpr int ST = 6;      // pipeline stages
constexpr int PLANE_A = BMR * BKR * 4;          // 8 KB: 128 x 16 fp32 (E hi or lo)
constexpr int PLANE_B = BNH * BKR * 4;          // 8 KB: 128 x 16 fp32 (tensor raw->hi or lo)
constexpr int OFF_ALO = PLANE_A, OFF_B = 2 * PLANE_A, OFF_BLO = 2 * PLANE_A + PLANE_B;
constexpr int STAGE_BYTES = 2 * PLANE_A + 2 * PLANE_B;
constexpr int TX_BYTES = 2 * PLANE_A + PLANE_B;  // bytes TMA lands per stage and CTA
constexpr int THREADS = 320;
constexpr int XSTAGE = 32 * 128;  // per epilogue warp: one 32 x 32-float (KC) or 16 x 32 (MC) output box
constexpr int SMEM_BYTES = ST * STAGE_BYTES + 1024 + 4 * XSTAGE + 1024;
constexpr int TMEM_COLS = 512;  // two 256-column accumulators

// layout: 4 = SWIZZLE_64B (K-major operands, 64-B rows), 1 = SWIZZLE_128B_BASE32B
// (the only shared-memory layout the tensor core takes for MN-major tf32 operands)
__device__ __forceinline__ uint64_t desc_sw(unsigned saddr, unsigned lbo, unsigned sbo, unsigned layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

// kind::tf32, fp32 accumulate, A K-major, B K- or MN-major, M = 256 (the CTA
// pair: 128 rows of A from each CTA), N = 256 (128 columns of B from each CTA)
__host__ __device__ constexpr uint32_t idesc_tf32(bool b_mn_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((b_mn_major ? 1u : 0u) << 16) | ((BNR >> 3) << 17) |
         (((2 * BMR) >> 4) << 24);
}

// issued by one thread of the pair's leader CTA; reads A and B from both CTAs'
// shared memory and writes each CTA's 128 accumulator rows into its own TMEM
__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(dtmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// MMA completion to the same barrier (offset) in both CTAs of the pair
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          tma::su32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
__device__ __forceinline__ unsigned cta_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
// arrive on the leader CTA's copy of a barrier.  The operands the MMA reads
// were ordered for the tensor core's (async) proxy by fence.proxy.async /
// tcgen05 fences before this; a cluster-scope release here would add a full
// memory barrier per arrive (measured: it halved the kernel's throughput).
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, 0;\n"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n"
      "}\n" ::"r"(tma::su32(bar))
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ float4 lds_f4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f4(unsigned a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void sts_f1(unsigned a, float v) {
  asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ float lds_f1(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ void store3(const CUtensorMap* m, unsigned src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];\n" ::"l"(m),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

}  // namespace tc32

// E's split planes: [KC hi (2m x 2K)][KC lo][MC hi (2m x K)][MC lo], fp32 row-major.
__global__ void prep_planes_kernel(const float2* __restrict__ L, float* __restrict__ planes, int m, int K) {
  const int64_t kc = static_cast<int64_t>(2 * m) * (2 * K);
  const int64_t mc = static_cast<int64_t>(2 * m) * K;
  pdl_wait();  // the planes buffer may still be read by the previous product
  float* kc_hi = planes;
  float* kc_lo = planes + kc;
  float* mc_hi = planes + 2 * kc;
  float* mc_lo = planes + 2 * kc + mc;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < static_cast<int64_t>(m) * K;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(idx / K), k = static_cast<int>(idx % K);
    const float2 e = L[idx];
    const float v[4] = {e.x, -e.y, e.y, e.x};  // E_blk[2n+r][2k+c]: [[Er, -Ei], [Ei, Er]]
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = q >> 1, c = q & 1;
      const int64_t o = static_cast<int64_t>(2 * n + r) * (2 * K) + 2 * k + c;
      const float hi = tc32::tf32_hi(v[q]);
      kc_hi[o] = hi;
      kc_lo[o] = v[q] - hi;
    }
    const float w[2] = {e.x, e.y};  // E'[2n+e][k]
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t o = static_cast<int64_t>(2 * n + q) * K + k;
      const float hi = tc32::tf32_hi(w[q]);
      mc_hi[o] = hi;
      mc_lo[o] = w[q] - hi;
    }
  }
}

template <bool KC, bool HALVES = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc32::THREADS, 1)
    mumode_tc32_kernel(const __grid_constant__ CUtensorMap mapAhi, const __grid_constant__ CUtensorMap mapAlo,
                       const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapOut, int64_t F,
                       int m, int K, int64_t nl) {
  using namespace tc32;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * STAGE_BYTES);
  uint64_t* ready = full + ST;
  uint64_t* empty = ready + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  unsigned char* xstage = smem + ST * STAGE_BYTES + 1024;  // 1024-B aligned (128-B swizzle)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned rank = cta_rank();  // 0 = leader of the CTA pair (issues the MMAs)
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      tma::mbar_init(&full[s], 1);    // this CTA's TMA bytes
      tma::mbar_init(&ready[s], 8);   // leader: 4 split warps of each CTA
      tma::mbar_init(&empty[s], 1);   // MMA commit (multicast to both CTAs)
    }
    for (int b = 0; b < 2; ++b) {
      tma::mbar_init(&tfull[b], 1);   // MMA commit (multicast)
      tma::mbar_init(&tempty[b], 8);  // leader: 4 epilogue warps of each CTA
    }
    tma::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tma::su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  fence_before();
  cluster_sync();  // barriers initialised and TMEM allocated in both CTAs before any remote arrive
  fence_after();
  pdl_wait();  // the previous kernel (prep_planes_kernel, the previous product) is done
  const uint32_t tmem = *tmem_slot;

  const int64_t fib_r = KC ? F : 2 * F;                // real columns of B
  const int nE = (2 * m + 2 * BMR - 1) / (2 * BMR);    // pair tiles along E's real rows (256 each)
  const int64_t nF = (fib_r + BNR - 1) / BNR;          // tiles along the real columns (256 each)
  const int64_t tiles = nE * nF;
  const int64_t pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;
  const int KR = KC ? 2 * K : K;                       // real contraction length
  const int KT = (KR + BKR - 1) / BKR;
  const int64_t my_tiles = tiles > pair ? (tiles - 1 - pair) / pairs + 1 : 0;
  const unsigned sbase = tma::su32(smem);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (each CTA: its A rows, its B half)
    if (lane == 0) {
      tma::prefetch_map(&mapAhi);
      tma::prefetch_map(&mapAlo);
      tma::prefetch_map(&mapB);
      int64_t q = 0;
      for (int64_t it = 0; it < my_tiles; ++it) {
        const int64_t tile = pair + it * pairs;
        const int e0 = static_cast<int>(tile % nE) * 2 * BMR + static_cast<int>(rank) * BMR;
        const int64_t c0 = (tile / nE) * BNR + rank * BNH;
        for (int kt = 0; kt < KT; ++kt, ++q) {
          const int s = static_cast<int>(q % ST);
          if (q >= ST) tma::mbar_wait(&empty[s], static_cast<unsigned>((q / ST - 1) & 1));
          unsigned char* st = smem + s * STAGE_BYTES;
          tma::mbar_expect_tx(&full[s], TX_BYTES);
          const int k0 = kt * BKR;
          tma::load3(st, &mapAhi, &full[s], k0, e0, 0);
          tma::load3(st + OFF_ALO, &mapAlo, &full[s], k0, e0, 0);
          if constexpr (KC) {
            tma::load3(st + OFF_B, &mapB, &full[s], k0, static_cast<int>(c0), 0);
          } else {
            const int64_t f0 = c0 / 2;  // fibers; the pair tile lies inside one n_left slab
            tma::load5(st + OFF_B, &mapB, &full[s], 0, k0, static_cast<int>((f0 % nl) / 16),
                       static_cast<int>(f0 / nl), 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA only)
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(!KC);
      int64_t q = 0;
      // HALVES: k-blocks [0, KH) accumulate into columns [0, 256), [KH, KT) into
      // [256, 512); whole tiles alternate between the two 256-column buffers
      const int KH = (KT + 1) / 2;
      for (int64_t it = 0; it < my_tiles; ++it) {
        for (int h = 0; h < (HALVES ? 2 : 1); ++h) {
          const int b = HALVES ? h : static_cast<int>(it & 1);
          if (HALVES ? it >= 1 : it >= 2)
            tma::mbar_wait(&tempty[b], static_cast<unsigned>((HALVES ? it - 1 : (it >> 1) - 1) & 1));
          fence_after();
          const uint32_t d = tmem + b * BNR;
          const int kb0 = HALVES && h ? KH : 0, kb1 = HALVES && !h ? KH : KT;
          for (int kt = kb0; kt < kb1; ++kt, ++q) {
            const int s = static_cast<int>(q % ST);
            tma::mbar_wait(&ready[s], static_cast<unsigned>((q / ST) & 1));
            fence_after();
            const unsigned st = sbase + s * STAGE_BYTES;
#pragma unroll
            for (int ks = 0; ks < BKR / 8; ++ks) {
              // A (E planes): K-major SW64 (8 rows x 64 B atoms, 512 B apart); 8 k = 32 B per step
              const uint64_t ahi = desc_sw(st + ks * 32, 16, 512, 4);
              const uint64_t alo = desc_sw(st + OFF_ALO + ks * 32, 16, 512, 4);
              uint64_t bhi, blo;
              if constexpr (KC) {  // K-major like A
                bhi = desc_sw(st + OFF_B + ks * 32, 16, 512, 4);
                blo = desc_sw(st + OFF_BLO + ks * 32, 16, 512, 4);
              } else {  // MN-major: 32-float column chunks 2048 B apart (LBO), 4-k groups 512 B apart (SBO)
                bhi = desc_sw(st + OFF_B + ks * 1024, 2048, 512, 1);
                blo = desc_sw(st + OFF_BLO + ks * 1024, 2048, 512, 1);
              }
              const uint32_t acc = (kt != kb0 || ks) ? 1u : 0u;
              mma_tf32(d, ahi, bhi, idesc, acc);
              mma_tf32(d, alo, bhi, idesc, 1u);
              mma_tf32(d, ahi, blo, idesc, 1u);
            }
            commit_pair(&empty[s]);
          }
          commit_pair(&tfull[b]);
        }
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ hi/lo split of this CTA's tensor half
    const int tt = threadIdx.x - 64;  // 0..127
    int64_t q = 0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      for (int kt = 0; kt < KT; ++kt, ++q) {
        const int s = static_cast<int>(q % ST);
        tma::mbar_wait(&full[s], static_cast<unsigned>((q / ST) & 1));
        const unsigned raw = sbase + s * STAGE_BYTES + OFF_B + tt * 16;
        const unsigned lo = sbase + s * STAGE_BYTES + OFF_BLO + tt * 16;
        constexpr int J = PLANE_B / 16 / 128;
        float4 x[J];
#pragma unroll
        for (int j = 0; j < J; ++j) x[j] = tc32::lds_f4(raw + j * 2048);
        // The tensor core reads an fp32 operand as tf32 by truncating the low 13
        // mantissa bits (verified: a rounding reader would leave ~5e-4 errors in
        // tests/test_gpu_tc32.py).  So the raw tile already is "hi" and only
        // lo = x - trunc(x) (exact in fp32) is written.
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const float4 h = make_float4(__uint_as_float(__float_as_uint(x[j].x) & 0xFFFFE000u),
                                       __uint_as_float(__float_as_uint(x[j].y) & 0xFFFFE000u),
                                       __uint_as_float(__float_as_uint(x[j].z) & 0xFFFFE000u),
                                       __uint_as_float(__float_as_uint(x[j].w) & 0xFFFFE000u));
          tc32::sts_f4(lo + j * 2048, make_float4(x[j].x - h.x, x[j].y - h.y, x[j].z - h.z, x[j].w - h.w));
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) arrive_leader(&ready[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // TMEM (this CTA's 128 rows x 256 columns) -> registers -> swizzled shared
    // staging (4 KB per warp) -> TMA store.  The staging layout is the output
    // box with the 128-B swizzle, so the staging writes are bank-conflict free
    // (KC) or 2-way (MC).
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
    const unsigned stg = tma::su32(xstage) + (warp - 6) * XSTAGE;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int64_t tile = pair + it * pairs;
      const int e0 = static_cast<int>(tile % nE) * 2 * BMR + static_cast<int>(rank) * BMR;
      const int64_t c0 = (tile / nE) * BNR;
      int b = static_cast<int>(it & 1);
      if constexpr (HALVES) {
        // fold the first half's accumulator into the second's (fp32 round-to-
        // nearest adds, tcgen05.st) and release it at once, so the next tile's
        // first half overlaps the output pass below
        b = 1;
        const uint32_t lanes = static_cast<uint32_t>(quarter * 32) << 16;
        tma::mbar_wait(&tfull[0], static_cast<unsigned>(it & 1));
        tma::mbar_wait(&tfull[1], static_cast<unsigned>(it & 1));
        fence_after();
#pragma unroll 1
        for (int ch = 0; ch < BNR / 32; ++ch) {
          float v0[32], v1[32];
          ld32(tmem + lanes + ch * 32, v0);
          ld32(tmem + lanes + BNR + ch * 32, v1);
#pragma unroll
          for (int j = 0; j < 32; ++j) v1[j] += v0[j];
          st32(tmem + lanes + BNR + ch * 32, v1);
        }
        st_wait();
        fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(&tempty[0]);
        fence_after();
      } else {
        tma::mbar_wait(&tfull[b], static_cast<unsigned>((it >> 1) & 1));
        fence_after();
      }
      const int nbase = (e0 >> 1) + quarter * 16;  // first output row (complex) of this warp
#pragma unroll 1
      for (int ch = 0; ch < BNR / 32; ++ch) {
        float v[32];
        ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + b * BNR + ch * 32, v);
        if (lane == 0) tc32::bulk_wait_read();  // the previous store from this staging buffer has read it
        __syncwarp();
        if constexpr (KC) {
          // D[2n+part][f]: lane = 2n'+part = the float column of the (f, 16 complex n) box
#pragma unroll
          for (int j = 0; j < 32; ++j)
            tc32::sts_f1(stg + j * 128 + ((((lane >> 2) ^ (j & 7))) << 4) + (lane & 3) * 4, v[j]);
        } else {
          // columns 2f+c; cr = D[2n][2f] - D[2n+1][2f+1], ci = D[2n][2f+1] + D[2n+1][2f]
          const int np = lane >> 1, part = lane & 1;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float x = __shfl_xor_sync(0xffffffffu, v[2 * j + 1], 1);
            const int c = 2 * j + part;
            tc32::sts_f1(stg + np * 128 + ((((c >> 2) ^ (np & 7))) << 4) + (c & 3) * 4,
                         part ? v[2 * j] + x : v[2 * j] - x);
          }
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          if constexpr (KC) {
            tc32::store3(&mapOut, stg, 2 * nbase, static_cast<int>(c0 + ch * 32), 0);
          } else {
            const int64_t ft = c0 / 2 + ch * 16, r = ft / nl;  // the tile lies inside one n_left slab
            tc32::store3(&mapOut, stg, static_cast<int>(2 * (ft - r * nl)), nbase, static_cast<int>(r));
          }
          tc32::bulk_commit();
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(&tempty[b]);
    }
    if (lane == 0) tc32::bulk_wait_all();
  }
  fence_before();
  cluster_sync();  // the peer's MMAs and arrivals are done before TMEM goes away
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
}

}  // namespace kmb
