// mumode_tc32_chunk_kernel — the tcgen05 complex64 product for long contractions.
//
// The tensor core accumulates tf32 products in fp32 with a truncating adder,
// so the error of one accumulation chain grows with its length (measured
// ~7e-9 relative per k', kmb200_tc32.cuh); mumode_tc32_kernel is therefore only
// used up to K' = 512.  This variant bounds the chain: the MMAs of a tile run
// in chunks of CKB k-blocks (64 k'), each into a fresh TMEM accumulator, and
// the epilogue warps drain every chunk into fp32 registers (round-to-nearest
// adds), so the error stays at the 64-k' level for any K (tests/test_gpu_tc32.py
// checks n_mu up to 1024 against the 1e-5 bar).
//
// Same CTA-pair structure as mumode_tc32_kernel (cta_group::2, leader issues
// M = 256 MMAs, split and epilogue warps of both CTAs arrive on the leader),
// with a 256 x 128 tile: the running sum of 128 columns per TMEM lane fits in
// the epilogue threads' registers, and the two 128-column chunk accumulators
// are double-buffered against the drain.  8 warps (producer, MMA, 2 split,
// 4 epilogue): with 10 warps three of them share a sub-partition's 16K
// registers and the running sums spill.
#pragma once
#include "kmb200_tc32.cuh"

namespace kmb {

namespace tc32k {

constexpr int BMR = 128;                  // real E rows per CTA (the pair covers 256)
constexpr int BNR = 128;                  // real columns of D per tile
constexpr int BNH = BNR / 2;              // tensor columns each CTA stages
constexpr int BKR = 16;                   // real k per stage
constexpr int ST = 8;                     // pipeline stages
constexpr int CKB = 4;                    // k-blocks (of BKR) per accumulation chunk: 64 k'
constexpr int PLANE_A = BMR * BKR * 4;    // 8 KB
constexpr int PLANE_B = BNH * BKR * 4;    // 4 KB
constexpr int OFF_ALO = PLANE_A, OFF_B = 2 * PLANE_A, OFF_BLO = 2 * PLANE_A + PLANE_B;
constexpr int STAGE_BYTES = 2 * PLANE_A + 2 * PLANE_B;
constexpr int TX_BYTES = 2 * PLANE_A + PLANE_B;
constexpr int THREADS = 256;  // 8 warps: 2 per SM sub-partition, so a thread may hold 255 registers
constexpr int XSTAGE = 32 * 128;
constexpr int SMEM_BYTES = ST * STAGE_BYTES + 1024 + 4 * XSTAGE + 1024;
constexpr int TMEM_COLS = 256;            // two 128-column chunk accumulators

__host__ __device__ constexpr uint32_t idesc(bool b_mn_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((b_mn_major ? 1u : 0u) << 16) | ((BNR >> 3) << 17) |
         (((2 * BMR) >> 4) << 24);
}

}  // namespace tc32k

template <bool KC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc32k::THREADS, 1)
    mumode_tc32_chunk_kernel(const __grid_constant__ CUtensorMap mapAhi, const __grid_constant__ CUtensorMap mapAlo,
                             const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapOut,
                             int64_t F, int m, int K, int64_t nl) {
  using namespace tc32k;
  using tc32::arrive_leader;
  using tc32::commit_pair;
  using tc32::desc_sw;
  using tc32::fence_after;
  using tc32::fence_before;
  using tc32::fence_proxy_async;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * STAGE_BYTES);
  uint64_t* ready = full + ST;
  uint64_t* empty = ready + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  unsigned char* xstage = smem + ST * STAGE_BYTES + 1024;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned rank = tc32::cta_rank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&ready[s], 4);   // leader: 2 split warps of each CTA
      tma::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tma::mbar_init(&tfull[b], 1);
      tma::mbar_init(&tempty[b], 8);
    }
    tma::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tma::su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  fence_before();
  tc32::cluster_sync();
  fence_after();
  pdl_wait();  // the previous kernel (prep_planes_kernel, the previous product) is done
  const uint32_t tmem = *tmem_slot;

  const int64_t fib_r = KC ? F : 2 * F;
  const int nE = (2 * m + 2 * BMR - 1) / (2 * BMR);
  const int64_t nF = (fib_r + BNR - 1) / BNR;
  const int64_t tiles = nE * nF;
  const int64_t pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;
  const int KR = KC ? 2 * K : K;
  const int KT = (KR + BKR - 1) / BKR;
  const int NCH = (KT + CKB - 1) / CKB;  // chunks per tile
  const int64_t my_tiles = tiles > pair ? (tiles - 1 - pair) / pairs + 1 : 0;
  const unsigned sbase = tma::su32(smem);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
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
            const int64_t f0 = c0 / 2;
            tma::load5(st + OFF_B, &mapB, &full[s], 0, k0, static_cast<int>((f0 % nl) / 16),
                       static_cast<int>(f0 / nl), 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader): one accumulator per chunk
    if (rank == 0 && lane == 0) {
      constexpr uint32_t id = idesc(!KC);
      int64_t q = 0, c = 0;  // stage counter, chunk counter
      for (int64_t it = 0; it < my_tiles; ++it) {
        for (int ch = 0; ch < NCH; ++ch, ++c) {
          const int b = static_cast<int>(c & 1);
          if (c >= 2) tma::mbar_wait(&tempty[b], static_cast<unsigned>(((c >> 1) - 1) & 1));
          fence_after();
          const uint32_t d = tmem + b * BNR;
          const int kt1 = (ch + 1) * CKB < KT ? (ch + 1) * CKB : KT;
          for (int kt = ch * CKB; kt < kt1; ++kt, ++q) {
            const int s = static_cast<int>(q % ST);
            tma::mbar_wait(&ready[s], static_cast<unsigned>((q / ST) & 1));
            fence_after();
            const unsigned st = sbase + s * STAGE_BYTES;
#pragma unroll
            for (int ks = 0; ks < BKR / 8; ++ks) {
              const uint64_t ahi = desc_sw(st + ks * 32, 16, 512, 4);
              const uint64_t alo = desc_sw(st + OFF_ALO + ks * 32, 16, 512, 4);
              uint64_t bhi, blo;
              if constexpr (KC) {
                bhi = desc_sw(st + OFF_B + ks * 32, 16, 512, 4);
                blo = desc_sw(st + OFF_BLO + ks * 32, 16, 512, 4);
              } else {
                bhi = desc_sw(st + OFF_B + ks * 1024, 2048, 512, 1);
                blo = desc_sw(st + OFF_BLO + ks * 1024, 2048, 512, 1);
              }
              const uint32_t acc = (kt != ch * CKB || ks) ? 1u : 0u;  // fresh accumulator per chunk
              tc32::mma_tf32(d, ahi, bhi, id, acc);
              tc32::mma_tf32(d, alo, bhi, id, 1u);
              tc32::mma_tf32(d, ahi, blo, id, 1u);
            }
            commit_pair(&empty[s]);
          }
          commit_pair(&tfull[b]);
        }
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ hi/lo split of this CTA's tensor half (2 warps)
    const int tt = threadIdx.x - 64;  // 0..63
    int64_t q = 0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      for (int kt = 0; kt < KT; ++kt, ++q) {
        const int s = static_cast<int>(q % ST);
        tma::mbar_wait(&full[s], static_cast<unsigned>((q / ST) & 1));
        const unsigned raw = sbase + s * STAGE_BYTES + OFF_B + tt * 16;
        const unsigned lo = sbase + s * STAGE_BYTES + OFF_BLO + tt * 16;
        constexpr int J = PLANE_B / 16 / 64;
        float4 x[J];
#pragma unroll
        for (int j = 0; j < J; ++j) x[j] = tc32::lds_f4(raw + j * 1024);
#pragma unroll
        for (int j = 0; j < J; ++j) {  // lo = x - trunc_tf32(x), exact (see mumode_tc32_kernel)
          const float4 h = make_float4(__uint_as_float(__float_as_uint(x[j].x) & 0xFFFFE000u),
                                       __uint_as_float(__float_as_uint(x[j].y) & 0xFFFFE000u),
                                       __uint_as_float(__float_as_uint(x[j].z) & 0xFFFFE000u),
                                       __uint_as_float(__float_as_uint(x[j].w) & 0xFFFFE000u));
          tc32::sts_f4(lo + j * 1024, make_float4(x[j].x - h.x, x[j].y - h.y, x[j].z - h.z, x[j].w - h.w));
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) arrive_leader(&ready[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ drain chunks into fp32 registers, then store
    const int quarter = warp & 3;  // warps 4-7: TMEM lanes 32*quarter .. +31
    const unsigned stg = tma::su32(xstage) + (warp - 4) * XSTAGE;
    int64_t c = 0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int64_t tile = pair + it * pairs;
      const int e0 = static_cast<int>(tile % nE) * 2 * BMR + static_cast<int>(rank) * BMR;
      const int64_t c0 = (tile / nE) * BNR;
      float tot[BNR];
#pragma unroll
      for (int i = 0; i < BNR; ++i) tot[i] = 0.0f;
      for (int ch = 0; ch < NCH; ++ch, ++c) {
        const int b = static_cast<int>(c & 1);
        tma::mbar_wait(&tfull[b], static_cast<unsigned>((c >> 1) & 1));
        fence_after();
#pragma unroll
        for (int q4 = 0; q4 < BNR / 32; ++q4) {
          float v[32];
          tc32::ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + b * BNR + q4 * 32, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) tot[q4 * 32 + j] = __fadd_rn(tot[q4 * 32 + j], v[j]);
        }
        fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(&tempty[b]);
      }
      const int nbase = (e0 >> 1) + quarter * 16;
#pragma unroll
      for (int q4 = 0; q4 < BNR / 32; ++q4) {
        if (lane == 0) tc32::bulk_wait_read();
        __syncwarp();
        if constexpr (KC) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            tc32::sts_f1(stg + j * 128 + ((((lane >> 2) ^ (j & 7))) << 4) + (lane & 3) * 4, tot[q4 * 32 + j]);
        } else {
          const int np = lane >> 1, part = lane & 1;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float x = __shfl_xor_sync(0xffffffffu, tot[q4 * 32 + 2 * j + 1], 1);
            const int cc = 2 * j + part;
            tc32::sts_f1(stg + np * 128 + ((((cc >> 2) ^ (np & 7))) << 4) + (cc & 3) * 4,
                         part ? tot[q4 * 32 + 2 * j] + x : tot[q4 * 32 + 2 * j] - x);
          }
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          if constexpr (KC) {
            tc32::store3(&mapOut, stg, 2 * nbase, static_cast<int>(c0 + q4 * 32), 0);
          } else {
            const int64_t ft = c0 / 2 + q4 * 16, r = ft / nl;
            tc32::store3(&mapOut, stg, static_cast<int>(2 * (ft - r * nl)), nbase, static_cast<int>(r));
          }
          tc32::bulk_commit();
        }
      }
    }
    if (lane == 0) tc32::bulk_wait_all();
  }
  fence_before();
  tc32::cluster_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
}

}  // namespace kmb
