// mumode_tma_kernel — warp-specialised, persistent complex128 μ-mode GEMM.
//
// Same GEMM view and DMMA arithmetic as mumode_kernel (kmb200_kernels.cuh),
// re-organised for the B200:
//   * TMA tile loads (cp.async.bulk.tensor, 128-B swizzle) for A (the tensor)
//     and B (the factor) into a 4-stage shared-memory ring, issued by ONE lane
//     (warp 0, lane 0) two k-blocks ahead of the compute and signalled on
//     per-stage "full" mbarriers with the expected byte count;
//   * all eight warps wait on "full", run their 4x4-tile DMMA.8x8x4 warp tiles
//     straight out of the swizzled stage, and release the stage with one
//     arrive per warp on its "empty" mbarrier — no __syncthreads in the loop.
//     (A dedicated producer warp puts a third warp on one SM sub-partition
//     and caps every thread at 168 registers; the complex accumulators alone
//     need 128, so only the real x real products, 64 accumulator registers,
//     use one: there it walks the whole ring and takes the load bookkeeping
//     off warp 0, which otherwise paces the CTA — 1.5 % on a 512^3 f64
//     product, tools/ab_probe.py.)
//   * the grid is persistent (one CTA per SM) and walks the tiles with a
//     static stride; the k-block counter runs across tiles, so the loads of
//     tile i+1 are in flight during the epilogue of tile i.
//
// Shared-memory tiles are the TMA boxes, 128-B rows with the hardware
// 16-B-chunk XOR swizzle (chunk ^= row % 8).  The DMMA k index of lane t in
// k-step s is mapped to stage row k = (s/2)*8 + 2t + (s%2) (the same
// permutation for A and B, so the sum is unchanged); with it, the 8 lanes of
// each LDS.128 phase hit 8 different 16-B bank groups — conflict free.
//
// A (tensor) boxes, in f64 elements (one complex = 2):
//   fiber-contiguous (n_left % 128 == 0): dims (16 [8 fibers], k-in-block,
//     n_left/8 fiber groups, n_right, k blocks), box (16, 16, 16, 1, 1)
//     → smem [fiber group][k][8 complex];
//   k-contiguous (n_left == 1): dims (16 [8 k], fibers, K/8), box (16, 128, 2)
//     → smem [k group][fiber][8 complex].
// B (row-major factor): dims (16 [8 k], rows, K/8), box (16, 64, 2)
//     → smem [k group][row][8 complex].
#pragma once
#include "kmb200_kernels.cuh"

#include <cuda.h>

namespace kmb {

#ifndef KMB_EPI_VEC
#define KMB_EPI_VEC 8
#endif
#ifndef KMB_TMA_AHEAD
#define KMB_TMA_AHEAD 2
#endif

namespace tma {

constexpr int BM = 128, BN = 64, BKS = 16, TSTAGES = 4, CONSUMERS = 8;
constexpr int THREADS = 32 * CONSUMERS;
constexpr int AHEAD = KMB_TMA_AHEAD;  // k-blocks between a stage's load and its use
constexpr int A_BYTES = BM * BKS * 16, B_BYTES = BN * BKS * 16, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = TSTAGES * STAGE_BYTES + 2 * TSTAGES * 8 + 1024;
#ifndef KMB_TMA_PRODUCER
#define KMB_TMA_PRODUCER 1
#endif
// a ninth (producer) warp issues the loads instead of warp 0's lane 0:
// 0 none, 1 real x real, 2 every real-factor product, 3 all
template <bool CL, bool CU>
constexpr bool producer_warp() {
  return KMB_TMA_PRODUCER == 3 || (KMB_TMA_PRODUCER == 2 && !CL) || (KMB_TMA_PRODUCER == 1 && !CL && !CU);
}
template <bool CL, bool CU>
constexpr int threads_for() { return THREADS + (producer_warp<CL, CU>() ? 32 : 0); }

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "KMB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra KMB_WAIT_%=;\n"
      "}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ double lds64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void prefetch_map(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(m) : "memory");
}
__device__ __forceinline__ void load3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];\n" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void load5(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3,
                                      int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, "
      "%7}], [%2];\n" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

}  // namespace tma

// Stream-K tail (host: inst_tma_c128.cu).  The first dp_waves * gridDim.x
// tiles are whole tiles, one CTA each; the k-blocks of the remaining tiles are
// cut into gridDim.x equal contiguous ranges, one per CTA, so every CTA does the
// same number of k-blocks.  A tile cut between CTAs is finished by the CTA
// holding its first k-block (the "owner"): the others store their partial
// accumulators (per warp, in piece order) with a release flag, and the owner
// adds them in piece order, so the result does not depend on timing.  The
// launch is cooperative (all CTAs resident), and a CTA only waits at the end
// of its range, after its own partial pieces are published: no cycles.
struct StreamK {
  int64_t dp_waves;  // whole-tile waves before the stream-K range (0 when iters == 0: all tiles whole)
  int64_t sk_base;   // first stream-K tile
  int64_t iters;     // k-blocks in the stream-K range (0 = none)
  double* part;      // partial accumulators: [sk tile][piece-1][warp][64 values][32 lanes]
  unsigned* flags;   // [sk tile][piece-1][warp] == epoch once published
  unsigned epoch;
  int slots;         // pieces per tile - 1
};

// CL = false: real factor (e.g. the Hermite Φ), 2 DMMA per complex multiply-add.
// Its box is (16 real k, 64 rows) in 128-B rows; one LDS.128 fetches the
// factor values of two consecutive k-steps (k = 2c, 2c+1 share a 16-B chunk
// under the k permutation above; 2-way bank conflicts on these reads, which the
// DMMA rate leaves room for: a conflict-free 64-B-swizzled layout measured < 1 %
// faster and was withdrawn).
// CU = false: real tensor (e.g. the f64 pipe-flow state).  Fiber-contiguous
// boxes are (16 fibers, 16 k, 8 fiber groups) in 128-B rows and read with one
// conflict-free LDS.64 per MMA tile; k-contiguous boxes are (16 k, 128 fibers)
// and read in k pairs with LDS.128 like the real factor.
template <bool KC, int OPK, bool CL = true, bool CU = true, bool SKT = false>
__global__ void __launch_bounds__(tma::threads_for<CL, CU>(), 1)
    mumode_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      typename El<double, CU || CL>::T* __restrict__ out, int64_t M, int N, int K, int64_t nl,
                      const OpDev op, const Split sp, const StreamK sk) {
  using namespace tma;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TSTAGES * STAGE_BYTES);
  uint64_t* empty = full + TSTAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], CONSUMERS);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();  // the previous product's output is this one's input

  const int nN = (N + BN - 1) / BN;
  const int64_t tiles = ((M + BM - 1) / BM) * nN;
  const int KT = (K + BKS - 1) / BKS;
  const int64_t S = gridDim.x, cta = blockIdx.x;
  // whole tiles of this CTA, then its stream-K range [sk_b, sk_e) of k-blocks
  // (SKT = false: the stream-K machinery is compiled out, whole tiles only)
  const int64_t n_dp = SKT ? sk.dp_waves : (tiles > cta ? (tiles - 1 - cta) / S + 1 : 0);
  const int64_t sk_b = SKT ? cta * sk.iters / S : 0, sk_e = SKT ? (cta + 1) * sk.iters / S : 0;
  const int64_t total = n_dp * KT + (sk_e - sk_b);  // k-blocks this CTA consumes
  auto sk_cta_of = [&](int64_t x) { return ((x + 1) * S + sk.iters - 1) / sk.iters - 1; };

  // one lane issues the loads of this CTA's k-block q
  // producer cursor (leader lane only): issue() runs for q = 0, 1, 2, ... in
  // order, so the k-block's tile and its TMA coordinates advance incrementally,
  // with the 64-bit divisions done once per tile instead of once per k-block
  int64_t pc_tile = cta, m0 = 0;
  int kt = -1, n0 = 0, a_grp = 0, a_slab = 0;
  auto set_tile = [&](int64_t tile) {
    pc_tile = tile;
    n0 = static_cast<int>(tile % nN) * BN;
    m0 = (tile / nN) * BM;
    if constexpr (!KC) {
      a_grp = static_cast<int>((m0 % nl) / (CU ? 8 : 16));
      a_slab = static_cast<int>(m0 / nl);
    }
  };
  auto issue = [&](int64_t q) {
    const int s = static_cast<int>(q % TSTAGES);
    if (q >= TSTAGES) tma::mbar_wait(&empty[s], static_cast<unsigned>((q / TSTAGES - 1) & 1));
    if (SKT && q == n_dp * KT) {  // first k-block of the stream-K range
      set_tile(sk.sk_base + sk_b / KT);
      kt = static_cast<int>(sk_b % KT);
    } else if (kt < 0) {
      set_tile(cta);
      kt = 0;
    } else if (++kt == KT) {
      kt = 0;
      set_tile(SKT && q > n_dp * KT ? pc_tile + 1 : pc_tile + S);
    }
    unsigned char* st = smem + s * STAGE_BYTES;
    tma::mbar_expect_tx(&full[s], (CU ? A_BYTES : A_BYTES / 2) + (CL ? B_BYTES : B_BYTES / 2));
    const int k0 = kt * BKS;
    if constexpr (KC && !CU) {
      tma::load3(st, &mapA, &full[s], k0, static_cast<int>(m0), 0);
    } else if constexpr (!CU) {
      const int kb = k0 / sp.kcb;
      tma::load5(st, &mapA, &full[s], 0, k0 - kb * sp.kcb, a_grp, a_slab, kb);
    } else if constexpr (KC) {
      tma::load3(st, &mapA, &full[s], 0, static_cast<int>(m0), k0 / 8);
    } else {
      const int kb = k0 / sp.kcb;
      tma::load5(st, &mapA, &full[s], 0, k0 - kb * sp.kcb, a_grp, a_slab, kb);
    }
    if constexpr (CL)
      tma::load3(st + A_BYTES, &mapB, &full[s], 0, n0, k0 / 8);
    else
      tma::load3(st + A_BYTES, &mapB, &full[s], k0, n0, 0);
  };
  constexpr bool PW = tma::producer_warp<CL, CU>();
  const bool leader = !PW && warp == 0 && lane == 0;
  if constexpr (PW) {
    // the producer warp walks the whole ring: a stage is refilled as soon as
    // all consumers have released it
    if (warp == CONSUMERS) {
      if (lane == 0) {
        tma::prefetch_map(&mapA);
        tma::prefetch_map(&mapB);
        for (int64_t q = 0; q < total; ++q) issue(q);
      }
      return;
    }
  } else if (leader) {
    tma::prefetch_map(&mapA);
    tma::prefetch_map(&mapB);
    for (int64_t q = 0; q < AHEAD && q < total; ++q) issue(q);
  }

  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  const int gx = g ^ (2 * t);
  // byte offsets of this lane's fragments inside a stage, for odd/even k-steps
  constexpr unsigned A_I = KC ? 8 * 128 : 16 * 128;     // next 8-row MMA tile
  constexpr unsigned A_KG = KC ? 128 * 128 : 8 * 128;   // next 8-k group
  const unsigned a0 = KC ? (wm + g) * 128 + gx * 16 : ((wm / 8) * 16 + 2 * t) * 128 + gx * 16;
  const unsigned a1 = KC ? (wm + g) * 128 + (gx ^ 1) * 16 : ((wm / 8) * 16 + 2 * t + 1) * 128 + (gx ^ 1) * 16;
  constexpr unsigned B_J = 8 * 128, B_KG = 64 * 128;
  const unsigned b0 = A_BYTES + (wn + g) * 128 + gx * 16;
  const unsigned b1 = A_BYTES + (wn + g) * 128 + (gx ^ 1) * 16;

  const unsigned sbase = tma::su32(smem);
  int64_t q = 0;
  // k-blocks [k0, k1) of one tile, then its epilogue (or its stream-K piece)
  auto run_tile = [&](const int64_t tile, const int k0, const int k1) {
    const int n0 = static_cast<int>(tile % nN) * BN;
    const int64_t m0 = (tile / nN) * BM;
    double cr[4][4][2], ci[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

    for (int kt = k0; kt < k1; ++kt, ++q) {
      if (!PW && leader && q + AHEAD < total) issue(q + AHEAD);
      const int s = static_cast<int>(q % TSTAGES);
      tma::mbar_wait(&full[s], static_cast<unsigned>((q / TSTAGES) & 1));
      const unsigned st = sbase + s * STAGE_BYTES;
      double2 breal[4], areal[4];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        double2 a[4];
        if constexpr (CU) {
          const unsigned ao = ((ks & 1) ? a1 : a0) + (ks >> 1) * A_KG;
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = tma::lds128(st + ao + i * A_I);
        } else if constexpr (KC) {
          // real, k-contiguous: row f = wm + 8i + g holds k 0..15; one LDS.128 per k pair
          if ((ks & 1) == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              areal[i] = tma::lds128(st + (wm + i * 8 + g) * 128 + ((((ks >> 1) * 4 + t) ^ g) << 4));
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = make_double2((ks & 1) ? areal[i].y : areal[i].x, 0.0);
        } else {
          // real, fiber-contiguous: [fiber group][k][16 fibers]; fiber c = 8*(i%2) + g of group wm/16 + i/2
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const unsigned row = (wm / 16 + (i >> 1)) * 16 + (ks >> 1) * 8 + 2 * t + (ks & 1);
            const unsigned chunk = ((i & 1) * 4 + (g >> 1)) ^ (2 * t + (ks & 1));
            a[i] = make_double2(tma::lds64(st + row * 128 + (chunk << 4) + (g & 1) * 8), 0.0);
          }
        }
        if constexpr (CL) {
          const unsigned bo = ((ks & 1) ? b1 : b0) + (ks >> 1) * B_KG;
          double2 b[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = tma::lds128(st + bo + j * B_J);
          if constexpr (CU) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                dmma(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
                dmma(ci[i][j][0], ci[i][j][1], a[i].x, b[j].y);
              }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                dmma(cr[i][j][0], cr[i][j][1], a[i].y, negate(b[j].y));
                dmma(ci[i][j][0], ci[i][j][1], a[i].y, b[j].x);
              }
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                dmma(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
                dmma(ci[i][j][0], ci[i][j][1], a[i].x, b[j].y);
              }
          }
        } else {
          if ((ks & 1) == 0) {
            // row n = wn + 8j + g holds k = 0..15; chunk (k/2) ^ (n % 8), k/2 = (ks/2)*4 + t
#pragma unroll
            for (int j = 0; j < 4; ++j)
              breal[j] = tma::lds128(st + A_BYTES + (wn + j * 8 + g) * 128 + ((((ks >> 1) * 4 + t) ^ g) << 4));
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const double bv = (ks & 1) ? breal[j].y : breal[j].x;
              dmma(cr[i][j][0], cr[i][j][1], a[i].x, bv);
              if constexpr (CU) dmma(ci[i][j][0], ci[i][j][1], a[i].y, bv);
            }
        }
      }
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[s]);
    }

    if (SKT && (k0 != 0 || k1 != KT)) {
      // a piece of a stream-K tile: publish it, or (owner) add the later pieces in order
      constexpr bool CO = CU || CL;
      const int64_t tstart = (tile - sk.sk_base) * KT;
      const int64_t owner = sk_cta_of(tstart);
      auto slot = [&](int64_t piece) {
        const int64_t idx = ((tile - sk.sk_base) * sk.slots + (piece - 1)) * CONSUMERS + warp;
        return idx;
      };
      if (k0 != 0) {
        const int64_t idx = slot(cta - owner);
        double* dst = sk.part + idx * 2048;
        int v = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              __stcg(dst + (v++) * 32 + lane, cr[i][j][h]);
              if constexpr (CO) __stcg(dst + (v++) * 32 + lane, ci[i][j][h]);
            }
        __threadfence();
        __syncwarp();
        if (lane == 0)
          asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(sk.flags + idx), "r"(sk.epoch) : "memory");
        return;
      }
      const int64_t last = sk_cta_of(tstart + KT - 1);
      for (int64_t piece = 1; piece <= last - owner; ++piece) {
        const int64_t idx = slot(piece);
        unsigned f = 0;
        long long spins = 0;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(f) : "l"(sk.flags + idx) : "memory");
          if (f != sk.epoch) {
            __nanosleep(64);
            if (++spins > (1ll << 28)) __trap();  // a lost partial must not hang the device
          }
        } while (f != sk.epoch);
        const double* src = sk.part + idx * 2048;
        int v = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              cr[i][j][h] += __ldcg(src + (v++) * 32 + lane);
              if constexpr (CO) ci[i][j][h] += __ldcg(src + (v++) * 32 + lane);
            }
      }
    }

    // epilogue (overlaps the producer's loads for the next tile)
    // fused ops run only where the host checked op_split_ok (inst_tma_c128.cu)
    const SplitOpCtx octx = split_ctx<OPK>(op);
    // fiber-contiguous tiles lie inside one n_left slab (nl % BM == 0, host-checked):
    // one 64-bit division per tile instead of one per output row
    // output rows in one block (no slab split, no peers): no per-column block division
    const bool plain_rows = sp.ncb >= N && !sp.peer[0];
    const int64_t f_q = KC ? 0 : m0 / nl;
    const int64_t f_rem = KC ? 0 : m0 - f_q * nl, f_slab = KC ? 0 : f_q * nl * sp.ncb;
    using TO = typename El<double, CU || CL>::T;
    double nacc = 0.0;  // optional epilogue two-norm (op.norm_ws), this warp's share of the tile
    // visit the output addresses of one 8-row block of the warp tile: fn(dst, p, j, h, col)
    // for every in-range element of row i
    auto visit_row = [&](const int i, auto&& fn) {
      const int64_t f = m0 + wm + i * 8 + g;
      if (f >= M) return;
      const int64_t cs = KC ? 1 : nl;
      TO* obase = out;
      int64_t ob;
      if constexpr (KC) {
        if (sp.fcb) {  // fiber blocks to peers
          const int64_t fb = f / sp.fcb;
          obase = static_cast<TO*>(sp.peer[fb]) + sp.peer_off;
          ob = (f - fb * sp.fcb) * N;
        } else {
          ob = f * N;
        }
      } else {
        ob = f_rem + (f - m0) + f_slab;  // (f % nl) + (f / nl) * nl * ncb, f in this tile's slab
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c8 = n0 + wn + j * 8;
        const int nblk = (KC || plain_rows) ? 0 : c8 / sp.ncb;
        TO* dst = obase;
        int64_t obj = ob - static_cast<int64_t>(nblk) * sp.ncb * cs;
        if (!KC && sp.peer[0]) dst = static_cast<TO*>(sp.peer[nblk]) + sp.peer_off;
        else if (!KC) obj += nblk * sp.nbs;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = c8 + 2 * t + h;
          if (col >= N) continue;
          fn(dst, obj + static_cast<int64_t>(col) * cs, j, h, col);
        }
      }
    };
    // accumulate-into-output (sp.acc): row i's accumulators += the stored values, as
    // numpy's `out += product` (the product rounded to f64 first: it is exact in the
    // accumulator), before any fused op sees them
    auto accum_row = [&](const int i, double (&crow)[4][2], double (&cirow)[4][2]) {
      visit_row(i, [&](TO* dst, int64_t p, int j, int h, int) {
        double re = crow[j][h], im = (CU || CL) ? cirow[j][h] : 0.0;
        KMB_ASSERT(p >= 0 && p < sp.out_ext);
        add_old(dst[p], re, im);
        crow[j][h] = re;
        if constexpr (CU || CL) cirow[j][h] = im;
      });
    };
    // one 8-row block of the warp tile: row i (runtime) with accumulators crow/cirow
    // (with_op false: the values were already transformed, gpe_rows below)
    auto emit_row = [&](const int i, const double (&crow)[4][2], const double (&cirow)[4][2], const bool with_op) {
      const int64_t f = m0 + wm + i * 8 + g;
      const double lf = (with_op && f < M) ? split_fiber_weight<OPK>(op, f) : 0.0;
      visit_row(i, [&](TO* dst, int64_t p, int j, int h, int col) {
        double re = crow[j][h], im = (CU || CL) ? cirow[j][h] : 0.0;
        if (with_op && sp.acc) add_old(dst[p], re, im);  // (other paths ran accum_row already)
        if constexpr (OPK != KM_OP_NONE && (CU || CL)) {
          if (with_op) apply_op_fast<OPK>(op, octx, lf, col, re, im);
        }
        KMB_ASSERT(p >= 0 && (sp.peer[0] ? true : p < sp.out_ext));
        dst[p] = narrow<TO>(re, im);
        if (op.norm_ws) nacc = fma(re, re, fma(im, im, nacc));  // |stored value|^2 (f64 output)
      });
    };
    if constexpr (OPK == KM_OP_NONE) {
      if (sp.acc) {
#pragma unroll
        for (int i = 0; i < 4; ++i) accum_row(i, cr[i], ci[i]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) emit_row(i, cr[i], ci[i], false);
    } else if constexpr (OPK == KM_OP_GPE_PHASE && (CU || CL)) {
      // GPE phase: the thread's 8 columns are fixed for the tile, so their
      // direction-d weights are loaded once; each 8-element row is rotated
      // as one vector (gpe_rotate_vec: 8 independent chains, one warp vote
      // for the reduction-free sin/cos).  Every lane takes part (out-of-range
      // elements compute on zeros and are not stored).
      double wl[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = n0 + wn + j * 8 + 2 * t + h;
          wl[j][h] = col < N ? __ldg(octx.wlast + col) : 1.0;
        }
#pragma unroll 1
      for (int i = 0; i < 4; ++i) {
        const int64_t f = m0 + wm + i * 8 + g;
        const double lf = f < M ? split_fiber_weight<OPK>(op, f) : 1.0;
        if (sp.acc) accum_row(i, cr[0], ci[0]);
        constexpr int EV = KMB_EPI_VEC;  // elements per gpe_rotate_vec call
#pragma unroll
        for (int hv = 0; hv < 8 / EV; ++hv) {
          double w[EV], vr[EV], vi[EV];
#pragma unroll
          for (int e = 0; e < EV; ++e) {
            const int x = hv * EV + e;
            w[e] = __dmul_rn(lf, wl[x >> 1][x & 1]);
            vr[e] = cr[0][x >> 1][x & 1];
            vi[e] = ci[0][x >> 1][x & 1];
          }
          gpe_rotate_vec<EV>(op.coef, w, vr, vi);
          if (op.repeat > 1) gpe_rotate_vec<EV>(op.coef, w, vr, vi);
#pragma unroll
          for (int e = 0; e < EV; ++e) {
            const int x = hv * EV + e;
            cr[0][x >> 1][x & 1] = vr[e];
            ci[0][x >> 1][x & 1] = vi[e];
          }
        }
        emit_row(i, cr[0], ci[0], false);
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              cr[r][j][h] = cr[r + 1][j][h];
              ci[r][j][h] = ci[r + 1][j][h];
            }
      }
    } else {
      // the phase math is ~80 instructions per element: emit the rows in a
      // rolled loop that rotates row i+1 into row 0, so the code holds 8 copies
      // of it instead of 32 (the unrolled version stalled on instruction fetch)
#pragma unroll 1
      for (int i = 0; i < 4; ++i) {
        emit_row(i, cr[0], ci[0], true);
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              cr[r][j][h] = cr[r + 1][j][h];
              ci[r][j][h] = ci[r + 1][j][h];
            }
      }
    }
    if (op.norm_ws) norm_slot(op.norm_ws, tile * CONSUMERS + warp, nacc, op.norm_count);
  };
  if (op.norm_ws) norm_count(op.norm_ws, tiles * CONSUMERS);

  if constexpr (!SKT) {
    for (int64_t tile = cta; tile < tiles; tile += S) run_tile(tile, 0, KT);
  } else {
    for (int64_t w = 0; w < n_dp; ++w) run_tile(cta + w * S, 0, KT);
    for (int64_t gk = sk_b; gk < sk_e;) {
      const int64_t tile = sk.sk_base + gk / KT;
      const int k0 = static_cast<int>(gk % KT);
      const int k1 = static_cast<int>(k0 + (sk_e - gk) < KT ? k0 + (sk_e - gk) : KT);
      gk += k1 - k0;
      run_tile(tile, k0, k1);
    }
  }
}

// Host side: tensor maps + launch.  Returns -1 when the shape is not eligible
// (the caller then uses the cp.async kernel).
int launch_tma_f64(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl, const OpDev& op,
                   const Split& sp, cudaStream_t st, bool complex_tensor, bool complex_factor);

}  // namespace kmb
