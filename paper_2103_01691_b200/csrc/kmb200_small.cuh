// mumode_steps_kernel — many exact steps of a small (L2-resident) complex128
// cube in ONE persistent launch: the d = 3 sweeps of every step fused into a
// dataflow of tiles with fine-grained dependency counters instead of one
// launch (or one grid barrier) per product.
//
// Reference: kron.step (kron.py:110-121) = tucker (tensor.py:143-166) applied
// `steps` times, i.e. the product chain ×_1 E_1 ×_2 E_2 ×_3 E_3 ×_1 E_1 ...
// (the loop of problems.py:597-598 / the config-1 benchmark).
//
// Why: at 64³ one product is 3.6 µs of DMMA work, but a per-product launch
// pays its pipeline fill, its 1.73-wave tile quantisation (256 tiles on 148
// SMs) and the launch gap every time (0.50 of the DMMA peak in a CUDA graph,
// DESIGN.md §2.5).  Here the tiles of all 3·steps products form one ordered
// list; CTA c (of G persistent CTAs, 2–3 per SM) takes tiles c, c+G, c+2G, ...
// A tile of product p waits only for the tiles of product p-1 it reads
// (counters per dependency group), so the next product's first tiles run in
// the current product's last partial wave.
//
// Tiles: 32 fibers × 32 output rows × the whole contraction (K = n_mu ≤ 96),
// staged in one shot with cp.async (the state is in L2).  The fibers of a tile
// are 32 consecutive indices of the faster "other" direction at one fixed
// index of the slower one:
//   dir 1: i2-block a, i3 = b      dir 2: i1-block a, i3 = b      dir 3: i1-block a, i2 = b
// Dependency groups (the producer tiles a consumer reads, all of them one
// counter):
//   dir 2 tile (a, b=i3)  <- dir 1 tiles with i3 = b, row block = a         (n2/32 tiles)
//   dir 3 tile (a, b=i2)  <- dir 2 tiles with i1-block a, row block b/32    (n3 tiles)
//   dir 1 tile (a, b=i3)  <- dir 3 tiles with i2-block a, row block b/32    (n1 tiles)
// Buffers rotate over three (product p reads buf[p%3], writes buf[(p+1)%3]);
// buf[0] is the state, so after 3·steps products the result is back in it.
// Before writing, a tile also waits until product p-2 (the last reader of its
// destination) is complete — write-after-read safety, normally long satisfied.
//
// Deadlock freedom: every dependency points to an earlier tile of the list,
// each CTA walks its tiles in list order, and the cooperative launch makes all
// CTAs co-resident; so the earliest unfinished tile always has its inputs.
#pragma once
#include "kmb200_tma.cuh"

namespace kmb {
namespace sm {

constexpr int BT = 32;          // tile edge: fibers and output rows
constexpr int THREADS = 128;    // 4 warps, 2 x 2 warp tiles of 16 x 16
constexpr int KMAX = 96;        // largest contraction staged in one shot
constexpr int CNT_STRIDE = 512; // counters per product (groups + the total)

struct Params {
  double2* buf[3];        // buf[0]: the state (in / out); buf[1], buf[2]: workspace
  const double2* E[3];    // row-major n_mu x n_mu factors
  int n[3];
  int products;           // 3 * steps
  unsigned* cnt;          // products x CNT_STRIDE counters, zeroed before the launch
  unsigned long long* trace;  // optional (KMB_STEPS_TRACE builds): 6 globaltimer stamps per tile
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int PM = BT + 2;      // pitch (complex elements) of the transposed A tile [k][fiber]

// A (either [fiber][k] with pitch K+4, or [k][fiber] with pitch PM), B [row][k] with
// pitch K+4, then two mbarriers
__host__ __device__ inline int a_elems(int kmax) { return BT * (kmax + 4) > kmax * PM ? BT * (kmax + 4) : kmax * PM; }
__host__ __device__ inline int smem_bytes(int kmax) { return (a_elems(kmax) + BT * (kmax + 4)) * 16 + 8 * (KMAX / BT); }

// one contiguous global -> shared bulk copy (TMA engine, no tensor map), completing on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   tma::su32(dst)),
               "l"(src), "r"(bytes), "r"(tma::su32(bar))
               : "memory");
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wait_count(const unsigned* p, unsigned need) {
  long long spins = 0;
  while (ld_acquire(p) < need) {
    __nanosleep(32);
    if (++spins > (1ll << 28)) __trap();  // a lost producer must not hang the device
  }
}

// tiles of one product of direction mu, and (a, b, r) of its t-th tile in list order
struct TileMap {
  int mu, na, nb, nr;  // a-blocks, b values, row blocks
  // (ternaries, not P.n[runtime index]: a dynamically indexed kernel parameter is
  // copied to local memory)
  __device__ TileMap(const Params& P, int mu_) : mu(mu_) {
    const int n1 = P.n[0], n2 = P.n[1], n3 = P.n[2];
    na = (mu == 0 ? n2 : n1) / BT;  // faster other direction
    nb = mu == 2 ? n2 : n3;         // slower other direction
    nr = (mu == 0 ? n1 : mu == 1 ? n2 : n3) / BT;
  }
  __device__ int count() const { return na * nb * nr; }
  // order: direction 1 b-major (i3 outer), directions 2 and 3 a-major (i1-block outer);
  // row blocks innermost, so a producer group's tiles are consecutive where possible
  __device__ void decode(int t, int& a, int& b, int& r) const {
    r = t % nr;
    const int q = t / nr;
    if (mu == 0) {
      a = q % na;
      b = q / na;
    } else {
      b = q % nb;
      a = q / nb;
    }
  }
};

__global__ void __launch_bounds__(THREADS) mumode_steps_kernel(const Params P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * 16, wn = (warp >> 1) * 16;
  const int n1 = P.n[0], n2 = P.n[1], n3 = P.n[2];

  const int kmax = n1 > n2 ? (n1 > n3 ? n1 : n3) : (n2 > n3 ? n2 : n3);
  double2* As = reinterpret_cast<double2*>(smem);
  double2* Bs = As + a_elems(kmax);
  uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + BT * (kmax + 4));
  if (tid == 0) {
    for (int c = 0; c < KMAX / BT; ++c) tma::mbar_init(&bars[c], 1);
    tma::fence_barrier_init();
  }
  __syncthreads();
  unsigned phases = 0;  // bit c: the parity chunk barrier c waits for next (each flips only when used)

  // list position of this CTA: product p, tile index within it
  int p = 0, ti = blockIdx.x;
  while (p < P.products) {
    const int mu = p % 3;
    const TileMap tm(P, mu);
    const int cnt_p = tm.count();
    if (ti >= cnt_p) {  // past this product: carry over into the next one
      ti -= cnt_p;
      ++p;
      continue;
    }
    int a, b, r;
    tm.decode(ti, a, b, r);
#ifdef KMB_STEPS_TRACE
    unsigned long long* tr = nullptr;
    if (P.trace && tid == 0) {
      int64_t gidx = ti;  // list index of this tile
      for (int q = 0; q < p; ++q) gidx += TileMap(P, q % 3).count();
      tr = P.trace + gidx * 6;
      tr[0] = gtimer();
      tr[5] = (static_cast<unsigned long long>(blockIdx.x) << 32) | static_cast<unsigned>(p);
    }
#define KMB_STAMP(i) if (tr) tr[i] = gtimer()
#else
#define KMB_STAMP(i)
#endif
    const int K = mu == 0 ? n1 : mu == 1 ? n2 : n3;
    const int PK = K + 4;  // smem pitch in complex elements (conflict-free fragment reads)

    // global addressing: element (j, k) of the A tile and (j, i) of the output at
    // base + j * sa + k * sk (the output has the input's shape: square factors)
    int64_t base, sa, sk;
    if (mu == 0) {
      base = (static_cast<int64_t>(a) * BT + static_cast<int64_t>(n2) * b) * n1;
      sa = n1;
      sk = 1;
    } else if (mu == 1) {
      base = static_cast<int64_t>(a) * BT + static_cast<int64_t>(b) * n1 * n2;
      sa = 1;
      sk = n1;
    } else {
      base = static_cast<int64_t>(a) * BT + static_cast<int64_t>(n1) * b;
      sa = 1;
      sk = static_cast<int64_t>(n1) * n2;
    }
    const int pi = p % 3;
    const double2* __restrict__ src = pi == 0 ? P.buf[0] : pi == 1 ? P.buf[1] : P.buf[2];
    double2* __restrict__ dst = pi == 0 ? P.buf[1] : pi == 1 ? P.buf[2] : P.buf[0];
    const double2* __restrict__ E = mu == 0 ? P.E[0] : mu == 1 ? P.E[1] : P.E[2];

    // 1-3: warp 0 stages the tile with bulk copies, one per lane: the factor rows at once,
    // the A tile once its producers have published (k-contiguous fibers for direction 1,
    // fiber-contiguous k-columns otherwise, stored transposed)
    // staged in chunks of 32 k (one mbarrier each), so the MMAs of chunk 0 start while the
    // later chunks are still in flight
    const int nch = K / BT;
    if (warp == 0) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // prior generic smem reads
        for (int c = 0; c < nch; ++c) tma::mbar_expect_tx(&bars[c], 2 * BT * BT * 16);
      }
      __syncwarp();
      for (int c = 0; c < nch; ++c)
        bulk_g2s(Bs + lane * PK + c * BT, E + static_cast<int64_t>(r * BT + lane) * K + c * BT, BT * 16, &bars[c]);
      if (lane == 0) {
        if (p >= 1) {  // the producer group of this tile
          const unsigned* cn = P.cnt + static_cast<int64_t>(p - 1) * CNT_STRIDE;
          int grp;
          unsigned need;
          if (mu == 1) {         // dir 1 tiles with i3 = b, row block a
            grp = b * (n1 / BT) + a;
            need = n2 / BT;
          } else if (mu == 2) {  // dir 2 tiles with i1-block a, row block b / 32
            grp = a * (n2 / BT) + b / BT;
            need = n3;
          } else {               // dir 3 tiles with i2-block a, row block b / 32
            grp = a * (n3 / BT) + b / BT;
            need = n1;
          }
          wait_count(cn + grp, need);
        }
        if (p >= 2) {  // the last reader of this tile's destination
          const TileMap t2(P, (p - 2) % 3);
          wait_count(P.cnt + static_cast<int64_t>(p - 2) * CNT_STRIDE + (CNT_STRIDE - 1), t2.count());
        }
        KMB_STAMP(1);
      }
      __syncwarp();
      KMB_ASSERT(base + (BT - 1) * sa + static_cast<int64_t>(K - 1) * sk < static_cast<int64_t>(n1) * n2 * n3);
      for (int c = 0; c < nch; ++c) {
        if (mu == 0) {
          bulk_g2s(As + lane * PK + c * BT, src + base + lane * sa + c * BT, BT * 16, &bars[c]);
        } else {
          const int k = c * BT + lane;
          bulk_g2s(As + k * PM, src + base + k * sk, BT * 16, &bars[c]);
        }
      }
    }
    if (tid == 0) KMB_STAMP(2);

    // 4. the tile's products: 2 x 2 DMMA tiles of 8 x 8 per warp, complex x complex
    double cr[2][2][2], ci[2][2][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        cr[x][y][0] = cr[x][y][1] = 0.0;
        ci[x][y][0] = ci[x][y][1] = 0.0;
      }
    // A fragment (fiber wm + 8x + g, k kk + t): [fiber][k] or [k][fiber]
    const int a_row = mu == 0 ? PK : 1, a_col = mu == 0 ? 1 : PM;
#pragma unroll 4
    for (int kk = 0; kk < K; kk += 4) {
      if ((kk & (BT - 1)) == 0) tma::mbar_wait(&bars[kk / BT], (phases >> (kk / BT)) & 1u);
      double2 av[2], bv[2];
#pragma unroll
      for (int x = 0; x < 2; ++x) av[x] = As[(wm + x * 8 + g) * a_row + (kk + t) * a_col];
#pragma unroll
      for (int y = 0; y < 2; ++y) bv[y] = Bs[(wn + y * 8 + g) * PK + kk + t];
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) {
          dmma(cr[x][y][0], cr[x][y][1], av[x].x, bv[y].x);
          dmma(ci[x][y][0], ci[x][y][1], av[x].x, bv[y].y);
        }
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) {
          dmma(cr[x][y][0], cr[x][y][1], av[x].y, negate(bv[y].y));
          dmma(ci[x][y][0], ci[x][y][1], av[x].y, bv[y].x);
        }
    }

    phases ^= (1u << nch) - 1u;  // the chunk barriers this tile used
    if (tid == 0) KMB_STAMP(3);
    // 5. store: C fragment (g, 2t + h) of each 8x8 tile -> (fiber j, row i)
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = wm + x * 8 + g;
          const int i = r * BT + wn + y * 8 + 2 * t + h;
          KMB_ASSERT(base + j * sa + static_cast<int64_t>(i) * sk < static_cast<int64_t>(n1) * n2 * n3);
          dst[base + j * sa + static_cast<int64_t>(i) * sk] = make_double2(cr[x][y][h], ci[x][y][h]);
        }
    __syncthreads();  // every store of the tile (and every shared-memory read) is done

    // 6. publish (as a grid barrier does: CTA barrier, one fence, one release add): the
    // consumer group this tile belongs to, and the product's total
    if (tid == 0) {
      __threadfence();
      unsigned* c = P.cnt + static_cast<int64_t>(p) * CNT_STRIDE;
      int grp;
      if (mu == 0) grp = b * (n1 / BT) + r;            // (i3, i1-block) for dir 2
      else if (mu == 1) grp = a * (n2 / BT) + r;       // (i1-block, i2-block) for dir 3
      else grp = (b / BT) * (n3 / BT) + r;             // (i2-block, i3-block) for dir 1
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(c + grp) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(c + CNT_STRIDE - 1) : "memory");
      KMB_STAMP(4);
    }
    ti += gridDim.x;
  }
}

}  // namespace sm
}  // namespace kmb
