// Host side of mumode_tma_kernel: eligibility, TMA tensor maps, persistent launch.
#include "kmb200_tma.cuh"

#include <cudaTypedefs.h>

#include <cstring>
#include <map>
#include <mutex>

namespace kmb {

bool g_tma_disabled = false;
bool g_streamk_disabled = false;

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

bool make_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
              const cuuint32_t* box) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Stream-K scratch: partial accumulators and publish flags, in a caller-owned
// device workspace bound to a stream (km_set_stream_workspace; the library
// never allocates).  Sized for the largest launch (2 * SMs stream-K tiles, 2
// extra pieces each); flags are zeroed at bind time and every launch publishes
// under a fresh epoch, so consecutive launches on the stream share it safely.
// A stream without a workspace runs whole tiles.
struct SkBinding {
  double* part = nullptr;
  unsigned* flags = nullptr;
  unsigned epoch = 0;
};

std::mutex g_sk_mu;
std::map<std::pair<int, cudaStream_t>, SkBinding> g_sk;

size_t sk_pieces() { return static_cast<size_t>(2 * num_sms()) * 2 * tma::CONSUMERS; }

}  // namespace

size_t streamk_workspace_bytes() { return sk_pieces() * (2048 * sizeof(double) + sizeof(unsigned)); }

int bind_streamk_workspace(cudaStream_t st, void* ws, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_sk_mu);
  if (!ws) {
    g_sk.erase({dev, st});
    return KM_OK;
  }
  const size_t need = streamk_workspace_bytes();
  if (bytes < need)
    return fail(KM_EINVAL, "km_set_stream_workspace: %zu bytes given, %zu needed", bytes, need);
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(KM_EINVAL, "km_set_stream_workspace: workspace not 256-B aligned");
  SkBinding b;
  b.part = static_cast<double*>(ws);
  b.flags = reinterpret_cast<unsigned*>(b.part + sk_pieces() * 2048);
  const cudaError_t e = cudaMemsetAsync(b.flags, 0, sk_pieces() * sizeof(unsigned), st);
  if (e != cudaSuccess) return fail(KM_ECUDA, "km_set_stream_workspace: %s", cudaGetErrorString(e));
  g_sk[{dev, st}] = b;
  return KM_OK;
}

namespace {

// the bound scratch of (current device, st) with a fresh epoch; false when none is bound
bool sk_scratch(cudaStream_t st, double** part, unsigned** flags, unsigned* epoch) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_sk_mu);
  auto it = g_sk.find({dev, st});
  if (it == g_sk.end()) return false;
  *part = it->second.part;
  *flags = it->second.flags;
  *epoch = ++it->second.epoch;
  return true;
}

template <typename Kern>
int set_smem(Kern k) {
  return ensure_smem(reinterpret_cast<const void*>(k), tma::SMEM_BYTES, "mumode_tma_kernel");
}

// Stream-K launch of a product (any real / complex mix).  Returns -1 when the
// shape or the stream does not call for it (the caller launches whole tiles).
// Stream-K pays for products whose tiles make 1-4 waves with a partial last
// one (e.g. the 256^3 state split over 4 or 8 GPUs): that wave plus one full
// wave is cut into equal k-ranges, so every CTA's range holds at least KT
// k-blocks.  Measured (tools/slab_probe.py): per-rank products at P = 4 / 8 go
// from 0.80 / 0.78 to 0.88 / 0.83 of the DMMA peak.  Between S/2 and S tiles
// all k-blocks are cut into S ranges (tools/pipe_probe.py: the 1024^2 f64
// pipe-flow step 189 -> 176 us, its complex128 variant 296 -> 283 us).
// Beyond 4 waves it is used only when the partial last wave wastes > 5 % of the
// slots (160^3: 4.05 waves); the 256^3 headline (13.8 waves, 1.2 % tail) keeps
// whole tiles.
template <bool KC, int OPK, bool CL, bool CU>
int launch_streamk(const CUtensorMap& ma, const CUtensorMap& mb, void* out, int64_t M, int N, int K, int64_t nl,
                   const OpDev& op, const Split& sp, cudaStream_t st) {
  using TO = typename El<double, CU || CL>::T;
  const int64_t tiles = ((M + tma::BM - 1) / tma::BM) * ((N + tma::BN - 1) / tma::BN);
  const int64_t KT = (K + tma::BKS - 1) / tma::BKS;
  const int64_t S = num_sms();
  // fewer tiles than SMs (down to S/2): every k-block goes to the stream-K
  // range, a tile spans at most 3 CTAs (slots <= 2)
  if (g_streamk_disabled || 2 * tiles < S || tiles % S == 0 || KT < 2) return -1;
  // many waves: only when the partial last wave wastes more than 5 % of the slots
  // (256^3, 13.8 waves: 1.2 %, whole tiles; 160^3, 4.05 waves: 19 %)
  const int64_t waves = (tiles + S - 1) / S;
  if (tiles > 4 * S && 20 * (waves * S - tiles) <= waves * S) return -1;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  if (cap != cudaStreamCaptureStatusNone) return -1;  // epochs would repeat on replay
  StreamK sk;
  memset(&sk, 0, sizeof(sk));
  sk.dp_waves = tiles > S ? tiles / S - 1 : 0;
  sk.sk_base = sk.dp_waves * S;
  sk.iters = (tiles - sk.sk_base) * KT;
  const int64_t per = sk.iters / S;  // >= KT (tiles > S: a tile spans at most 2 CTAs) or >= KT/2
  sk.slots = static_cast<int>((KT + per - 1) / per);
  if (!sk_scratch(st, &sk.part, &sk.flags, &sk.epoch)) return -1;
  auto kern = mumode_tma_kernel<KC, OPK, CL, CU, true>;
  if (int rc = set_smem(kern)) return rc;
  TO* outp = static_cast<TO*>(out);
  void* args[] = {const_cast<CUtensorMap*>(&ma), const_cast<CUtensorMap*>(&mb), &outp, &M, &N, &K, &nl,
                  const_cast<OpDev*>(&op), const_cast<Split*>(&sp), &sk};
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(static_cast<unsigned>(S)),
                                              dim3(tma::threads_for<CL, CU>()), args, tma::SMEM_BYTES, st);
  return e == cudaSuccess ? KM_OK : fail(KM_ECUDA, "mumode_tma_kernel (stream-K): %s", cudaGetErrorString(e));
}

template <bool KC, int OPK, bool CL, bool CU>
int launch(const CUtensorMap& ma, const CUtensorMap& mb, void* out, int64_t M, int N, int K, int64_t nl,
           const OpDev& op, const Split& sp, cudaStream_t st) {
  using TO = typename El<double, CU || CL>::T;
  {
    const int rc = launch_streamk<KC, OPK, CL, CU>(ma, mb, out, M, N, K, nl, op, sp, st);
    if (rc >= 0) return rc;
  }
  auto kern = mumode_tma_kernel<KC, OPK, CL, CU, false>;
  if (int rc = set_smem(kern)) return rc;
  const int64_t tiles = ((M + tma::BM - 1) / tma::BM) * ((N + tma::BN - 1) / tma::BN);
  const int64_t S = num_sms();
  StreamK none;
  memset(&none, 0, sizeof(none));
  const int grid = static_cast<int>(tiles < S ? tiles : S);
  const cudaError_t e = launch_pdl(kern, dim3(grid), dim3(tma::threads_for<CL, CU>()), tma::SMEM_BYTES, st, ma, mb,
                                   static_cast<TO*>(out), M, N, K, nl, op, sp, none);
  if (e != cudaSuccess) return fail(KM_ECUDA, "mumode_tma_kernel: %s", cudaGetErrorString(e));
  return check_launch("mumode_tma_kernel");
}

}  // namespace


int launch_tma_f64(const void* u, const void* L, void* out, int64_t M, int N, int K, int64_t nl, const OpDev& op,
                   const Split& sp, cudaStream_t st, bool complex_tensor, bool complex_factor) {
  if (g_tma_disabled) return -1;
  const bool kc = (nl == 1);
  const int64_t tiles = ((M + tma::BM - 1) / tma::BM) * ((N + tma::BN - 1) / tma::BN);
  // persistent: worth it once the tiles cover ~3/4 of the SMs (smaller problems use
  // the cp.async kernel's 4x finer tiles)
  // below two waves of tiles the cp.async kernel's finer tiles win for short K or
  // padded row tiles (tools/mid_probe.py: 96^3 step 105 -> 80 us, 128^3 230 -> 216
  // us); the stream-K cut keeps this kernel ahead for full-width tiles with K >= 256
  // (P = 8 slab products, the 1024^2 pipe-flow step)
  if (K % 8 != 0 || 4 * tiles < 3 * num_sms()) return -1;
  if (tiles < 2 * num_sms() && (K <= 128 || N % tma::BN != 0)) return -1;
  if ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(L)) & 15) return -1;
  if (!kc && (nl % tma::BM != 0 || (sp.kcb != K && sp.kcb % tma::BKS != 0))) return -1;
  if (static_cast<int64_t>(K) * 16 >= (int64_t(1) << 40) || M >= (int64_t(1) << 32)) return -1;

  CUtensorMap ma, mb;
  if (complex_factor) {  // B: row-major complex factor, dims (16 f64 = 8 complex k, rows, k groups)
    cuuint64_t dims[3] = {16, static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(K / 8)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(K) * 16, 128};
    cuuint32_t box[3] = {16, tma::BN, 2};
    if (!make_map(&mb, L, 3, dims, strides, box)) return -1;
  } else {  // real factor: dims (k, rows), 128-B rows of 16 k
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N), 1};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(K) * 8, static_cast<cuuint64_t>(K) * 8 * N};
    cuuint32_t box[3] = {16, tma::BN, 1};
    if (!make_map(&mb, L, 3, dims, strides, box)) return -1;
  }
  if (kc && !complex_tensor) {  // real, k-contiguous: dims (k, fibers), 128-B rows of 16 k
    if (K % 2 != 0) return -1;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M), 1};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(K) * 8, static_cast<cuuint64_t>(K) * 8 * M};
    cuuint32_t box[3] = {16, tma::BM, 1};
    if (!make_map(&ma, u, 3, dims, strides, box)) return -1;
  } else if (kc) {  // complex, k-contiguous: dims (16 f64 = 8 complex k, fibers, k groups)
    cuuint64_t dims[3] = {16, static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(K / 8)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(K) * 16, 128};
    cuuint32_t box[3] = {16, tma::BM, 2};
    if (!make_map(&ma, u, 3, dims, strides, box)) return -1;
  } else {
    const int64_t nr = (M + nl - 1) / nl;  // M < nl: a fiber range of one slab (km_mumode_fibers)
    const int64_t nblk = (K + sp.kcb - 1) / sp.kcb;
    const int64_t es = complex_tensor ? 16 : 8;  // element bytes
    const int64_t kbs = nblk > 1 ? sp.kbs : static_cast<int64_t>(nl) * sp.kcb * nr;
    // (one 128-B row of fibers, k in block, fiber rows, n_right, k blocks)
    const cuuint64_t fib_per_row = 128 / es;
    cuuint64_t dims[5] = {16, static_cast<cuuint64_t>(sp.kcb), static_cast<cuuint64_t>(nl / fib_per_row),
                          static_cast<cuuint64_t>(nr), static_cast<cuuint64_t>(nblk)};
    cuuint64_t strides[4] = {static_cast<cuuint64_t>(nl * es), 128, static_cast<cuuint64_t>(nl * sp.kcb * es),
                             static_cast<cuuint64_t>(kbs * es)};
    cuuint32_t box[5] = {16, tma::BKS, static_cast<cuuint32_t>(tma::BM / fib_per_row), 1, 1};
    if (!make_map(&ma, u, 5, dims, strides, box)) return -1;
  }
  const bool ops = op.kind != KM_OP_NONE;
  // fused ops: c x c, strided layout, and only where (fiber, row) is the op's (l, i_last) split
  if (ops && (kc || !(complex_tensor && complex_factor) || !op_split_ok(op, M, nl))) return -1;
  if (!complex_tensor) {
    if (complex_factor) {
      if (kc) return launch<true, KM_OP_NONE, true, false>(ma, mb, out, M, N, K, nl, op, sp, st);
      return launch<false, KM_OP_NONE, true, false>(ma, mb, out, M, N, K, nl, op, sp, st);
    }
    if (kc) return launch<true, KM_OP_NONE, false, false>(ma, mb, out, M, N, K, nl, op, sp, st);
    return launch<false, KM_OP_NONE, false, false>(ma, mb, out, M, N, K, nl, op, sp, st);
  }
  if (!complex_factor) {
    if (kc) return launch<true, KM_OP_NONE, false, true>(ma, mb, out, M, N, K, nl, op, sp, st);
    return launch<false, KM_OP_NONE, false, true>(ma, mb, out, M, N, K, nl, op, sp, st);
  }
  if (kc) return launch<true, KM_OP_NONE, true, true>(ma, mb, out, M, N, K, nl, op, sp, st);
  switch (op.kind) {
    case KM_OP_GPE_PHASE: return launch<false, KM_OP_GPE_PHASE, true, true>(ma, mb, out, M, N, K, nl, op, sp, st);
    case KM_OP_DIAG: return launch<false, KM_OP_DIAG, true, true>(ma, mb, out, M, N, K, nl, op, sp, st);
    default: return launch<false, KM_OP_NONE, true, true>(ma, mb, out, M, N, K, nl, op, sp, st);
  }
}

}  // namespace kmb
