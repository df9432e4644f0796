// libkmb200 C ABI (include/kmb200.h): argument checks, dtype dispatch, the
// standalone pointwise pass and the Tucker/step driver.  Kernels live in
// kmb200_kernels.cuh; each dtype combination is instantiated in inst_*.cu.
#include "kmb200_plane.cuh"
#include "kmb200_launch.cuh"

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>

namespace kmb {

extern bool g_tma_disabled;     // inst_tma_c128.cu
extern bool g_streamk_disabled;  // inst_tma_c128.cu
extern bool g_tc_halves_disabled;  // inst_tc32_c64.cu
extern bool g_plane_disabled;      // inst_plane.cu
size_t tc32_workspace_bytes(int64_t m, int64_t K);  // inst_tc32_c64.cu
size_t streamk_workspace_bytes();                    // inst_tma_c128.cu
int bind_streamk_workspace(cudaStream_t st, void* ws, size_t bytes);  // inst_tma_c128.cu
int norm_epilogue_finish(const km_pointop* op, bool fused, const void* out, int out_dt, int64_t n,
                         cudaStream_t st);  // norm.cu
int64_t norm_epilogue_slots(int64_t m, int64_t fibers);  // norm.cu
int steps_small_workspace(int64_t n1, int64_t n2, int64_t n3, int64_t steps, size_t* bytes);  // inst_small.cu
int launch_steps_small(void* state, const void* E1, const void* E2, const void* E3, int64_t n1, int64_t n2,
                       int64_t n3, int64_t steps, void* ws, size_t ws_bytes, cudaStream_t st);  // inst_small.cu
int launch_tc32_c64(const void* u, const void* L, void* out, int64_t m, int64_t nl, int64_t K, int64_t nr, void* ws,
                    size_t ws_bytes, cudaStream_t st);
thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(KM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return KM_OK;
}

OpDev to_dev(const km_pointop* op) {
  OpDev o;
  memset(&o, 0, sizeof(o));
  if (!op) return o;
  o.kind = op->kind;
  o.d = op->d;
  for (int i = 0; i < KM_MAX_D; ++i) {
    o.dims[i] = op->dims[i];
    o.w[i] = op->weights[i];
  }
  o.coef = op->coef;
  o.diag = static_cast<const double2*>(op->diag);
  o.diag_dir = op->diag_dir;
  int64_t s = 1;
  for (int i = 0; i < op->diag_dir && i < op->d; ++i) s *= op->dims[i];
  o.diag_stride = s;
  o.winner = op->inner_weights;
  o.repeat = op->repeat > 1 ? 2 : 1;
  int64_t in = 1;
  for (int i = 0; i + 1 < op->d; ++i) in *= op->dims[i];
  o.inner = in;
  o.norm_ws = op->norm_result ? op->norm_ws : nullptr;
  o.norm_count = op->norm_ws_count;
  return o;
}

int validate_op(const km_pointop* op, const char* where) {
  if (op && op->norm_result && (!op->norm_ws || op->norm_ws_count < 1))
    return fail(KM_EINVAL, "%s: epilogue norm without a partial-sum workspace", where);
  if (!op || op->kind == KM_OP_NONE) return KM_OK;
  if (op->d < 1 || op->d > KM_MAX_D) return fail(KM_EINVAL, "%s: op order %d outside 1..%d", where, op->d, KM_MAX_D);
  if (op->kind == KM_OP_GPE_PHASE) {
    if (op->repeat < 0 || op->repeat > 2) return fail(KM_EINVAL, "%s: GPE phase repeat %d outside 0..2", where, op->repeat);
    for (int i = 0; i < op->d; ++i)
      if (!op->weights[i]) return fail(KM_EINVAL, "%s: GPE phase weight %d is NULL", where, i);
    return KM_OK;
  }
  if (op->kind == KM_OP_DIAG) {
    if (!op->diag) return fail(KM_EINVAL, "%s: diagonal factor is NULL", where);
    if (op->diag_dir < 0 || op->diag_dir >= op->d)
      return fail(KM_EINVAL, "%s: diagonal direction %d outside 0..%d", where, op->diag_dir, op->d - 1);
    return KM_OK;
  }
  return fail(KM_EINVAL, "%s: unknown pointwise op kind %d", where, op->kind);
}

bool is_complex(int dt) { return dt == KM_C64 || dt == KM_C128; }
bool is_double(int dt) { return dt == KM_F64 || dt == KM_C128; }
size_t elem_bytes(int dt) { return dt == KM_F32 ? 4 : (dt == KM_C128 ? 16 : 8); }
int promote(int a, int b) {
  const bool c = is_complex(a) || is_complex(b);
  const bool d = is_double(a) || is_double(b);
  return c ? (d ? KM_C128 : KM_C64) : (d ? KM_F64 : KM_F32);
}

namespace {
std::mutex g_memo_mu;
std::map<std::pair<int, const void*>, int> g_memo;
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
constexpr int MAX_DEVICES = 64;
std::atomic<int> g_num_sms[MAX_DEVICES];
}  // namespace

bool memo_get(const void* key, int* value) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_memo_mu);
  auto it = g_memo.find({dev, key});
  if (it == g_memo.end()) return false;
  *value = it->second;
  return true;
}

void memo_put(const void* key, int value) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_memo_mu);
  g_memo[{dev, key}] = value;
}

int ensure_smem(const void* func, int bytes, const char* what) {
  int have = 0;
  if (memo_get(func, &have) && have >= bytes) return KM_OK;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return fail(KM_ECUDA, "cudaFuncSetAttribute(%s): %s", what, cudaGetErrorString(e));
  memo_put(func, bytes);
  return KM_OK;
}

int num_sms() {
  const int dev = current_device();
  if (dev < 0 || dev >= MAX_DEVICES) return 148;
  int n = g_num_sms[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    g_num_sms[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

int pointwise_impl(const void* in, void* out, int dt, int64_t n, const km_pointop* op, cudaStream_t st);

int mumode_impl(const void* u, int udt, const void* L, int ldt, void* out, int64_t m, int64_t nl, int64_t nmu,
                int64_t nr, const km_pointop* post, cudaStream_t st, const Split* split = nullptr,
                int64_t fibers = -1) {
  if (udt < KM_F32 || udt > KM_C128 || ldt < KM_F32 || ldt > KM_C128)
    return fail(KM_EINVAL, "km_mumode: unknown dtype (u=%d, L=%d)", udt, ldt);
  if (is_double(udt) != is_double(ldt))
    return fail(KM_EINVAL, "km_mumode: operands must share one precision (u=%d, L=%d)", udt, ldt);
  if (m < 1 || nl < 1 || nmu < 1 || nr < 1)
    return fail(KM_EINVAL, "km_mumode: extents must be positive (m=%lld, n_left=%lld, n_mu=%lld, n_right=%lld)",
                (long long)m, (long long)nl, (long long)nmu, (long long)nr);
  if (m > 0x7fffffffLL || nmu > 0x7fffffffLL) return fail(KM_EINVAL, "km_mumode: matrix too large");
  if (!u || !L || !out) return fail(KM_EINVAL, "km_mumode: NULL pointer");
  int rc0 = validate_op(post, "km_mumode");
  if (rc0) return rc0;
  if (post && post->kind != KM_OP_NONE && !(is_complex(udt) || is_complex(ldt)))
    return fail(KM_EINVAL, "km_mumode: pointwise op needs a complex result");
  const OpDev op = to_dev(post);
  // fibers >= 0: only the first `fibers` fibers of an n_right == 1 product
  // (km_mumode_fibers passes u and out already offset to its first fiber)
  const int64_t M = fibers >= 0 ? fibers : nl * nr;
  const int N = static_cast<int>(m), K = static_cast<int>(nmu);
  Split sp{K, 0, N, 0};
  if (split) {
    const bool ksplit = split->kcb != K, nsplit = split->ncb != N, fsplit = split->fcb > 0;
    if (split->kcb < 1 || split->kcb > K || split->ncb < 1 || split->ncb > N)
      return fail(KM_EINVAL, "km_mumode_split: block sizes (%d, %d) outside (1..%d, 1..%d)", split->kcb,
                  split->ncb, K, N);
    if ((ksplit || nsplit) && nl == 1)
      return fail(KM_EINVAL, "km_mumode_split: blocked layouts need n_left > 1");
    if (split->acc && split->peer[0])
      return fail(KM_EINVAL, "km_mumode_peer: no accumulation into peer outputs");
    if (fsplit && (nl != 1 || nsplit || !split->peer[0]))
      return fail(KM_EINVAL, "km_mumode_peer: fiber blocks need n_left == 1, unsplit rows and peer outputs");
    if (ksplit && split->kcb % BK != 0)
      return fail(KM_EINVAL, "km_mumode_split: input block %d is not a multiple of %d", split->kcb, BK);
    if (nsplit && split->ncb % 8 != 0)
      return fail(KM_EINVAL, "km_mumode_split: output block %d is not a multiple of 8", split->ncb);
    // a blocked INPUT only changes the loads; the fused op needs the plain output layout
    if ((nsplit || fsplit) && op.kind != KM_OP_NONE)
      return fail(KM_EINVAL, "km_mumode_split: pointwise ops are not supported on blocked output layouts");
    if (split->peer[0]) {
      const int64_t blocks = fsplit ? (M + split->fcb - 1) / split->fcb : (N + split->ncb - 1) / split->ncb;
      if (blocks > MAX_PEERS) return fail(KM_EINVAL, "km_mumode_peer: %lld output blocks exceed %d peers",
                                          (long long)blocks, MAX_PEERS);
      for (int64_t b = 0; b < blocks; ++b)
        if (!split->peer[b]) return fail(KM_EINVAL, "km_mumode_peer: peer %lld is NULL", (long long)b);
    }
    sp = *split;
    if (!ksplit) sp.kbs = 0;
    if (!nsplit) sp.nbs = 0;
  }
  {  // logical extents (one past the largest index the layouts address), for KMB_CHECK builds
    const int64_t nr_ = (M + nl - 1) / nl;  // M < nl: a fiber range of one slab (km_mumode_fibers)
    const int64_t lmax = (M < nl ? M : nl) - 1;
    auto extent = [&](int64_t len, int64_t blk, int64_t bstride) {
      const int64_t j = len - 1;
      const int64_t b = blk < len ? j / blk : 0, w = blk < len ? blk : len;
      return b * (blk < len ? bstride : 0) + lmax + nl * (j - b * w) + nl * w * (nr_ - 1) + 1;
    };
    sp.in_ext = nl == 1 ? M * static_cast<int64_t>(K) : extent(K, sp.kcb, sp.kbs);
    sp.out_ext = nl == 1 ? M * static_cast<int64_t>(N) : extent(N, sp.ncb, sp.nbs);
  }
  const bool cu = is_complex(udt), cl = is_complex(ldt);
  auto launcher = is_double(udt) ? (cu ? (cl ? launch_d_cc : launch_d_cr) : (cl ? launch_d_rc : launch_d_rr))
                                 : (cu ? (cl ? launch_f_cc : launch_f_cr) : (cl ? launch_f_rc : launch_f_rr));
  const bool want_norm = post && post->norm_result;
  if (want_norm && post->norm_ws_count < norm_epilogue_slots(N, M))
    return fail(KM_EINVAL, "km_mumode: epilogue norm workspace of %lld slots, %lld needed",
                (long long)post->norm_ws_count, (long long)norm_epilogue_slots(N, M));
  int rc = launcher(u, L, out, M, N, K, nl, op, sp, st);
  if (rc >= 0) return rc ? rc : norm_epilogue_finish(post, true, out, promote(udt, ldt), M * N, st);
  // op not fusable for this layout/dtype: plain product, then the op in place (and the norm
  // as a separate pass)
  OpDev none;
  memset(&none, 0, sizeof(none));
  if ((rc = launcher(u, L, out, M, N, K, nl, none, sp, st))) return rc;
  if ((rc = pointwise_impl(out, out, promote(udt, ldt), M * N, post, st))) return rc;
  return norm_epilogue_finish(post, false, out, promote(udt, ldt), M * N, st);
}

// complex64 -> complex128, exact
__global__ void widen_kernel(const float2* __restrict__ in, double2* __restrict__ out, int64_t n) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[p] = widen(in[p]);
}

template <typename TI, typename TO>
int pointwise_t(const void* in, void* out, int64_t n, const OpDev& op, cudaStream_t st) {
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  dim3 grid(static_cast<unsigned>(blocks));
  const bool split = (op.kind == KM_OP_GPE_PHASE && op.winner) ||
                     (op.kind == KM_OP_DIAG && op.diag_dir == op.d - 1);
  if (split && op.inner > 0 && n % op.inner == 0) {
    // 2-D grid: x over directions 1..d-1, y over the last direction
    const int64_t nlast = n / op.inner;
    int64_t bx = (op.inner + KMB_PW * threads - 1) / (KMB_PW * threads);  // KMB_PW elements per thread (pointwise_kernel)
    int64_t by = nlast;
    if (by > 65535) by = 65535;
    while (bx * by > cap && bx > 1) bx = (bx + 1) / 2;
    while (bx * by > cap && by > 1) by = (by + 1) / 2;
    grid = dim3(static_cast<unsigned>(bx), static_cast<unsigned>(by));
  }
  if (op.kind == KM_OP_GPE_PHASE)
    pointwise_kernel<TI, TO, KM_OP_GPE_PHASE><<<grid, threads, 0, st>>>(static_cast<const TI*>(in),
                                                                         static_cast<TO*>(out), n, op);
  else
    pointwise_kernel<TI, TO, KM_OP_DIAG><<<grid, threads, 0, st>>>(static_cast<const TI*>(in), static_cast<TO*>(out),
                                                                    n, op);
  return check_launch("pointwise_kernel");
}

int pointwise_cast_impl(const void* in, int idt, void* out, int odt, int64_t n, const km_pointop* op,
                        cudaStream_t st) {
  if (!is_complex(idt) || !is_complex(odt))
    return fail(KM_EINVAL, "km_pointwise: dtypes %d -> %d are not complex", idt, odt);
  if (idt == KM_C128 && odt == KM_C64)
    return fail(KM_EINVAL, "km_pointwise: complex128 -> complex64 would round the state");
  if (idt != odt && in == out) return fail(KM_EINVAL, "km_pointwise: a widening pass cannot run in place");
  if ((!op || op->kind == KM_OP_NONE) && idt == odt) {
    if (in != out && n > 0) {
      cudaError_t e = cudaMemcpyAsync(out, in, n * elem_bytes(idt), cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return fail(KM_ECUDA, "km_pointwise copy: %s", cudaGetErrorString(e));
    }
    return KM_OK;
  }
  if (!op || op->kind == KM_OP_NONE) {  // plain widening
    op = nullptr;
  } else {
    int rc = validate_op(op, "km_pointwise");
    if (rc) return rc;
  }
  if (n <= 0) return KM_OK;
  if (!op) {
    if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 7)
      return fail(KM_EINVAL, "km_pointwise: misaligned buffers");
    widen_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 8 * num_sms())), 256, 0, st>>>(
        static_cast<const float2*>(in), static_cast<double2*>(out), n);
    return check_launch("widen_kernel");
  }
  const OpDev o = to_dev(op);
  if (idt == KM_C128) return pointwise_t<double2, double2>(in, out, n, o, st);
  if (odt == KM_C128) return pointwise_t<float2, double2>(in, out, n, o, st);
  return pointwise_t<float2, float2>(in, out, n, o, st);
}

int pointwise_impl(const void* in, void* out, int dt, int64_t n, const km_pointop* op, cudaStream_t st) {
  return pointwise_cast_impl(in, dt, out, dt, n, op, st);
}

int tucker_plan(int udt, int d, const int64_t* dims, const void* const* mats, const int* mdt, const int64_t* rows,
                size_t* ws_bytes, int* final_dt) {
  if (d < 1 || d > KM_MAX_D) return fail(KM_EINVAL, "km_tucker: order %d outside 1..%d", d, KM_MAX_D);
  if (!dims) return fail(KM_EINVAL, "km_tucker: NULL dims");
  int64_t cur[KM_MAX_D];
  for (int i = 0; i < d; ++i) {
    if (dims[i] < 1) return fail(KM_EINVAL, "km_tucker: extent %d is %lld", i, (long long)dims[i]);
    cur[i] = dims[i];
  }
  int dt = udt;
  size_t ws = 0;
  for (int mu = 0; mu < d; ++mu) {
    if (!mats || !mats[mu]) continue;
    if (!rows || rows[mu] < 1) return fail(KM_EINVAL, "km_tucker: direction %d has no row count", mu + 1);
    dt = promote(dt, mdt[mu]);
    cur[mu] = rows[mu];
    int64_t n = 1;
    for (int i = 0; i < d; ++i) n *= cur[i];
    const size_t b = static_cast<size_t>(n) * elem_bytes(dt);
    if (b > ws) ws = b;
  }
  {  // a standalone pre-pass writes an input-sized copy into the workspace
    int64_t n = 1;
    for (int i = 0; i < d; ++i) n *= dims[i];
    const size_t b = static_cast<size_t>(n) * elem_bytes(udt);
    if (b > ws) ws = b;
  }
  *ws_bytes = ws;
  *final_dt = dt;
  return KM_OK;
}

}  // namespace kmb

using namespace kmb;

// ================================================================== C ABI
extern "C" {

int km_abi_version(void) { return KMB200_ABI_VERSION; }

int km_set_kernel_policy(int policy) {
  if (policy < 0 ||
      policy > (KM_POLICY_NO_TMA | KM_POLICY_NO_STREAMK | KM_POLICY_NO_TC_HALVES | KM_POLICY_NO_PLANE_FUSION))
    return fail(KM_EINVAL, "km_set_kernel_policy: unknown policy %d", policy);
  g_tma_disabled = (policy & KM_POLICY_NO_TMA) != 0;
  g_streamk_disabled = (policy & KM_POLICY_NO_STREAMK) != 0;
  g_tc_halves_disabled = (policy & KM_POLICY_NO_TC_HALVES) != 0;
  g_plane_disabled = (policy & KM_POLICY_NO_PLANE_FUSION) != 0;
  return KM_OK;
}

const char* km_build_info(void) {
  return "libkmb200 sm_100a: mumode_tma_kernel (TMA + mbarrier ring, DMMA.8x8x4, stream-K tail), "
         "mumode_tc32_kernel (tcgen05 kind::tf32 3xTF32, CTA pairs), mumode_plane12_kernel (fused planes), "
         "cp.async DMMA kernels, fused phase / norm / accumulate epilogues"
#ifdef KMB_CHECK
         "; KMB_CHECK bounds asserts"
#endif
      ;
}

const char* km_last_error(void) { return g_err; }

int km_mumode(const void* u, int u_dtype, const void* L, int L_dtype, void* out, int64_t m, int64_t n_left,
              int64_t n_mu, int64_t n_right, const km_pointop* post, void* stream) {
  return mumode_impl(u, u_dtype, L, L_dtype, out, m, n_left, n_mu, n_right, post,
                     static_cast<cudaStream_t>(stream));
}

int km_mumode_fibers(const void* u, int u_dtype, const void* L, int L_dtype, void* out, int64_t m, int64_t n_left,
                     int64_t n_mu, int64_t fiber0, int64_t fibers, void* stream) {
  if (u_dtype < KM_F32 || u_dtype > KM_C128 || L_dtype < KM_F32 || L_dtype > KM_C128)
    return fail(KM_EINVAL, "km_mumode_fibers: unknown dtype (u=%d, L=%d)", u_dtype, L_dtype);
  if (fiber0 < 0 || fibers < 1 || fiber0 + fibers > n_left)
    return fail(KM_EINVAL, "km_mumode_fibers: fibers [%lld, %lld) outside [0, %lld)", (long long)fiber0,
                (long long)(fiber0 + fibers), (long long)n_left);
  if (!u || !out) return fail(KM_EINVAL, "km_mumode_fibers: NULL pointer");
  const int64_t ue = elem_bytes(u_dtype), oe = elem_bytes(promote(u_dtype, L_dtype));
  return mumode_impl(static_cast<const char*>(u) + fiber0 * ue, u_dtype, L, L_dtype,
                     static_cast<char*>(out) + fiber0 * oe, m, n_left, n_mu, 1, nullptr,
                     static_cast<cudaStream_t>(stream), nullptr, fibers);
}

int km_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height, void* stream) {
  if (!dst || !src) return fail(KM_EINVAL, "km_copy_2d: NULL pointer");
  const cudaError_t e =
      cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? KM_OK : fail(KM_ECUDA, "km_copy_2d: %s", cudaGetErrorString(e));
}

int km_mumode_split(const void* u, int u_dtype, const void* L, int L_dtype, void* out, int64_t m, int64_t n_left,
                    int64_t n_mu, int64_t n_right, int32_t in_block, int64_t in_block_stride, int32_t out_block,
                    int64_t out_block_stride, int32_t accumulate, const km_pointop* post, void* stream) {
  if (accumulate != 0 && accumulate != 1)
    return fail(KM_EINVAL, "km_mumode_split: accumulate must be 0 or 1, got %d", accumulate);
  Split sp{in_block, in_block_stride, out_block, out_block_stride};
  sp.acc = accumulate;
  return mumode_impl(u, u_dtype, L, L_dtype, out, m, n_left, n_mu, n_right, post,
                     static_cast<cudaStream_t>(stream), &sp);
}

int km_steps_paired(const void* u, const void* E1, const void* E2, const void* E3, int64_t n1, int64_t n2,
                    int64_t n3, int64_t steps, void* out, void* ws, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!u || !E1 || !E2 || !E3 || !out || !ws) return fail(KM_EINVAL, "km_steps_paired: NULL pointer");
  if (steps < 1) return fail(KM_EINVAL, "km_steps_paired: steps must be >= 1");
  if (out == u || ws == u || ws == out) return fail(KM_EINVAL, "km_steps_paired: u, out and ws must not alias");
  const int64_t nfib = n1 * n2;
  // the plane launches need a row split that fits, the pencil launch 32-fiber blocks
  if (!plane12_shape_ok(n1, n2, n3) || (steps > 1 && !pencil33_supported(nfib, n3))) return fail(KM_EINVAL, "km_steps_paired: extents must be 32, 48 or 64 (got %lld x %lld x %lld)",
                       static_cast<long long>(n1), static_cast<long long>(n2), static_cast<long long>(n3));
  // launch list: per two steps (1,2)(3,3)(1,2) -- step s+1 runs 3, 1, 2 -- and a last odd step (1,2)(3)
  enum { PLANE, PENCIL, DIR3 };
  const int64_t launches = (steps / 2) * 3 + (steps % 2) * 2;
  int64_t k = 0;
  const void* src = u;
  auto next_dst = [&]() { return ((launches - 1 - k) % 2 == 0) ? out : ws; };
  for (int64_t s = 0; s < steps; s += 2) {
    const bool pair = s + 1 < steps;
    const int kinds[3] = {PLANE, pair ? PENCIL : DIR3, PLANE};
    for (int i = 0; i < (pair ? 3 : 2); ++i, ++k) {
      void* dst = next_dst();
      int rc = KM_OK;
      if (kinds[i] == PLANE) {
        rc = launch_plane12(src, E1, E2, dst, n1, n2, n3, st);
      } else if (kinds[i] == PENCIL) {
        rc = launch_pencil33(src, E3, E3, dst, nfib, n3, st);
      } else {
        rc = mumode_impl(src, KM_C128, E3, KM_C128, dst, n3, nfib, n3, 1, nullptr, st);
      }
      if (rc) return rc;
      src = dst;
    }
  }
  return KM_OK;
}

int km_steps_small_workspace_bytes(int64_t n1, int64_t n2, int64_t n3, int64_t steps, size_t* bytes) {
  return steps_small_workspace(n1, n2, n3, steps, bytes);
}

int km_steps_small(void* state, const void* E1, const void* E2, const void* E3, int64_t n1, int64_t n2, int64_t n3,
                   int64_t steps, void* workspace, size_t workspace_bytes, void* stream) {
  return launch_steps_small(state, E1, E2, E3, n1, n2, n3, steps, workspace, workspace_bytes,
                            static_cast<cudaStream_t>(stream));
}

int km_stream_workspace_bytes(size_t* bytes) {
  if (!bytes) return fail(KM_EINVAL, "km_stream_workspace_bytes: NULL output");
  *bytes = streamk_workspace_bytes();
  return KM_OK;
}

int km_set_stream_workspace(void* stream, void* workspace, size_t bytes) {
  return bind_streamk_workspace(static_cast<cudaStream_t>(stream), workspace, bytes);
}

int km_tc_workspace_bytes(int64_t m, int64_t n_mu, size_t* bytes) {
  if (!bytes || m < 1 || n_mu < 1) return fail(KM_EINVAL, "km_tc_workspace_bytes: bad arguments");
  *bytes = tc32_workspace_bytes(m, n_mu);
  return KM_OK;
}

int km_mumode_c64_tc(const void* u, const void* L, void* out, int64_t m, int64_t n_left, int64_t n_mu,
                     int64_t n_right, void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!u || !L || !out) return fail(KM_EINVAL, "km_mumode_c64_tc: NULL pointer");
  if (m < 1 || n_left < 1 || n_mu < 1 || n_right < 1) return fail(KM_EINVAL, "km_mumode_c64_tc: bad extents");
  if (!g_tma_disabled) {
    const int rc = launch_tc32_c64(u, L, out, m, n_left, n_mu, n_right, workspace, workspace_bytes, st);
    if (rc >= 0) return rc;
  }
  return mumode_impl(u, KM_C64, L, KM_C64, out, m, n_left, n_mu, n_right, nullptr, st);
}

int km_mumode_peer(const void* u, int u_dtype, const void* L, int L_dtype, int64_t m, int64_t n_left, int64_t n_mu,
                   int64_t n_right, int32_t in_block, int64_t in_block_stride, int32_t out_block,
                   int64_t fiber_block, void* const* peers, int32_t npeers, int64_t peer_offset, void* stream) {
  if (!peers || npeers < 1 || npeers > MAX_PEERS)
    return fail(KM_EINVAL, "km_mumode_peer: need 1..%d peer buffers, got %d", MAX_PEERS, npeers);
  Split sp{in_block, in_block_stride, out_block, 0, static_cast<int>(fiber_block), peer_offset, {}};
  for (int b = 0; b < npeers; ++b) sp.peer[b] = peers[b];
  return mumode_impl(u, u_dtype, L, L_dtype, peers[0], m, n_left, n_mu, n_right, nullptr,
                     static_cast<cudaStream_t>(stream), &sp);
}

int km_tucker_workspace(int u_dtype, int d, const int64_t* dims, const void* const* mats, const int* mat_dtypes,
                        const int64_t* rows, size_t* bytes) {
  int fdt = 0;
  if (!bytes) return fail(KM_EINVAL, "km_tucker_workspace: NULL output");
  return tucker_plan(u_dtype, d, dims, mats, mat_dtypes, rows, bytes, &fdt);
}

int km_pointwise(const void* in, void* out, int dtype, int64_t n, const km_pointop* op, void* stream) {
  return pointwise_impl(in, out, dtype, n, op, static_cast<cudaStream_t>(stream));
}

int km_pointwise_cast(const void* in, int in_dtype, void* out, int out_dtype, int64_t n, const km_pointop* op,
                      void* stream) {
  return pointwise_cast_impl(in, in_dtype, out, out_dtype, n, op, static_cast<cudaStream_t>(stream));
}

int km_tucker(const void* u, int u_dtype, int d, const int64_t* dims, const void* const* mats,
              const int* mat_dtypes, const int64_t* rows, void* out, void* ws0, void* ws1, const km_pointop* pre,
              const km_pointop* post, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  size_t ws = 0;
  int fdt = 0;
  int rc = tucker_plan(u_dtype, d, dims, mats, mat_dtypes, rows, &ws, &fdt);
  if (rc) return rc;
  if ((rc = validate_op(pre, "km_tucker pre"))) return rc;
  if ((rc = validate_op(post, "km_tucker post"))) return rc;
  const bool has_pre = pre && pre->kind != KM_OP_NONE;
  const bool has_post_op = post && post->kind != KM_OP_NONE;
  const bool has_post = has_post_op || (post && post->norm_result);  // an op and/or the epilogue norm
  if ((has_pre && !is_complex(u_dtype)) || (has_post_op && !is_complex(fdt)))
    return fail(KM_EINVAL, "km_tucker: pointwise ops need complex tensors");

  int active[KM_MAX_D];
  int na = 0;
  for (int mu = 0; mu < d; ++mu)
    if (mats && mats[mu]) active[na++] = mu;
  int64_t n_in = 1;
  for (int i = 0; i < d; ++i) n_in *= dims[i];

  if (na == 0) {
    if (has_pre) {
      if ((rc = pointwise_impl(u, out, u_dtype, n_in, pre, st))) return rc;
    } else if (u != out && n_in > 0) {
      cudaError_t e = cudaMemcpyAsync(out, u, n_in * elem_bytes(u_dtype), cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return fail(KM_ECUDA, "km_tucker copy: %s", cudaGetErrorString(e));
    }
    if (has_post_op && (rc = pointwise_impl(out, out, fdt, n_in, post, st))) return rc;
    return norm_epilogue_finish(post, false, out, fdt, n_in, st);
  }
  if ((na > 1 || has_pre) && !ws0) return fail(KM_EINVAL, "km_tucker: NULL workspace");
  if ((ws0 && (ws0 == u || ws0 == out)) || (ws1 && (ws1 == u || ws1 == out || ws1 == ws0)))
    return fail(KM_EINVAL, "km_tucker: a workspace aliases the input, the output or the other workspace");
  // Destinations are assigned backwards from the last product (which writes
  // out): ws0 and a second buffer alternate.  With ws1 == NULL the second
  // buffer is `out` itself — legal because the product reading it never
  // writes it — so a step needs one workspace, not two, when every
  // intermediate fits in out (always true for square factors).
  int64_t cur[KM_MAX_D];
  for (int i = 0; i < d; ++i) cur[i] = dims[i];
  size_t out_bytes = 0;
  {
    int64_t n = 1;
    for (int i = 0; i < d; ++i) n *= (mats && mats[i]) ? rows[i] : dims[i];
    out_bytes = static_cast<size_t>(n) * elem_bytes(fdt);
  }
  void* alt = ws1 ? ws1 : out;
  void* dst[KM_MAX_D];
  size_t dst_bytes[KM_MAX_D];
  {
    int64_t c[KM_MAX_D];
    for (int i = 0; i < d; ++i) c[i] = dims[i];
    int t = u_dtype;
    for (int a = 0; a < na; ++a) {
      c[active[a]] = rows[active[a]];
      t = promote(t, mat_dtypes[active[a]]);
      int64_t n = 1;
      for (int i = 0; i < d; ++i) n *= c[i];
      dst_bytes[a] = static_cast<size_t>(n) * elem_bytes(t);
    }
  }
  dst[na - 1] = out;
  for (int a = na - 2; a >= 0; --a) {
    dst[a] = (dst[a + 1] == ws0) ? alt : ws0;
    if (dst[a] == out && dst_bytes[a] > out_bytes)
      return fail(KM_EINVAL, "km_tucker: intermediate %d does not fit in out; pass ws1", a + 1);
  }
  // small planes: the first two products fused per i3-plane (kmb200_plane.cuh).  The
  // fused launch writes dst[1] (ws0), so a pre-pass must not land there: it takes alt
  // (ws1 or out; out is read by the fused launch before the last product writes it).
  const bool fuse = d == 3 && na == 3 && u_dtype == KM_C128 && mat_dtypes[0] == KM_C128 &&
                    mat_dtypes[1] == KM_C128 && rows[0] == dims[0] && rows[1] == dims[1] &&
                    plane12_supported(dims[0], dims[1], dims[2]) &&
                    !((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(mats[0]) |
                       reinterpret_cast<uintptr_t>(mats[1]) | reinterpret_cast<uintptr_t>(ws0) |
                       reinterpret_cast<uintptr_t>(alt)) & 15);
  const void* src = u;
  if (has_pre) {
    void* pd = fuse ? alt : (dst[0] == ws0) ? alt : ws0;
    if (pd == out && static_cast<size_t>(n_in) * elem_bytes(u_dtype) > out_bytes)
      return fail(KM_EINVAL, "km_tucker: the pre-pass does not fit in out; pass ws1");
    if ((rc = pointwise_impl(u, pd, u_dtype, n_in, pre, st))) return rc;
    src = pd;
  }
  int dt = u_dtype;
  int a0 = 0;
  if (fuse) {
    if ((rc = launch_plane12(src, mats[0], mats[1], dst[1], dims[0], dims[1], dims[2], st))) return rc;
    a0 = 2;
    src = dst[1];
  }
  for (int a = a0; a < na; ++a) {
    const int mu = active[a];
    int64_t nl = 1, nr = 1;
    for (int i = 0; i < mu; ++i) nl *= cur[i];
    for (int i = mu + 1; i < d; ++i) nr *= cur[i];
    const bool last = (a == na - 1);
    km_pointop post_here;
    const km_pointop* pp = nullptr;
    if (last && has_post) {
      post_here = *post;
      pp = &post_here;
    }
    if ((rc = mumode_impl(src, dt, mats[mu], mat_dtypes[mu], dst[a], rows[mu], nl, cur[mu], nr, pp, st))) return rc;
    dt = promote(dt, mat_dtypes[mu]);
    cur[mu] = rows[mu];
    src = dst[a];
  }
  return KM_OK;
}

}  // extern "C"
