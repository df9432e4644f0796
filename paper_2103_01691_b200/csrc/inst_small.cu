// Host side of mumode_steps_kernel (kmb200_small.cuh): eligibility, workspace
// layout, counters, cooperative persistent launch.
#include "kmb200_small.cuh"

namespace kmb {

#ifdef KMB_STEPS_TRACE
unsigned long long* g_steps_trace = nullptr;  // set by km_steps_small_trace (probe builds only)
#endif

namespace {
bool steps_eligible(int64_t n1, int64_t n2, int64_t n3, int64_t steps) {
  const int64_t n[3] = {n1, n2, n3};
  for (int i = 0; i < 3; ++i)
    if (n[i] < sm::BT || n[i] > sm::KMAX || n[i] % sm::BT != 0) return false;
  return steps >= 1 && 3 * steps <= (int64_t(1) << 20);
}
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

int steps_small_workspace(int64_t n1, int64_t n2, int64_t n3, int64_t steps, size_t* bytes) {
  if (!bytes) return fail(KM_EINVAL, "km_steps_small_workspace_bytes: NULL output");
  if (!steps_eligible(n1, n2, n3, steps))
    return fail(KM_EINVAL,
                "km_steps_small: extents (%lld, %lld, %lld) must be multiples of %d in [%d, %d], steps >= 1",
                (long long)n1, (long long)n2, (long long)n3, sm::BT, sm::BT, sm::KMAX);
  const size_t state = static_cast<size_t>(n1 * n2 * n3) * 16;
  *bytes = 2 * align256(state) + static_cast<size_t>(3 * steps) * sm::CNT_STRIDE * sizeof(unsigned);
  return KM_OK;
}

int launch_steps_small(void* state, const void* E1, const void* E2, const void* E3, int64_t n1, int64_t n2,
                       int64_t n3, int64_t steps, void* ws, size_t ws_bytes, cudaStream_t st) {
  size_t need = 0;
  if (int rc = steps_small_workspace(n1, n2, n3, steps, &need)) return rc;
  if (!state || !E1 || !E2 || !E3 || !ws) return fail(KM_EINVAL, "km_steps_small: NULL pointer");
  if (ws_bytes < need) return fail(KM_EINVAL, "km_steps_small: workspace %zu bytes, %zu needed", ws_bytes, need);
  if ((reinterpret_cast<uintptr_t>(state) | reinterpret_cast<uintptr_t>(ws) | reinterpret_cast<uintptr_t>(E1) |
       reinterpret_cast<uintptr_t>(E2) | reinterpret_cast<uintptr_t>(E3)) & 15)
    return fail(KM_EINVAL, "km_steps_small: buffers must be 16-B aligned");
  const size_t sbytes = align256(static_cast<size_t>(n1 * n2 * n3) * 16);
  sm::Params P;
  P.buf[0] = static_cast<double2*>(state);
  P.buf[1] = reinterpret_cast<double2*>(static_cast<char*>(ws));
  P.buf[2] = reinterpret_cast<double2*>(static_cast<char*>(ws) + sbytes);
  P.E[0] = static_cast<const double2*>(E1);
  P.E[1] = static_cast<const double2*>(E2);
  P.E[2] = static_cast<const double2*>(E3);
  P.n[0] = static_cast<int>(n1);
  P.n[1] = static_cast<int>(n2);
  P.n[2] = static_cast<int>(n3);
  P.products = static_cast<int>(3 * steps);
  P.cnt = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + 2 * sbytes);
  P.trace = nullptr;
#ifdef KMB_STEPS_TRACE
  P.trace = g_steps_trace;
#endif
  const size_t cbytes = static_cast<size_t>(P.products) * sm::CNT_STRIDE * sizeof(unsigned);
  cudaError_t e = cudaMemsetAsync(P.cnt, 0, cbytes, st);
  if (e != cudaSuccess) return fail(KM_ECUDA, "km_steps_small counters: %s", cudaGetErrorString(e));
  int kmax = static_cast<int>(n1 > n2 ? (n1 > n3 ? n1 : n3) : (n2 > n3 ? n2 : n3));
  const int smem = sm::smem_bytes(kmax);
  auto kern = sm::mumode_steps_kernel;
  if (int rc = ensure_smem(reinterpret_cast<const void*>(kern), smem, "mumode_steps_kernel")) return rc;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, sm::THREADS, smem) != cudaSuccess || per_sm < 1)
    return fail(KM_ECUDA, "km_steps_small: no resident CTA (%d B of shared memory)", smem);
  // persistent, at most one CTA per tile of the largest product: CTA c then takes tile c of
  // every product (more CTAs than tiles would queue a product's last tiles behind the
  // previous product's on the same CTAs, measured: every product then costs two tile latencies)
  const int64_t t1 = (n2 / sm::BT) * n3 * (n1 / sm::BT), t2 = (n1 / sm::BT) * n3 * (n2 / sm::BT),
                t3 = (n1 / sm::BT) * n2 * (n3 / sm::BT);
  const int64_t tmax = t1 > t2 ? (t1 > t3 ? t1 : t3) : (t2 > t3 ? t2 : t3);
  const int64_t resident = static_cast<int64_t>(per_sm) * num_sms();
  const int grid = static_cast<int>(tmax < resident ? tmax : resident);
  sm::Params* pp = &P;
  void* args[] = {pp};
  e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(sm::THREADS), args, smem, st);
  if (e != cudaSuccess) return fail(KM_ECUDA, "mumode_steps_kernel: %s", cudaGetErrorString(e));
  return KM_OK;
}

}  // namespace kmb

#ifdef KMB_STEPS_TRACE
extern "C" void km_steps_small_trace(void* buf) { kmb::g_steps_trace = static_cast<unsigned long long*>(buf); }
#endif
