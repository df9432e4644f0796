// FP64 peak microbenchmark for the B200 roofline denominator.
// Measures (a) mma.sync m8n8k4 f64 (SASS DMMA.8x8x4) and (b) scalar DFMA
// throughput with register-resident operands, at several warps/SM, timed with
// CUDA events. Output: one line per variant, TFLOP/s (2 flop per FMA).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double acc[CHAINS][2];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { acc[c][0] = 0.0; acc[c][1] = c * 1e-12; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(acc[c][0]), "+d"(acc[c][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = c * 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(a, b, acc[c]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// half the warps of each CTA run DMMA chains, the other half DFMA chains: does the FP64
// datapath serve both at once (sum of the two rates) or share one pipe?
__global__ void mixed_loop(double* out, int iters, double seed) {
  const int warp = threadIdx.x >> 5;
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double acc[8][2];
#pragma unroll
  for (int c = 0; c < 8; ++c) { acc[c][0] = 0.0; acc[c][1] = c * 1e-12; }
  if (warp % 2 == 0) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
  } else {
    for (int it = 0; it < iters * 4; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c][0] = fma(a, b, acc[c][0]);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

static int run_mixed(int warps) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 4096 * sizeof(double)));
  const int iters = 20000;
  dim3 grid(sms), block(32 * warps);
  mixed_loop<<<grid, block>>>(out, iters, 1.0);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    mixed_loop<<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  // per SM: warps/2 DMMA warps x iters x 8 chains x 512 flop; warps/2 DFMA warps x 4 iters x 8 x 64 flop
  const double dmma = double(sms) * (warps / 2) * iters * 8 * 512.0;
  const double dfma = double(sms) * (warps / 2) * iters * 4.0 * 8 * 64.0;
  printf("mixed DMMA + DFMA warps/SM=%3d  %.3f ms  DMMA part %.2f + DFMA part %.2f = %.2f TFLOP/s\n", warps, best,
         dmma / (best * 1e-3) / 1e12, dfma / (best * 1e-3) / 1e12, (dmma + dfma) / (best * 1e-3) / 1e12);
  cudaFree(out);
  return 0;
}

template <typename K>
static int run(const char* name, K kern, int warps_per_cta, int ctas_per_sm, int iters, double flop_per_thread_iter) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 4096 * sizeof(double)));
  dim3 grid(sms * ctas_per_sm), block(32 * warps_per_cta);
  kern<<<grid, block>>>(out, iters, 1.0);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double flops = double(grid.x) * block.x * iters * flop_per_thread_iter;
  printf("%-28s warps/SM=%3d  %.3f ms  %.2f TFLOP/s\n", name, warps_per_cta * ctas_per_sm, best,
         flops / (best * 1e-3) / 1e12);
  cudaFree(out);
  return 0;
}

// back-to-back launches for ~seconds: the power-capped sustained rate
static int sustained(double seconds) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 4096 * sizeof(double)));
  dim3 grid(sms), block(256);
  const int iters = 20000;
  dmma_loop<8><<<grid, block>>>(out, iters, 1.0);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  // calibrate launches per second
  cudaEventRecord(e0);
  for (int i = 0; i < 10; ++i) dmma_loop<8><<<grid, block>>>(out, iters, 1.0);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int n = (int)(seconds * 1000.0 / (ms / 10));
  cudaEventRecord(e0);
  for (int i = 0; i < n; ++i) dmma_loop<8><<<grid, block>>>(out, iters, 1.0);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = double(grid.x) * block.x * iters * 8 * 16.0 * n;
  printf("SUSTAINED dmma m8n8k4 %d launches %.3f s  %.2f TFLOP/s\n", n, ms / 1e3, flops / (ms * 1e-3) / 1e12);
  cudaFree(out);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1) return sustained(atof(argv[1]));
  const int iters = 20000;
  // one m8n8k4 = 256 FMA per warp = 8 FMA per thread = 16 flop per thread.
  for (int w : {4, 8, 16, 32}) run("dmma m8n8k4 chains=8", dmma_loop<8>, w, 1, iters, 8 * 16.0);
  run("dmma m8n8k4 chains=16", dmma_loop<16>, 8, 1, iters / 2, 16 * 16.0);
  run("dmma m8n8k4 chains=2", dmma_loop<2>, 16, 1, iters * 4, 2 * 16.0);
  for (int w : {8, 16, 32}) run("dfma chains=8", dfma_loop<8>, w, 1, iters * 4, 8 * 2.0);
  for (int w : {8, 16}) run_mixed(w);
  return 0;
}
