// FP64 peak micro-benchmark for the roofline denominator (MEASURED_PEAKS.json has
// no FP64 entry). Measures: DMMA (mma.sync m8n8k4 f64) and DFMA throughput, and a
// plain device copy (HBM GB/s). Timed with CUDA events after warm-up.
#include <cstdio>
#include <cuda_runtime.h>

#define CHK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  int sms; CHK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CHK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int iters = 4096;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dmma_loop<8><<<sms * 2, warps * 32>>>(out, iters);
      cudaEventRecord(e1); CHK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)sms * 2 * warps * iters * 8 * (8.0 * 8 * 4 * 2);
    printf("{\"kind\":\"dmma_m8n8k4\",\"warps_per_cta\":%d,\"tflops\":%.2f}\n", warps, flops / ms / 1e9);
  }
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dfma_loop<8><<<sms * 2, warps * 32>>>(out, iters);
      cudaEventRecord(e1); CHK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)sms * 2 * warps * 32 * iters * 8 * 2.0;
    printf("{\"kind\":\"dfma\",\"warps_per_cta\":%d,\"tflops\":%.2f}\n", warps, flops / ms / 1e9);
  }
  size_t bytes = (size_t)2 << 30;
  double2 *a, *b; CHK(cudaMalloc(&a, bytes)); CHK(cudaMalloc(&b, bytes));
  cudaMemset(a, 0, bytes);
  size_t n = bytes / 16;
  float best = 1e9;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0);
    copy_k<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); CHK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("{\"kind\":\"copy\",\"gbs\":%.1f}\n", 2.0 * bytes / best / 1e6);
  return 0;
}
