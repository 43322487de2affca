// FP64 peak probe for B200 (sm_100a): DFMA (CUDA-core) vs DMMA (mma.sync f64 tensor path).
// Prints achieved TFLOP/s per variant; used to pick the roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  // m8n8k4: A 8x4 (1 f64/lane), B 4x8 (1 f64/lane), C/D 8x8 (2 f64/lane)
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; CK(cudaMalloc(&d, 8));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("device %s SMs %d\n", p.name, sms);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int iters = 20000;
      dfma_kernel<8><<<sms * bps, threads>>>(d, 100, 1.0000001, 1e-9);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_kernel<8><<<sms * bps, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * iters * (double)threads * sms * bps;
      printf("DFMA  threads=%d blocks/SM=%d : %.2f TFLOP/s (%.3f ms)\n", threads, bps, flops / ms / 1e9, ms);
    }
  }
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int iters = 5000;
      dmma_kernel<4><<<sms * bps, threads>>>(d, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_kernel<4><<<sms * bps, threads>>>(d, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 8 * 4 * 4 * iters * (double)(threads / 32) * sms * bps;
      printf("DMMA  threads=%d blocks/SM=%d : %.2f TFLOP/s (%.3f ms)\n", threads, bps, flops / ms / 1e9, ms);
    }
  }
  return 0;
}
