// Inner-loop ceiling of the 3M complex DMMA GEMM (zgemm3m_kernel) on B200: the same warp tile
// (32 x 16, 4 x 2 DMMA.8x8x4 sub-tiles x 3 Gauss products), fragments read from shared memory,
// no global traffic.  Variants isolate what the real kernel adds to pure DMMA issue:
//   v0  DMMA only (fragments loaded once)                 -> pipe ceiling with this register use
//   v1  + LDS.128 fragment loads per k-step (6 per 24 DMMA)
//   v2  + the 3M operand sums (6 DADD per k-step)
//   v3  + a __syncthreads every 2 k-steps (the cp.async kernel's per-stage barrier)
//   v4  the v2 DADDs, but their results feed a side accumulator instead of the DMMAs (pipe sharing
//       without the LDS -> DADD -> DMMA dependency)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_loop_probe tools/dmma_loop_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int V, int MINB>
__global__ void __launch_bounds__(256, MINB) loop_kernel(double* out, int iters) {
  __shared__ double2 sA[4 * 8 * 16 * 2];  // a few KB of fragments, cycled
  __shared__ double2 sB[4 * 8 * 16 * 2];
  for (int i = threadIdx.x; i < 4 * 8 * 16 * 2; i += blockDim.x) {
    sA[i] = make_double2(1.0 + i * 1e-7, 1e-7 * i);
    sB[i] = make_double2(1.0 - i * 1e-7, 2e-7 * i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[4][2][3][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[a][b][c][0] = acc[a][b][c][1] = 0.0;
  double ar[4], ai[4], as[4], br[2], bi[2], bs[2];
  double side = 0.0;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) { ar[mi] = sA[lane + mi].x; ai[mi] = sA[lane + mi].y; as[mi] = ar[mi] + ai[mi]; }
#pragma unroll
  for (int ni = 0; ni < 2; ++ni) { br[ni] = sB[lane + ni].x; bi[ni] = sB[lane + ni].y; bs[ni] = br[ni] + bi[ni]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      if (V >= 1) {
        const int base = ((it * 2 + ks) & 15) * 32 + (warp & 1) * 8;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const double2 a = sA[(base + lane + mi * 37) & 1023];
          ar[mi] = a.x; ai[mi] = a.y;
          as[mi] = (V >= 2 && V != 4) ? a.x + a.y : a.x;
          if (V == 4) side += a.x + a.y;
        }
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          const double2 b = sB[(base + lane + ni * 41) & 1023];
          br[ni] = b.x; bi[ni] = b.y;
          bs[ni] = (V >= 2 && V != 4) ? b.x + b.y : b.y;
          if (V == 4) side += b.x + b.y;
        }
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          dmma(acc[mi][ni][0][0], acc[mi][ni][0][1], ar[mi], br[ni]);
          dmma(acc[mi][ni][1][0], acc[mi][ni][1][1], ai[mi], bi[ni]);
          dmma(acc[mi][ni][2][0], acc[mi][ni][2][1], as[mi], bs[ni]);
        }
    }
    if (V == 3) __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) s += acc[a][b][c][0] + acc[a][b][c][1];
  if (s + side == 12345.678) out[0] = s;
}

template <int V, int MINB>
int run(int sms, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  loop_kernel<V, MINB><<<sms * MINB, 256>>>(d, 10);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  loop_kernel<V, MINB><<<sms * MINB, 256>>>(d, iters);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * 48.0 * iters * 8 * sms * MINB;  // 48 DMMA per iter per warp
  printf("v%d CTAs/SM=%d : %.2f TFLOP/s executed DMMA (%.3f ms)\n", V, MINB, flops / ms / 1e9, ms);
  return 0;
}

int main() {
  double* d;
  CK(cudaMalloc(&d, 8));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  run<0, 2>(sms, d); run<1, 2>(sms, d); run<2, 2>(sms, d); run<3, 2>(sms, d); run<4, 2>(sms, d);
  run<0, 1>(sms, d); run<1, 1>(sms, d); run<2, 1>(sms, d); run<3, 1>(sms, d); run<4, 1>(sms, d);
  return 0;
}
