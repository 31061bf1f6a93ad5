// FP64 peak probe: DMMA (mma.sync m8n8k4 f64, SASS DMMA.8x8x4) and DFMA, register-resident.
// Used to establish the FP64 roofline denominator on the B200 box (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int ACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int bps = 1; bps <= 2; ++bps) {
      dim3 grid(sms * bps), block(32 * warps);
      dmma_loop<8><<<grid, block>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<8><<<grid, block>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid.x * warps;
      printf("DMMA warps/cta=%2d ctas/sm=%d: %.2f TFLOP/s (%.3f ms)\n", warps, bps, flops / ms / 1e9, ms);
    }
  }
  for (int warps = 4; warps <= 16; warps *= 2) {
    dim3 grid(sms * 2), block(32 * warps);
    dfma_loop<8><<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<8><<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8.0 * iters * (double)grid.x * 32 * warps;
    printf("DFMA warps/cta=%2d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s sms=%d\n", cudaGetErrorString(err), sms);
  return 0;
}
