// Standalone probe of the tcgen05 3xTF32 GEMM (tc_gemm.cuh): small shapes, prints errors.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cudaTypedefs.h>
#include "../../paper_2601_14466_b200/csrc/tc_gemm.cuh"
namespace bcmg { void note_launch() {} }
using namespace bcmg;
static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* f; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)f;
}
static CUtensorMap mk(const void* base, int64_t rows, int64_t cols, int64_t ld) {
  CUtensorMap m; cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols}; cuuint64_t str[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)tc::BK}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode failed %d\n", (int)r);
  return m;
}
int main(int argc, char** argv) {
  int M = argc > 1 ? atoi(argv[1]) : 256, N = argc > 2 ? atoi(argv[2]) : 128, K = argc > 3 ? atoi(argv[3]) : 32;
  std::vector<float> A((size_t)M * K), B((size_t)N * K), Cc((size_t)M * N, 0.f);
  srand(1);
  for (auto& x : A) x = (float)(rand() % 9 - 4);
  for (auto& x : B) x = (float)(rand() % 9 - 4);
  float *dA, *dB, *dC; cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, Cc.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, Cc.size() * 4);
  CUtensorMap ma = mk(dA, M, K, M), mb = mk(dB, N, K, N);
  cudaFuncSetAttribute(tc3_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::SMEM_BYTES);
  int nb = ((M + 127) / 128) * ((N + 127) / 128);
  tc3_gemm_kernel<<<nb, tc::THREADS, tc::SMEM_BYTES>>>(ma, mb, M, N, K, dC, M, 1.f, 0.f, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  printf("M=%d N=%d K=%d err=%s\n", M, N, K, cudaGetErrorString(e));
  cudaMemcpy(Cc.data(), dC, Cc.size() * 4, cudaMemcpyDeviceToHost);
  double maxd = 0, maxr = 0; int bad = 0, firsti = -1, firstj = -1;
  for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
    double r = 0; for (int k = 0; k < K; ++k) r += (double)A[i + (size_t)k * M] * B[j + (size_t)k * N];
    double d = fabs(r - Cc[i + (size_t)j * M]); maxr = fmax(maxr, fabs(r));
    if (d > 1e-3) { if (!bad) { firsti = i; firstj = j; } ++bad; }
    maxd = fmax(maxd, d);
  }
  printf("maxdiff %.3f maxref %.1f bad %d first (%d,%d) got %f\n", maxd, maxr, bad, firsti, firstj, firsti >= 0 ? Cc[firsti + (size_t)firstj * M] : 0.f);
  for (int i = 0; i < 4; ++i) { for (int j = 0; j < 6; ++j) printf("%7.1f ", Cc[i + (size_t)j * M]); printf("\n"); }
  return 0;
}
