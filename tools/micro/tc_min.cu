// Minimal tcgen05.mma kind::tf32 probe: A = B = 1 in smem, one MMA, read TMEM.
#include <cstdio>
#include <cstdint>
#include "../../paper_2601_14466_b200/csrc/tc_gemm.cuh"
namespace bcmg { void note_launch() {} }
using namespace bcmg;
__global__ void k(float* out, int variant) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* base = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  float* A = reinterpret_cast<float*>(base);           // 128 x 32 (4 atoms of 4 KB)
  float* B = reinterpret_cast<float*>(base + 16384);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { A[i] = 1.f; B[i] = (variant == 2) ? (float)(i % 7) : 1.f; }
  if (variant == 5) for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
    reinterpret_cast<uint32_t*>(A)[i] = 0x3f803f80u; reinterpret_cast<uint32_t*>(B)[i] = 0x3f803f80u; }
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc::fence_before(); __syncthreads(); tc::fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(A), b = smem_u32(B);
    uint64_t da = tc::sdesc(a), db = tc::sdesc(b);
    if (variant == 1) {  // K-major, no swizzle: core matrices 8 rows x 16 B
      da = (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
      db = (uint64_t)((b >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
    }
    printf("idesc=%08x da=%016llx db=%016llx tmem=%08x\n", tc::IDESC, (unsigned long long)da, (unsigned long long)db, tmem);
    if (variant == 3) {
      // tcgen05.st path check is done below by all threads; just commit
    } else if (variant == 5) {
      // kind::f16 with bf16 ones (A, B buffers reinterpreted: bf16 1.0 = 0x3f80)
      const uint32_t idesc_bf16 = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | (16u << 17) | (8u << 24);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc_bf16), "r"(0));
    } else if (variant >= 6) {
      uint32_t id = tc::IDESC;
      if (variant == 6) id &= ~((1u << 15) | (1u << 16));                 // K-major A and B
      if (variant == 7) id = (id & ~(0x3Fu << 17)) | ((64u >> 3) << 17);   // N = 64
      if (variant == 8) id &= ~(1u << 15);                                  // A K-major only
      if (variant == 9) id &= ~(1u << 16);                                  // B K-major only
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(id), "r"(0));
    } else if (variant == 4) {
      uint32_t m0 = 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(tc::IDESC), "r"(0), "r"(m0));
    } else {
      tc::mma_tf32(tmem, da, db, 0);
    }
    tc::commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  if (variant == 3) {
    uint32_t val = __float_as_uint(7.0f + threadIdx.x);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(tmem + ((uint32_t)(32 * warp) << 16)), "r"(val));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  tc::fence_after();
  float v[32];
  tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), v);
  if (threadIdx.x % 32 == 0) printf("warp %d row %d: %f %f %f %f\n", warp, threadIdx.x, v[0], v[1], v[2], v[31]);
  out[threadIdx.x] = v[0];
  tc::fence_before(); __syncthreads();
  if (warp == 0) { tc::fence_after(); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256)); }
}
int main() {
  float* out; cudaMalloc(&out, 4096);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int v = 6; v < 10; ++v) { printf("variant %d\n", v); k<<<1, 128, 64 * 1024>>>(out, v); printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize())); }
}
