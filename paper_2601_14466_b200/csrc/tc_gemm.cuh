// float32 contractions on the 5th-gen tensor cores: tcgen05.mma kind::tf32
// with a 3xTF32 split (a = a_hi + a_lo, a*b ~= a_hi*b_hi + a_hi*b_lo +
// a_lo*b_hi, FP32 accumulation in TMEM) -- FP32-level accuracy at tensor-core
// rate, as the north star asks for float32 / complex64.
//
// Warp-specialised persistent kernel, 12 warps:
//   warp 0        TMA producer: fp32 boxes {32 rows, BK} (SWIZZLE_128B) of
//                 the operands as stored (rows contiguous) into a raw ring
//   warp 1        TMEM allocator + single-thread MMA issuer
//   warps 2,3,8-11 splitters: raw -> K-major SW128 "hi" = rna_tf32(x) and
//                 "lo" = x - hi planes (kind::tf32 takes K-major operands
//                 only), then fence.proxy.async for the tensor core
//   warps 4-7     epilogue warpgroup: tcgen05.ld 32x32b accumulator rows,
//                 C := alpha*acc + beta*C, coalesced along the column
// Pipelines: raw stages (TMA tx -> split), split stages (split -> MMA commit),
// two TMEM accumulators (commit -> epilogue), so TMA, splitting, MMA and the
// epilogue of the previous tile all overlap.
#pragma once

#include "gemm_tma.cuh"

namespace bcmg {

namespace tc {

constexpr int BM = 128, BN = 128, BK = 32;
constexpr int RAW_STAGES = 2, SPL_STAGES = 2;
constexpr int THREADS = 384;                         // 12 warps (see the role map above)
constexpr int SPLIT_WARPS = 6;                       // warps 2, 3, 8, 9, 10, 11
constexpr int ATOM_BYTES = 32 * 4 * BK;              // raw: one 32-row MN chunk x BK k-rows
constexpr int PLANE_A = BM * BK * 4, PLANE_B = BN * BK * 4;  // 16 KB each
constexpr int RAW_BYTES = PLANE_A + PLANE_B;         // raw stage (TMA, MN-major)
constexpr int SPL_BYTES = 2 * (PLANE_A + PLANE_B);   // split stage: A hi, A lo, B hi, B lo (K-major)
constexpr int TMEM_COLS = 2 * BN;                    // two accumulators
constexpr size_t SMEM_BYTES = 1024 /*align slack*/ + (size_t)RAW_STAGES * RAW_BYTES + (size_t)SPL_STAGES * SPL_BYTES + 256;

// UMMA instruction descriptor: D f32, A/B tf32, both K-major (kind::tf32 on
// sm_100a accepts only K-major operands -- measured: MN-major writes nothing),
// M=128, N=128.
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

// Shared-memory matrix descriptor, K-major SWIZZLE_128B: rows of 128 B (32 k),
// 8-row 1 KB atoms stacked along M/N (SBO = 1 KB), LBO unused (16 B).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)((1024 >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | (2ull << 61);
}

// raw (TMA, MN-major SW128) byte offset of element (i, k) of a 128 x BK tile
__device__ __forceinline__ int raw_off(int i, int k) {
  return (i >> 5) * ATOM_BYTES + k * 128 + ((((i & 31) >> 2) ^ (k & 7)) << 4) + ((i & 3) << 2);
}
// K-major SW128 byte offset of the 16-byte chunk holding (i, 4c .. 4c+3)
__device__ __forceinline__ int kmaj_off(int i, int c) { return (i >> 3) * 1024 + (i & 7) * 128 + ((c ^ (i & 7)) << 4); }

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Block of work: output rows [m0, m0+BM) x cols [n0, n0+BN); TMA row
// coordinates of its A and B panels; epilogue target.
struct Blk {
  int a_row, b_row;
  int64_t m0, n0, M, N;
  float* C;
  int64_t ldc;
  float alpha, beta;
  float* fan[MAX_FAN];  // peer copies of C (Epilogue::fan)
  int nfan;
  // TMA epilogue (tck_loop_epi): C's tensor map (local device) and the map
  // coordinates of the item's row / column 0 (the block adds m0 / n0)
  int cdev;
  int64_t crow0, ccol0;
  // 2-SM pair kernel (tck_loop_pair): B rows of CTA rank 1 (< 0: b_row + 128), and
  // a second output column tile for tile columns >= 128 (C2, same row base as C;
  // its rows < skip2 lie above that tile column's diagonal and are not written)
  int b_row1 = -1;
  float* C2 = nullptr;
  int64_t skip2 = 0;
  int cdev2 = 0;        // TMA epilogue: C2's local device and map column
  int64_t ccol02 = 0;
};

template <class Next>
__device__ __forceinline__ void tc3_loop(const CUtensorMap* mapA, const CUtensorMap* mapB, int K, Next&& next) {
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  // 1024-byte aligned base for the SWIZZLE_128B atoms
  unsigned char* base = tc_smem_raw + ((1024 - (smem_u32(tc_smem_raw) & 1023)) & 1023);
  unsigned char* raw = base;                                       // RAW_STAGES x RAW_BYTES
  unsigned char* spl = base + (size_t)RAW_STAGES * RAW_BYTES;      // SPL_STAGES x SPL_BYTES
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(spl + (size_t)SPL_STAGES * SPL_BYTES);
  uint64_t* raw_free = raw_full + RAW_STAGES;
  uint64_t* spl_ready = raw_free + RAW_STAGES;
  uint64_t* spl_empty = spl_ready + SPL_STAGES;
  uint64_t* tfull = spl_empty + SPL_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RAW_STAGES; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_free[s], SPLIT_WARPS);
    }
    for (int s = 0; s < SPL_STAGES; ++s) {
      mbar_init(&spl_ready[s], SPLIT_WARPS);
      mbar_init(&spl_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      uint32_t g = 0;
      Blk blk;
      for (int64_t item = blockIdx.x; next(item, blk); item += gridDim.x) {
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int s = g % RAW_STAGES;
          mbar_wait(&raw_free[s], ((g / RAW_STAGES) & 1) ^ 1);
          unsigned char* st = raw + (size_t)s * RAW_BYTES;
          mbar_expect_tx(&raw_full[s], RAW_BYTES);
#pragma unroll
          for (int c = 0; c < BM / 32; ++c)
            tma_load_2d(st + c * ATOM_BYTES, mapA, blk.a_row + (int)blk.m0 + 32 * c, kt * BK, &raw_full[s]);
#pragma unroll
          for (int c = 0; c < BN / 32; ++c)
            tma_load_2d(st + PLANE_A + c * ATOM_BYTES, mapB, blk.b_row + (int)blk.n0 + 32 * c, kt * BK,
                        &raw_full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      uint32_t g = 0, t = 0;
      Blk blk;
      for (int64_t item = blockIdx.x; next(item, blk); item += gridDim.x, ++t) {
        const int b = t & 1;
        mbar_wait(&tempty[b], ((t >> 1) & 1) ^ 1);
        fence_after();
        const uint32_t d = tmem + b * BN;
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int s = g % SPL_STAGES;
          mbar_wait(&spl_ready[s], (g / SPL_STAGES) & 1);
          fence_after();
          const uint32_t st = smem_u32(spl + (size_t)s * SPL_BYTES);
          const uint32_t ahi = st, alo = st + PLANE_A, bhi = st + 2 * PLANE_A, blo = bhi + PLANE_B;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint32_t off = ks * 32;  // 8 tf32 k = 32 bytes along the 128-byte K-major row
            // small terms first, then the dominant hi*hi product
            mma_tf32(d, sdesc(alo + off), sdesc(bhi + off), (kt | ks) != 0);
            mma_tf32(d, sdesc(ahi + off), sdesc(blo + off), 1);
            mma_tf32(d, sdesc(ahi + off), sdesc(bhi + off), 1);
          }
          commit(&spl_empty[s]);  // split stage reusable once these MMAs have read it
        }
        commit(&tfull[b]);  // accumulator b complete
      }
    }
  } else if (warp < 4 || warp >= 8) {
    // ---------------------------------------------------------- splitters
    // raw MN-major (TMA) -> K-major SW128 hi / lo planes.  A warp takes 32
    // consecutive rows i of one 4-wide k chunk: the four scalar raw loads and
    // the 16-byte hi / lo stores are all bank-conflict free.
    const int sw = warp < 4 ? warp - 2 : warp - 6;  // 0..5
    // A warp owns whole 32-row groups (operand x 4 groups = 8 per k-step): the
    // lane's row is fixed, so the swizzle terms of its raw reads and K-major
    // writes are computed once (xo / wo) and every access in the fully
    // unrolled k loop is a register base plus an immediate.
    const int xr = (lane >> 2) & 7;  // raw swizzle row phase ((i & 31) >> 2)
    uint32_t g = 0;
    Blk blk;
    for (int64_t item = blockIdx.x; next(item, blk); item += gridDim.x) {
      for (int kt = 0; kt < KT; ++kt, ++g) {
        const int rs = g % RAW_STAGES, ss = g % SPL_STAGES;
        mbar_wait(&raw_full[rs], (g / RAW_STAGES) & 1);
        mbar_wait(&spl_empty[ss], ((g / SPL_STAGES) & 1) ^ 1);
        const unsigned char* rst = raw + (size_t)rs * RAW_BYTES;
        unsigned char* sst = spl + (size_t)ss * SPL_BYTES;
        for (int rg = sw; rg < 8; rg += SPLIT_WARPS) {
          const int op = rg >> 2, grp = rg & 3;
          const int i = grp * 32 + lane, xw = i & 7;
          const unsigned char* rsrc = rst + op * PLANE_A + grp * ATOM_BYTES + ((lane & 3) << 2);
          unsigned char* dst = sst + op * 2 * PLANE_A + (i >> 3) * 1024 + (i & 7) * 128;
          const unsigned char* rb[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) rb[j] = rsrc + ((xr ^ j) << 4);
#pragma unroll
          for (int c = 0; c < BK / 4; ++c) {
            float x[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int k = 4 * c + e;
              x[e] = *reinterpret_cast<const float*>(rb[k & 7] + k * 128);
            }
            const float4 h = make_float4(tf32_rna(x[0]), tf32_rna(x[1]), tf32_rna(x[2]), tf32_rna(x[3]));
            const float4 l = make_float4(x[0] - h.x, x[1] - h.y, x[2] - h.z, x[3] - h.w);
            unsigned char* d = dst + ((c ^ xw) << 4);
            *reinterpret_cast<float4*>(d) = h;
            *reinterpret_cast<float4*>(d + PLANE_A) = l;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&spl_ready[ss]);
          mbar_arrive(&raw_free[rs]);
        }
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    const int q = warp - 4;  // TMEM lane quarter
    const int row = 32 * q + lane;
    uint32_t t = 0;
    Blk blk;
    for (int64_t item = blockIdx.x; next(item, blk); item += gridDim.x, ++t) {
      const int b = t & 1;
      const int64_t r = blk.m0 + row;
      float* __restrict__ crow = blk.C + r;
      auto load_chunk = [&](int c0, float* dst) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int64_t col = blk.n0 + c0 + j;
          dst[j] = (blk.beta != 0.f && r < blk.M && col < blk.N) ? crow[col * blk.ldc] : 0.f;
        }
      };
      // C does not depend on this tile's MMAs: pull the warp's 32 x 128 block into
      // L2 and load its first chunk while they run (short K leaves little MMA time
      // to hide the read-modify-write behind)
      if (blk.beta != 0.f) {
#pragma unroll
        for (int j = 0; j < BN / 32; ++j) {
          const int64_t col = blk.n0 + 4 * lane + j, r0 = blk.m0 + 32 * q;
          if (col < blk.N && r0 < blk.M) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(blk.C + r0 + col * blk.ldc));
        }
      }
      float old[32], nxt[32];
      load_chunk(0, old);
      mbar_wait(&tfull[b], (t >> 1) & 1);
      fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        // next chunk's C loads are in flight while this chunk is read from TMEM and stored
        if (c0 + 32 < BN) load_chunk(c0 + 32, nxt);
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + b * BN + c0, v);
        if (r < blk.M) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int64_t col = blk.n0 + c0 + j;
            if (col < blk.N) {
              const float o = blk.alpha * v[j] + blk.beta * old[j];
              crow[col * blk.ldc] = o;
              for (int e = 0; e < blk.nfan; ++e) fan_at(blk.fan, e)[r + col * blk.ldc] = o;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) old[j] = nxt[j];
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

}  // namespace tc

// C := alpha * A * B^T + beta * C, A (M x K) and B (N x K) M-/N-contiguous fp32.
__global__ void __launch_bounds__(tc::THREADS, 1)
    tc3_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int64_t M,
                    int64_t N, int64_t K, float* C, int64_t ldc, float alpha, float beta, const int* info) {
  if (ld_flag(info)) return;
  const int64_t nbm = (M + tc::BM - 1) / tc::BM, nbn = (N + tc::BN - 1) / tc::BN;
  tc::tc3_loop(&mapA, &mapB, (int)K, [&](int64_t item, tc::Blk& blk) -> bool {
    if (item >= nbm * nbn) return false;
    blk.a_row = 0;
    blk.b_row = 0;
    blk.m0 = (item % nbm) * tc::BM;
    blk.n0 = (item / nbm) * tc::BN;
    blk.M = M;
    blk.N = N;
    blk.C = C;
    blk.ldc = ldc;
    blk.alpha = alpha;
    blk.beta = beta;
    blk.nfan = 0;
    return true;
  });
}

// potrf trailing update for float32 shards (see trail_kernel): stateless
// decode (every role walks the same item sequence independently).
// complex64 (p.cplx): the real embedding of TrailParams (A = [P | -iP] as a
// (2 rows) x (2K) float matrix, B = planar [Re P | Im P]); a 128-row tile then
// covers 64 complex rows (TrapH enumeration) and C is addressed as floats.
__global__ void __launch_bounds__(tc::THREADS, 1)
    tc3_trail_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     TrailParams p, const int* info) {
  using TZ = Trap<tc::BM, tc::BN>;
  using TZC = TrapH<tc::BM / 2, tc::BN>;
  if (ld_flag(info)) return;
  int64_t cm = p.m_first, cbase = 0, ccnt = -1;  // per-thread monotone cursor
  tc::tc3_loop(&mapA, &mapB, (int)(p.cplx ? 2 * p.K : p.K), [&](int64_t item, tc::Blk& blk) -> bool {
    for (;;) {
      if (cm >= p.m_last) return false;
      const int dev = (int)(cm % p.D);
      if (dev >= p.dev0 && dev < p.dev0 + p.nloc) {
        if (ccnt < 0) {
          const int64_t ms = cm * p.T, tcm = p.T < p.N - ms ? p.T : p.N - ms;
          ccnt = p.cplx ? TZC::count(p.N - ms, tcm) : TZ::count(p.N - ms, tcm);
        }
        if (item < cbase + ccnt) break;
        cbase += ccnt;
      }
      ++cm;
      ccnt = -1;
    }
    const int64_t ms = cm * p.T, rows = p.N - ms, tcw = p.T < rows ? p.T : rows;
    int64_t rb, cb;
    const int dev = (int)(cm % p.D);
    float* shard = reinterpret_cast<float*>(p.shards[dev - p.dev0]);
    const int64_t loc = (cm / p.D) * p.T;
    if (p.cplx) {
      TZC::decode(item - cbase, tcw, rb, cb);
      blk.a_row = (int)(2 * (ms - p.prow0));
      blk.b_row = (int)(ms - p.prow0);
      blk.m0 = rb * tc::BM;
      blk.n0 = cb * tc::BN;
      blk.M = 2 * rows;
      blk.N = tcw;
      blk.C = shard + 2 * (ms + loc * p.N);
      blk.ldc = 2 * p.N;
      blk.alpha = -1.f;
      blk.beta = 1.f;
      blk.nfan = 0;
      return true;
    }
    TZ::decode(item - cbase, tcw, rb, cb);
    blk.a_row = (int)(ms - p.prow0);
    blk.b_row = (int)(ms - p.prow0);
    blk.m0 = rb * tc::BM;
    blk.n0 = cb * tc::BN;
    blk.M = rows;
    blk.N = tcw;
    blk.C = shard + ms + loc * p.N;
    blk.ldc = p.N;
    blk.alpha = -1.f;
    blk.beta = 1.f;
    blk.nfan = 0;
    return true;
  });
}

}  // namespace bcmg
