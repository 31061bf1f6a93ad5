// 3xTF32 tcgen05 GEMM on PRE-SPLIT operands.
//
// tc_gemm.cuh splits every operand tile into tf32 hi / lo planes inside the
// CTA, and that splitting (raw read + two plane writes per element, every
// time a tile is used) plus the tensor core's own operand reads saturate the
// SM's shared-memory bandwidth at ~1/3 of the tf32 MMA rate.  Here each
// operand is split ONCE in global memory (split_tf32 kernel, K-major rows:
// hi = rna_tf32(x), lo = x - hi) and TMA delivers the hi / lo tiles straight
// into the canonical K-major SWIZZLE_128B layout the UMMA descriptors
// describe; no splitter warps remain:
//   warp 0        TMA producer: A hi, A lo, B hi, B lo boxes {32 k, 128 rows}
//   warp 1        TMEM allocator + single-thread MMA issuer (3 MMAs per k8:
//                 lo*hi, hi*lo, hi*hi into an FP32 accumulator)
//   warps 4-11    epilogue: two warpgroups, each owns half of the accumulator
//                 columns (TMEM lane quarter = warp % 4)
// Stages: 3 x 64 KB operand ring (TMA tx -> MMA commit), two TMEM
// accumulators (MMA commit -> epilogue).
#pragma once

#include "tc_gemm.cuh"

namespace bcmg {
struct FloatFan {  // peer copies of a tcgen05 GEMM's output (Epilogue::fan)
  float* p[MAX_FAN];
  int n;
};
namespace tck {

using tc::BM;
using tc::BK;
// BNT: 128 or 256 output columns per tile (UMMA M=128, N=BNT).  N=256 halves
// the A-operand traffic (TMA and tensor-core shared-memory reads) per flop.
template <int BNT>
struct Cfg {
  static_assert(BNT == 128 || BNT == 256, "tile width");
  static constexpr int PLANE_A = BM * BK * 4, PLANE_B = BNT * BK * 4;
  static constexpr int STAGE_BYTES = 2 * (PLANE_A + PLANE_B);   // A hi, A lo, B hi, B lo
  static constexpr int STAGES = BNT == 256 ? 2 : 3;
  static constexpr int TMEM_COLS = 2 * BNT;
  static constexpr size_t SMEM_BYTES = 1024 + (size_t)STAGES * STAGE_BYTES + 256;
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BNT >> 3) << 17) |
                                    ((uint32_t)(BM >> 4) << 24);
};
constexpr int THREADS = 384;

__device__ __forceinline__ void mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// CTA-pair helpers (CL = 2: two CTAs of a cluster share the B operand, see tck_loop)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// TMA box into the same shared-memory offset of every CTA in `mask`; each
// destination CTA's mbarrier at the same offset receives its bytes
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// MMA completion arrives on the mbarrier at the same offset in every CTA of `mask`
__device__ __forceinline__ void commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// CL = 1: one CTA per 128-row item.  CL = 2: a cluster of two CTAs per
// 256-row item, CTA r computing rows [128 r, 128 r + 128) with its own A rows
// but the SAME B tile, which each CTA loads half of and multicasts to both:
// per SM the operand traffic from L2 drops from A + B to A + B/2 (96 -> 64 KB
// per k-tile at BNT = 256), the resource the 3xTF32 pre-split operands
// saturate.  A stage is refilled only once both CTAs' MMAs released it (the
// MMA commit arrives on both CTAs' empty barriers, count 2).
template <int BNT, int CL = 1, class Next>
__device__ __forceinline__ void tck_loop(const CUtensorMap* mAh, const CUtensorMap* mAl, const CUtensorMap* mBh,
                                         const CUtensorMap* mBl, int K, Next&& next) {
  static_assert(CL == 1 || CL == 2, "cluster size");
  using CF = Cfg<BNT>;
  constexpr int STAGES = CF::STAGES, STAGE_BYTES = CF::STAGE_BYTES, PLANE_A = CF::PLANE_A, PLANE_B = CF::PLANE_B;
  constexpr int BN = BNT;
  extern __shared__ __align__(1024) unsigned char tck_smem_raw[];
  unsigned char* base = tck_smem_raw + ((1024 - (smem_u32(tck_smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = (K + BK - 1) / BK;
  const int rank = CL == 2 ? (int)cluster_rank() : 0;
  const int64_t first = blockIdx.x / CL, stride = gridDim.x / CL;  // items per cluster

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);  // released by this CTA's MMAs and (CL = 2) the peer's
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);  // 8 epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc::fence_before();
  __syncthreads();
  if constexpr (CL == 2) cluster_sync_all();  // the peer's barriers exist before anything is multicast to them
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mAh) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mAl) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mBh) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mBl) : "memory");
      uint32_t g = 0;
      tc::Blk blk;
      const int arow = rank * BM;  // this CTA's rows of a (CL x 128)-row item
      for (int64_t item = first; next(item, blk); item += stride) {
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int s = g % STAGES;
          mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
          unsigned char* st = base + (size_t)s * STAGE_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);  // A (own) + the whole B tile (half from the peer when CL = 2)
          // box {32 k, 128 rows}: coordinates (k, row)
          tma_load_2d(st, mAh, kt * BK, blk.a_row + (int)blk.m0 + arow, &full[s]);
          tma_load_2d(st + PLANE_A, mAl, kt * BK, blk.a_row + (int)blk.m0 + arow, &full[s]);
          if constexpr (CL == 1) {
            tma_load_2d(st + 2 * PLANE_A, mBh, kt * BK, blk.b_row + (int)blk.n0, &full[s]);
            tma_load_2d(st + 2 * PLANE_A + PLANE_B, mBl, kt * BK, blk.b_row + (int)blk.n0, &full[s]);
          } else {  // B rows [rank BNT/2, ...) of the tile, into both CTAs (box {32 k, BNT/2 rows})
            const int brow = blk.b_row + (int)blk.n0 + rank * (BN / 2);
            const size_t boff = (size_t)rank * (PLANE_B / 2);  // whole 1 KB swizzle atoms
            tma_load_2d_mc(st + 2 * PLANE_A + boff, mBh, kt * BK, brow, &full[s], 0x3);
            tma_load_2d_mc(st + 2 * PLANE_A + PLANE_B + boff, mBl, kt * BK, brow, &full[s], 0x3);
          }
        }
      }
      if constexpr (CL == 2) {
        // the peer's last MMA commits arrive on our empty barriers: let them land before exit
        for (uint32_t q = g > (uint32_t)STAGES ? g - STAGES : 0; q < g; ++q)
          mbar_wait(&empty[q % STAGES], (q / STAGES) & 1);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      uint32_t g = 0, t = 0;
      tc::Blk blk;
      for (int64_t item = first; next(item, blk); item += stride, ++t) {
        const int b = t & 1;
        mbar_wait(&tempty[b], ((t >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t d = tmem + b * BN;
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int s = g % STAGES;
          mbar_wait(&full[s], (g / STAGES) & 1);
          tc::fence_after();
          const uint32_t st = smem_u32(base + (size_t)s * STAGE_BYTES);
          const uint32_t ahi = st, alo = st + PLANE_A, bhi = st + 2 * PLANE_A, blo = bhi + PLANE_B;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint32_t off = ks * 32;  // 8 tf32 k = 32 bytes along the 128-byte K-major row
            mma(d, tc::sdesc(alo + off), tc::sdesc(bhi + off), CF::IDESC, (kt | ks) != 0);
            mma(d, tc::sdesc(ahi + off), tc::sdesc(blo + off), CF::IDESC, 1);
            mma(d, tc::sdesc(ahi + off), tc::sdesc(bhi + off), CF::IDESC, 1);
          }
          if constexpr (CL == 1) tc::commit(&empty[s]);  // stage reusable once these MMAs have read it
          else commit_mc(&empty[s], 0x3);              // ... in both CTAs (the B half came from the peer)
        }
        tc::commit(&tfull[b]);
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------- epilogue (8 warps)
    const int q = warp & 3;             // TMEM lane quarter
    const int ch = (warp - 4) >> 2;     // column half
    const int row = 32 * q + lane;
    uint32_t t = 0;
    tc::Blk blk;
    for (int64_t item = first; next(item, blk); item += stride, ++t) {
      const int b = t & 1;
      const int64_t r = blk.m0 + rank * BM + row;
      float* __restrict__ crow = blk.C + r;
      auto load_chunk = [&](int c0, float* dst) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int64_t col = blk.n0 + c0 + j;
          dst[j] = (blk.beta != 0.f && r < blk.M && col < blk.N) ? crow[col * blk.ldc] : 0.f;
        }
      };
      const int cbeg = ch * (BN / 2), cend = cbeg + BN / 2;
      if (blk.beta != 0.f) {  // pull this warp's 32-row block into L2 during the MMAs
        constexpr int PER = BN / 2 / 32;
        const int64_t col = blk.n0 + cbeg + PER * lane, r0 = blk.m0 + rank * BM + 32 * q;
#pragma unroll
        for (int j = 0; j < PER; ++j)
          if (col + j < blk.N && r0 < blk.M) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(blk.C + r0 + (col + j) * blk.ldc));
      }
      float old[32], nxt[32];
      load_chunk(cbeg, old);
      mbar_wait(&tfull[b], (t >> 1) & 1);
      tc::fence_after();
#pragma unroll 1
      for (int c0 = cbeg; c0 < cend; c0 += 32) {
        if (c0 + 32 < cend) load_chunk(c0 + 32, nxt);
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + b * BN + c0, v);
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
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }
  __syncthreads();
  if constexpr (CL == 2) cluster_sync_all();  // no CTA leaves while its peer may still write to it
  if (warp == 1) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(CF::TMEM_COLS));
  }
}

// ----------------------------------------------------------------- 2-SM UMMA
// CTA pair on one 256 x 256 output tile with tcgen05.mma.cta_group::2 (M = 256,
// N = 256): CTA r holds rows [128 r, 128 r + 128) of A and rows
// [128 r, 128 r + 128) of B (the tile's output columns) in its own shared
// memory, and its 128 rows of the accumulator in its own TMEM; the leader
// (rank 0) issues the MMAs over both CTAs' operands.  Per SM the tensor core
// reads 4 + 4 KB per k8 MMA instead of 4 + 8 KB, TMA writes 64 instead of 96
// KB per k-tile, and a stage is 64 KB so three fit (two at N = 256 in one CTA):
// the shared-memory bandwidth and pipeline depth that bound the one-CTA
// 128 x 256 kernel.
//   both CTAs  warp 0: TMA of their A / B halves, completion on the LEADER's
//              full barrier (.cta_group::2); stage refilled after the leader's
//              MMA commit arrives on this CTA's empty barrier (multicast)
//   leader     warp 1: MMA issuer; commits to both CTAs' empty / tfull
//   both CTAs  warps 4-11: epilogue of their 128 rows; "TMEM drained" arrives
//              on the leader's tempty (count 16)
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(bar_cluster) : "memory");
}

struct CMaps {
  CUtensorMap m[MAX_LOCAL_DEV];  // per local device: its shard as (rows, columns), box {128, 128}
  int mode;                      // EPI_PREFETCH | EPI_DIRECT (BCMG_EPI_MODE)
};
enum : int {
  EPI_PREFETCH = 1,  // the producer prefetches an item's C tile into L2 when it starts the item's operands
  EPI_DIRECT = 2,    // results stored straight from registers (coalesced 128 B per warp and column):
                     // cbuf is free for the next item's C as soon as every warp has read it
};
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(map), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map), "r"(c0),
               "r"(c1), "r"(smem_u32(src))
               : "memory");
}

// EPI: the TMA read-modify-write epilogue (see tck_loop_epi).  1: in two
// 128-column halves per CTA through one 64 KB C buffer; 2: in 64-column
// quarters through a ring of three 32 KB buffers, so up to three loads are in
// flight while a quarter is combined and stored.  Two operand stages then fit.
template <int EPI = 0>
struct PairT {
  static constexpr int BN = 256;                      // output columns per tile (UMMA N)
  static constexpr int PA = BM * BK * 4;              // 16 KB: 128 A rows x 32 k
  static constexpr int PB = (BN / 2) * BK * 4;        // 16 KB: this CTA's 128 B rows
  static constexpr int STAGE_BYTES = 2 * (PA + PB);   // A hi, A lo, B hi, B lo
  static constexpr int STAGES = EPI ? 2 : 3;
  static constexpr int NCB = EPI == 2 ? 3 : 1;        // C buffers (and their barriers)
  static constexpr int CBUF = EPI == 1 ? BM * 128 * 4 : EPI == 2 ? NCB * BM * 64 * 4 : 0;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr size_t SMEM_BYTES = 1024 + (size_t)STAGES * STAGE_BYTES + CBUF + 256;
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)(256 >> 4) << 24);
};
using Pair = PairT<0>;

template <int EPI = 0, class Next>
__device__ __forceinline__ void tck_loop_pair(const CUtensorMap* mAh, const CUtensorMap* mAl, const CUtensorMap* mBh,
                                              const CUtensorMap* mBl, const CMaps* cmaps, int K, Next&& next) {
  using P = PairT<EPI>;
  constexpr int STAGES = P::STAGES, STAGE_BYTES = P::STAGE_BYTES, PA = P::PA, PB = P::PB, BN = P::BN;
  extern __shared__ __align__(1024) unsigned char tck_smem_raw[];
  unsigned char* base = tck_smem_raw + ((1024 - (smem_u32(tck_smem_raw) & 1023)) & 1023);
  float* cbuf = reinterpret_cast<float*>(base + (size_t)STAGES * STAGE_BYTES);  // EPI: 128 x 128, column-major
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)STAGES * STAGE_BYTES + P::CBUF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* cfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfull + P::NCB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = (K + BK - 1) / BK;
  const int rank = (int)cluster_rank();
  const bool leader = rank == 0;
  const int64_t first = blockIdx.x / 2, stride = gridDim.x / 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's arrive.expect_tx (both CTAs' bytes)
      mbar_init(&empty[s], 1);  // the leader's MMA commit (multicast)
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 16);  // leader: 8 epilogue warps of each CTA
    }
    for (int i = 0; i < P::NCB; ++i) mbar_init(&cfull[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {  // pair allocation: the same columns in both CTAs' TMEM
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(P::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc::fence_before();
  __syncthreads();
  cluster_sync_all();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer (both CTAs)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mAh) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mAl) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mBh) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mBl) : "memory");
      uint32_t g = 0;
      tc::Blk blk;
      const int arow = rank * BM;
      for (int64_t item = first; next(item, blk); item += stride) {
        const int brow = (rank == 0 ? blk.b_row : blk.b_row1 >= 0 ? blk.b_row1 : blk.b_row + BN / 2) + (int)blk.n0;
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int s = g % STAGES;
          mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
          unsigned char* st = base + (size_t)s * STAGE_BYTES;
          const uint32_t fb = mapa_u32(smem_u32(&full[s]), 0);  // the leader's full barrier
          if (leader) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
          tma_load_2d_pair(st, mAh, kt * BK, blk.a_row + (int)blk.m0 + arow, fb);
          tma_load_2d_pair(st + PA, mAl, kt * BK, blk.a_row + (int)blk.m0 + arow, fb);
          tma_load_2d_pair(st + 2 * PA, mBh, kt * BK, brow, fb);
          tma_load_2d_pair(st + 2 * PA + PB, mBl, kt * BK, brow, fb);
        }
      }
      // the leader's last commits arrive on our empty barriers: let them land before exit
      for (uint32_t q = g > (uint32_t)STAGES ? g - STAGES : 0; q < g; ++q)
        mbar_wait(&empty[q % STAGES], (q / STAGES) & 1);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer (leader)
    if (lane == 0 && leader) {
      uint32_t g = 0, t = 0;
      tc::Blk blk;
      for (int64_t item = first; next(item, blk); item += stride, ++t) {
        const int b = t & 1;
        mbar_wait(&tempty[b], ((t >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t d = tmem + b * BN;
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int s = g % STAGES;
          mbar_wait(&full[s], (g / STAGES) & 1);
          tc::fence_after();
          const uint32_t st = smem_u32(base + (size_t)s * STAGE_BYTES);
          const uint32_t ahi = st, alo = st + PA, bhi = st + 2 * PA, blo = bhi + PB;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint32_t off = ks * 32;
            mma_pair(d, tc::sdesc(alo + off), tc::sdesc(bhi + off), P::IDESC, (kt | ks) != 0);
            mma_pair(d, tc::sdesc(ahi + off), tc::sdesc(blo + off), P::IDESC, 1);
            mma_pair(d, tc::sdesc(ahi + off), tc::sdesc(bhi + off), P::IDESC, 1);
          }
          commit_pair(&empty[s]);  // both CTAs' stage s reusable once these MMAs read it
        }
        commit_pair(&tfull[b]);    // both CTAs' accumulator b ready
      }
    }
  } else if (EPI == 2 && warp >= 4) {
    // ------------------------ TMA epilogue, quarter ring (8 warps, both CTAs)
    // A CTA's 128 rows of an item in 64-column quarters (the live halves in
    // order, two quarters each).  The leader keeps up to NB quarter loads in
    // flight -- the rest of this item, then the next item's -- and refills a
    // buffer as soon as its store has read it.
    constexpr int NB = P::NCB, QF = BM * 64;
    float* qb = cbuf;
    const int q = warp & 3, ch = (warp - 4) >> 2, row = 32 * q + lane;
    const bool lead = warp == 4 && lane == 0;
    const uint32_t te = mapa_u32(smem_u32(&tempty[0]), 0);
    auto live = [&](const tc::Blk& bk, int h) {
      const int64_t r0 = bk.m0 + rank * BM;
      if (r0 >= bk.M) return false;
      if (h == 0) return true;
      return bk.C2 != nullptr ? r0 >= bk.skip2 : bk.n0 + 128 < bk.N;
    };
    auto nquarters = [&](const tc::Blk& bk) { return (live(bk, 0) ? 2 : 0) + (live(bk, 1) ? 2 : 0); };
    auto quarter = [&](const tc::Blk& bk, int i, int& h, int& qq) {
      h = (i >> 1) == 0 && live(bk, 0) ? 0 : 1;
      qq = i & 1;
    };
    auto coord = [&](const tc::Blk& bk, int h, int qq, int& dev, int& r, int& c) {
      dev = h && bk.C2 ? bk.cdev2 : bk.cdev;
      r = (int)(bk.crow0 + bk.m0 + rank * BM);
      c = (int)(h && bk.C2 ? bk.ccol02 : bk.ccol0 + bk.n0 + h * 128) + qq * 64;
    };
    auto issue = [&](const tc::Blk& bk, int i, uint32_t slot) {  // leader: quarter i of bk into buffer slot % NB
      int h, qq, dev, r, c;
      quarter(bk, i, h, qq);
      coord(bk, h, qq, dev, r, c);
      mbar_expect_tx(&cfull[slot % NB], QF * 4);
      tma_load_2d(qb + (slot % NB) * QF, &cmaps->m[dev], r, c, &cfull[slot % NB]);
    };
    uint32_t t = 0, g = 0, gi = 0;  // items, quarters consumed, quarters issued (leader)
    int pend = 0;                   // leader: next quarter to issue, counted from the current item's first
    tc::Blk blk, nblk;
    bool have = next(first, blk);
    for (int64_t item = first; have; item += stride, ++t) {
      const int b = t & 1;
      const bool more = next(item + stride, nblk);
      const int ncur = nquarters(blk), nnext = more ? nquarters(nblk) : 0;
      if (lead && pend < ncur && gi < g + NB) {
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // every buffer read by its store
        while (pend < ncur && gi < g + NB) issue(blk, pend++, gi++);
      }
      mbar_wait(&tfull[b], (t >> 1) & 1);
      tc::fence_after();
      for (int i = 0; i < ncur; ++i, ++g) {
        int h, qq;
        quarter(blk, i, h, qq);
        const uint32_t s = g % NB;
        mbar_wait(&cfull[s], (g / NB) & 1);
        float* cb = qb + s * QF;
        {
          const int c0 = ch * 32;
          float v[32];
          tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + b * BN + h * 128 + qq * 64 + c0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float* cp = cb + row + (c0 + j) * BM;
            *cp = blk.alpha * v[j] + blk.beta * *cp;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // cb writes -> the TMA store
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        if (lead) {
          int dev, r, c;
          coord(blk, h, qq, dev, r, c);
          tma_store_2d(&cmaps->m[dev], r, c, cb);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          // this quarter's store may still be reading cb: the refill goes into the
          // buffer of the previous quarter, whose store has been read
          asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
          if (gi < g + NB) {  // a buffer is free: the next quarter in order, this item or the next
            if (pend < ncur) issue(blk, pend++, gi++);
            else if (pend - ncur < nnext) issue(nblk, pend++ - ncur, gi++);
          }
        }
        __syncwarp();  // warp 4 reconverges before the next warp-collective tcgen05.ld
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(te + 8 * b);  // TMEM accumulator b drained
      if (lead) pend -= ncur;  // what was issued from the next item carries over
      have = more;
      blk = nblk;
    }
    if (lead) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // stores complete before exit
  } else if (EPI == 1 && warp >= 4) {
    // ------------------------------------- TMA epilogue (8 warps, both CTAs)
    // Each CTA updates its 128 rows of the item in two 128-column halves
    // (h = 0: the item's first tile column; h = 1: columns 128.. or, for a
    // two-column item, the second tile column C2), each through cbuf: the
    // leader TMA-loads the half, the warps combine it with TMEM, the leader
    // TMA-stores it and loads the next live half.  Halves whose rows lie
    // outside the matrix or above C2's diagonal are skipped by both sides.
    const int q = warp & 3, ch = (warp - 4) >> 2, row = 32 * q + lane;
    const bool lead = warp == 4 && lane == 0;
    const uint32_t te = mapa_u32(smem_u32(&tempty[0]), 0);
    auto live = [&](const tc::Blk& bk, int h) {
      const int64_t r0 = bk.m0 + rank * BM;
      if (r0 >= bk.M) return false;
      if (h == 0) return true;
      return bk.C2 != nullptr ? r0 >= bk.skip2 : bk.n0 + 128 < bk.N;
    };
    auto coord = [&](const tc::Blk& bk, int h, int& dev, int& r, int& c) {
      dev = h && bk.C2 ? bk.cdev2 : bk.cdev;
      r = (int)(bk.crow0 + bk.m0 + rank * BM);
      c = (int)(h && bk.C2 ? bk.ccol02 : bk.ccol0 + bk.n0 + h * 128);
    };
    auto load_half = [&](const tc::Blk& bk, int h) {
      int dev, r, c;
      coord(bk, h, dev, r, c);
      mbar_expect_tx(cfull, P::CBUF);
      tma_load_2d(cbuf, &cmaps->m[dev], r, c, cfull);
    };
    auto load_first = [&](const tc::Blk& bk) {
      for (int h = 0; h < 2; ++h)
        if (live(bk, h)) {
          load_half(bk, h);
          return;
        }
    };
    uint32_t t = 0, nw = 0;
    tc::Blk blk, nblk;
    bool have = next(first, blk);
    if (lead && have) load_first(blk);
    for (int64_t item = first; have; item += stride, ++t) {
      const int b = t & 1;
      const bool more = next(item + stride, nblk);
      mbar_wait(&tfull[b], (t >> 1) & 1);
      tc::fence_after();
      bool any = false;
      for (int h = 0; h < 2; ++h) {
        if (!live(blk, h)) continue;
        any = true;
        mbar_wait(cfull, nw & 1);
        ++nw;
#pragma unroll 1
        for (int c0 = ch * 64; c0 < ch * 64 + 64; c0 += 32) {
          float v[32];
          tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + b * BN + h * 128 + c0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float* cp = cbuf + row + (c0 + j) * BM;
            *cp = blk.alpha * v[j] + blk.beta * *cp;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // cbuf writes -> the TMA store
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        if (lead) {
          int dev, r, c;
          coord(blk, h, dev, r, c);
          tma_store_2d(&cmaps->m[dev], r, c, cbuf);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // cbuf read by the store
          if (h == 0 && live(blk, 1)) load_half(blk, 1);
          else if (more) load_first(nblk);
        }
        __syncwarp();  // warp 4 reconverges before the next warp-collective tcgen05.ld
      }
      if (lead && !any && more) load_first(nblk);  // nothing of this item is ours: keep the chain going
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(te + 8 * b);  // TMEM accumulator b drained (both halves read)
      have = more;
      blk = nblk;
    }
    if (lead) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // stores complete before exit
  } else if (EPI == 0 && warp >= 4) {
    // ---------------------------------------------------------- epilogue (8 warps, both CTAs)
    const int q = warp & 3;
    const int ch = (warp - 4) >> 2;
    const int row = 32 * q + lane;
    const uint32_t te = mapa_u32(smem_u32(&tempty[0]), 0);  // the leader's tempty[0]; [1] is 8 bytes on
    uint32_t t = 0;
    tc::Blk blk;
    for (int64_t item = first; next(item, blk); item += stride, ++t) {
      const int b = t & 1;
      const int64_t r = blk.m0 + rank * BM + row;
      // columns >= 128 of a two-column item go to the second tile column (C2)
      const bool second = blk.C2 != nullptr && ch == 1;
      const int64_t coff = second ? BN / 2 : 0;
      float* __restrict__ crow = (second ? blk.C2 : blk.C) + r;
      const bool rok = r < blk.M && (!second || r >= blk.skip2);
      auto load_chunk = [&](int c0, float* dst) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int64_t col = blk.n0 + c0 + j;
          dst[j] = (blk.beta != 0.f && rok && col < blk.N) ? crow[(col - coff) * blk.ldc] : 0.f;
        }
      };
      const int cbeg = ch * (BN / 2), cend = cbeg + BN / 2;
      if (blk.beta != 0.f) {
        constexpr int PER = BN / 2 / 32;
        const int64_t col = blk.n0 + cbeg + PER * lane, r0 = blk.m0 + rank * BM + 32 * q;
        const bool live = r0 < blk.M && (!second || r0 + 32 > blk.skip2);
#pragma unroll
        for (int j = 0; j < PER; ++j)
          if (col + j < blk.N && live)
            asm volatile("prefetch.global.L2 [%0];\n" ::"l"((second ? blk.C2 : blk.C) + r0 + (col + j - coff) * blk.ldc));
      }
      float old[32], nxt[32];
      load_chunk(cbeg, old);
      mbar_wait(&tfull[b], (t >> 1) & 1);
      tc::fence_after();
#pragma unroll 1
      for (int c0 = cbeg; c0 < cend; c0 += 32) {
        if (c0 + 32 < cend) load_chunk(c0 + 32, nxt);
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + b * BN + c0, v);
        if (rok) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int64_t col = blk.n0 + c0 + j;
            if (col < blk.N) crow[(col - coff) * blk.ldc] = blk.alpha * v[j] + blk.beta * old[j];
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) old[j] = nxt[j];
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(te + 8 * b);
    }
  }
  __syncthreads();
  cluster_sync_all();  // both CTAs done with the pair's TMEM and with each other's barriers
  if (warp == 1) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(P::TMEM_COLS));
  }
}

// ----------------------------------------------------------------- TMA epilogue
// One CTA per 128 x 128 tile (the narrow-tile trailing update, T_A = 128) with
// the read-modify-write of C done by TMA instead of per-thread loads: the
// epilogue leader TMA-loads the next item's C tile (64 KB, column-major, no
// swizzle) into shared memory as soon as the previous tile's TMA store has
// read it, i.e. while the MMAs run; the eight epilogue warps combine it with
// the accumulator in shared memory (row r, 32 consecutive columns per thread:
// conflict-free), and the leader TMA-stores the tile back.  The per-thread
// scalar loads of the default epilogue keep only ~32 KB in flight per SM and
// leave HBM ~35 % busy at T_A = 128; the bulk copies keep a whole tile in
// flight.  Two 64 KB operand stages + the C tile fill 192 KB.
struct Epi {
  static constexpr int BN = 128;
  static constexpr int PA = BM * BK * 4, PB = BN * BK * 4;  // 16 KB each
  static constexpr int STAGE_BYTES = 2 * (PA + PB);         // 64 KB
  static constexpr int STAGES = 2;
  static constexpr int CBUF = BM * BN * 4;                  // 64 KB
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr size_t SMEM_BYTES = 1024 + (size_t)STAGES * STAGE_BYTES + CBUF + 256;
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)(BM >> 4) << 24);
};
template <class Next>
__device__ __forceinline__ void tck_loop_epi(const CUtensorMap* mAh, const CUtensorMap* mAl, const CUtensorMap* mBh,
                                             const CUtensorMap* mBl, const CMaps* cmaps, int K, Next&& next) {
  using E = Epi;
  constexpr int STAGES = E::STAGES, STAGE_BYTES = E::STAGE_BYTES, PA = E::PA, PB = E::PB, BN = E::BN;
  extern __shared__ __align__(1024) unsigned char tck_smem_raw[];
  unsigned char* base = tck_smem_raw + ((1024 - (smem_u32(tck_smem_raw) & 1023)) & 1023);
  float* cbuf = reinterpret_cast<float*>(base + (size_t)STAGES * STAGE_BYTES);  // C tile, column-major 128 x 128
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)STAGES * STAGE_BYTES + E::CBUF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* cfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = (K + BK - 1) / BK;
  const int64_t first = blockIdx.x, stride = gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    mbar_init(cfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(E::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mAh) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mAl) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mBh) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(mBl) : "memory");
      uint32_t g = 0;
      tc::Blk blk;
      for (int64_t item = first; next(item, blk); item += stride) {
        if (cmaps->mode & EPI_PREFETCH)
          tma_prefetch_2d(&cmaps->m[blk.cdev], (int)(blk.crow0 + blk.m0), (int)(blk.ccol0 + blk.n0));
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int s = g % STAGES;
          mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
          unsigned char* st = base + (size_t)s * STAGE_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(st, mAh, kt * BK, blk.a_row + (int)blk.m0, &full[s]);
          tma_load_2d(st + PA, mAl, kt * BK, blk.a_row + (int)blk.m0, &full[s]);
          tma_load_2d(st + 2 * PA, mBh, kt * BK, blk.b_row + (int)blk.n0, &full[s]);
          tma_load_2d(st + 2 * PA + PB, mBl, kt * BK, blk.b_row + (int)blk.n0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      uint32_t g = 0, t = 0;
      tc::Blk blk;
      for (int64_t item = first; next(item, blk); item += stride, ++t) {
        const int b = t & 1;
        mbar_wait(&tempty[b], ((t >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t d = tmem + b * BN;
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int s = g % STAGES;
          mbar_wait(&full[s], (g / STAGES) & 1);
          tc::fence_after();
          const uint32_t st = smem_u32(base + (size_t)s * STAGE_BYTES);
          const uint32_t ahi = st, alo = st + PA, bhi = st + 2 * PA, blo = bhi + PB;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint32_t off = ks * 32;
            mma(d, tc::sdesc(alo + off), tc::sdesc(bhi + off), E::IDESC, (kt | ks) != 0);
            mma(d, tc::sdesc(ahi + off), tc::sdesc(blo + off), E::IDESC, 1);
            mma(d, tc::sdesc(ahi + off), tc::sdesc(bhi + off), E::IDESC, 1);
          }
          tc::commit(&empty[s]);
        }
        tc::commit(&tfull[b]);
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------- epilogue (8 warps)
    const int q = warp & 3, ch = (warp - 4) >> 2, row = 32 * q + lane;
    const bool leader = warp == 4 && lane == 0;
    auto load_c = [&](const tc::Blk& bk) {  // leader: C tile of an item into cbuf
      mbar_expect_tx(cfull, E::CBUF);
      tma_load_2d(cbuf, &cmaps->m[bk.cdev], (int)(bk.crow0 + bk.m0), (int)(bk.ccol0 + bk.n0), cfull);
    };
    uint32_t t = 0;
    tc::Blk blk, nblk;
    bool have = next(first, blk);
    if (leader && have) load_c(blk);
    for (int64_t item = first; have; item += stride, ++t) {
      const int b = t & 1;
      mbar_wait(&tfull[b], (t >> 1) & 1);
      tc::fence_after();
      mbar_wait(cfull, t & 1);  // C of this item in cbuf
      const int cbeg = ch * (BN / 2), cend = cbeg + BN / 2;
      const bool direct = cmaps->mode & EPI_DIRECT;
      float* gc = blk.C + blk.m0 + row + blk.n0 * blk.ldc;
      const bool live = blk.m0 + row < blk.M;
#pragma unroll 1
      for (int c0 = cbeg; c0 < cend; c0 += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + b * BN + c0, v);
        if (direct) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float out = blk.alpha * v[j] + blk.beta * cbuf[row + (c0 + j) * BM];
            if (live && c0 + j < blk.N) gc[(int64_t)(c0 + j) * blk.ldc] = out;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float* cp = cbuf + row + (c0 + j) * BM;
            *cp = blk.alpha * v[j] + blk.beta * *cp;
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);  // TMEM accumulator b drained
      if (!direct) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // cbuf writes -> the TMA store
      asm volatile("bar.sync 1, 256;\n" ::: "memory");  // all eight warps are done with cbuf
      have = next(item + stride, nblk);
      if (leader) {
        if (!direct) {
          tma_store_2d(&cmaps->m[blk.cdev], (int)(blk.crow0 + blk.m0), (int)(blk.ccol0 + blk.n0), cbuf);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // cbuf read by the store
        }
        if (have) load_c(nblk);
      }
      __syncwarp();  // warp 4 reconverges before the next warp-collective tcgen05.ld
      blk = nblk;
    }
    if (leader) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // stores complete before exit
  }
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(E::TMEM_COLS));
  }
}

}  // namespace tck

// C := alpha * A * B^T + beta * C on pre-split K-major planes (rows x Kp).
// CL = 3: CTA pairs on 256 x 256 tiles with the 2-SM UMMA (no fan-out)
template <int BNT, int CL = 1>
__global__ void __launch_bounds__(tck::THREADS, 1)
    tck_gemm_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                    const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl, int64_t M,
                    int64_t N, int64_t K, float* C, int64_t ldc, float alpha, float beta, const int* info,
                    FloatFan fan) {
  static_assert(CL == 1 || (CL == 3 && BNT == 256), "pair GEMM tiles are 256 x 256");
  if ((CL == 1 || CL == 4) && ld_flag(info)) return;  // (a CTA pair must not split on the flag)
  constexpr int64_t BMX = CL == 1 ? tc::BM : 2 * tc::BM;
  const int64_t nbm = (M + BMX - 1) / BMX, nbn = (N + BNT - 1) / BNT;
  auto next = [&](int64_t item, tc::Blk& blk) -> bool {
    if (item >= nbm * nbn) return false;
    blk.a_row = 0;
    blk.b_row = 0;
    blk.m0 = (item % nbm) * BMX;
    blk.n0 = (item / nbm) * BNT;
    blk.M = M;
    blk.N = N;
    blk.C = C;
    blk.ldc = ldc;
    blk.alpha = alpha;
    blk.beta = beta;
    blk.nfan = fan.n;
#pragma unroll
    for (int e = 0; e < MAX_FAN; ++e) blk.fan[e] = e < fan.n ? fan.p[e] : nullptr;
    return true;
  };
  if constexpr (CL == 3) tck::tck_loop_pair(&mAh, &mAl, &mBh, &mBl, nullptr, (int)K, next);
  else tck::tck_loop<BNT>(&mAh, &mAl, &mBh, &mBl, (int)K, next);
}

// potrf trailing update on the pre-split panel (TrailParams::split_*): same
// item decode as tc3_trail_kernel (real, or the complex64 embedding).
template <int BNT, int CL = 1>
__global__ void __launch_bounds__(tck::THREADS, 1)
    tck_trail_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                     const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl, TrailParams p,
                     const int* info, const __grid_constant__ tck::CMaps cmaps) {
  static_assert(CL != 4 || BNT == 128, "the TMA-epilogue tile is 128 x 128");
  static_assert((CL != 3 && CL != 6 && CL != 7) || BNT == 256, "the 2-SM UMMA tile is 256 x 256");
  constexpr int64_t BMX = (CL == 1 || CL == 4 ? 1 : 2) * tc::BM;  // rows per item (a CTA pair covers 256)
  using TZ = TrapR<BMX, BNT>;
  using TZC = TrapR<BMX / 2, BNT>;
  // (a CTA pair must not split on a flag another stream may be writing: only single CTAs skip)
  if ((CL == 1 || CL == 4) && ld_flag(info)) return;
  int64_t cm = p.m_first, cbase = 0, ccnt = -1;
  // band mode (see TrailParams::band).  The band interleaves "units" that all
  // end at row N: owned tile columns (T <= BNT, spaced sc tiles), or, with one
  // process owning every column and T a multiple of BNT, the BNT-wide column
  // blocks of consecutive tiles (spaced BNT rows).
  const int64_t sc = p.nloc == p.D ? 1 : p.D;
  const int64_t ncb = p.T > BNT ? p.T / BNT : 1;
  // CL = 3 at T_A = 128: a unit is two owned tile columns (c, c + sc), one 256-wide item
  const int64_t cpu = (CL == 3 || CL == 6 || CL == 7) && ncb == 1 && p.cpu > 1 ? p.cpu : 1, usp = cpu * sc;
  if (p.band > 0 && sc > 1) cm += ((p.dev0 - cm % p.D) + p.D) % p.D;  // first owned column
  const int64_t nunits = ncb == 1 ? ((p.m_last - cm + sc - 1) / sc + cpu - 1) / cpu : (p.m_last - p.m_first) * ncb;
  const int64_t cm0 = cm;
  auto unit_row = [&](int64_t k) { return ncb == 1 ? (cm0 + k * usp) * p.T : (p.m_first * ncb + k) * BNT; };
  // row blocks are counted from roff (units start a multiple of RB rows apart)
  const int64_t roff = unit_row(0) % (p.cplx ? BMX / 2 : BMX);
  int64_t ku = 0, bg = 0, ba0 = 0, btop = 0;
  auto next = [&](int64_t item, tc::Blk& blk) -> bool {
    if (p.band > 0) {
      const int64_t RB = p.cplx ? BMX / 2 : BMX;  // matrix rows per row block (complex64: embedded pairs)
      const int64_t step = (ncb == 1 ? usp * p.T : (int64_t)BNT) / RB, aend = (p.N - roff + RB - 1) / RB;
      for (;;) {
        if (ku >= nunits) return false;
        if (ccnt < 0) {
          bg = nunits - ku < p.band ? nunits - ku : p.band;
          ba0 = (unit_row(ku) - roff) / RB;
          btop = step * bg * (bg - 1) / 2;
          ccnt = bg * (aend - ba0) - btop;
        }
        if (item < cbase + ccnt) break;
        cbase += ccnt;
        ku += bg;
        ccnt = -1;
      }
      int64_t o = item - cbase, A, i;
      if (o < btop) {  // level j: row blocks [ba0 + j step, ba0 + (j+1) step) of units 0..j
        int64_t j = 0;
        while (step * (j + 1) * (j + 2) / 2 <= o) ++j;
        o -= step * j * (j + 1) / 2;
        A = ba0 + j * step + o / (j + 1);
        i = o % (j + 1);
      } else {
        o -= btop;
        A = ba0 + (bg - 1) * step + o / bg;
        i = o % bg;
      }
      const int64_t k = ku + i;
      const int64_t c = ncb == 1 ? cm0 + k * usp : (p.m_first * ncb + k) / ncb;
      const int64_t cb = ncb == 1 ? 0 : (p.m_first * ncb + k) % ncb;
      const int64_t ms = c * p.T, rows = p.N - ms;
      const int dev = (int)(c % p.D);
      float* shard = reinterpret_cast<float*>(p.shards[dev - p.dev0]);
      const int64_t cx = p.cplx ? 2 : 1;
      blk.a_row = (int)(cx * (ms - p.prow0));
      blk.b_row = (int)(ms - p.prow0);
      blk.m0 = (A - (ms - roff) / RB) * BMX;
      blk.n0 = cb * BNT;
      blk.M = cx * rows;
      blk.N = p.T < rows ? p.T : rows;
      blk.C = shard + cx * (ms + (c / p.D) * p.T * p.N);
      blk.ldc = cx * p.N;
      blk.cdev = dev - p.dev0;
      blk.crow0 = cx * ms;
      blk.ccol0 = (c / p.D) * p.T;
      blk.alpha = -1.f;
      blk.beta = 1.f;
      blk.nfan = 0;
      blk.C2 = nullptr;
      blk.b_row1 = -1;
      if (cpu > 1 && c + sc < p.m_last) {  // the unit's second tile column
        const int64_t c2 = c + sc;
        float* shard2 = reinterpret_cast<float*>(p.shards[(int)(c2 % p.D) - p.dev0]);
        blk.C2 = shard2 + cx * (ms + (c2 / p.D) * p.T * p.N);
        blk.skip2 = cx * (c2 - c) * p.T;
        blk.b_row1 = (int)(c2 * p.T - p.prow0);
        blk.N = 2 * p.T;
        blk.cdev2 = (int)(c2 % p.D) - p.dev0;
        blk.ccol02 = (c2 / p.D) * p.T;
      }
      return true;
    }
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
      blk.m0 = rb * BMX;
      blk.n0 = cb * BNT;
      blk.M = 2 * rows;
      blk.N = tcw;
      blk.C = shard + 2 * (ms + loc * p.N);
      blk.ldc = 2 * p.N;
      blk.crow0 = 2 * ms;
    } else {
      TZ::decode(item - cbase, tcw, rb, cb);
      blk.a_row = (int)(ms - p.prow0);
      blk.b_row = (int)(ms - p.prow0);
      blk.m0 = rb * BMX;
      blk.n0 = cb * BNT;
      blk.M = rows;
      blk.N = tcw;
      blk.C = shard + ms + loc * p.N;
      blk.ldc = p.N;
      blk.crow0 = ms;
    }
    blk.cdev = dev - p.dev0;
    blk.ccol0 = loc;
    blk.alpha = -1.f;
    blk.beta = 1.f;
    blk.nfan = 0;
    return true;
  };
  const int Kx = (int)(p.cplx ? 2 * p.K : p.K);
  if constexpr (CL == 3) tck::tck_loop_pair(&mAh, &mAl, &mBh, &mBl, nullptr, Kx, next);
  else if constexpr (CL == 6) tck::tck_loop_pair<1>(&mAh, &mAl, &mBh, &mBl, &cmaps, Kx, next);
  else if constexpr (CL == 7) tck::tck_loop_pair<2>(&mAh, &mAl, &mBh, &mBl, &cmaps, Kx, next);
  else if constexpr (CL == 4) tck::tck_loop_epi(&mAh, &mAl, &mBh, &mBl, &cmaps, Kx, next);
  else tck::tck_loop<BNT, CL>(&mAh, &mAl, &mBh, &mBl, Kx, next);
}

}  // namespace bcmg
