// Hot-path FP64 GEMM: TMA-fed, mbarrier-pipelined, persistent DMMA kernel.
//
// Operands are real double, stored i-contiguous (column-major M x K for A,
// N x K for B): the potrf trailing update C_m -= P P_m^H and the panel solve
// P = A21 X11^H.  One elected thread issues cp.async.bulk.tensor (TMA, SASS
// UTMALDG) boxes of {132 rows, BK columns} into a STAGES-deep ring; the box
// is 4 rows taller than the tile so every smem row is 132 words long -- the
// same conflict-free pad as the cp.async path, produced by TMA itself (TMA
// cannot pad, but it can over-fetch).  Consumers wait on the stage's "full"
// mbarrier (complete_tx) and release it with one arrive per warp on its
// "empty" mbarrier, so warps never meet at a CTA-wide barrier inside the K
// loop.  The kernel is persistent: the producer runs STAGES-1 slices ahead
// across work-item boundaries, so the next tile's operands stream in while
// the current tile's epilogue updates C.
#pragma once

#include <cuda.h>

#include "gemm.cuh"

namespace bcmg {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Box rows fetched per operand tile (tile rows + 4-row pad).
template <class TL>
constexpr int tma_box_rows_a() { return TL::LDA; }
template <class TL>
constexpr int tma_box_rows_b() { return TL::LDB; }
// TBK: B stored k-contiguous (N x K with K innermost): its tile is [BN][LDT]
template <class TL, bool TBK = false>
constexpr int tma_stage_words() { return TL::BK * TL::LDA + (TBK ? TL::BN * TL::LDT : TL::BK * TL::LDB); }
template <class TL, bool TBK = false>
constexpr unsigned tma_stage_bytes() { return (unsigned)(tma_stage_words<TL, TBK>() * 8); }
// One output block: rows [a_row + m0 ...) of A's map, [b_row + n0 ...) of B's map.
struct TmaBlock {
  int a_row, b_row;      // tensor-map row coordinate of the block's first A / B row
  int64_t m0, n0;        // block origin inside the output (for the epilogue)
  int64_t M, N;          // output extent (rows >= M / cols >= N are not stored)
  Epilogue ep;
  int live;              // 0: no more items (sentinel slot)
  int bmap;              // B tensor map of the item (multi-map kernels; MB)
};
// Dynamic shared memory: STAGES operand stages | 2*STAGES mbarriers | aux area:
// producer state [0,384), caller state [384,512), then a ring of decoded work
// items [512, ...) -- the producer decodes every item once and publishes it
// here, so neither the producer's bookkeeping nor the consumers' view of the
// current item occupies registers next to the DMMA accumulators.
constexpr int TMA_RING = 8;
constexpr int TMA_AUX_BYTES = 512 + TMA_RING * (int)sizeof(TmaBlock);
template <class TL, bool TBK = false>
constexpr size_t tma_smem_bytes() {
  return (size_t)TL::STAGES * tma_stage_bytes<TL, TBK>() + 2 * TL::STAGES * 8 + TMA_AUX_BYTES;
}
extern __shared__ __align__(1024) unsigned char tma_dyn_smem[];
template <class TL, bool TBK = false>
__device__ __forceinline__ unsigned char* tma_aux() {
  return tma_dyn_smem + (size_t)TL::STAGES * tma_stage_bytes<TL, TBK>() + 2 * TL::STAGES * 8;
}

// One BK slice with B k-contiguous ([BN][LDT] tile, TBK): thread (r, q) takes
// k = kk + 2q + j in DMMA step j of each 8-wide k block, so both of its B
// values are one 16-byte load (conflict-free at LDT = 36: rows 2r + c land on
// 16-byte bank groups 4r + q); A keeps the paired-row loads of mma_slice.
template <class TL>
__device__ __forceinline__ void mma_slice_tbk(Acc<TL, false>& acc, const double* __restrict__ As,
                                              const double* __restrict__ Bs, int wm0, int wn0, int lane) {
  static_assert(TL::PAIR && TL::BK % 8 == 0, "paired fragments, 8-wide k blocks");
  const int r = lane >> 2, q = lane & 3;
#pragma unroll
  for (int kk = 0; kk < TL::BK; kk += 8) {
    double b0[TL::FN], b1[TL::FN];
#pragma unroll
    for (int f = 0; f < TL::FN; ++f) {
      const double2 v = *reinterpret_cast<const double2*>(Bs + (wn0 + frag_row<TL>(f, r)) * TL::LDT + kk + 2 * q);
      b0[f] = v.x;
      b1[f] = v.y;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double a[TL::FM];
#pragma unroll
      for (int f = 0; f < TL::FM; f += 2) {
        const double2 v =
            *reinterpret_cast<const double2*>(As + (kk + 2 * q + j) * TL::LDA + wm0 + frag_row<TL>(f, r));
        a[f] = v.x;
        a[f + 1] = v.y;
      }
#pragma unroll
      for (int fm = 0; fm < TL::FM; ++fm)
#pragma unroll
        for (int fn = 0; fn < TL::FN; ++fn) dmma(acc.re[fm][fn][0], acc.re[fm][fn][1], a[fm], j ? b1[fn] : b0[fn]);
    }
  }
}

// Persistent producer/consumer loop.  `next_p(item, blk)` fills the block of
// work item `item` (called by the producer thread only, items increasing) and
// returns false when there is none.  The producer publishes each decoded item
// in the aux ring before issuing its first slice; the consumers read it after
// waiting for that slice (mbarrier release / acquire orders the ring store).
// When the items run out the producer publishes a sentinel (live = 0) and
// completes the next stage's barrier without a transfer.
template <class TL, bool FAN = true, bool COPY = false, bool TBK = false, bool MB = false, class NextP>
__device__ __forceinline__ void tma_gemm_loop(const CUtensorMap* mapA, const CUtensorMap* mapB, int K, NextP&& next_p,
                                              long long stagger_ns = 0) {
  double* smem = reinterpret_cast<double*>(tma_dyn_smem);
  constexpr int NW = TL::THREADS / 32;
  constexpr unsigned STAGE_BYTES = tma_stage_bytes<TL, TBK>();
  constexpr int STAGE_WORDS = tma_stage_words<TL, TBK>();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TL::STAGES * STAGE_WORDS);
  uint64_t* empty = full + TL::STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % TL::WARPS_M) * TL::WM, wn0 = (warp / TL::WARPS_M) * TL::WN;
  const int KT = (K + TL::BK - 1) / TL::BK;
  if (tid == 0) {
    for (int s = 0; s < TL::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(mapB) : "memory");
  }
  __syncthreads();

  // producer state (thread 0 only) lives in shared memory so it costs the
  // consumer warps no registers: slice counter gp over (item, kt)
  struct Prod {
    int64_t item;
    uint32_t gp, seq;
    int kt, live, done;
  };
  static_assert(sizeof(Prod) <= 384, "producer state must fit its aux slot");
  Prod& ps = *reinterpret_cast<Prod*>(tma_aux<TL, TBK>());
  TmaBlock* ring = reinterpret_cast<TmaBlock*>(tma_aux<TL, TBK>() + 512);
  auto produce_one = [&]() {
    if (ps.done) return;
    const uint32_t gp = ps.gp;
    const int s = gp % TL::STAGES, kt = ps.kt;
    mbar_wait(&empty[s], ((gp / TL::STAGES) & 1) ^ 1);
    TmaBlock& blk = ring[ps.seq % TMA_RING];
    if (!ps.live) {  // sentinel: the consumers find live == 0 behind this stage's barrier
      blk.live = 0;
      mbar_arrive(&full[s]);
      ps.done = 1;
      return;
    }
    double* st = smem + s * STAGE_WORDS;
    mbar_expect_tx(&full[s], STAGE_BYTES);
    tma_load_2d(st, mapA, blk.a_row + (int)blk.m0, kt * TL::BK, &full[s]);
    const CUtensorMap* mb = MB ? mapB + blk.bmap : mapB;
    if constexpr (TBK) tma_load_2d(st + TL::BK * TL::LDA, mb, kt * TL::BK, blk.b_row + (int)blk.n0, &full[s]);
    else tma_load_2d(st + TL::BK * TL::LDA, mb, blk.b_row + (int)blk.n0, kt * TL::BK, &full[s]);
    ps.gp = gp + 1;
    if (kt + 1 == KT) {
      ps.kt = 0;
      ps.item += gridDim.x;
      ps.seq += 1;
      TmaBlock& nb = ring[ps.seq % TMA_RING];  // consumed TMA_RING items ago (ring > stages)
      ps.live = next_p(ps.item, nb);
      nb.live = ps.live;
    } else {
      ps.kt = kt + 1;
    }
  };
  static_assert(TMA_RING > TL::STAGES, "a ring slot must outlive the producer's run-ahead");
  if (tid == 0) {
    ps.item = blockIdx.x;
    ps.gp = 0;
    ps.seq = 0;
    ps.kt = 0;
    ps.done = 0;
    ps.live = next_p(ps.item, ring[0]);
    ring[0].live = ps.live;
    for (int i = 0; i < TL::STAGES - 1; ++i) produce_one();
  }

  uint32_t g = 0;
  // C tile prefetch into L2 a few slices before the epilogue: all CTAs reach
  // their epilogues at nearly the same time (uniform items), and without it
  // the read-modify-write of 128 KB per CTA would stall every SM on HBM.
  constexpr int PREFETCH_AHEAD = 6;
  auto prefetch_c = [&](const TmaBlock& blk) {
    if (blk.ep.beta == 0.0) return;
    const double* C = reinterpret_cast<const double*>(blk.ep.C);
    constexpr int SEGS = TL::BM * 8 / 128;  // 128-byte lines per column of the tile
    for (int i = tid; i < TL::BN * SEGS; i += TL::THREADS) {
      const int64_t col = blk.n0 + i / SEGS, row = blk.m0 + (i % SEGS) * 16;
      if (col < blk.N && row < blk.M)
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(C + row + col * blk.ep.ldc));
    }
  };
  // Two co-resident CTAs per SM start in lockstep and, with uniform items,
  // would hit their epilogues together; delaying the second half of the grid
  // by about half an item makes one CTA's epilogue overlap the other's DMMAs.
  if (stagger_ns > 0 && blockIdx.x >= gridDim.x / 2) {
    const long long t0 = clock64();
    while (clock64() - t0 < stagger_ns * 2) __nanosleep(1000);  // ~2 cycles per ns at ~2 GHz
  }
  for (uint32_t seq = 0;; ++seq) {
    const TmaBlock& cb = ring[seq % TMA_RING];
    Acc<TL, false> acc;
    acc.zero();
    for (int kt = 0; kt < KT; ++kt) {
      if (tid == 0) produce_one();
      const int s = g % TL::STAGES;
      mbar_wait(&full[s], (g / TL::STAGES) & 1);
      if (kt == 0 && !cb.live) return;  // sentinel (published before this barrier completed)
      if (kt == (KT > PREFETCH_AHEAD ? KT - PREFETCH_AHEAD : 0)) prefetch_c(cb);
      const double* st = smem + s * STAGE_WORDS;
      if constexpr (TBK) mma_slice_tbk<TL>(acc, st, st + TL::BK * TL::LDA, wm0, wn0, lane);
      else mma_slice<TL, false, false, false>(acc, st, st + TL::BK * TL::LDA, nullptr, nullptr, wm0, wn0, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++g;
    }
    if constexpr (COPY) {  // the item's geometry in registers for the epilogue
      const Epilogue ep = cb.ep;
      const int64_t M = cb.M, N = cb.N, m0 = cb.m0, n0 = cb.n0;
      store_block<double, TL, false, FAN>(acc, ep, M, N, m0, n0, wm0, wn0, lane);
    } else {  // read from the ring as the epilogue needs it
      store_block<double, TL, false, FAN>(acc, cb.ep, cb.M, cb.N, cb.m0, cb.n0, wm0, wn0, lane);
    }
  }
}

// Lower-trapezoid enumeration of one trailing tile (rows x tc, row blocks of
// BM, column blocks of BN, BM a multiple of BN): row block rb keeps the
// column blocks that reach the diagonal, min(ncb, (rb+1)*BM/BN) of them.
template <int BM, int BN>
struct Trap {
  static_assert(BM % BN == 0, "BM must be a multiple of BN");
  static constexpr int64_t R = BM / BN;
  __host__ __device__ static int64_t count(int64_t rows, int64_t tc) {
    const int64_t nrb = (rows + BM - 1) / BM, ncb = (tc + BN - 1) / BN;
    const int64_t r0 = (ncb + R - 1) / R - 1;  // rows [0, r0) have fewer than ncb blocks
    const int64_t t = nrb < r0 ? nrb : r0;
    return R * t * (t + 1) / 2 + (nrb > r0 ? (nrb - r0) * ncb : 0);
  }
  __host__ __device__ static void decode(int64_t b, int64_t tc, int64_t& rb, int64_t& cb) {
    const int64_t ncb = (tc + BN - 1) / BN, r0 = (ncb + R - 1) / R - 1, tri = R * r0 * (r0 + 1) / 2;
    if (b < tri) {
      rb = 0;
      while (R * (rb + 1) * (rb + 2) / 2 <= b) ++rb;
      cb = b - R * rb * (rb + 1) / 2;
    } else {
      rb = r0 + (b - tri) / ncb;
      cb = (b - tri) % ncb;
    }
  }
};

// Same enumeration with column blocks twice as wide as row blocks (BN = 2 BM):
// row block rb keeps min(ncb, rb/2 + 1) column blocks (complex embedding on
// the 128x128 tcgen05 tile: 128 real rows = 64 complex rows).
template <int BM, int BN>
struct TrapH {
  static_assert(BN == 2 * BM, "TrapH is for BN == 2 BM");
  __host__ __device__ static int64_t tri(int64_t t) {  // sum_{rb < t} (rb/2 + 1)
    const int64_t p = t / 2;
    return p * (p + 1) + (t & 1) * (p + 1);
  }
  __host__ __device__ static int64_t count(int64_t rows, int64_t tc) {
    const int64_t nrb = (rows + BM - 1) / BM, ncb = (tc + BN - 1) / BN, r0 = 2 * (ncb - 1);
    return nrb <= r0 ? tri(nrb) : tri(r0) + (nrb - r0) * ncb;
  }
  __host__ __device__ static void decode(int64_t b, int64_t tc, int64_t& rb, int64_t& cb) {
    const int64_t ncb = (tc + BN - 1) / BN, r0 = 2 * (ncb - 1), t0 = tri(r0);
    if (b < t0) {  // pair g of row blocks (2g, 2g+1) holds 2(g+1) items, g(g+1) before it
      int64_t g = 0;
      while ((g + 1) * (g + 2) <= b) ++g;
      const int64_t o = b - g * (g + 1);
      rb = 2 * g + o / (g + 1);
      cb = o % (g + 1);
    } else {
      rb = r0 + (b - t0) / ncb;
      cb = (b - t0) % ncb;
    }
  }
};

// General form for column blocks R = BN / BM times as wide as row blocks:
// row block rb keeps min(ncb, rb / R + 1) column blocks.
template <int BM, int BN>
struct TrapR {
  static_assert(BN % BM == 0, "BN must be a multiple of BM");
  static constexpr int64_t R = BN / BM;
  __host__ __device__ static int64_t tri(int64_t t) {  // sum_{rb < t} (rb / R + 1)
    const int64_t p = t / R;
    return R * p * (p + 1) / 2 + (t % R) * (p + 1);
  }
  __host__ __device__ static int64_t count(int64_t rows, int64_t tc) {
    const int64_t nrb = (rows + BM - 1) / BM, ncb = (tc + BN - 1) / BN, r0 = R * (ncb - 1);
    return nrb <= r0 ? tri(nrb) : tri(r0) + (nrb - r0) * ncb;
  }
  __host__ __device__ static void decode(int64_t b, int64_t tc, int64_t& rb, int64_t& cb) {
    const int64_t ncb = (tc + BN - 1) / BN, r0 = R * (ncb - 1), t0 = tri(r0);
    if (b < t0) {  // group g of R row blocks holds R(g+1) items, R g(g+1)/2 before it
      int64_t g = 0;
      while (R * (g + 1) * (g + 2) / 2 <= b) ++g;
      const int64_t o = b - R * g * (g + 1) / 2;
      rb = R * g + o / (g + 1);
      cb = o % (g + 1);
    } else {
      rb = r0 + (b - t0) / ncb;
      cb = (b - t0) % ncb;
    }
  }
};

template <class TL>
constexpr int min_blocks() { return 65536 / (TL::THREADS * 128) > 0 ? 65536 / (TL::THREADS * 128) : 1; }

// Trailing update (see trail_kernel in gemm.cuh) over one panel tensor map.
template <class TL, bool COPY = false>
__global__ void __launch_bounds__(TL::THREADS, min_blocks<TL>())
    trail_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, TrailParams p,
                     const int* info) {
  using TZ = Trap<TL::BM, TL::BN>;
  // complex embedding: real rows 2r, 2r+1 = re, im of complex row r, so a block
  // of BM real rows covers BM/2 complex rows of the lower trapezoid
  using TZC = Trap<(TL::BM / 2 >= TL::BN ? TL::BM / 2 : TL::BN), TL::BN>;
  if (ld_flag(info)) return;
  // tile cursor: items only grow for a given caller, so the walk over tiles is
  // amortised O(1); producer and consumer each own one
  struct Cursor {
    int64_t m, base, cnt;
  };
  auto decode = [&p](Cursor& cur, int64_t item, TmaBlock& blk) -> bool {
    for (;;) {
      if (cur.m >= p.m_last) return false;
      const int dev = (int)(cur.m % p.D);
      const bool local = dev >= p.dev0 && dev < p.dev0 + p.nloc;
      if (local) {
        if (cur.cnt < 0) {
          const int64_t ms = cur.m * p.T, tcm = p.T < p.N - ms ? p.T : p.N - ms;
          cur.cnt = p.cplx ? TZC::count(p.N - ms, tcm) : TZ::count(p.N - ms, tcm);
        }
        if (item < cur.base + cur.cnt) break;
        cur.base += cur.cnt;
      }
      ++cur.m;
      cur.cnt = -1;
    }
    const int64_t m = cur.m, ms = m * p.T, rows = p.N - ms, tc = p.T < rows ? p.T : rows;
    int64_t rb, cbk;
    const int dev = (int)(m % p.D);
    double* shard = reinterpret_cast<double*>(p.shards[dev - p.dev0]);
    const int64_t loc = (m / p.D) * p.T;
    if (p.cplx) {
      TZC::decode(item - cur.base, tc, rb, cbk);
      blk.a_row = (int)(2 * (ms - p.prow0));
      blk.b_row = (int)(ms - p.prow0);
      blk.m0 = rb * TL::BM;
      blk.n0 = cbk * TL::BN;
      blk.M = 2 * rows;
      blk.N = tc;
      blk.ep = Epilogue{shard + 2 * (ms + loc * p.N), 2 * p.N, -1.0, 1.0, 0, 0};
      return true;
    }
    TZ::decode(item - cur.base, tc, rb, cbk);
    blk.a_row = (int)(ms - p.prow0);
    blk.b_row = (int)(ms - p.prow0);
    blk.m0 = rb * TL::BM;
    blk.n0 = cbk * TL::BN;
    blk.M = rows;
    blk.N = tc;
    blk.ep = Epilogue{shard + ms + loc * p.N, p.N, -1.0, 1.0, 0, 0};
    return true;
  };
  // producer's cursor (thread 0 only) in the caller aux slot: no registers in the consumers
  Cursor& cp = *reinterpret_cast<Cursor*>(tma_aux<TL>() + 384);
  if (threadIdx.x == 0) cp = Cursor{p.m_first, 0, -1};
  tma_gemm_loop<TL, false, COPY>(  // trailing updates never fan out
      &mapA, &mapB, (int)(p.cplx ? 2 * p.K : p.K), [&](int64_t item, TmaBlock& blk) { return decode(cp, item, blk); },
      p.stagger_ns);
}

// Round-1 persistent loop (consumer-side decode), used by trail_tma_kernel_v1.
// Persistent producer/consumer loop.  `next_p(item, blk)` / `next_c(item, blk)`
// fill the block of work item `item` (producer / consumer view; separate so
// stateful cursors stay monotone) and return false when there is none.
template <class TL, bool FAN = true, bool TBK = false, bool MB = false, class NextP, class NextC>
__device__ __forceinline__ void tma_gemm_loop_v1(const CUtensorMap* mapA, const CUtensorMap* mapB, int K, NextP&& next_p,
                                              NextC&& next_c, long long stagger_ns = 0) {
  double* smem = reinterpret_cast<double*>(tma_dyn_smem);
  constexpr int NW = TL::THREADS / 32;
  constexpr unsigned STAGE_BYTES = tma_stage_bytes<TL, TBK>();
  constexpr int STAGE_WORDS = tma_stage_words<TL, TBK>();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TL::STAGES * STAGE_WORDS);
  uint64_t* empty = full + TL::STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % TL::WARPS_M) * TL::WM, wn0 = (warp / TL::WARPS_M) * TL::WN;
  const int KT = (K + TL::BK - 1) / TL::BK;
  if (tid == 0) {
    for (int s = 0; s < TL::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(mapB) : "memory");
  }
  __syncthreads();

  // producer state (thread 0 only) lives in shared memory so it costs the
  // consumer warps no registers: slice counter gp over (item, kt)
  struct Prod {
    int64_t item;
    TmaBlock blk;
    uint32_t gp;
    int kt, live;
  };
  static_assert(sizeof(Prod) <= 384, "producer state must fit its aux slot");
  Prod& ps = *reinterpret_cast<Prod*>(tma_aux<TL, TBK>());
  auto produce_one = [&]() {
    if (!ps.live) return;
    const uint32_t gp = ps.gp;
    const int s = gp % TL::STAGES, kt = ps.kt;
    mbar_wait(&empty[s], ((gp / TL::STAGES) & 1) ^ 1);
    double* st = smem + s * STAGE_WORDS;
    mbar_expect_tx(&full[s], STAGE_BYTES);
    tma_load_2d(st, mapA, ps.blk.a_row + (int)ps.blk.m0, kt * TL::BK, &full[s]);
    const CUtensorMap* mb = MB ? mapB + ps.blk.bmap : mapB;
    if constexpr (TBK) tma_load_2d(st + TL::BK * TL::LDA, mb, kt * TL::BK, ps.blk.b_row + (int)ps.blk.n0, &full[s]);
    else tma_load_2d(st + TL::BK * TL::LDA, mb, ps.blk.b_row + (int)ps.blk.n0, kt * TL::BK, &full[s]);
    ps.gp = gp + 1;
    if (kt + 1 == KT) {
      ps.kt = 0;
      ps.item += gridDim.x;
      ps.live = next_p(ps.item, ps.blk);
    } else {
      ps.kt = kt + 1;
    }
  };
  if (tid == 0) {
    ps.item = blockIdx.x;
    ps.gp = 0;
    ps.kt = 0;
    ps.live = next_p(ps.item, ps.blk);
    for (int i = 0; i < TL::STAGES - 1; ++i) produce_one();
  }

  uint32_t g = 0;
  TmaBlock cb;
  // C tile prefetch into L2 a few slices before the epilogue: all CTAs reach
  // their epilogues at nearly the same time (uniform items), and without it
  // the read-modify-write of 128 KB per CTA would stall every SM on HBM.
  constexpr int PREFETCH_AHEAD = 6;
  auto prefetch_c = [&](const TmaBlock& blk) {
    if (blk.ep.beta == 0.0) return;
    const double* C = reinterpret_cast<const double*>(blk.ep.C);
    constexpr int SEGS = TL::BM * 8 / 128;  // 128-byte lines per column of the tile
    for (int i = tid; i < TL::BN * SEGS; i += TL::THREADS) {
      const int64_t col = blk.n0 + i / SEGS, row = blk.m0 + (i % SEGS) * 16;
      if (col < blk.N && row < blk.M)
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(C + row + col * blk.ep.ldc));
    }
  };
  // Two co-resident CTAs per SM start in lockstep and, with uniform items,
  // would hit their epilogues together; delaying the second half of the grid
  // by about half an item makes one CTA's epilogue overlap the other's DMMAs.
  if (stagger_ns > 0 && blockIdx.x >= gridDim.x / 2) {
    const long long t0 = clock64();
    while (clock64() - t0 < stagger_ns * 2) __nanosleep(1000);  // ~2 cycles per ns at ~2 GHz
  }
  for (int64_t item = blockIdx.x; next_c(item, cb); item += gridDim.x) {
    Acc<TL, false> acc;
    acc.zero();
    for (int kt = 0; kt < KT; ++kt) {
      if (kt == (KT > PREFETCH_AHEAD ? KT - PREFETCH_AHEAD : 0)) prefetch_c(cb);
      if (tid == 0) produce_one();
      const int s = g % TL::STAGES;
      mbar_wait(&full[s], (g / TL::STAGES) & 1);
      const double* st = smem + s * STAGE_WORDS;
      if constexpr (TBK) mma_slice_tbk<TL>(acc, st, st + TL::BK * TL::LDA, wm0, wn0, lane);
      else mma_slice<TL, false, false, false>(acc, st, st + TL::BK * TL::LDA, nullptr, nullptr, wm0, wn0, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++g;
    }
    store_block<double, TL, false, FAN>(acc, cb.ep, cb.M, cb.N, cb.m0, cb.n0, wm0, wn0, lane);
  }
}

// Round-1 form of trail_tma_kernel (consumers decode their own items; kept for A/B
// measurement; the default, BCMG_TRAIL_VARIANT=1).
template <class TL>
__global__ void __launch_bounds__(TL::THREADS, min_blocks<TL>())
    trail_tma_kernel_v1(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, TrailParams p,
                     const int* info) {
  using TZ = Trap<TL::BM, TL::BN>;
  // complex embedding: real rows 2r, 2r+1 = re, im of complex row r, so a block
  // of BM real rows covers BM/2 complex rows of the lower trapezoid
  using TZC = Trap<(TL::BM / 2 >= TL::BN ? TL::BM / 2 : TL::BN), TL::BN>;
  if (ld_flag(info)) return;
  // tile cursor: items only grow for a given caller, so the walk over tiles is
  // amortised O(1); producer and consumer each own one
  struct Cursor {
    int64_t m, base, cnt;
  };
  auto decode = [&p](Cursor& cur, int64_t item, TmaBlock& blk) -> bool {
    for (;;) {
      if (cur.m >= p.m_last) return false;
      const int dev = (int)(cur.m % p.D);
      const bool local = dev >= p.dev0 && dev < p.dev0 + p.nloc;
      if (local) {
        if (cur.cnt < 0) {
          const int64_t ms = cur.m * p.T, tcm = p.T < p.N - ms ? p.T : p.N - ms;
          cur.cnt = p.cplx ? TZC::count(p.N - ms, tcm) : TZ::count(p.N - ms, tcm);
        }
        if (item < cur.base + cur.cnt) break;
        cur.base += cur.cnt;
      }
      ++cur.m;
      cur.cnt = -1;
    }
    const int64_t m = cur.m, ms = m * p.T, rows = p.N - ms, tc = p.T < rows ? p.T : rows;
    int64_t rb, cbk;
    const int dev = (int)(m % p.D);
    double* shard = reinterpret_cast<double*>(p.shards[dev - p.dev0]);
    const int64_t loc = (m / p.D) * p.T;
    if (p.cplx) {
      TZC::decode(item - cur.base, tc, rb, cbk);
      blk.a_row = (int)(2 * (ms - p.prow0));
      blk.b_row = (int)(ms - p.prow0);
      blk.m0 = rb * TL::BM;
      blk.n0 = cbk * TL::BN;
      blk.M = 2 * rows;
      blk.N = tc;
      blk.ep = Epilogue{shard + 2 * (ms + loc * p.N), 2 * p.N, -1.0, 1.0, 0, 0};
      return true;
    }
    TZ::decode(item - cur.base, tc, rb, cbk);
    blk.a_row = (int)(ms - p.prow0);
    blk.b_row = (int)(ms - p.prow0);
    blk.m0 = rb * TL::BM;
    blk.n0 = cbk * TL::BN;
    blk.M = rows;
    blk.N = tc;
    blk.ep = Epilogue{shard + ms + loc * p.N, p.N, -1.0, 1.0, 0, 0};
    return true;
  };
  // producer's cursor (thread 0 only) in the caller aux slot: no registers in the consumers
  Cursor& cp = *reinterpret_cast<Cursor*>(tma_aux<TL>() + 384);
  if (threadIdx.x == 0) cp = Cursor{p.m_first, 0, -1};
  Cursor cc{p.m_first, 0, -1};
  tma_gemm_loop_v1<TL, false>(  // trailing updates never fan out
      &mapA, &mapB, (int)(p.cplx ? 2 * p.K : p.K), [&](int64_t item, TmaBlock& blk) { return decode(cp, item, blk); },
      [&](int64_t item, TmaBlock& blk) { return decode(cc, item, blk); }, p.stagger_ns);
}

// Single GEMM C := alpha A B^H (+ beta C) with A (M x K) i-contiguous and B
// (N x K) i-contiguous (TBK = false) or k-contiguous (TBK = true) real double,
// persistent over the ceil(M/BM) x ceil(N/BN) blocks.
template <class TL, bool TBK = false>
__global__ void __launch_bounds__(TL::THREADS, min_blocks<TL>())
    gemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int64_t M,
                    int64_t N, int64_t K, Epilogue ep, const int* info) {
  if (ld_flag(info)) return;
  const int64_t nbm = (M + TL::BM - 1) / TL::BM, nbn = (N + TL::BN - 1) / TL::BN;
  auto decode = [&](int64_t item, TmaBlock& blk) -> bool {
    if (item >= nbm * nbn) return false;
    // column-block-major: co-resident CTAs share the B (N x K) tile in L2
    blk.a_row = 0;
    blk.b_row = 0;
    blk.m0 = (item % nbm) * TL::BM;
    blk.n0 = (item / nbm) * TL::BN;
    blk.M = M;
    blk.N = N;
    blk.ep = ep;
    return true;
  };
  tma_gemm_loop<TL, true, false, TBK>(&mapA, &mapB, (int)K, decode);
}

// Several GEMMs sharing A in one persistent launch: group g is
// C[:, col0[g] + j] := alpha A Bg(j, :)^T (+ beta C), Bg k-contiguous (TBK)
// with its own tensor map; column blocks never straddle groups.  (The complex
// embedding's product sweep: one B per local device, one wave-filling launch.)
struct BMaps {
  static constexpr int MAX = 8;
  CUtensorMap m[MAX];
  int64_t col0[MAX + 1];  // output column of each group; col0[n] = total
  char* cbase[MAX];       // nullptr: group g writes ep.C + col0[g] * ldc; else its own C
  int n;
};
template <class TL, bool TBK = true>
__global__ void __launch_bounds__(TL::THREADS, min_blocks<TL>())
    gemm_tma_grouped_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ BMaps bm, int64_t M,
                            int64_t K, Epilogue ep, const int* info) {
  if (ld_flag(info)) return;
  const int64_t nbm = (M + TL::BM - 1) / TL::BM;
  auto decode = [&](int64_t item, TmaBlock& blk) -> bool {
    int64_t cb = item / nbm;  // column-block-major, as gemm_tma_kernel
    for (int g = 0; g < bm.n; ++g) {
      const int64_t ng = bm.col0[g + 1] - bm.col0[g], nbg = (ng + TL::BN - 1) / TL::BN;
      if (cb < nbg) {
        blk.a_row = 0;
        blk.b_row = 0;
        blk.bmap = g;
        blk.m0 = (item % nbm) * TL::BM;
        blk.n0 = cb * TL::BN;
        blk.M = M;
        blk.N = ng;
        blk.ep = ep;
        blk.ep.C = bm.cbase[g] ? bm.cbase[g] : static_cast<char*>(ep.C) + bm.col0[g] * ep.ldc * 8;
        return true;
      }
      cb -= nbg;
    }
    return false;
  };
  // i-contiguous B (potri's W sweep): the consumer-decoded loop of
  // trail_tma_kernel_v1, 2.3 % faster there (10.86 vs 11.12 s at config 4);
  // k-contiguous B (product sweep): the item ring, 1.7 % faster there
  if constexpr (TBK) tma_gemm_loop<TL, true, false, true, true>(&mapA, &bm.m[0], (int)K, decode);
  else tma_gemm_loop_v1<TL, false, false, true>(&mapA, &bm.m[0], (int)K, decode, decode);
}

}  // namespace bcmg
