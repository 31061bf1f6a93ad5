// FP64 tensor-core (DMMA) block GEMM for sm_100a.
//
// The only dense contraction of the Cholesky path is a GEMM of the form
//     C := alpha * Ahat * Bhat^T + beta * C
// where Ahat (M x K) and Bhat (N x K) are logical views of column-major
// storage (see Operand).  On sm_100a there is no tcgen05 kind::f64, so FP64
// tensor work is warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), fed from
// shared memory laid out k-major ([k][i], i contiguous) with a 4-word row
// pad so every 8x4 fragment load is bank-conflict free.  Complex operands are
// split into re/im planes and contracted with 4 real DMMAs per step;
// float/complex64 storage is widened to FP64 on the way into shared memory.
//
// Two operand feeders:
//   * CP  : cp.async 16-byte copies into a STAGES-deep ring (real double,
//           natural orientation, 16-byte aligned) -- the hot trailing update
//           and panel TRSM of potrf;
//   * REG : register-staged loads with conversion / conjugation /
//           transposition / triangular masks, double buffered -- every other
//           shape.
#pragma once

#include "common.cuh"

namespace bcmg {

enum Op : int { OP_N = 0, OP_C = 1 };

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ int ld_flag(const int* p) { return p ? *(volatile const int*)p : 0; }

// Logical operand: element (i, k) of Xhat.
struct Operand {
  const void* ptr;
  int64_t ld;
  int trans;         // 0: Xhat(i,k) = X[i + k*ld]   1: Xhat(i,k) = X[k + i*ld]
  int conj;          // conjugate on load
  int mask;          // 1: element read as 0 unless storage_row + mask_off >= storage_col
  int64_t mask_off;  //    (a lower-triangular view of the stored matrix)
};

// op(A): A is M x K (op N) or K x M (op C) column-major.
inline Operand opA(const void* p, int64_t ld, int op) {
  return Operand{p, ld, op == OP_C ? 1 : 0, op == OP_C ? 1 : 0, 0, 0};
}
// op(B): B is K x N (op N) or N x K (op C) column-major.
inline Operand opB(const void* p, int64_t ld, int op) {
  return Operand{p, ld, op == OP_N ? 1 : 0, op == OP_C ? 1 : 0, 0, 0};
}

constexpr int MAX_FAN = 7;  // peers of an 8-GPU node
struct Epilogue {
  void* C;
  int64_t ldc;
  double alpha, beta;
  int lower_only;      // store only where row - col >= lower_off
  int64_t lower_off;
  // fan-out: every stored element is also written at the same offset from
  // each fan[e] (peer GPUs' copies of C over NVLink: a GEMM fused with its
  // broadcast, see Session::potrf's peer-memory mode)
  void* fan[MAX_FAN];
  int nfan;
};

// fan[e] through constant offsets only: indexing a fan array with a runtime e
// would move a kernel's local Epilogue / Blk copy into local memory
template <class P>
__device__ __forceinline__ P fan_at(P const (&fan)[MAX_FAN], int e) {
  static_assert(MAX_FAN == 7, "fan_at enumerates MAX_FAN entries");
  switch (e) {
    case 0: return fan[0];
    case 1: return fan[1];
    case 2: return fan[2];
    case 3: return fan[3];
    case 4: return fan[4];
    case 5: return fan[5];
    default: return fan[6];
  }
}

// PAIR: fragment f covers rows {16(f/2) + 2r + f%2 : r = 0..7} instead of
// {8f + r}, so a thread's rows for fragments 2p and 2p+1 are adjacent and one
// LDS.128 feeds two DMMA fragments (rows of a GEMM are independent: the
// permutation changes no arithmetic, only where the epilogue stores).
template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, bool PAIR_ = false>
struct Tile {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr bool PAIR = PAIR_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static_assert(!PAIR || (FM % 2 == 0 && FN % 2 == 0), "paired fragments need even counts");
  // i-contiguous tiles [BK][BI+4] (operand stored with i contiguous) and
  // k-contiguous tiles [BI][BK+4] (operand stored with k contiguous); the
  // 4-word pad keeps both fragment read patterns bank-conflict free.
  static constexpr int LDA = BM + 4, LDB = BN + 4, LDT = BK + 4;  // 8-byte words; == 4 (mod 16)
  static_assert(LDA % 16 == 4 && LDB % 16 == 4 && LDT % 16 == 4, "row pad must be 4 words mod 16");
  static constexpr int A_WORDS = (BK * LDA > BM * LDT) ? BK * LDA : BM * LDT;
  static constexpr int B_WORDS = (BK * LDB > BN * LDT) ? BK * LDB : BN * LDT;
  static constexpr int STAGE_WORDS = A_WORDS + B_WORDS;
};

template <class TL, bool CPLX, bool CP>
constexpr size_t gemm_smem_bytes() {
  return CP ? (size_t)TL::STAGES * TL::STAGE_WORDS * 8 : (size_t)2 * TL::STAGE_WORDS * 8 * (CPLX ? 2 : 1);
}

// ----------------------------------------------------------------- accumulators
template <class TL, bool CPLX>
struct Acc {
  double re[TL::FM][TL::FN][2];
  double im[CPLX ? TL::FM : 1][CPLX ? TL::FN : 1][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int a = 0; a < TL::FM; ++a)
#pragma unroll
      for (int b = 0; b < TL::FN; ++b) {
        re[a][b][0] = re[a][b][1] = 0.0;
        if constexpr (CPLX) im[a][b][0] = im[a][b][1] = 0.0;
      }
  }
};

template <class TL>
__device__ __forceinline__ int frag_row(int f, int r) {
  return TL::PAIR ? 16 * (f >> 1) + 2 * r + (f & 1) : 8 * f + r;
}

// One BK slice of DMMAs out of shared memory (planes: real or re/im).
template <class TL, bool CPLX, bool TA, bool TB>
__device__ __forceinline__ void mma_slice(Acc<TL, CPLX>& acc, const double* __restrict__ As,
                                          const double* __restrict__ Bs, const double* __restrict__ Asi,
                                          const double* __restrict__ Bsi, int wm0, int wn0, int lane) {
  const int r = lane >> 2, q = lane & 3;
#pragma unroll
  for (int kk = 0; kk < TL::BK; kk += 4) {
    double a[TL::FM], b[TL::FN];
    double ai[CPLX ? TL::FM : 1], bi[CPLX ? TL::FN : 1];
    if constexpr (TL::PAIR && !TA && !CPLX) {
#pragma unroll
      for (int f = 0; f < TL::FM; f += 2) {
        const double2 v = *reinterpret_cast<const double2*>(As + (kk + q) * TL::LDA + wm0 + frag_row<TL>(f, r));
        a[f] = v.x;
        a[f + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int f = 0; f < TL::FM; ++f) {
        const int m = wm0 + frag_row<TL>(f, r);
        const int o = TA ? m * TL::LDT + kk + q : (kk + q) * TL::LDA + m;
        a[f] = As[o];
        if constexpr (CPLX) ai[f] = Asi[o];
      }
    }
    if constexpr (TL::PAIR && !TB && !CPLX) {
#pragma unroll
      for (int f = 0; f < TL::FN; f += 2) {
        const double2 v = *reinterpret_cast<const double2*>(Bs + (kk + q) * TL::LDB + wn0 + frag_row<TL>(f, r));
        b[f] = v.x;
        b[f + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int f = 0; f < TL::FN; ++f) {
        const int nn = wn0 + frag_row<TL>(f, r);
        const int o = TB ? nn * TL::LDT + kk + q : (kk + q) * TL::LDB + nn;
        b[f] = Bs[o];
        if constexpr (CPLX) bi[f] = Bsi[o];
      }
    }
#pragma unroll
    for (int fm = 0; fm < TL::FM; ++fm)
#pragma unroll
      for (int fn = 0; fn < TL::FN; ++fn) {
        dmma(acc.re[fm][fn][0], acc.re[fm][fn][1], a[fm], b[fn]);
        if constexpr (CPLX) {
          dmma(acc.re[fm][fn][0], acc.re[fm][fn][1], -ai[fm], bi[fn]);
          dmma(acc.im[fm][fn][0], acc.im[fm][fn][1], a[fm], bi[fn]);
          dmma(acc.im[fm][fn][0], acc.im[fm][fn][1], ai[fm], b[fn]);
        }
      }
  }
}

// ----------------------------------------------------------------- REG feeder
// Holds the raw storage elements between load() and store(): widening and
// conjugation happen in store(), after the MMAs of the current slice, so the
// predicated loads of a slice are all in flight at once (converting inside the
// guarded load made every element wait for its own load: ~4 us per slice).
template <class S, int BI, int BK, int THREADS>
struct RegFeed {
  static constexpr bool CPLX = Traits<S>::cplx;
  static constexpr int E = BI * BK / THREADS;
  static_assert(E * THREADS == BI * BK, "tile not divisible by threads");
  S raw[E];

  __device__ __forceinline__ void load(const Operand& op, int64_t I, int64_t K, int64_t i0, int64_t k0, int tid) {
    const S* base = reinterpret_cast<const S*>(op.ptr);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int idx = tid + e * THREADS;
      const int il = op.trans ? idx / BK : idx % BI;
      const int kl = op.trans ? idx % BK : idx / BI;
      const int64_t i = i0 + il, k = k0 + kl;
      // storage coordinates: natural (row i, col k), transposed (row k, col i)
      const int64_t srow = op.trans ? k : i, scol = op.trans ? i : k;
      const bool ok = i < I && k < K && (!op.mask || srow + op.mask_off >= scol);
      raw[e] = from_c<S>(make_double2(0.0, 0.0));
      if (ok) raw[e] = base[op.trans ? (k + i * op.ld) : (i + k * op.ld)];
    }
  }
  // LD: row length of the i-contiguous layout; LDT: of the k-contiguous one
  __device__ __forceinline__ void store(const Operand& op, double* Xs, double* Xsi, int LD, int LDT, int tid) const {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int idx = tid + e * THREADS;
      const int il = op.trans ? idx / BK : idx % BI;
      const int kl = op.trans ? idx % BK : idx / BI;
      const int o = op.trans ? il * LDT + kl : kl * LD + il;
      const double2 v = to_c(raw[e]);
      Xs[o] = v.x;
      if constexpr (CPLX) Xsi[o] = op.conj ? -v.y : v.y;
    }
  }
};

// ----------------------------------------------------------------- CP feeder
// Real double, natural orientation (Xhat(i,k) = X[i + k*ld]), X 16B aligned,
// ld even.  Out-of-range elements are zero-filled by cp.async src-size.
template <int BI, int BK, int THREADS>
__device__ __forceinline__ void cp_feed(const Operand& op, int64_t I, int64_t K, int64_t i0, int64_t k0,
                                        double* Xs, int LD, int tid) {
  constexpr int CH = (BI / 2) * BK;  // 16-byte chunks per stage
  static_assert(CH % THREADS == 0, "chunks not divisible by threads");
  const double* base = reinterpret_cast<const double*>(op.ptr);
#pragma unroll
  for (int c = 0; c < CH / THREADS; ++c) {
    const int idx = tid + c * THREADS;
    const int il = (idx % (BI / 2)) * 2, kl = idx / (BI / 2);
    const int64_t i = i0 + il, k = k0 + kl;
    int64_t rem = I - i;
    int bytes = (k < K && rem > 0) ? (rem >= 2 ? 16 : 8) : 0;
    const double* src = bytes ? base + i + k * op.ld : base;
    cp_async16(Xs + kl * LD + il, src, bytes);
  }
}

// k-contiguous operand (Xhat(i,k) = X[k + i*ld]) into [BI][BK+4].
template <int BI, int BK, int LDT, int THREADS>
__device__ __forceinline__ void cp_feed_t(const Operand& op, int64_t I, int64_t K, int64_t i0, int64_t k0,
                                          double* Xs, int tid) {
  constexpr int CH = BI * (BK / 2);
  static_assert(CH % THREADS == 0, "chunks not divisible by threads");
  const double* base = reinterpret_cast<const double*>(op.ptr);
#pragma unroll
  for (int c = 0; c < CH / THREADS; ++c) {
    const int idx = tid + c * THREADS;
    const int kl = (idx % (BK / 2)) * 2, il = idx / (BK / 2);
    const int64_t i = i0 + il, k = k0 + kl;
    int64_t rem = K - k;
    int bytes = (i < I && rem > 0) ? (rem >= 2 ? 16 : 8) : 0;
    const double* src = bytes ? base + k + i * op.ld : base;
    cp_async16(Xs + il * LDT + kl, src, bytes);
  }
}

template <bool T, int BI, int BK, int LD, int LDT, int THREADS>
__device__ __forceinline__ void cp_feed_any(const Operand& op, int64_t I, int64_t K, int64_t i0, int64_t k0,
                                            double* Xs, int tid) {
  if constexpr (T) cp_feed_t<BI, BK, LDT, THREADS>(op, I, K, i0, k0, Xs, tid);
  else cp_feed<BI, BK, THREADS>(op, I, K, i0, k0, Xs, LD, tid);
}

// ----------------------------------------------------------------- epilogue
template <class S, class TL, bool CPLX, bool FAN = true>
__device__ __forceinline__ void store_block(const Acc<TL, CPLX>& acc, const Epilogue& ep, int64_t M, int64_t N,
                                            int64_t m0, int64_t n0, int wm0, int wn0, int lane) {
  const int r = lane >> 2, q = lane & 3;
  S* __restrict__ C = reinterpret_cast<S*>(ep.C);
  // One fragment row at a time: issue all of its C loads before any store, so
  // the read-modify-write pays one memory latency per row group instead of one
  // per element (the compiler cannot reorder loads across the stores itself).
#pragma unroll
  for (int fm = 0; fm < TL::FM; ++fm) {
    const int64_t row = m0 + wm0 + frag_row<TL>(fm, r);
    bool ok[TL::FN][2];
    S old[TL::FN][2];
#pragma unroll
    for (int fn = 0; fn < TL::FN; ++fn)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t col = n0 + wn0 + (TL::PAIR ? 16 * (fn >> 1) + 2 * (2 * q + j) + (fn & 1) : fn * 8 + 2 * q + j);
        ok[fn][j] = row < M && col < N && (!ep.lower_only || row - col >= ep.lower_off);
        old[fn][j] = from_c<S>(make_double2(0.0, 0.0));
        if (ok[fn][j] && ep.beta != 0.0) old[fn][j] = C[row + col * ep.ldc];
      }
#pragma unroll
    for (int fn = 0; fn < TL::FN; ++fn)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (!ok[fn][j]) continue;
        const int64_t col = n0 + wn0 + (TL::PAIR ? 16 * (fn >> 1) + 2 * (2 * q + j) + (fn & 1) : fn * 8 + 2 * q + j);
        double2 v = make_double2(ep.alpha * acc.re[fm][fn][j], 0.0);
        if constexpr (CPLX) v.y = ep.alpha * acc.im[fm][fn][j];
        if (ep.beta != 0.0) {
          const double2 o = to_c(old[fn][j]);
          v.x += ep.beta * o.x;
          v.y += ep.beta * o.y;
        }
        const S out = from_c<S>(v);
        C[row + col * ep.ldc] = out;
        if constexpr (FAN)
          for (int e = 0; e < ep.nfan; ++e) static_cast<S*>(fan_at(ep.fan, e))[row + col * ep.ldc] = out;
      }
  }
}

// ----------------------------------------------------------------- block GEMM
// Computes the BM x BN block at (m0, n0) of C := alpha*Ahat*Bhat^T + beta*C.
template <class S, class TL, bool CP, bool TA, bool TB>
__device__ __forceinline__ void gemm_block(const Operand& A, const Operand& B, int64_t M, int64_t N, int64_t K,
                                           int64_t m0, int64_t n0, const Epilogue& ep, double* smem) {
  constexpr bool CPLX = Traits<S>::cplx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % TL::WARPS_M) * TL::WM, wn0 = (warp / TL::WARPS_M) * TL::WN;
  const int KT = (int)((K + TL::BK - 1) / TL::BK);
  Acc<TL, CPLX> acc;
  acc.zero();

  if constexpr (CP) {
    static_assert(!CPLX, "cp.async feeder is real-only");
    // prologue: STAGES-1 slices in flight
#pragma unroll
    for (int s = 0; s < TL::STAGES - 1; ++s) {
      if (s < KT) {
        double* st = smem + s * TL::STAGE_WORDS;
        cp_feed_any<TA, TL::BM, TL::BK, TL::LDA, TL::LDT, TL::THREADS>(A, M, K, m0, (int64_t)s * TL::BK, st, tid);
        cp_feed_any<TB, TL::BN, TL::BK, TL::LDB, TL::LDT, TL::THREADS>(B, N, K, n0, (int64_t)s * TL::BK,
                                                                        st + TL::A_WORDS, tid);
      }
      cp_async_commit();
    }
    for (int kt = 0; kt < KT; ++kt) {
      cp_async_wait<TL::STAGES - 2>();
      __syncthreads();
      const int nk = kt + TL::STAGES - 1;
      if (nk < KT) {
        double* st = smem + (nk % TL::STAGES) * TL::STAGE_WORDS;
        cp_feed_any<TA, TL::BM, TL::BK, TL::LDA, TL::LDT, TL::THREADS>(A, M, K, m0, (int64_t)nk * TL::BK, st, tid);
        cp_feed_any<TB, TL::BN, TL::BK, TL::LDB, TL::LDT, TL::THREADS>(B, N, K, n0, (int64_t)nk * TL::BK,
                                                                        st + TL::A_WORDS, tid);
      }
      cp_async_commit();
      const double* st = smem + (kt % TL::STAGES) * TL::STAGE_WORDS;
      mma_slice<TL, false, TA, TB>(acc, st, st + TL::A_WORDS, nullptr, nullptr, wm0, wn0, lane);
    }
    cp_async_wait<0>();
    __syncthreads();
  } else {
    RegFeed<S, TL::BM, TL::BK, TL::THREADS> fa;
    RegFeed<S, TL::BN, TL::BK, TL::THREADS> fb;
    constexpr int PLANE = TL::STAGE_WORDS;  // re plane size per buffer
    auto bufA = [&](int b) { return smem + b * PLANE * (CPLX ? 2 : 1); };
    fa.load(A, M, K, m0, 0, tid);
    fb.load(B, N, K, n0, 0, tid);
    {
      double* s0 = bufA(0);
      fa.store(A, s0, s0 + PLANE, TL::LDA, TL::LDT, tid);
      fb.store(B, s0 + TL::A_WORDS, s0 + PLANE + TL::A_WORDS, TL::LDB, TL::LDT, tid);
    }
    __syncthreads();
    for (int kt = 0; kt < KT; ++kt) {
      const bool more = kt + 1 < KT;
      if (more) {
        fa.load(A, M, K, m0, (int64_t)(kt + 1) * TL::BK, tid);
        fb.load(B, N, K, n0, (int64_t)(kt + 1) * TL::BK, tid);
      }
      const double* s = bufA(kt & 1);
      mma_slice<TL, CPLX, TA, TB>(acc, s, s + TL::A_WORDS, s + PLANE, s + PLANE + TL::A_WORDS, wm0, wn0, lane);
      if (more) {
        double* d = bufA((kt + 1) & 1);
        fa.store(A, d, d + PLANE, TL::LDA, TL::LDT, tid);
        fb.store(B, d + TL::A_WORDS, d + PLANE + TL::A_WORDS, TL::LDB, TL::LDT, tid);
      }
      __syncthreads();
    }
  }
  store_block<S, TL, CPLX>(acc, ep, M, N, m0, n0, wm0, wn0, lane);
}

// ----------------------------------------------------------------- front-ends
// Single GEMM: grid (ceil(M/BM), ceil(N/BN)).
template <class S, class TL, bool CP, bool TA, bool TB>
__global__ void __launch_bounds__(TL::THREADS) gemm_kernel(Operand A, Operand B, int64_t M, int64_t N, int64_t K,
                                                            Epilogue ep, const int* info) {
  if (ld_flag(info)) return;
  extern __shared__ __align__(16) double smem[];
  gemm_block<S, TL, CP, TA, TB>(A, B, M, N, K, (int64_t)blockIdx.x * TL::BM, (int64_t)blockIdx.y * TL::BN, ep,
                                smem);
}

// Split-K GEMM: part z = blockIdx.z contracts k in [z*kchunk, (z+1)*kchunk)
// into its own M x N slab of `parts` (ld M); a fixed-order reduction sums
// the slabs afterwards, so the result does not depend on scheduling.
template <class S, class TL, bool CP, bool TA, bool TB>
__global__ void __launch_bounds__(TL::THREADS) gemm_splitk_kernel(Operand A, Operand B, int64_t M, int64_t N,
                                                                   int64_t K, int64_t kchunk, S* parts) {
  extern __shared__ __align__(16) double smem[];
  const int64_t k0 = (int64_t)blockIdx.z * kchunk;
  const int64_t kz = (K - k0 < kchunk) ? K - k0 : kchunk;
  if (kz <= 0) return;
  // advance both operands by k0 along their k dimension
  A.ptr = reinterpret_cast<const S*>(A.ptr) + (A.trans ? k0 : k0 * A.ld);
  B.ptr = reinterpret_cast<const S*>(B.ptr) + (B.trans ? k0 : k0 * B.ld);
  A.mask_off += A.trans ? k0 : -k0;
  B.mask_off += B.trans ? k0 : -k0;
  Epilogue ep{parts + (int64_t)blockIdx.z * M * N, M, 1.0, 0.0, 0, 0};
  gemm_block<S, TL, CP, TA, TB>(A, B, M, N, kz, (int64_t)blockIdx.x * TL::BM, (int64_t)blockIdx.y * TL::BN, ep,
                                smem);
}

// Trailing update of potrf step k on this process's shards:
//   for every local tile m in [m_first, m_last):
//     A_m[ms:N, :] -= P[ms:N, :] * P[ms:ms+tc_m, :]^H
// (reference solvers.py:395-405, restricted to the rows the lower triangle
// reads).  Persistent grid, static round-robin over the lower-trapezoid
// blocks of all tiles, tile-major so co-resident CTAs share panel rows.
constexpr int MAX_LOCAL_DEV = 16;
struct TrailParams {
  const void* P;      // panel, element (r, c) at P[r + c*ldp], r = global row - prow0
  // complex128 through the real FP64 TMA kernel (cplx = 1): P holds [P | -iP]
  // (ld = ldp = panel rows) and PB the planar [Re P | Im P] (real, ld ldp);
  // the update is then one real GEMM with interleaved re/im output rows
  const void* PB;
  int cplx;
  // float32 / complex64 on tcgen05: the panel pre-split into tf32 hi / lo
  // planes, K-major (row-major rows x ld): A hi, A lo, B hi, B lo (A == B for
  // real input; complex64: A = [P | -iP] with 2x the rows, B = [Re P | Im P])
  const float* split[4];
  int64_t split_ld[2];
  int64_t ldp, prow0;
  int64_t N, T, K;    // matrix order, tile width, panel width
  int D, dev0, nloc;  // logical devices; this launch owns dev0 .. dev0+nloc-1
  void* shards[MAX_LOCAL_DEV];
  int64_t m_first, m_last;
  int max_ctas;       // host-side: persistent grid cap (0 = all SMs)
  long long stagger_ns;  // delay of the second half of the grid (two CTAs per SM)
  // tcgen05 trailing update with one column block per tile (T <= tile width):
  // items of `band` consecutive owned tile columns are interleaved by absolute
  // row block, so a wave reuses each panel row block across the band from L2
  // instead of streaming the whole panel from HBM once per tile column (0 = off)
  int band;
  // tcgen05 pair kernel at T_A = 128 (cpu = 2): each item covers two owned tile
  // columns (c, c + spacing) as one 256-wide UMMA tile; 0 / 1 = one column
  int cpu;
};

template <int B>
__device__ __forceinline__ int64_t trail_blocks(int64_t rows, int64_t tc) {
  const int64_t nrb = (rows + B - 1) / B, ncb = (tc + B - 1) / B;
  return nrb <= ncb ? nrb * (nrb + 1) / 2 : ncb * (ncb + 1) / 2 + (nrb - ncb) * ncb;
}

template <class S, class TL, bool CP>
__global__ void __launch_bounds__(TL::THREADS) trail_kernel(TrailParams p, const int* info) {
  static_assert(TL::BM == TL::BN, "trailing decode assumes square blocks");
  constexpr int B = TL::BM;
  if (ld_flag(info)) return;
  extern __shared__ __align__(16) double smem[];
  const S* P = reinterpret_cast<const S*>(p.P);
  int64_t m = p.m_first, base = 0, cnt = -1;
  for (int64_t item = blockIdx.x;; item += gridDim.x) {
    // advance the tile cursor (monotone: items only grow)
    for (;;) {
      if (m >= p.m_last) return;
      const int dev = (int)(m % p.D);
      const bool local = dev >= p.dev0 && dev < p.dev0 + p.nloc;
      if (local) {
        if (cnt < 0) {
          const int64_t ms = m * p.T;
          cnt = trail_blocks<B>(p.N - ms, (p.T < p.N - ms ? p.T : p.N - ms));
        }
        if (item < base + cnt) break;
        base += cnt;
      }
      ++m;
      cnt = -1;
    }
    const int64_t ms = m * p.T, rows = p.N - ms, tc = p.T < rows ? p.T : rows;
    const int64_t ncb = (tc + B - 1) / B;
    int64_t b = item - base, rb, cb;
    const int64_t tri = ncb * (ncb + 1) / 2;
    if (b < tri) {
      rb = 0;
      while ((rb + 1) * (rb + 2) / 2 <= b) ++rb;
      cb = b - rb * (rb + 1) / 2;
    } else {
      rb = ncb + (b - tri) / ncb;
      cb = (b - tri) % ncb;
    }
    const int dev = (int)(m % p.D);
    S* shard = reinterpret_cast<S*>(p.shards[dev - p.dev0]);
    const int64_t loc = (m / p.D) * p.T;
    Operand A{P + (ms - p.prow0), p.ldp, 0, 0, 0, 0};
    Operand Bo{P + (ms - p.prow0), p.ldp, 0, 1, 0, 0};
    Epilogue ep{shard + ms + loc * p.N, p.N, -1.0, 1.0, 0, 0};
    gemm_block<S, TL, CP, false, false>(A, Bo, rows, tc, p.K, rb * B, cb * B, ep, smem);
    __syncthreads();
  }
}

}  // namespace bcmg
