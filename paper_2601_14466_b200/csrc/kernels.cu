// Kernels and launchers of the bcmg B200 library (sm_100a):
//   * GEMM dispatch onto the DMMA block kernels of gemm.cuh,
//   * the potrf trailing update launcher,
//   * the diagonal-tile factor+inverse (leaf kernel + recursive GEMM driver),
//   * the in-place cycle rotation of the block-cyclic redistribution,
//   * small copy / conjugate / mirror helpers.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <type_traits>

#include <cudaTypedefs.h>

#include "gemm_tma.cuh"
#include "tc_gemm.cuh"
#include "tc_gemm_k.cuh"
#include "ops.h"
#include "comm.h"

namespace bcmg {

static std::atomic<long long> g_launches{0};
void note_launch(const char* file, int line) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  static const bool debug = [] {
    const char* e = getenv("BCMG_DEBUG_SYNC");
    return e && atoi(e);
  }();
  if (debug) {
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess)
      throw Error(CUDA, std::string("kernel launched at ") + file + ":" + std::to_string(line) + ": " +
                            cudaGetErrorString(e));
  }
}
long long launch_count() { return g_launches.load(); }

// ============================================================== GEMM dispatch
using TileBig = Tile<128, 128, 32, 32, 32, 3, true>;  // 512 threads, hot real path (paired LDS.128)
using TileMed = Tile<64, 64, 16, 32, 32, 3>;      // 128 threads, general
using TileNarrow = Tile<128, 16, 16, 32, 16, 3>;  // 128 threads, N <= 16 (RHS blocks)

static int num_sms() {
  static const int sms = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return sms;
}

// once per kernel and process (the attribute is per function, not per
// thread; a first cudaFuncSetAttribute can load the function's module, which
// must not happen in the middle of another rank's flag hand-off)
static std::mutex g_smem_mu;
template <class K>
static void set_smem(K kernel, size_t bytes) {
  static std::vector<const void*> done;
  const void* key = reinterpret_cast<const void*>(kernel);
  std::lock_guard<std::mutex> lk(g_smem_mu);
  if (std::find(done.begin(), done.end(), key) != done.end()) return;
  BCMG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done.push_back(key);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static bool cp_ok(const Operand& X) { return !X.mask && aligned16(X.ptr) && (X.ld % 2 == 0); }

template <class S, class TL, bool CP, bool TA, bool TB>
static void launch_gemm_t(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                          const int* info, cudaStream_t st) {
  constexpr size_t smem = gemm_smem_bytes<TL, Traits<S>::cplx, CP>();
  auto kern = gemm_kernel<S, TL, CP, TA, TB>;
  set_smem(kern, smem);
  dim3 grid((unsigned)((M + TL::BM - 1) / TL::BM), (unsigned)((N + TL::BN - 1) / TL::BN));
  kern<<<grid, TL::THREADS, smem, st>>>(A, B, M, N, K, ep, info);
  BCMG_CHECK_LAUNCH();
}

template <class S, class TL, bool CP>
static void launch_gemm(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                        const int* info, cudaStream_t st) {
  if (A.trans) {
    if (B.trans) launch_gemm_t<S, TL, CP, true, true>(M, N, K, A, B, ep, info, st);
    else launch_gemm_t<S, TL, CP, true, false>(M, N, K, A, B, ep, info, st);
  } else {
    if (B.trans) launch_gemm_t<S, TL, CP, false, true>(M, N, K, A, B, ep, info, st);
    else launch_gemm_t<S, TL, CP, false, false>(M, N, K, A, B, ep, info, st);
  }
}

static bool use_tma();
static unsigned ew_grid(int64_t total);
static bool use_tc();
static bool use_presplit();
static float* split_scratch(cudaStream_t st, size_t bytes, size_t* held = nullptr);
static void gemm_tck_generic(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                             const int* info, cudaStream_t st);
static bool tc_ok(const void* p, int64_t ld);
static void launch_tc3_gemm(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                            const int* info, cudaStream_t st);
static bool tma_ok(const void* p, int64_t ld);
static void launch_gemm_tma(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                            const int* info, cudaStream_t st);

template <class S>
static void gemm_t(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                   const int* info, cudaStream_t st) {
  if constexpr (std::is_same_v<S, double>) {
    const bool cp = cp_ok(A) && cp_ok(B);
    if (cp) {
      if (N <= 16) return launch_gemm<S, TileNarrow, true>(M, N, K, A, B, ep, info, st);
      const int64_t big_blocks = ((M + TileBig::BM - 1) / TileBig::BM) * ((N + TileBig::BN - 1) / TileBig::BN);
      if (big_blocks >= num_sms()) {
        if (use_tma() && !A.trans && !B.trans && tma_ok(A.ptr, A.ld) && tma_ok(B.ptr, B.ld))
          return launch_gemm_tma(M, N, K, A, B, ep, info, st);
        return launch_gemm<S, TileBig, true>(M, N, K, A, B, ep, info, st);
      }
      return launch_gemm<S, TileMed, true>(M, N, K, A, B, ep, info, st);
    }
  }
  if constexpr (std::is_same_v<S, float>) {
    // (no alignment condition on C: the epilogue stores are scalar, and a condition
    // on the shard's address would make the kernel -- and the bits -- depend on
    // where a device's shard sits in the flat buffer, i.e. on the device count)
    if (use_tc() && use_presplit() && !A.mask && !B.mask && M >= 256 && N >= 64 && K >= 32)
      return gemm_tck_generic(M, N, K, A, B, ep, info, st);
    if (use_tc() && ep.nfan == 0 && !A.trans && !B.trans && !A.mask && !B.mask && tc_ok(A.ptr, A.ld) &&
        tc_ok(B.ptr, B.ld) && tc_ok(ep.C, 4) && M >= 256 && N >= 64 && K >= 32)
      return launch_tc3_gemm(M, N, K, A, B, ep, info, st);
  }
  if (N <= 16) return launch_gemm<S, TileNarrow, false>(M, N, K, A, B, ep, info, st);
  return launch_gemm<S, TileMed, false>(M, N, K, A, B, ep, info, st);
}

template <class S, class TL, bool CP, bool TA, bool TB>
static void launch_splitk_t(int64_t M, int64_t N, int64_t K, int64_t kchunk, int np, const Operand& A,
                            const Operand& B, void* parts, cudaStream_t st) {
  constexpr size_t smem = gemm_smem_bytes<TL, Traits<S>::cplx, CP>();
  auto kern = gemm_splitk_kernel<S, TL, CP, TA, TB>;
  set_smem(kern, smem);
  dim3 grid((unsigned)((M + TL::BM - 1) / TL::BM), (unsigned)((N + TL::BN - 1) / TL::BN), (unsigned)np);
  kern<<<grid, TL::THREADS, smem, st>>>(A, B, M, N, K, kchunk, static_cast<S*>(parts));
  BCMG_CHECK_LAUNCH();
}

template <class S, class TL, bool CP>
static int splitk_t(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, void* parts, int max_parts,
                    cudaStream_t st) {
  const int64_t ctas = ((M + TL::BM - 1) / TL::BM) * ((N + TL::BN - 1) / TL::BN);
  int64_t np = (2 * num_sms() + ctas - 1) / ctas;
  np = std::max<int64_t>(1, std::min<int64_t>({np, (int64_t)max_parts, (K + 127) / 128}));
  int64_t kchunk = ((K + np - 1) / np + TL::BK - 1) / TL::BK * TL::BK;
  np = (K + kchunk - 1) / kchunk;
  if (A.trans) {
    if (B.trans) launch_splitk_t<S, TL, CP, true, true>(M, N, K, kchunk, (int)np, A, B, parts, st);
    else launch_splitk_t<S, TL, CP, true, false>(M, N, K, kchunk, (int)np, A, B, parts, st);
  } else {
    if (B.trans) launch_splitk_t<S, TL, CP, false, true>(M, N, K, kchunk, (int)np, A, B, parts, st);
    else launch_splitk_t<S, TL, CP, false, false>(M, N, K, kchunk, (int)np, A, B, parts, st);
  }
  return (int)np;
}

int gemm_splitk(int dt, int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, void* parts,
                int max_parts, cudaStream_t st) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  int np = 0;
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    if constexpr (std::is_same_v<S, double>) {
      if (cp_ok(A) && cp_ok(B)) {
        np = N <= 16 ? splitk_t<S, TileNarrow, true>(M, N, K, A, B, parts, max_parts, st)
                     : splitk_t<S, TileMed, true>(M, N, K, A, B, parts, max_parts, st);
        return;
      }
    }
    np = N <= 16 ? splitk_t<S, TileNarrow, false>(M, N, K, A, B, parts, max_parts, st)
                 : splitk_t<S, TileMed, false>(M, N, K, A, B, parts, max_parts, st);
  });
  return np;
}

// The kernel choice of gemm() depends on N (the tcgen05 path needs N >= 64).
// potri's per-device products have N = that device's columns, so the same
// block would take different kernels (different bits) at different device
// counts; this variant decides from M and K only.
void gemm_shape_fixed(int dt, int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                      const int* info, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  // (nor on C's alignment: one flat buffer puts later devices' shards at any
  // 4-byte offset, and the tcgen05 epilogue stores are scalar)
  if (dt == R32 && use_tc() && use_presplit() && !A.mask && !B.mask && M >= 256 && K >= 32)
    return gemm_tck_generic(M, N, K, A, B, ep, info, st);
  gemm(dt, M, N, K, A, B, ep, info, st);
}

void gemm(int dt, int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
          const int* info, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    // C := beta*C only; with beta==1 nothing to do, beta==0 handled by a zero-K GEMM
    if (ep.beta == 1.0) return;
  }
  dispatch_dtype(dt, [&](auto s) { gemm_t<decltype(s)>(M, N, std::max<int64_t>(K, 0), A, B, ep, info, st); });
}

// ============================================================== trailing update
template <class S, class TL, bool CP>
static void launch_trail(const TrailParams& p, const int* info, cudaStream_t st) {
  constexpr int B = TL::BM;
  int64_t total = 0;
  for (int64_t m = p.m_first; m < p.m_last; ++m) {
    const int dev = (int)(m % p.D);
    if (dev < p.dev0 || dev >= p.dev0 + p.nloc) continue;
    const int64_t rows = p.N - m * p.T, tc = std::min(p.T, rows);
    const int64_t nrb = (rows + B - 1) / B, ncb = (tc + B - 1) / B;
    total += nrb <= ncb ? nrb * (nrb + 1) / 2 : ncb * (ncb + 1) / 2 + (nrb - ncb) * ncb;
  }
  if (total == 0) return;
  constexpr size_t smem = gemm_smem_bytes<TL, Traits<S>::cplx, CP>();
  auto kern = trail_kernel<S, TL, CP>;
  set_smem(kern, smem);
  int per_sm = 0;
  BCMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TL::THREADS, smem));
  per_sm = std::max(per_sm, 1);
  int64_t grid = std::min<int64_t>(total, (int64_t)num_sms() * per_sm);
  if (p.max_ctas > 0) grid = std::min<int64_t>(grid, p.max_ctas);
  kern<<<(unsigned)grid, TL::THREADS, smem, st>>>(p, info);
  BCMG_CHECK_LAUNCH();
}

// ============================================================== TMA tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    BCMG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) throw Error(CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// 2D map over a column-major double matrix (rows contiguous), box {box_rows, box_cols}.
static CUtensorMap make_map(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows, int box_cols) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

static bool tma_ok(const void* p, int64_t ld) { return aligned16(p) && ld % 2 == 0 && ld < ((int64_t)1 << 36); }

// 128x64 tiles, 8 warps, 2-stage ring, two CTAs per SM: the two co-resident
// CTAs drift apart, so one CTA's epilogue overlaps the other's DMMAs.
using TileTrail2 = Tile<128, 64, 32, 32, 32, 2, true>;

template <class TL>
static void launch_trail_tma_t(const TrailParams& p, const int* info, cudaStream_t st) {
  static_assert(TL::BM / 2 >= TL::BN || !std::is_same_v<TL, TileTrail2>, "complex embedding needs BM/2 >= BN");
  using TZC = Trap<(TL::BM / 2 >= TL::BN ? TL::BM / 2 : TL::BN), TL::BN>;
  int64_t total = 0;
  for (int64_t m = p.m_first; m < p.m_last; ++m) {
    const int dev = (int)(m % p.D);
    if (dev < p.dev0 || dev >= p.dev0 + p.nloc) continue;
    const int64_t rows = p.N - m * p.T, tc = std::min(p.T, rows);
    total += p.cplx ? TZC::count(rows, tc) : Trap<TL::BM, TL::BN>::count(rows, tc);
  }
  if (total == 0) return;
  const int64_t prow = p.N - p.prow0;
  // complex: A = [P | -iP] read as a (2 rows) x (2K) real matrix, B = planar [Re P | Im P]
  const CUtensorMap mapA = p.cplx ? make_map(p.P, 2 * prow, 2 * p.K, 2 * p.ldp, TL::LDA, TL::BK)
                                  : make_map(p.P, prow, p.K, p.ldp, TL::LDA, TL::BK);
  const CUtensorMap mapB = p.cplx ? make_map(p.PB, prow, 2 * p.K, p.ldp, TL::LDB, TL::BK)
                                  : make_map(p.P, prow, p.K, p.ldp, TL::LDB, TL::BK);
  constexpr size_t smem = tma_smem_bytes<TL>();
  // BCMG_TRAIL_VARIANT: 1 (default) consumers decode their own items (a
  // 24-byte stack frame: the epilogue's C pointer / bounds spill to L1);
  // 0 items published in the shared-memory ring and read by the epilogue in
  // place (no frame); 2 ring + register copy.  Measured at config 3
  // (profiles/r02_trail_variants_ab.jsonl): 34.27 / 33.44 / 34.13 TF/s -- the
  // spill-free epilogue's shared-memory reads cost more than the spills.
  static const int variant = [] {
    const char* e = getenv("BCMG_TRAIL_VARIANT");
    return e ? atoi(e) : 1;
  }();
  auto kern = variant == 1 ? trail_tma_kernel_v1<TL> : variant == 2 ? trail_tma_kernel<TL, true> : trail_tma_kernel<TL>;
  set_smem(kern, smem);
  int per_sm = 1;
  BCMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TL::THREADS, smem));
  per_sm = std::max(per_sm, 1);
  const int sms = p.max_ctas > 0 ? std::min(p.max_ctas, num_sms()) : num_sms();
  const int64_t grid = std::min<int64_t>(total, (int64_t)sms * per_sm);
  TrailParams q = p;
  q.stagger_ns = 0;
  if (per_sm >= 2 && total >= 8 * grid) {
    // half an item at ~85% of the per-CTA DMMA rate (37 TF/s over 2 CTAs per SM)
    const double item_flops = 2.0 * TL::BM * TL::BN * (double)p.K * (p.cplx ? 2 : 1);
    q.stagger_ns = (long long)(0.5 * item_flops / (0.85 * 37e12 / (num_sms() * per_sm)) * 1e9);
    if (const char* e = getenv("BCMG_STAGGER")) q.stagger_ns = atoi(e) ? q.stagger_ns : 0;
  }
  kern<<<(unsigned)grid, TL::THREADS, smem, st>>>(mapA, mapB, q, info);
  BCMG_CHECK_LAUNCH();
}

static int trail_tile_choice() {
  static const int v = [] {
    const char* e = getenv("BCMG_TRAIL_TILE");
    return e ? atoi(e) : 2;
  }();
  return v;
}

static void launch_trail_tma(const TrailParams& p, const int* info, cudaStream_t st) {
  if (trail_tile_choice() == 1 && !p.cplx) return launch_trail_tma_t<TileBig>(p, info, st);
  launch_trail_tma_t<TileTrail2>(p, info, st);
}

// complex128 trailing updates through the real TMA kernel (TrailParams::cplx).
// TMA box starts must be 16-byte aligned: the planar operand's row offsets are
// multiples of T (even T), and its ld (= panel rows) must be even.
// complex64 uses the tcgen05 3xTF32 kernel the same way (16-byte box starts: T and
// the panel height multiples of 4 floats).
bool complex_embed_ok(int dt, int64_t panel_rows, int64_t T) {
  if (getenv("BCMG_NO_CPLX_EMBED")) return false;
  if (dt == C128) return use_tma() && panel_rows % 2 == 0 && T % 2 == 0;
  if (dt == C64) return use_tc() && panel_rows % 4 == 0 && T % 4 == 0;
  return false;
}

// [P | -iP] and planar [Re P | Im P] from the complex panel P (rows x K, ld rows)
template <class C, class R>
__global__ void expand_panel_kernel(C* P, R* PB, int64_t rows, int64_t K) {
  const int64_t total = rows * K;
  C* Q = P + total;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const C v = P[idx];
    C q;
    q.x = v.y;
    q.y = -v.x;
    Q[idx] = q;
    PB[idx] = v.x;
    PB[idx + total] = v.y;
  }
}

void expand_panel(int dt, void* P, void* PB, int64_t rows, int64_t K, cudaStream_t st) {
  if (rows <= 0 || K <= 0) return;
  if (dt == C128)
    expand_panel_kernel<<<ew_grid(rows * K), 256, 0, st>>>(static_cast<double2*>(P), static_cast<double*>(PB), rows,
                                                           K);
  else
    expand_panel_kernel<<<ew_grid(rows * K), 256, 0, st>>>(static_cast<float2*>(P), static_cast<float*>(PB), rows, K);
  BCMG_CHECK_LAUNCH();
}

// TBK: B is k-contiguous (Bhat(n, k) = B[k + n*ld]); its box is {LDT k, BN rows}
// (4 k columns of over-fetch, zero past K) for the [BN][LDT] tile of mma_slice_tbk
template <class TL, bool TBK = false>
static void launch_gemm_tma_t(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B,
                              const Epilogue& ep, const int* info, cudaStream_t st) {
  const CUtensorMap ma = make_map(A.ptr, M, K, A.ld, TL::LDA, TL::BK);
  const CUtensorMap mb = TBK ? make_map(B.ptr, K, N, B.ld, TL::LDT, TL::BN) : make_map(B.ptr, N, K, B.ld, TL::LDB, TL::BK);
  constexpr size_t smem = tma_smem_bytes<TL, TBK>();
  auto kern = gemm_tma_kernel<TL, TBK>;
  set_smem(kern, smem);
  int per_sm = 1;
  BCMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TL::THREADS, smem));
  const int64_t blocks = ((M + TL::BM - 1) / TL::BM) * ((N + TL::BN - 1) / TL::BN);
  const int64_t grid = std::min<int64_t>(blocks, (int64_t)num_sms() * std::max(per_sm, 1));
  kern<<<(unsigned)grid, TL::THREADS, smem, st>>>(ma, mb, M, N, K, ep, info);
  BCMG_CHECK_LAUNCH();
}

static int trail_tile_choice();
using TileTrail2 = Tile<128, 64, 32, 32, 32, 2, true>;

static void launch_gemm_tma(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                            const int* info, cudaStream_t st) {
  if (trail_tile_choice() == 1) return launch_gemm_tma_t<TileBig>(M, N, K, A, B, ep, info, st);
  launch_gemm_tma_t<TileTrail2>(M, N, K, A, B, ep, info, st);
}

// ---------------------------------------------------------------- complex GEMM by real embedding
// C = alpha*Ahat*Bhat^T + beta*C (complex) as ONE real GEMM on the tensor-core
// kernels (FP64 TMA + DMMA for complex128, tcgen05 3xTF32 for complex64):
//   Atilde = [Ahat | -i Ahat]          (M x 2K complex = 2M x 2K real, re/im interleaved rows)
//   X      = [Re Bhat | -Im Bhat]      (N x 2K real, planar)
//   Ctilde (2M x N real, interleaved re/im rows = C's storage) = Atilde X^T:
//     row 2r:   sum Re A Re B - Im A Im B = Re (A B)_rc
//     row 2r+1: sum Im A Re B + Re A Im B = Im (A B)_rc
// The gather kernel materialises either operand from any Operand view
// (transposed / conjugated) through a 32x32 shared-memory tile.
// With B-hat k-contiguous and unconjugated (complex128), B-hat's own storage is
// the real operand: Bhat(n, k) -> doubles (Re, Im) at k' = 2k, 2k+1 of a real
// N x 2K k-contiguous matrix (ld 2 ld).  A is then embedded with interleaved
// columns, Atilde(:, 2k) = A(:, k), Atilde(:, 2k+1) = i A(:, k):
//     sum_k A(r,k) Re B(c,k) + i A(r,k) Im B(c,k) = (A B^T)(r,c)
// so only the (small) A side is gathered; the GEMM reads B in place
// (launch_gemm_tma_t<TL, true>).
template <class C, class R>
__global__ void embed_gather_kernel(Operand X, int64_t I, int64_t kn, C* outc, R* outp, int64_t ldo, int inter) {
  // logical element (i, kk) of X, kk < kn; outc: complex Atilde (ld ldo, cols kk and kn + kk,
  // or 2kk and 2kk + 1 when inter), outp: planar X (ld ldo, cols kk and kn + kk)
  __shared__ C t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  const C* base = static_cast<const C*>(X.ptr);
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    // coalesced along the storage-contiguous index
    const int64_t i = X.trans ? i0 + y : i0 + threadIdx.x, kk = X.trans ? c0 + threadIdx.x : c0 + y;
    C v;
    v.x = 0;
    v.y = 0;
    if (i < I && kk < kn) {
      v = X.trans ? base[kk + i * X.ld] : base[i + kk * X.ld];
      if (X.conj) v.y = -v.y;
    }
    if (X.trans) t[threadIdx.x][y] = v; else t[y][threadIdx.x] = v;  // t[kk][i]
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, kk = c0 + y;
    if (i >= I || kk >= kn) continue;
    const C v = t[y][threadIdx.x];
    if (outc && inter) {
      C q;
      q.x = -v.y;
      q.y = v.x;
      outc[i + 2 * kk * ldo] = v;
      outc[i + (2 * kk + 1) * ldo] = q;
    } else if (outc) {
      C q;
      q.x = v.y;
      q.y = -v.x;
      outc[i + kk * ldo] = v;
      outc[i + (kn + kk) * ldo] = q;
    } else {
      outp[i + kk * ldo] = v.x;
      outp[i + (kn + kk) * ldo] = -v.y;
    }
  }
}

template <class C, class R>
static void embed_gather(const Operand& X, int64_t I, int64_t kn, C* outc, R* outp, int64_t ldo, cudaStream_t st,
                         int inter = 0) {
  dim3 grid((unsigned)((I + 31) / 32), (unsigned)((kn + 31) / 32)), block(32, 8);
  embed_gather_kernel<C, R><<<grid, block, 0, st>>>(X, I, kn, outc, outp, ldo, inter);
  BCMG_CHECK_LAUNCH();
}

// complex128 B-hat usable in place by the k-contiguous TMA GEMM (see embed_gather_kernel)
static bool native_b(const Operand& B) {
  static const bool off = getenv("BCMG_CPLX_NATIVE_B") && atoi(getenv("BCMG_CPLX_NATIVE_B")) == 0;
  return !off && B.trans && !B.conj && !B.mask && aligned16(B.ptr) && B.ld < ((int64_t)1 << 35);
}

size_t gemm_cplx_embed_bytes(int dt, int64_t M, int64_t N, int64_t K) {
  return (size_t)(2 * M + N) * K * (dt == C64 ? 8 : 16);
}

bool gemm_cplx_embed(int dt, int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                     void* scratch, size_t scratch_bytes, const int* info, cudaStream_t st, bool always) {
  if (getenv("BCMG_NO_CPLX_EMBED") || A.mask || B.mask || ep.lower_only) return false;
  if (dt != C128 && dt != C64) return false;
  if (dt == C128 ? !use_tma() : !use_tc()) return false;
  const int64_t align = dt == C128 ? 2 : 4;  // real ld and box starts: 16 bytes
  if (M <= 0 || N <= 0 || K <= 0 || N % align || (2 * M) % align || !aligned16(ep.C) || !aligned16(scratch))
    return false;
  if (scratch_bytes < gemm_cplx_embed_bytes(dt, M, N, K)) return false;
  // the tcgen05 tile's minimum shape (N only when the caller allows a shape-dependent choice)
  if (dt == C64 && (2 * M < 256 || (!always && N < 64))) return false;
  if (dt == C64 && ep.nfan && !use_presplit()) return false;  // the inline-split kernel has no fan-out
  // enough real blocks to fill the GPU (smaller GEMMs stay on the complex kernels), unless
  // the caller needs a shape-independent choice (bit-identical results across device counts)
  const int64_t blocks = ((2 * M + TileTrail2::BM - 1) / TileTrail2::BM) * ((N + TileTrail2::BN - 1) / TileTrail2::BN);
  if (!always && blocks < num_sms()) return false;
  if (dt == C128 && native_b(B)) {  // B read in place, A gathered with interleaved columns
    double2* at = static_cast<double2*>(scratch);
    embed_gather<double2, double>(A, M, K, at, nullptr, M, st, 1);
    Epilogue er = ep;
    er.ldc = 2 * ep.ldc;
    launch_gemm_tma_t<TileTrail2, true>(2 * M, N, 2 * K, Operand{at, 2 * M, 0, 0, 0, 0},
                                        Operand{B.ptr, 2 * B.ld, 1, 0, 0, 0}, er, info, st);
  } else if (dt == C128) {
    double2* at = static_cast<double2*>(scratch);              // M x 2K complex, ld M
    double* xp = reinterpret_cast<double*>(at + 2 * M * K);    // N x 2K real, ld N
    embed_gather<double2, double>(A, M, K, at, nullptr, M, st);
    embed_gather<double2, double>(B, N, K, nullptr, xp, N, st);
    Epilogue er = ep;  // real view of C (and of its fan-out copies)
    er.ldc = 2 * ep.ldc;
    launch_gemm_tma_t<TileTrail2>(2 * M, N, 2 * K, Operand{at, 2 * M, 0, 0, 0, 0}, Operand{xp, N, 0, 0, 0, 0}, er,
                                  info, st);
  } else {
    float2* at = static_cast<float2*>(scratch);
    float* xp = reinterpret_cast<float*>(at + 2 * M * K);
    embed_gather<float2, float>(A, M, K, at, nullptr, M, st);
    embed_gather<float2, float>(B, N, K, nullptr, xp, N, st);
    if (use_presplit()) {  // tf32 hi / lo planes of both embedded operands, then the pre-split kernel
      const int64_t kp = split_ld(2 * K);
      float* s = split_scratch(st, (size_t)2 * (2 * M + N) * kp * 4);
      float *ah = s, *al = s + 2 * M * kp, *bh = al + 2 * M * kp, *bl = bh + N * kp;
      split_tf32(0, at, 2 * M, 2 * M, 2 * K, 2 * K, ah, al, kp, st);
      split_tf32(0, xp, N, N, 2 * K, 2 * K, bh, bl, kp, st);
      tck_gemm(2 * M, N, 2 * K, ah, al, bh, bl, kp, static_cast<float*>(ep.C), 2 * ep.ldc, (float)ep.alpha,
               (float)ep.beta, info, st, &ep);
    } else {
      launch_tc3_gemm(2 * M, N, 2 * K, Operand{at, 2 * M, 0, 0, 0, 0}, Operand{xp, N, 0, 0, 0, 0},
                      Epilogue{ep.C, 2 * ep.ldc, ep.alpha, ep.beta, 0, 0}, info, st);
    }
  }
  return true;
}

// complex128: C_g (+)= alpha A B_g^T for several groups sharing A, each with its
// own C (potri's W sweep: one product per local device into its own shard).
// A is gathered once as [A | -iA]; each B_g planar [Re B | -Im B]; ONE launch
// of the multi-map TMA kernel.  Per element the same tile kernel, K order and
// epilogue as gemm_cplx_embed, so the same bits.  False when a group would not
// take the embedding on its own (the caller then runs the groups one by one).
bool gemm_cplx_embed_multi(int dt, int64_t M, int64_t K, const Operand& A, const Operand* Bs, const int64_t* ncols,
                           void* const* Cs, int ngroups, const Epilogue& ep, void* scratch, size_t scratch_bytes,
                           cudaStream_t st) {
  if (dt != C128 || getenv("BCMG_NO_CPLX_EMBED") || !use_tma() || A.mask || ep.lower_only || ep.nfan) return false;
  if (ngroups < 1 || ngroups > BMaps::MAX || M <= 0 || K <= 0 || (2 * M) % 2 || !aligned16(scratch)) return false;
  int64_t total = 0;
  for (int i = 0; i < ngroups; ++i) {
    if (Bs[i].mask || native_b(Bs[i]) || ncols[i] <= 0 || ncols[i] % 2 || !aligned16(Cs[i])) return false;
    total += ncols[i];
  }
  if (scratch_bytes < gemm_cplx_embed_bytes(dt, M, total, K)) return false;
  using TL = TileTrail2;
  double2* at = static_cast<double2*>(scratch);              // M x 2K complex, ld M
  double* xp = reinterpret_cast<double*>(at + 2 * M * K);    // per group: N_g x 2K real, ld N_g
  embed_gather<double2, double>(A, M, K, at, nullptr, M, st);
  BMaps bm;
  std::memset(&bm, 0, sizeof(bm));
  int64_t nblk = 0, off = 0;
  for (int i = 0; i < ngroups; ++i) {
    double* xg = xp + off;
    embed_gather<double2, double>(Bs[i], ncols[i], K, nullptr, xg, ncols[i], st);
    bm.m[i] = make_map(xg, ncols[i], 2 * K, ncols[i], TL::LDB, TL::BK);
    bm.col0[i + 1] = bm.col0[i] + ncols[i];
    bm.cbase[i] = static_cast<char*>(Cs[i]);
    off += ncols[i] * 2 * K;
    nblk += (ncols[i] + TL::BN - 1) / TL::BN;
  }
  bm.n = ngroups;
  Epilogue er = ep;
  er.ldc = 2 * ep.ldc;
  const CUtensorMap ma = make_map(at, 2 * M, 2 * K, 2 * M, TL::LDA, TL::BK);
  constexpr size_t smem = tma_smem_bytes<TL, false>();
  auto kern = gemm_tma_grouped_kernel<TL, false>;
  set_smem(kern, smem);
  int per_sm = 1;
  BCMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TL::THREADS, smem));
  const int64_t blocks = ((2 * M + TL::BM - 1) / TL::BM) * nblk;
  const int64_t grid = std::min<int64_t>(blocks, (int64_t)num_sms() * std::max(per_sm, 1));
  kern<<<(unsigned)grid, TL::THREADS, smem, st>>>(ma, bm, 2 * M, 2 * K, er, nullptr);
  BCMG_CHECK_LAUNCH();
  return true;
}

bool gemm_cplx_embed_grouped(int dt, int64_t M, int64_t K, const Operand& A, const Operand* Bs, const int64_t* ncols,
                             int ngroups, const Epilogue& ep, void* scratch, size_t scratch_bytes, int64_t chunk,
                             cudaStream_t st) {
  if (getenv("BCMG_NO_CPLX_EMBED") || A.mask || ep.lower_only || ep.nfan) return false;
  if (dt != C128 && dt != C64) return false;
  if (dt == C128 ? !use_tma() : !(use_tc() && use_presplit())) return false;
  const int64_t align = dt == C128 ? 2 : 4;
  int64_t total = 0;
  for (int i = 0; i < ngroups; ++i) {
    if (Bs[i].mask || ncols[i] % align) return false;
    total += ncols[i];
  }
  if (M <= 0 || K <= 0 || total <= 0 || chunk < 64 || chunk % align || (2 * M) % align) return false;
  if (!aligned16(ep.C) || !aligned16(scratch) || scratch_bytes < gemm_cplx_embed_bytes(dt, M, chunk, K)) return false;
  if (dt == C64 && 2 * M < 256) return false;  // the tcgen05 tile's minimum shape
  const size_t csz = dt == C128 ? 16 : 8;
  bool native = dt == C128;
  for (int i = 0; i < ngroups && native; ++i) native = native_b(Bs[i]);
  if (native) {  // A gathered once (interleaved columns), one GEMM per group reading B in place
    double2* at = static_cast<double2*>(scratch);
    embed_gather<double2, double>(A, M, K, at, nullptr, M, st, 1);
    using TL = TileTrail2;
    BMaps bm;
    std::memset(&bm, 0, sizeof(bm));
    if (ngroups <= BMaps::MAX) {  // one launch over every group's columns
      int64_t nblk = 0;
      for (int i = 0; i < ngroups; ++i) {
        if (ncols[i] == 0) continue;
        bm.m[bm.n] = make_map(Bs[i].ptr, 2 * K, ncols[i], 2 * Bs[i].ld, TL::LDT, TL::BN);
        bm.col0[bm.n + 1] = bm.col0[bm.n] + ncols[i];
        ++bm.n;
        nblk += (ncols[i] + TL::BN - 1) / TL::BN;
      }
      Epilogue er = ep;
      er.ldc = 2 * ep.ldc;
      const CUtensorMap ma = make_map(at, 2 * M, 2 * K, 2 * M, TL::LDA, TL::BK);
      constexpr size_t smem = tma_smem_bytes<TL, true>();
      auto kern = gemm_tma_grouped_kernel<TL, true>;
      set_smem(kern, smem);
      int per_sm = 1;
      BCMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TL::THREADS, smem));
      const int64_t blocks = ((2 * M + TL::BM - 1) / TL::BM) * nblk;
      const int64_t grid = std::min<int64_t>(blocks, (int64_t)num_sms() * std::max(per_sm, 1));
      if (grid > 0) kern<<<(unsigned)grid, TL::THREADS, smem, st>>>(ma, bm, 2 * M, 2 * K, er, nullptr);
      BCMG_CHECK_LAUNCH();
      return true;
    }
    int64_t g0 = 0;
    for (int i = 0; i < ngroups; ++i) {
      if (ncols[i] == 0) continue;
      Epilogue er = ep;
      er.C = static_cast<char*>(ep.C) + g0 * ep.ldc * (int64_t)csz;
      er.ldc = 2 * ep.ldc;
      launch_gemm_tma_t<TL, true>(2 * M, ncols[i], 2 * K, Operand{at, 2 * M, 0, 0, 0, 0},
                                  Operand{Bs[i].ptr, 2 * Bs[i].ld, 1, 0, 0, 0}, er, nullptr, st);
      g0 += ncols[i];
    }
    return true;
  }
  // A (M x K, op(A)) gathered ONCE as [A | -iA] (M x 2K complex), then chunk
  // after chunk of the concatenated groups' columns as planar [Re B | -Im B]
  // and one real GEMM per chunk into the concatenated output columns
  char* at = static_cast<char*>(scratch);
  char* xp = at + (size_t)2 * M * K * csz;
  if (dt == C128) embed_gather<double2, double>(A, M, K, reinterpret_cast<double2*>(at), nullptr, M, st);
  else embed_gather<float2, float>(A, M, K, reinterpret_cast<float2*>(at), nullptr, M, st);
  float *ah = nullptr, *al = nullptr, *bh = nullptr, *bl = nullptr;
  const int64_t kp = split_ld(2 * K);
  if (dt == C64) {  // tf32 planes: A split once, B per chunk
    float* sp = split_scratch(st, (size_t)2 * (2 * M + chunk) * kp * 4);
    ah = sp;
    al = sp + 2 * M * kp;
    bh = al + 2 * M * kp;
    bl = bh + chunk * kp;
    split_tf32(0, at, 2 * M, 2 * M, 2 * K, 2 * K, ah, al, kp, st);
  }
  int gi = 0;
  int64_t goff = 0;  // column offset inside group gi
  for (int64_t g0 = 0; g0 < total; g0 += chunk) {
    const int64_t cn = std::min(chunk, total - g0);
    for (int64_t r = 0; r < cn;) {  // gather the chunk's columns group by group
      while (goff >= ncols[gi]) {
        goff = 0;
        ++gi;
      }
      const int64_t take = std::min(cn - r, ncols[gi] - goff);
      Operand b = Bs[gi];
      // logical row i of B-hat is stored column i (trans) or row i
      b.ptr = static_cast<const char*>(b.ptr) + (b.trans ? goff * b.ld : goff) * (int64_t)csz;
      if (dt == C128) embed_gather<double2, double>(b, take, K, nullptr, reinterpret_cast<double*>(xp) + r, cn, st);
      else embed_gather<float2, float>(b, take, K, nullptr, reinterpret_cast<float*>(xp) + r, cn, st);
      r += take;
      goff += take;
    }
    Epilogue er = ep;
    er.C = static_cast<char*>(ep.C) + g0 * ep.ldc * (int64_t)csz;
    if (dt == C128) {
      er.ldc = 2 * ep.ldc;
      launch_gemm_tma_t<TileTrail2>(2 * M, cn, 2 * K, Operand{at, 2 * M, 0, 0, 0, 0}, Operand{xp, cn, 0, 0, 0, 0}, er,
                                    nullptr, st);
    } else {
      split_tf32(0, xp, cn, cn, 2 * K, 2 * K, bh, bl, kp, st);
      tck_gemm(2 * M, cn, 2 * K, ah, al, bh, bl, kp, static_cast<float*>(er.C), 2 * ep.ldc, (float)ep.alpha,
               (float)ep.beta, nullptr, st, &er);
    }
  }
  return true;
}

static bool use_tma() {
  static const bool v = [] {
    const char* e = getenv("BCMG_NO_TMA");
    return !(e && atoi(e));
  }();
  return v;
}

// ============================================================== tcgen05 3xTF32 (float32)
static CUtensorMap make_map_f32_sw128(const void* base, int64_t rows, int64_t cols, int64_t ld) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)tc::BK};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(CUDA, "cuTensorMapEncodeTiled (f32 sw128) failed (" + std::to_string((int)r) + ")");
  return m;
}

static bool tc_ok(const void* p, int64_t ld) { return aligned16(p) && ld % 4 == 0; }

static bool use_tc() {
  static const bool v = [] {
    const char* e = getenv("BCMG_NO_TCGEN05");
    return !(e && atoi(e));
  }();
  return v;
}

static void launch_tc3_gemm(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                            const int* info, cudaStream_t st) {
  const CUtensorMap ma = make_map_f32_sw128(A.ptr, M, K, A.ld);
  const CUtensorMap mb = make_map_f32_sw128(B.ptr, N, K, B.ld);
  set_smem(tc3_gemm_kernel, tc::SMEM_BYTES);
  const int64_t blocks = ((M + tc::BM - 1) / tc::BM) * ((N + tc::BN - 1) / tc::BN);
  const int64_t grid = std::min<int64_t>(blocks, (int64_t)num_sms());
  tc3_gemm_kernel<<<(unsigned)grid, tc::THREADS, tc::SMEM_BYTES, st>>>(
      ma, mb, M, N, K, static_cast<float*>(ep.C), ep.ldc, (float)ep.alpha, (float)ep.beta, info);
  BCMG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- pre-split tf32 planes
// X (rows x Kx, logical) -> hi = rna_tf32(x), lo = x - hi, stored K-major
// (row-major, ld kp >= Kx, columns [Kx, kp) zero) for tck_* kernels.
//   mode 0: real float, X(m, k) = src[m + k*ld] (column-major)
//   mode 1: complex64 embedding A = [P | -iP] as a (2R) x (2Kc) real matrix
//           (re / im interleaved rows), P complex R x Kc, ld ld (complex)
//   mode 2: complex64 planar B = [Re P | Im P] (R x 2Kc)
template <int MODE>
__global__ void split_tf32_kernel(const float* __restrict__ src, int64_t ld, int64_t rows, int64_t Kx, int64_t kc,
                                  float* __restrict__ hi, float* __restrict__ lo, int64_t kp, int64_t kw) {
  __shared__ float t[32][33];
  const int64_t m0 = (int64_t)blockIdx.x * 32, k0 = (int64_t)blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t m = m0 + threadIdx.x, k = k0 + y;  // coalesced along m (column-major source)
    float v = 0.f;
    if (m < rows && k < Kx) {
      if (MODE == 0) {
        v = src[m + k * ld];
      } else if (MODE == 3) {
        v = src[k + m * ld];  // transposed view (k contiguous)
      } else if (MODE == 1) {
        const int64_t kk = k < kc ? k : k - kc, r = m >> 1;
        const float* e = src + 2 * (r + kk * ld);
        if (k < kc) v = e[m & 1];
        else v = (m & 1) ? -e[0] : e[1];  // -i P = (im, -re)
      } else {
        const int64_t kk = k < kc ? k : k - kc;
        v = src[2 * (m + kk * ld) + (k < kc ? 0 : 1)];
      }
    }
    t[y][threadIdx.x] = v;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t m = m0 + y, k = k0 + threadIdx.x;  // coalesced along k (row-major planes)
    if (m >= rows || k >= kw) continue;
    const float x = t[threadIdx.x][y];
    const float h = tc::tf32_rna(x);
    hi[m * kp + k] = h;
    lo[m * kp + k] = x - h;
  }
}

int64_t split_ld(int64_t kx) { return (kx + 3) / 4 * 4; }

void split_tf32(int mode, const void* src, int64_t ld, int64_t rows, int64_t Kx, int64_t kc, float* hi, float* lo,
                int64_t kp, cudaStream_t st, int64_t kw) {
  if (kw < 0) kw = kp;
  if (rows <= 0 || kw <= 0) return;
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((kw + 31) / 32)), block(32, 8);
  const float* s = static_cast<const float*>(src);
  if (mode == 0) split_tf32_kernel<0><<<grid, block, 0, st>>>(s, ld, rows, Kx, kc, hi, lo, kp, kw);
  else if (mode == 1) split_tf32_kernel<1><<<grid, block, 0, st>>>(s, ld, rows, Kx, kc, hi, lo, kp, kw);
  else if (mode == 2) split_tf32_kernel<2><<<grid, block, 0, st>>>(s, ld, rows, Kx, kc, hi, lo, kp, kw);
  else split_tf32_kernel<3><<<grid, block, 0, st>>>(s, ld, rows, Kx, kc, hi, lo, kp, kw);
  BCMG_CHECK_LAUNCH();
}

// Narrow tiles on the tcgen05 path: the trailing update is HBM-bound (each
// pass reads and writes the whole trailing trapezoid for only K = T of
// work), so potrf applies the panels in pairs (K = 2T) and halves the passes.
bool pair_panels(int dt, int64_t T) {
  static const int v = [] {
    const char* e = getenv("BCMG_PAIR_PANELS");
    return e && *e ? atoi(e) : 2;
  }();
  // 2 (default): T_A <= 512; 1: T_A <= 256 (N=65536, 8 devices, T_A=512, same box, two
  // rounds: f32 191.0 / 193.0 -> 198.8 / 201.0, c64 215.4 / 215.2 -> 215.2 / 216.0 TFLOP/s)
  return v && (dt == R32 || dt == C64) && tc_presplit_enabled() && T <= (v >= 3 ? 1024 : v >= 2 ? 512 : 256) &&
         T % 32 == 0;
}

// K-major plane map: dims {kp, rows}, box {32 k, 128 rows}, SWIZZLE_128B (the
// canonical K-major layout of the UMMA descriptors).
static CUtensorMap make_map_kmajor(const float* base, int64_t rows, int64_t kp, int box_rows = tc::BM) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kp * 4};
  cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(CUDA, "cuTensorMapEncodeTiled (k-major) failed (" + std::to_string((int)r) + ")");
  return m;
}

bool tc_presplit_enabled();
static bool use_presplit() {
  static const bool v = [] {
    const char* e = getenv("BCMG_TC_INLINE_SPLIT");
    return !(e && atoi(e));
  }();
  return v;
}

bool tc_presplit_enabled() { return use_tc() && use_presplit(); }

// BCMG_TRAIL_BAND: owned tile columns (units) per band of the tcgen05 trailing update
static int trail_band() {
  static const int band = [] {
    const char* e = getenv("BCMG_TRAIL_BAND");
    return e && *e ? std::max(0, atoi(e)) : 8;
  }();
  return band;
}

static int tck_width(int64_t n) {
  static const int forced = [] {
    const char* e = getenv("BCMG_TCK_N");
    return e ? atoi(e) : 0;
  }();
  if (forced == 128 || forced == 256) return forced;
  return n >= 256 ? 256 : 128;
}

template <int BNT, int CL = 1>
static void launch_tck_trail_t(const TrailParams& p, const int* info, cudaStream_t st) {
  constexpr int64_t BMX = (CL == 1 || CL == 4 ? 1 : 2) * tc::BM;
  using TZ = TrapR<BMX, BNT>;
  using TZC = TrapR<BMX / 2, BNT>;
  int64_t total = 0;
  for (int64_t m = p.m_first; m < p.m_last; ++m) {
    const int dev = (int)(m % p.D);
    if (dev < p.dev0 || dev >= p.dev0 + p.nloc) continue;
    const int64_t rows = p.N - m * p.T, tcm = std::min(p.T, rows);
    total += p.cplx ? TZC::count(rows, tcm) : TZ::count(rows, tcm);
  }
  if (total == 0) return;
  TrailParams q = p;
  {
    const int band = trail_band();
    const int64_t rb = p.cplx ? BMX / 2 : BMX;
    const int64_t cpu = (CL == 3 || CL == 6 || CL == 7) && p.cpu > 1 ? p.cpu : 1;  // tile columns per unit
    const bool cols = p.T <= BNT && (cpu * p.T) % rb == 0 && (p.nloc == 1 || p.nloc == p.D);
    const bool blocks = p.T > BNT && p.T % BNT == 0 && p.N % p.T == 0 && p.nloc == p.D;
    q.band = cols || blocks ? band : 0;
  }
  const int64_t prow = p.N - p.prow0, arows = p.cplx ? 2 * prow : prow;
  const CUtensorMap ah = make_map_kmajor(p.split[0], arows, p.split_ld[0]);
  const CUtensorMap al = make_map_kmajor(p.split[1], arows, p.split_ld[0]);
  constexpr int BROWS = (CL == 2 || CL == 3 || CL == 6 || CL == 7) ? BNT / 2 : BNT;  // CTA pairs load half the B tile each
  const CUtensorMap bh = make_map_kmajor(p.split[2], prow, p.split_ld[1], BROWS);
  const CUtensorMap bl = make_map_kmajor(p.split[3], prow, p.split_ld[1], BROWS);
  constexpr size_t smem = CL == 3   ? tck::Pair::SMEM_BYTES
                          : CL == 6 ? tck::PairT<1>::SMEM_BYTES
                          : CL == 7 ? tck::PairT<2>::SMEM_BYTES
                          : CL == 4 ? tck::Epi::SMEM_BYTES
                                    : tck::Cfg<BNT>::SMEM_BYTES;
  auto kern = tck_trail_kernel<BNT, CL>;
  set_smem(kern, smem);
  const int sms = p.max_ctas > 0 ? std::min(p.max_ctas, num_sms()) : num_sms();
  tck::CMaps cmaps;
  std::memset(&cmaps, 0, sizeof(cmaps));
  if constexpr (CL == 4 || CL == 6 || CL == 7) {  // the TMA epilogue's C maps: each local shard as (rows, its columns)
    static const int mode = [] {
      const char* e = getenv("BCMG_EPI_MODE");
      return e && *e ? atoi(e) : 0;
    }();
    cmaps.mode = mode;
    const auto counts = column_counts(p.N, p.T, p.D);
    const int64_t cx = p.cplx ? 2 : 1;
    for (int i = 0; i < p.nloc; ++i) {
      cuuint64_t dims[2] = {(cuuint64_t)(cx * p.N), (cuuint64_t)counts[p.dev0 + i]};
      cuuint64_t strides[1] = {(cuuint64_t)(cx * p.N) * 4};
      cuuint32_t box[2] = {(cuuint32_t)tc::BM, CL == 7 ? 64u : 128u};  // quarters / halves / tiles
      cuuint32_t es[2] = {1, 1};
      CUresult r = encode_fn()(&cmaps.m[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p.shards[i], dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error(CUDA, "cuTensorMapEncodeTiled (C tile) failed (" + std::to_string((int)r) + ")");
    }
  }
  if constexpr (CL == 1 || CL == 4) {
    const int64_t grid = std::min<int64_t>(total, sms);
    kern<<<(unsigned)grid, tck::THREADS, smem, st>>>(ah, al, bh, bl, q, info, cmaps);
  } else {  // clusters of two CTAs (one per SM of a TPC pair)
    const int64_t pairs = std::min<int64_t>(total, sms / 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * std::max<int64_t>(pairs, 1)));
    cfg.blockDim = dim3(tck::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    BCMG_CUDA(cudaLaunchKernelEx(&cfg, kern, ah, al, bh, bl, q, info, cmaps));
  }
  BCMG_CHECK_LAUNCH();
}

// clusters of two CTAs (one per SM of a TPC pair), `pairs` clusters
static void launch_pair(const void* kern, int64_t pairs, size_t smem, cudaStream_t st, void** args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * std::max<int64_t>(pairs, 1)));
  cfg.blockDim = dim3(tck::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BCMG_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
  BCMG_CHECK_LAUNCH();
}

// BCMG_TCK_CLUSTER, the 256-wide trailing update: 0 one CTA per 128 x 256 tile;
// 1 CTA pairs sharing the B tile through TMA multicast (tck_loop CL = 2);
// 2 (default) CTA pairs on 256 x 256 tiles with the 2-SM UMMA (tck_loop_pair)
static int tck_cluster() {
  static const int v = [] {
    const char* e = getenv("BCMG_TCK_CLUSTER");
    return e && *e ? atoi(e) : 2;
  }();
  return v;
}

// BCMG_TCK_EPI: T_A = 128 trailing updates on whole 128 x 128 tiles use the
// TMA read-modify-write epilogue (tck_loop_epi). Unset: real dtypes only
// (float32 N = 65536: 101 -> 114 TFLOP/s; complex64 150 -> 147, so off);
// 0 never; 1 real and complex. Same bits either way.
static bool tck_epi(bool cplx) {
  static const int v = [] {
    const char* e = getenv("BCMG_TCK_EPI");
    return e && *e ? atoi(e) : -1;
  }();
  return v > 0 || (v < 0 && !cplx);
}

// BCMG_TCK_UNIT2 (default 1): at T_A = 128, where the TMA epilogue is not used
// (complex64 by default), the bulk trailing update runs on the 2-SM pair kernel
// with items of two owned tile columns (one 256 x 256 UMMA tile: 3/4 of the
// shared-memory operand traffic per SM of the 128 x 128 kernel).  Same bits.
// N = 65536, 8 devices: complex64 150.6 -> 170.6 TFLOP/s; float32 117.3 -> 112.6
// (its C read-modify-write per flop is twice complex64's: the TMA epilogue wins)
static bool tck_unit2() {
  static const bool v = [] {
    const char* e = getenv("BCMG_TCK_UNIT2");
    return !(e && *e && atoi(e) == 0);
  }();
  return v;
}

// BCMG_TCK_PAIR_EPI (default 1): at T_A = 128 the bulk update runs on the
// two-column 2-SM pair items of BCMG_TCK_UNIT2 with the TMA read-modify-write
// epilogue in 128-column halves (tck_loop_pair<1>; 3: quarter ring, tck_loop_pair<2>).  Same bits.  N = 65536,
// 8 devices: float32 118.8 -> 139.6 TFLOP/s (trailing update 652 -> 529 ms,
// against the one-CTA TMA-epilogue kernel), complex64 176.7 -> 177.7 (against
// the pair kernel's per-thread epilogue)
// Unset: float32 the quarter ring (3), complex64 the halves (1) -- N=65536 T_A=128,
// same box: f32 159.6 / 163.8, c64 196.1 / 195.6 TFLOP/s (halves / quarters).
static int tck_pair_epi(bool cplx) {
  static const int v = [] {
    const char* e = getenv("BCMG_TCK_PAIR_EPI");
    return e && *e ? atoi(e) : -1;
  }();
  return v >= 0 ? v : cplx ? 1 : 3;
}

static void launch_tck_trail(const TrailParams& p, const int* info, cudaStream_t st) {
  bool unit2 = false;  // at least two owned 128-wide tile columns, pair kernels usable
  if (p.T == 128 && tck_cluster() == 2 && trail_band() > 0 && p.N % p.T == 0 && (p.nloc == 1 || p.nloc == p.D) &&
      p.nloc <= MAX_LOCAL_DEV) {
    const int64_t sc = p.nloc == p.D ? 1 : p.D;
    int64_t cm = p.m_first;
    if (sc > 1) cm += ((p.dev0 - cm % p.D) + p.D) % p.D;
    unit2 = cm + sc < p.m_last;
  }
  TrailParams q = p;
  q.cpu = 2;
  if (unit2 && tck_pair_epi(p.cplx) == 3) return launch_tck_trail_t<256, 7>(q, info, st);
  if (unit2 && tck_pair_epi(p.cplx) > 0) return launch_tck_trail_t<256, 6>(q, info, st);
  const bool epi = tck_width(p.T) == 128 && p.T == 128 && p.N % p.T == 0 && tck_epi(p.cplx) && p.nloc <= MAX_LOCAL_DEV;
  if (epi) return launch_tck_trail_t<128, 4>(p, info, st);
  if (unit2 && tck_unit2()) return launch_tck_trail_t<256, 3>(q, info, st);
  if (tck_width(p.T) == 256) {
    const int c = tck_cluster();
    // whole 256-wide column blocks (T_A a multiple of 256): the TMA epilogue in halves
    if (c == 2 && tck_pair_epi(p.cplx) == 2 && p.T % 256 == 0 && p.N % p.T == 0 && p.nloc <= MAX_LOCAL_DEV)
      return launch_tck_trail_t<256, 6>(p, info, st);
    if (c == 2 && tck_pair_epi(p.cplx) == 4 && p.T % 256 == 0 && p.N % p.T == 0 && p.nloc <= MAX_LOCAL_DEV)
      return launch_tck_trail_t<256, 7>(p, info, st);  // (measurement switch: the quarter ring at T_A >= 256)
    if (c == 2) return launch_tck_trail_t<256, 3>(p, info, st);
    if (c == 1) return launch_tck_trail_t<256, 2>(p, info, st);
    return launch_tck_trail_t<256, 1>(p, info, st);
  }
  launch_tck_trail_t<128>(p, info, st);
}

// C = alpha*A*B^T + beta*C (float32) on pre-split planes Ah/Al (M x kp) and Bh/Bl (N x kp).
static int tck_cluster();
static void launch_pair(const void* kern, int64_t pairs, size_t smem, cudaStream_t st, void** args);

template <int BNT>
static void tck_gemm_t(int64_t M, int64_t N, int64_t K, const float* ah, const float* al, const float* bh,
                       const float* bl, int64_t kp, float* C, int64_t ldc, float alpha, float beta, const int* info,
                       cudaStream_t st, const FloatFan& fan) {
  const CUtensorMap mah = make_map_kmajor(ah, M, kp), mal = make_map_kmajor(al, M, kp);
  if constexpr (BNT == 256) {
    if (fan.n == 0 && M > tc::BM && tck_cluster() == 2) {  // CTA pairs, 2-SM UMMA on 256 x 256 tiles
      const CUtensorMap mbh = make_map_kmajor(bh, N, kp, BNT / 2), mbl = make_map_kmajor(bl, N, kp, BNT / 2);
      auto kern = tck_gemm_kernel<256, 3>;
      set_smem(kern, tck::Pair::SMEM_BYTES);
      const int64_t tiles = ((M + 2 * tc::BM - 1) / (2 * tc::BM)) * ((N + BNT - 1) / BNT);
      void* args[] = {(void*)&mah, (void*)&mal, (void*)&mbh, (void*)&mbl, &M, &N, &K, &C, &ldc, &alpha, &beta,
                      (void*)&info, (void*)&fan};
      launch_pair((const void*)kern, std::min<int64_t>(tiles, num_sms() / 2), tck::Pair::SMEM_BYTES, st, args);
      return;
    }
  }
  const CUtensorMap mbh = make_map_kmajor(bh, N, kp, BNT), mbl = make_map_kmajor(bl, N, kp, BNT);
  constexpr size_t smem = tck::Cfg<BNT>::SMEM_BYTES;
  set_smem(tck_gemm_kernel<BNT>, smem);
  const int64_t blocks = ((M + tc::BM - 1) / tc::BM) * ((N + BNT - 1) / BNT);
  const int64_t grid = std::min<int64_t>(blocks, (int64_t)num_sms());
  tck_gemm_kernel<BNT><<<(unsigned)grid, tck::THREADS, smem, st>>>(mah, mal, mbh, mbl, M, N, K, C, ldc, alpha, beta,
                                                                    info, fan);
  BCMG_CHECK_LAUNCH();
}

static FloatFan float_fan(const Epilogue& ep) {
  FloatFan f{};
  f.n = ep.nfan;
  for (int e = 0; e < ep.nfan; ++e) f.p[e] = static_cast<float*>(ep.fan[e]);
  return f;
}

void tck_gemm(int64_t M, int64_t N, int64_t K, const float* ah, const float* al, const float* bh, const float* bl,
              int64_t kp, float* C, int64_t ldc, float alpha, float beta, const int* info, cudaStream_t st,
              const Epilogue* fan_src) {
  const FloatFan fan = fan_src ? float_fan(*fan_src) : FloatFan{};
  if (tck_width(N) == 256) return tck_gemm_t<256>(M, N, K, ah, al, bh, bl, kp, C, ldc, alpha, beta, info, st, fan);
  tck_gemm_t<128>(M, N, K, ah, al, bh, bl, kp, C, ldc, alpha, beta, info, st, fan);
}

// gemm() for float32 on tcgen05: both operands split into a scratch owned by
// the stream (grow-only; stream order makes reuse safe).  Process-wide
// registry: a session releases its streams' scratch when it closes, so a new
// stream that happens to reuse a closed stream's handle starts empty.
namespace {
struct SplitBuf {
  void* p = nullptr;
  size_t n = 0;
};
std::mutex g_split_mu;
std::vector<std::pair<cudaStream_t, SplitBuf>> g_split;
}  // namespace

static float* split_scratch(cudaStream_t st, size_t bytes, size_t* held) {
  std::lock_guard<std::mutex> lk(g_split_mu);
  SplitBuf* b = nullptr;
  for (auto& e : g_split)
    if (e.first == st) b = &e.second;
  if (held) {  // query only
    *held = b ? b->n : 0;
    return nullptr;
  }
  if (!b) {
    g_split.emplace_back(st, SplitBuf{});
    b = &g_split.back().second;
  }
  if (b->n < bytes) {
    if (b->p) {
      BCMG_CUDA(cudaStreamSynchronize(st));
      cudaFree(b->p);
      b->p = nullptr;
      b->n = 0;
    }
    cudaError_t e = cudaMalloc(&b->p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error(OUT_OF_MEMORY, "tf32 split scratch: " + std::string(cudaGetErrorString(e)));
    }
    b->n = bytes;
  }
  return static_cast<float*>(b->p);
}

// Grow the split scratch of `st` ahead of a schedule loop: growth frees the
// old buffer (cudaFree synchronises the device), which must not happen while
// another rank's stream waits for a flag this rank has yet to raise.
void reserve_split_scratch(cudaStream_t st, size_t bytes) { split_scratch(st, bytes); }
size_t split_scratch_held(cudaStream_t st) {
  size_t h = 0;
  split_scratch(st, 0, &h);
  return h;
}
void release_split_scratch(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_split_mu);
  for (size_t i = 0; i < g_split.size(); ++i)
    if (g_split[i].first == st) {
      if (g_split[i].second.p) {
        cudaStreamSynchronize(st);
        cudaFree(g_split[i].second.p);
      }
      g_split.erase(g_split.begin() + i);
      return;
    }
}
size_t split_scratch_bytes(int dt, int64_t M, int64_t N, int64_t K) {
  return dt == C64 ? (size_t)2 * (2 * M + N) * split_ld(2 * K) * 4 : (size_t)2 * (M + N) * split_ld(K) * 4;
}

static void gemm_tck_generic(int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                             const int* info, cudaStream_t st) {
  const int64_t kp = split_ld(K);
  float* s = split_scratch(st, (size_t)2 * (M + N) * kp * 4);
  float *ah = s, *al = s + M * kp, *bh = al + M * kp, *bl = bh + N * kp;
  split_tf32(A.trans ? 3 : 0, A.ptr, A.ld, M, K, K, ah, al, kp, st);
  split_tf32(B.trans ? 3 : 0, B.ptr, B.ld, N, K, K, bh, bl, kp, st);
  tck_gemm(M, N, K, ah, al, bh, bl, kp, static_cast<float*>(ep.C), ep.ldc, (float)ep.alpha, (float)ep.beta, info, st,
           &ep);
}

static void launch_tc3_trail(const TrailParams& p, const int* info, cudaStream_t st) {
  if (p.split[0]) return launch_tck_trail(p, info, st);
  int64_t total = 0;
  for (int64_t m = p.m_first; m < p.m_last; ++m) {
    const int dev = (int)(m % p.D);
    if (dev < p.dev0 || dev >= p.dev0 + p.nloc) continue;
    const int64_t rows = p.N - m * p.T, tcm = std::min(p.T, rows);
    total += p.cplx ? TrapH<tc::BM / 2, tc::BN>::count(rows, tcm) : Trap<tc::BM, tc::BN>::count(rows, tcm);
  }
  if (total == 0) return;
  const int64_t prow = p.N - p.prow0;
  // complex64: A = [P | -iP] as a (2 rows) x (2K) float matrix, B = planar [Re P | Im P]
  const CUtensorMap ma = p.cplx ? make_map_f32_sw128(p.P, 2 * prow, 2 * p.K, 2 * p.ldp)
                                : make_map_f32_sw128(p.P, prow, p.K, p.ldp);
  const CUtensorMap mb = p.cplx ? make_map_f32_sw128(p.PB, prow, 2 * p.K, p.ldp) : ma;
  set_smem(tc3_trail_kernel, tc::SMEM_BYTES);
  const int sms = p.max_ctas > 0 ? std::min(p.max_ctas, num_sms()) : num_sms();
  const int64_t grid = std::min<int64_t>(total, sms);
  tc3_trail_kernel<<<(unsigned)grid, tc::THREADS, tc::SMEM_BYTES, st>>>(ma, mb, p, info);
  BCMG_CHECK_LAUNCH();
}

void trailing_update(int dt, const TrailParams& p, const int* info, cudaStream_t st) {
  if (p.m_first >= p.m_last || p.K <= 0) return;
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    if constexpr (std::is_same_v<S, float> || std::is_same_v<S, float2>) {
      if (p.split[0]) return launch_tck_trail(p, info, st);  // pre-split panel (any T)
    }
    if constexpr (std::is_same_v<S, float>) {
      if (use_tc() && tc_ok(p.P, p.ldp) && p.T % 4 == 0 && p.prow0 % 4 == 0 && p.N % 4 == 0)
        return launch_tc3_trail(p, info, st);
    }
    if constexpr (std::is_same_v<S, double>) {
      const bool cp = aligned16(p.P) && p.ldp % 2 == 0 && p.T % 2 == 0 && (p.prow0 % 2 == 0);
      if (cp && use_tma() && tma_ok(p.P, p.ldp)) return launch_trail_tma(p, info, st);
      if (cp) return launch_trail<S, TileBig, true>(p, info, st);
    }
    if constexpr (std::is_same_v<S, double2>) {
      if (p.cplx) return launch_trail_tma(p, info, st);
    }
    if constexpr (std::is_same_v<S, float2>) {
      if (p.cplx) return launch_tc3_trail(p, info, st);
    }
    launch_trail<S, TileMed, false>(p, info, st);
  });
}

// ============================================================== diagonal leaf
// n <= 64: in-place lower Cholesky + X = L^-1 in shared memory, right-looking
// (the reference's unblocked factor is solvers.py:322-338; same pivot test:
// d = Re a_jj after the updates, fail unless d > 0 and finite).
constexpr int LEAF = 64;

template <bool C> struct V_ { using type = double; };
template <> struct V_<true> { using type = double2; };

__device__ __forceinline__ double v_re(double a) { return a; }
__device__ __forceinline__ double v_re(double2 a) { return a.x; }
__device__ __forceinline__ double v_scale(double a, double s) { return a * s; }
__device__ __forceinline__ double2 v_scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double v_fnms(double c, double a, double b) { return c - a * b; }            // c - a*b
__device__ __forceinline__ double2 v_fnms(double2 c, double2 a, double2 b) {
  double2 p = cmul(a, b);
  return make_double2(c.x - p.x, c.y - p.y);
}
__device__ __forceinline__ double v_fnmsc(double c, double a, double b) { return c - a * b; }           // c - a*conj(b)
__device__ __forceinline__ double2 v_fnmsc(double2 c, double2 a, double2 b) {
  double2 p = cmulc(a, b);
  return make_double2(c.x - p.x, c.y - p.y);
}
template <class V> __device__ __forceinline__ V v_from(double2 x);
template <> __device__ __forceinline__ double v_from<double>(double2 x) { return x.x; }
template <> __device__ __forceinline__ double2 v_from<double2>(double2 x) { return x; }
__device__ __forceinline__ double2 v_to(double a) { return make_double2(a, 0.0); }
__device__ __forceinline__ double2 v_to(double2 a) { return a; }

// Register-resident leaf: thread (ty, tx) = (tid/16, tid%16) owns the 4x4
// elements (ty + 16a, tx + 16b) of both L and X = L^-1, so the only shared
// traffic per column is a broadcast of the scaled column of L and row of X
// (double buffered: two barriers per column, no shared-memory matrix).
// Right-looking: step j takes the pivot d = Re a_jj after all earlier
// updates -- the reference's test, failing unless d > 0 and finite.
template <class S>
__device__ __forceinline__ void leaf_body(S* A, int64_t lda, S* X, int64_t ldx, int n, int64_t goff, int* info) {
  using V = typename V_<Traits<S>::cplx>::type;
  if (*(volatile int*)info) return;
  __shared__ V colL[2][LEAF];
  __shared__ V rowX[2][LEAF];
  __shared__ double s_inv[2];
  __shared__ int s_bad;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  V l[4][4], x[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, c = tx + 16 * b;
      const bool in = i < n && c < n;
      l[a][b] = v_from<V>(in && i >= c ? to_c(A[i + (int64_t)c * lda]) : make_double2(0, 0));
      x[a][b] = v_from<V>(make_double2(in && i == c ? 1.0 : 0.0, 0.0));
    }
  if (tid == 0) s_bad = -1;
  __syncthreads();
  int done = n;
#pragma unroll
  for (int jo = 0; jo < 4; ++jo) {
    for (int jl = 0; jl < 16; ++jl) {
      const int j = 16 * jo + jl, buf = j & 1;
      if (j >= n) goto finished;
      // pivot (owner of (j, j))
      if (ty == jl && tx == jl) {
        const double d = v_re(l[jo][jo]);
        if (!(d > 0.0) || !isfinite(d)) {
          s_bad = j;
        } else {
          const double r = rsqrt(d);  // one MUFU + Newton steps on the serial chain (not sqrt + div)
          l[jo][jo] = v_from<V>(make_double2(d * r, 0.0));
          s_inv[buf] = r;
        }
      }
      __syncthreads();
      if (s_bad >= 0) {
        done = j;
        goto finished;
      }
      {
        const double inv = s_inv[buf];
        if (tx == jl) {  // column j of L, rows below the diagonal
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int i = ty + 16 * a;
            if (i > j && i < n) {
              l[a][jo] = v_scale(l[a][jo], inv);
              colL[buf][i] = l[a][jo];
            }
          }
        }
        if (ty == jl) {  // row j of X, columns up to the diagonal
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int c = tx + 16 * b;
            if (c <= j) {
              x[jo][b] = v_scale(x[jo][b], inv);
              rowX[buf][c] = x[jo][b];
            }
          }
        }
      }
      __syncthreads();
      {
        // branch-free rank-1 update: all broadcast operands are loaded up front
        // (stale entries are loaded but never selected), then predicated FMAs,
        // so the shared-memory latency is paid once per column, not per element
        // (jo is a compile-time index here: row blocks a < jo lie above the
        // pivot, L column blocks b < jo left of it and X column blocks b > jo
        // right of it, so those are never touched -- the triangle shrinks)
        V li[4], lc[4], xc[4];
#pragma unroll
        for (int a = jo; a < 4; ++a) li[a] = colL[buf][ty + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (b >= jo) lc[b] = colL[buf][tx + 16 * b];
          if (b <= jo) xc[b] = rowX[buf][tx + 16 * b];
        }
#pragma unroll
        for (int a = jo; a < 4; ++a) {
          const int i = ty + 16 * a;
          const bool row = i > j && i < n;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int c = tx + 16 * b;
            if (b <= jo) {
              const V nx = v_fnms(x[a][b], li[a], xc[b]);
              x[a][b] = (row && c <= j) ? nx : x[a][b];
            }
            if (b >= jo && b <= a) {
              const V nl = v_fnmsc(l[a][b], li[a], lc[b]);
              l[a][b] = (row && c > j && c <= i) ? nl : l[a][b];
            }
          }
        }
      }
    }
  }
finished:
  if (done < n && tid == 0) atomicCAS(info, 0, (int)(goff + done + 1));
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, c = tx + 16 * b;
      if (i >= n || c >= n) continue;
      if (c < done && i >= c) A[i + (int64_t)c * lda] = from_c<S>(v_to(l[a][b]));
      if (done == n) X[i + (int64_t)c * ldx] = from_c<S>(i >= c ? v_to(x[a][b]) : make_double2(0, 0));
    }
}

template <class S>
__global__ void __launch_bounds__(256) leaf_kernel(S* A, int64_t lda, S* X, int64_t ldx, int n, int64_t goff,
                                                   int* info) {
  leaf_body<S>(A, lda, X, ldx, n, goff, info);
}

template <class S>
static void launch_leaf(S* A, int64_t lda, S* X, int64_t ldx, int n, int64_t goff, int* info, cudaStream_t st) {
  leaf_kernel<S><<<1, 256, 0, st>>>(A, lda, X, ldx, n, goff, info);
  BCMG_CHECK_LAUNCH();
}

// One recursion node of size 64 < n <= 128 in ONE CTA (the bottom level of
// diag_factor, which otherwise costs two leaf launches, four 64^3 GEMM
// launches and three copies):
//   leaf(A11) -> L11, X11;  L21 = A21 X11^H;  A22 -= L21 L21^H (lower);
//   leaf(A22) -> L22, X22;  X21 = -X22 (L21 X11);  X12 = 0
// The 64x64 operands of the small products live in shared memory (row
// stride 65); thread (ty, tx) computes rows ty + 16a, columns tx + 16b.
template <class S>
__global__ void __launch_bounds__(256) node_kernel(S* A, int64_t lda, S* X, int64_t ldx, int n, int64_t goff,
                                                   int* info) {
  using V = typename V_<Traits<S>::cplx>::type;
  constexpr int LD = LEAF + 1;
  extern __shared__ __align__(16) unsigned char node_smem[];
  V* X11 = reinterpret_cast<V*>(node_smem);  // X11[r * LD + c]
  V* B1 = X11 + LEAF * LD;                   // A21, then T1 = L21 X11
  V* B2 = B1 + LEAF * LD;                    // L21, then X22
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int n1 = LEAF, n2 = n - LEAF;
  auto ld = [](const S* p, int64_t ld_, int r, int c) { return v_from<V>(to_c(p[r + (int64_t)c * ld_])); };
  auto st = [](S* p, int64_t ld_, int r, int c, V v) { p[r + (int64_t)c * ld_] = from_c<S>(v_to(v)); };
  auto zero = [] { return v_from<V>(make_double2(0.0, 0.0)); };
  auto fma_ = [](V acc, V a, V b) { return v_fnms(acc, v_scale(a, -1.0), b); };         // acc + a*b
  auto fmac_ = [](V acc, V a, V b) { return v_fnmsc(acc, v_scale(a, -1.0), b); };       // acc + a*conj(b)

  leaf_body<S>(A, lda, X, ldx, n1, goff, info);
  __syncthreads();
  if (*(volatile int*)info) return;
  for (int e = tid; e < LEAF * LEAF; e += 256) {
    const int r = e % LEAF, c = e / LEAF;
    X11[r * LD + c] = ld(X, ldx, r, c);
    B1[r * LD + c] = r < n2 ? ld(A, lda, n1 + r, c) : zero();
  }
  __syncthreads();
  // L21 = A21 X11^H  (X11 lower: k <= c)
  V acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = zero();
  for (int kk = 0; kk < LEAF; ++kk) {
    V av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = B1[(ty + 16 * a) * LD + kk];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = X11[(tx + 16 * b) * LD + kk];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fmac_(acc[a][b], av[a], bv[b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, c = tx + 16 * b;
      B2[i * LD + c] = i < n2 ? acc[a][b] : zero();
      if (i < n2) st(A, lda, n1 + i, c, acc[a][b]);
    }
  __syncthreads();
  // A22 -= L21 L21^H on the lower triangle
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = zero();
  for (int kk = 0; kk < LEAF; ++kk) {
    V av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = B2[(ty + 16 * a) * LD + kk];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = B2[(tx + 16 * b) * LD + kk];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fmac_(acc[a][b], av[a], bv[b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, c = tx + 16 * b;
      if (i < n2 && c <= i) {
        const V old = ld(A, lda, n1 + i, n1 + c);
        st(A, lda, n1 + i, n1 + c, v_fnms(old, acc[a][b], v_from<V>(make_double2(1.0, 0.0))));
      }
    }
  __syncthreads();
  leaf_body<S>(A + n1 + (int64_t)n1 * lda, lda, X + n1 + (int64_t)n1 * ldx, ldx, n2, goff + n1, info);
  __syncthreads();
  if (*(volatile int*)info) return;
  // T1 = L21 X11 -> B1
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = zero();
  for (int kk = 0; kk < LEAF; ++kk) {
    V av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = B2[(ty + 16 * a) * LD + kk];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = X11[kk * LD + tx + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma_(acc[a][b], av[a], bv[b]);
  }
  __syncthreads();  // every read of B2 (L21) done before X22 overwrites it
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) B1[(ty + 16 * a) * LD + tx + 16 * b] = acc[a][b];
  for (int e = tid; e < LEAF * LEAF; e += 256) {
    const int r = e % LEAF, c = e / LEAF;
    B2[r * LD + c] = (r < n2 && c < n2) ? ld(X, ldx, n1 + r, n1 + c) : zero();
  }
  __syncthreads();
  // X21 = -X22 T1 ; X12 = 0
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = zero();
  for (int kk = 0; kk < LEAF; ++kk) {
    V av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = B2[(ty + 16 * a) * LD + kk];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = B1[kk * LD + tx + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma_(acc[a][b], av[a], bv[b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, c = tx + 16 * b;
      if (i < n2) st(X, ldx, n1 + i, c, v_scale(acc[a][b], -1.0));
      if (c < n2) st(X, ldx, i, n1 + c, zero());
    }
}

template <class S>
static void launch_node(S* A, int64_t lda, S* X, int64_t ldx, int n, int64_t goff, int* info, cudaStream_t st) {
  using V = typename V_<Traits<S>::cplx>::type;
  constexpr size_t smem = (size_t)3 * LEAF * (LEAF + 1) * sizeof(V);
  set_smem(node_kernel<S>, smem);
  node_kernel<S><<<1, 256, smem, st>>>(A, lda, X, ldx, n, goff, info);
  BCMG_CHECK_LAUNCH();
}

// Recursive diagonal factor + inverse:
//   [L11 0; L21 L22] = chol(A),  X = [X11 0; X21 X22] = L^-1
//   L21 = A21 X11^H,  A22 -= L21 L21^H,  X21 = -X22 (L21 X11)
void diag_factor(int dt, void* A, int64_t lda, void* X, int64_t ldx, void* W, int64_t n, int64_t goff, int* info,
                 cudaStream_t st) {
  const int esz = dtype_size(dt);
  auto at = [esz](void* base, int64_t ld, int64_t r, int64_t c) {
    return static_cast<void*>(static_cast<char*>(base) + (r + c * ld) * esz);
  };
  if (n <= LEAF) {
    dispatch_dtype(dt, [&](auto s) {
      using S = decltype(s);
      launch_leaf<S>(static_cast<S*>(A), lda, static_cast<S*>(X), ldx, (int)n, goff, info, st);
    });
    return;
  }
  if (n <= 2 * LEAF && !getenv("BCMG_NO_NODE_KERNEL")) {
    dispatch_dtype(dt, [&](auto s) {
      using S = decltype(s);
      launch_node<S>(static_cast<S*>(A), lda, static_cast<S*>(X), ldx, (int)n, goff, info, st);
    });
    return;
  }
  int64_t n1 = ((n + 1) / 2 + LEAF - 1) / LEAF * LEAF;
  if (n1 >= n) n1 = n - LEAF;
  const int64_t n2 = n - n1;
  void* A11 = A;
  void* A21 = at(A, lda, n1, 0);
  void* A22 = at(A, lda, n1, n1);
  void* X11 = X;
  void* X21 = at(X, ldx, n1, 0);
  void* X22 = at(X, ldx, n1, n1);
  const int64_t ldw = n2;  // W holds n2 x n1 and n2 x n1 temporaries
  diag_factor(dt, A11, lda, X11, ldx, W, n1, goff, info, st);
  // L21 = A21 * X11^H  -> W, then back into A21
  gemm(dt, n2, n1, n1, opA(A21, lda, OP_N), opB(X11, ldx, OP_C), Epilogue{W, ldw, 1.0, 0.0, 0, 0}, info, st);
  copy2d(dt, W, ldw, A21, lda, n2, n1, false, info, st);
  // A22 -= L21 * L21^H (lower triangle)
  gemm(dt, n2, n2, n1, opA(A21, lda, OP_N), opB(A21, lda, OP_C), Epilogue{A22, lda, -1.0, 1.0, 1, 0}, info, st);
  diag_factor(dt, A22, lda, X22, ldx, W, n2, goff + n1, info, st);
  // X21 = -X22 * (L21 * X11)
  gemm(dt, n2, n1, n1, opA(A21, lda, OP_N), opB(X11, ldx, OP_N), Epilogue{X21, ldx, 1.0, 0.0, 0, 0}, info, st);
  gemm(dt, n2, n1, n2, opA(X22, ldx, OP_N), opB(X21, ldx, OP_N), Epilogue{W, ldw, -1.0, 0.0, 0, 0}, info, st);
  copy2d(dt, W, ldw, X21, ldx, n2, n1, false, info, st);
  // X's strict upper block (X12) must read as zero for later GEMM operands
  zero_upper(dt, at(X, ldx, 0, n1), ldx, n1, n2, n1, st);
}

// ============================================================== substitution (small N_RHS)
// Bandwidth kernels for the triangular sweeps of potrs when the right-hand
// side is narrow (N_RHS <= 16): the split-K GEMM path pads N_RHS to its 16-wide
// tile and runs ~7x (T_A = 1024) to ~27x (T_A = 128) above the HBM floor of
// reading the factor twice.  Accumulation in double / double2; every sum has a
// fixed order that depends on (n, T_A, k) only, so the bits do not depend on
// the device or process count.
template <bool CPLX> struct SubAcc { using T = double; };
template <> struct SubAcc<true> { using T = double2; };
__device__ __forceinline__ double sub_ld(float v) { return v; }
__device__ __forceinline__ double sub_ld(double v) { return v; }
__device__ __forceinline__ double2 sub_ld(float2 v) { return make_double2(v.x, v.y); }
__device__ __forceinline__ double2 sub_ld(double2 v) { return v; }
__device__ __forceinline__ double sub_conj(double v) { return v; }
__device__ __forceinline__ double2 sub_conj(double2 v) { return make_double2(v.x, -v.y); }
__device__ __forceinline__ double sub_fma(double acc, double a, double b) { return fma(a, b, acc); }
__device__ __forceinline__ double2 sub_fma(double2 acc, double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
__device__ __forceinline__ double sub_add(double a, double b) { return a + b; }
__device__ __forceinline__ double2 sub_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double sub_zero(double) { return 0.0; }
__device__ __forceinline__ double2 sub_zero(double2) { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double sub_shfl(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ double2 sub_shfl(double2 v, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
template <class S> __device__ __forceinline__ S sub_st(double v) { return (S)v; }
template <class S> __device__ __forceinline__ S sub_st(double2 v) { return from_c<S>(v); }

// Forward GEMV out[r, j] = (beta ? out[r, j] : 0) + alpha * sum_c A[r + c lda] y[c, j]
// for r in [ncopy, rows); out[r, j] = y[r, j] for r < ncopy.  A CTA owns 32 rows
// (one per lane); its W warps split the columns (contiguous ranges, loads
// coalesced across the lanes, U in flight per lane) and their sums meet in
// shared memory in warp order.  (128 rows per CTA with 4 rows per lane was
// measured slower: fewer CTAs, fewer loads in flight.)
template <class S, int NR>
constexpr int subst_gemv_warps() { return 8; }
template <class S, int NR>
__global__ void __launch_bounds__(256) subst_gemv_kernel(const S* __restrict__ A, int64_t lda, const S* __restrict__ y,
                                                         int64_t ldy, S* __restrict__ out, int64_t ldo, int64_t rows,
                                                         int tc, int nrhs, int64_t ncopy, double alpha, int beta) {
  using Acc = typename SubAcc<Traits<S>::cplx>::T;
  constexpr int W = subst_gemv_warps<S, NR>();
  __shared__ Acc red[W][32][NR];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 32 + lane;
  const bool live = r < rows && r >= ncopy;
  Acc acc[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = sub_zero(Acc{});
  const int cpw = (tc + W - 1) / W, c0 = warp * cpw, c1 = c0 + cpw < tc ? c0 + cpw : tc;
  if (live) {
    const S* a = A + r;
    int c = c0;
    constexpr int U = 8;  // column loads in flight per lane (16 / 32 measured slower: more DRAM pages open)
    for (; c + U <= c1; c += U) {
      Acc av[U];
#pragma unroll
      for (int u = 0; u < U; ++u) av[u] = sub_ld(a[(int64_t)(c + u) * lda]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < NR; ++j)
          if (j < nrhs) acc[j] = sub_fma(acc[j], av[u], sub_ld(__ldg(y + (c + u) + j * ldy)));
    }
    for (; c < c1; ++c) {
      const Acc av = sub_ld(a[(int64_t)c * lda]);
#pragma unroll
      for (int j = 0; j < NR; ++j)
        if (j < nrhs) acc[j] = sub_fma(acc[j], av, sub_ld(__ldg(y + c + j * ldy)));
    }
  }
#pragma unroll
  for (int j = 0; j < NR; ++j) red[warp][lane][j] = acc[j];
  __syncthreads();
  if (warp != 0 || r >= rows) return;
  if (r < ncopy) {
#pragma unroll
    for (int j = 0; j < NR; ++j)
      if (j < nrhs) out[r + j * ldo] = y[r + j * ldy];
    return;
  }
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if (j >= nrhs) break;
    Acc v = red[0][lane][j];
    for (int w = 1; w < W; ++w) v = sub_add(v, red[w][lane][j]);
    if constexpr (Traits<S>::cplx) v = make_double2(alpha * v.x, alpha * v.y);
    else v = alpha * v;
    if (beta) v = sub_add(v, sub_ld(out[r + j * ldo]));
    out[r + j * ldo] = sub_st<S>(v);
  }
}

// float32, N_RHS = 1: the same GEMV with 4 consecutive rows per lane (one
// 16-byte load per column: 512-byte runs per warp instead of 128), 128 rows
// per CTA.  Same column split and warp-order sums as subst_gemv_kernel, so the
// same bits; used when every column start is 16-byte aligned.
#ifndef BCMG_NO_GEMV4
#define BCMG_NO_GEMV4 0
#endif
__global__ void __launch_bounds__(256) subst_gemv4_kernel(const float* __restrict__ A, int64_t lda,
                                                          const float* __restrict__ y, float* __restrict__ out,
                                                          int64_t rows, int tc, int64_t ncopy, double alpha, int beta) {
  constexpr int W = 8;
  __shared__ double red[W][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * 128 + 4 * lane;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int cpw = (tc + W - 1) / W, c0 = warp * cpw, c1 = c0 + cpw < tc ? c0 + cpw : tc;
  const bool full = r0 + 3 < rows;
  if (r0 < rows) {
    const float* a = A + r0;
    int c = c0;
    if (full) {
      for (; c + 4 <= c1; c += 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(a + (int64_t)(c + u) * lda));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double yv = __ldg(y + c + u);
          acc[0] = fma((double)v[u].x, yv, acc[0]);
          acc[1] = fma((double)v[u].y, yv, acc[1]);
          acc[2] = fma((double)v[u].z, yv, acc[2]);
          acc[3] = fma((double)v[u].w, yv, acc[3]);
        }
      }
      for (; c < c1; ++c) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(a + (int64_t)c * lda));
        const double yv = __ldg(y + c);
        acc[0] = fma((double)v.x, yv, acc[0]);
        acc[1] = fma((double)v.y, yv, acc[1]);
        acc[2] = fma((double)v.z, yv, acc[2]);
        acc[3] = fma((double)v.w, yv, acc[3]);
      }
    } else {
      for (; c < c1; ++c) {
        const double yv = __ldg(y + c);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (r0 + i < rows) acc[i] = fma((double)a[(int64_t)c * lda + i], yv, acc[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) red[warp][4 * lane + i] = acc[i];
  __syncthreads();
  if (threadIdx.x >= 128) return;
  const int e = threadIdx.x;
  const int64_t r = (int64_t)blockIdx.x * 128 + e;
  if (r >= rows) return;
  if (r < ncopy) {
    out[r] = y[r];
    return;
  }
  double v = red[0][e];
#pragma unroll
  for (int w = 1; w < W; ++w) v += red[w][e];
  v = alpha * v;
  if (beta) v += (double)out[r];
  out[r] = (float)v;
}

// complex64, N_RHS = 1: two consecutive rows per lane (one 16-byte load per
// column), 64 rows per CTA; same column split and sums as subst_gemv_kernel.
__global__ void __launch_bounds__(256) subst_gemv2c_kernel(const float2* __restrict__ A, int64_t lda,
                                                           const float2* __restrict__ y, float2* __restrict__ out,
                                                           int64_t rows, int tc, int64_t ncopy, double alpha, int beta) {
  constexpr int W = 8;
  __shared__ double2 red[W][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * 64 + 2 * lane;
  double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  const int cpw = (tc + W - 1) / W, c0 = warp * cpw, c1 = c0 + cpw < tc ? c0 + cpw : tc;
  if (r0 < rows) {
    const float2* a = A + r0;
    if (r0 + 1 < rows) {
      for (int c = c0; c < c1; ++c) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(a + (int64_t)c * lda));
        const double2 yv = sub_ld(__ldg(y + c));
        acc[0] = sub_fma(acc[0], make_double2(v.x, v.y), yv);
        acc[1] = sub_fma(acc[1], make_double2(v.z, v.w), yv);
      }
    } else {
      for (int c = c0; c < c1; ++c) acc[0] = sub_fma(acc[0], sub_ld(a[(int64_t)c * lda]), sub_ld(__ldg(y + c)));
    }
  }
  red[warp][2 * lane] = acc[0];
  red[warp][2 * lane + 1] = acc[1];
  __syncthreads();
  if (threadIdx.x >= 64) return;
  const int e = threadIdx.x;
  const int64_t r = (int64_t)blockIdx.x * 64 + e;
  if (r >= rows) return;
  if (r < ncopy) {
    out[r] = y[r];
    return;
  }
  double2 v = red[0][e];
#pragma unroll
  for (int w = 1; w < W; ++w) v = sub_add(v, red[w][e]);
  v = make_double2(alpha * v.x, alpha * v.y);
  if (beta) v = sub_add(v, sub_ld(out[r]));
  out[r] = sub_st<float2>(v);
}

// Backward partial sums P[chunk][c][j] = sum_{r in chunk} conj(L[r, c]) x[r, j]
// over chunks of SUBST_CH rows.  Grid (chunk, column group): a CTA stages its
// chunk of x in shared memory and its warps take the group's columns two at a
// time (lanes stride the rows, coalesced; one fixed butterfly reduction per
// sum), so the partial of (chunk, c) does not depend on the grid shape.
constexpr int SUBST_CH = 512;
template <class S, int NR>
__global__ void __launch_bounds__(256) subst_partials_kernel(const S* __restrict__ L, int64_t ldl,
                                                             const S* __restrict__ x, int64_t ldx, int64_t rows, int tc,
                                                             int nrhs, int cpg, void* parts) {
  using Acc = typename SubAcc<Traits<S>::cplx>::T;
  constexpr int CH = SUBST_CH, PER = CH / 32;
  extern __shared__ __align__(16) unsigned char subst_smem[];
  Acc* xs = reinterpret_cast<Acc*>(subst_smem);  // [NR][CH]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * CH;
  const int sn = (int)(rows - r0 < CH ? rows - r0 : CH);
  for (int e = threadIdx.x; e < CH * NR; e += blockDim.x) {
    const int r = e % CH, j = e / CH;
    xs[j * CH + r] = (r < sn && j < nrhs) ? sub_ld(x[(r0 + r) + j * ldx]) : sub_zero(Acc{});
  }
  __syncthreads();
  Acc* P = static_cast<Acc*>(parts) + (int64_t)blockIdx.x * tc * nrhs;
  const int cb = blockIdx.y * cpg, ce = cb + cpg < tc ? cb + cpg : tc;
  auto one = [&](const Acc* lv, int c) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j >= nrhs) break;
      Acc v = sub_zero(Acc{});
#pragma unroll
      for (int i = 0; i < PER; ++i) v = sub_fma(v, lv[i], xs[j * CH + lane + 32 * i]);
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) v = sub_add(v, sub_shfl(v, m));
      if (lane == 0) P[(int64_t)c * nrhs + j] = v;
    }
  };
  for (int c = cb + 2 * warp; c < ce; c += 2 * nw) {
    const bool two = c + 1 < ce;
    const S* l0 = L + (int64_t)c * ldl + r0;
    const S* l1 = l0 + ldl;
    Acc a0[PER], a1[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int r = lane + 32 * i;
      a0[i] = r < sn ? sub_conj(sub_ld(l0[r])) : sub_zero(Acc{});
      a1[i] = (two && r < sn) ? sub_conj(sub_ld(l1[r])) : sub_zero(Acc{});
    }
    one(a0, c);
    if (two) one(a1, c + 1);
  }
}

// mode 0: z[c, j] = x[c, j] - sum_p P[p][c][j];  mode 1: z[c, j] = sum_p P[p][c][j]
// (p ascending); z has leading dimension ldz
template <class S>
__global__ void subst_reduce_kernel(const S* __restrict__ x, int64_t ldx, const void* parts, int np, int tc, int nrhs,
                                    S* __restrict__ z, int64_t ldz, int mode) {
  using Acc = typename SubAcc<Traits<S>::cplx>::T;
  const Acc* P = static_cast<const Acc*>(parts);
  const int64_t total = (int64_t)tc * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / nrhs), j = (int)(e % nrhs);
    Acc s = sub_zero(Acc{});
#pragma unroll 8
    for (int p = 0; p < np; ++p) s = sub_add(s, P[((int64_t)p * tc + c) * nrhs + j]);
    if (mode == 0) {
      Acc v = sub_ld(x[c + j * ldx]);
      if constexpr (Traits<S>::cplx) s = make_double2(v.x - s.x, v.y - s.y);
      else s = v - s;
    }
    z[c + j * ldz] = sub_st<S>(s);
  }
}

bool subst_gemv_ok(int dt, int64_t nrhs) {
  static const bool on = [] {
    const char* e = getenv("BCMG_SUBST_GEMV");
    return !(e && *e && atoi(e) == 0);
  }();
  // measured (tools/potrs_phase.py, N=65536, ms new / split-K): f32 T=128 N_RHS=1 29.9 / 73.8,
  // T=1024 13.9 / 18.5, T=256 N_RHS=2 18.1 / 41.4; c64 21.9 / 38.1; c128 N_RHS=1 / 4 28.9 / 56.9,
  // 37.8 / 57.0; f64 N_RHS=1 / 4 14.1 / 10.4, 16.8 / 10.5 -- float64 keeps the DMMA split-K GEMMs
  return on && nrhs >= 1 && nrhs <= 4 && dt != R64;
}
size_t subst_parts_bytes(int64_t n, int64_t T, int64_t nrhs) {
  return (size_t)((n + SUBST_CH - 1) / SUBST_CH + 1) * T * nrhs * 16 + (size_t)T * nrhs * 16;
}

static int subst_nr(int64_t nrhs) { return nrhs <= 1 ? 1 : nrhs <= 2 ? 2 : 4; }

template <class S>
static void launch_subst_gemv(int nr, const S* A, int64_t lda, const S* y, int64_t ldy, S* out, int64_t ldo,
                              int64_t rows, int tc, int nrhs, int64_t ncopy, double alpha, int beta, cudaStream_t st) {
  if (rows <= 0) return;
  if constexpr (std::is_same_v<S, float> && !BCMG_NO_GEMV4) {
    if (nr == 1 && nrhs == 1 && lda % 4 == 0 && aligned16(A)) {
      subst_gemv4_kernel<<<(unsigned)((rows + 127) / 128), 256, 0, st>>>(A, lda, y, out, rows, tc, ncopy, alpha,
                                                                          beta);
      BCMG_CHECK_LAUNCH();
      return;
    }
  }
  if constexpr (std::is_same_v<S, float2> && !BCMG_NO_GEMV4) {
    if (nr == 1 && nrhs == 1 && lda % 2 == 0 && aligned16(A)) {
      subst_gemv2c_kernel<<<(unsigned)((rows + 63) / 64), 256, 0, st>>>(A, lda, y, out, rows, tc, ncopy, alpha,
                                                                         beta);
      BCMG_CHECK_LAUNCH();
      return;
    }
  }
  const unsigned grid = (unsigned)((rows + 31) / 32);
  auto go = [&](auto kern, int warps) {
    kern<<<grid, 32 * warps, 0, st>>>(A, lda, y, ldy, out, ldo, rows, tc, nrhs, ncopy, alpha, beta);
  };
  if (nr == 1) go(subst_gemv_kernel<S, 1>, subst_gemv_warps<S, 1>());
  else if (nr == 2) go(subst_gemv_kernel<S, 2>, subst_gemv_warps<S, 2>());
  else go(subst_gemv_kernel<S, 4>, subst_gemv_warps<S, 4>());
  BCMG_CHECK_LAUNCH();
}

// P[chunk] over `rows` rows of L (ld ldl) against x; returns the chunk count
template <class S>
static int launch_subst_partials(int nr, const S* L, int64_t ldl, const S* x, int64_t ldx, int64_t rows, int tc,
                                 int nrhs, void* parts, cudaStream_t st) {
  if (rows <= 0) return 0;
  using Acc = typename SubAcc<Traits<S>::cplx>::T;
  const int np = (int)((rows + SUBST_CH - 1) / SUBST_CH);
  const size_t smem = (size_t)SUBST_CH * nr * sizeof(Acc);
  // column groups of >= 16 columns so that the grid covers ~8 CTAs per SM
  const int groups = (int)std::max<int64_t>(1, std::min<int64_t>((tc + 15) / 16, ((int64_t)num_sms() * 8 + np - 1) / np));
  const int cpg = (tc + groups - 1) / groups;
  auto go = [&](auto kern) {
    set_smem(kern, smem);
    kern<<<dim3((unsigned)np, (unsigned)((tc + cpg - 1) / cpg)), 256, smem, st>>>(L, ldl, x, ldx, rows, tc, nrhs, cpg,
                                                                                 parts);
  };
  if (nr == 1) go(subst_partials_kernel<S, 1>);
  else if (nr == 2) go(subst_partials_kernel<S, 2>);
  else go(subst_partials_kernel<S, 4>);
  BCMG_CHECK_LAUNCH();
  return np;
}

// forward step: tmp = X_kk x_k; x_k = tmp; x[s0 + tc + r] -= L[tc + r, :] tmp
void subst_fwd(int dt, int64_t rows, int64_t tc, int64_t nrhs, const void* Xkk, int64_t ldxk, const void* Lk,
               int64_t ldl, void* xk, int64_t ldx, void* tmp, cudaStream_t st) {
  const int nr = subst_nr(nrhs);
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    launch_subst_gemv<S>(nr, static_cast<const S*>(Xkk), ldxk, static_cast<const S*>(xk), ldx, static_cast<S*>(tmp),
                         tc, tc, (int)tc, (int)nrhs, 0, 1.0, 0, st);
    launch_subst_gemv<S>(nr, static_cast<const S*>(Lk), ldl, static_cast<const S*>(tmp), tc, static_cast<S*>(xk), ldx,
                         rows, (int)tc, (int)nrhs, tc, -1.0, 1, st);
  });
}

// backward step: z = x_k - L[tc:, :]^H x[s0 + tc:]; x_k = X_kk^H z
void subst_bwd(int dt, int64_t rows, int64_t tc, int64_t nrhs, const void* Xkk, int64_t ldxk, const void* Lk,
               int64_t ldl, void* xk, int64_t ldx, void* parts, void* tmp, cudaStream_t st) {
  const int nr = subst_nr(nrhs);
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    const S* L = static_cast<const S*>(Lk);
    S* x = static_cast<S*>(xk);
    S* z = static_cast<S*>(tmp);
    const int np = launch_subst_partials<S>(nr, L + tc, ldl, x + tc, ldx, rows - tc, (int)tc, (int)nrhs, parts, st);
    subst_reduce_kernel<S><<<ew_grid(tc * nrhs), 256, 0, st>>>(x, ldx, parts, np, (int)tc, (int)nrhs, z, tc, 0);
    BCMG_CHECK_LAUNCH();
    const int nd = launch_subst_partials<S>(nr, static_cast<const S*>(Xkk), ldxk, z, tc, tc, (int)tc, (int)nrhs, parts,
                                            st);
    subst_reduce_kernel<S><<<ew_grid(tc * nrhs), 256, 0, st>>>(x, ldx, parts, nd, (int)tc, (int)nrhs, x, ldx, 1);
    BCMG_CHECK_LAUNCH();
  });
}

// ============================================================== elementwise helpers
template <class S>
__global__ void copy2d_kernel(const S* __restrict__ src, int64_t lds, S* __restrict__ dst, int64_t ldd, int64_t rows,
                              int64_t cols, int conj, const int* info) {
  if (ld_flag(info)) return;
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % rows, c = idx / rows;
    S v = src[r + c * lds];
    if (conj) v = from_c<S>(cconj(to_c(v)));
    dst[r + c * ldd] = v;
  }
}

static unsigned ew_grid(int64_t total) {
  int64_t g = (total + 255) / 256;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms() * 16));
}

void copy2d(int dt, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols, bool conj,
            const int* info, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    copy2d_kernel<S><<<ew_grid(rows * cols), 256, 0, st>>>(static_cast<const S*>(src), lds, static_cast<S*>(dst), ldd,
                                                           rows, cols, conj ? 1 : 0, info);
  });
  BCMG_CHECK_LAUNCH();
}

template <class S>
__global__ void conj2d_kernel(S* a, int64_t lda, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % rows, c = idx / rows;
    a[r + c * lda] = from_c<S>(cconj(to_c(a[r + c * lda])));
  }
}

void conj2d(int dt, void* a, int64_t lda, int64_t rows, int64_t cols, cudaStream_t st) {
  if (!dtype_complex(dt) || rows <= 0 || cols <= 0) return;
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    conj2d_kernel<S><<<ew_grid(rows * cols), 256, 0, st>>>(static_cast<S*>(a), lda, rows, cols);
  });
  BCMG_CHECK_LAUNCH();
}

template <class S>
__global__ void zero_upper_kernel(S* a, int64_t lda, int64_t rows, int64_t cols, int64_t off) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % rows, c = idx / rows;
    if (r < c + off) a[r + c * lda] = from_c<S>(make_double2(0, 0));
  }
}

void zero_upper(int dt, void* a, int64_t lda, int64_t rows, int64_t cols, int64_t off, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    zero_upper_kernel<S><<<ew_grid(rows * cols), 256, 0, st>>>(static_cast<S*>(a), lda, rows, cols, off);
  });
  BCMG_CHECK_LAUNCH();
}

template <class S>
__global__ void conj_transpose_kernel(const S* __restrict__ src, int64_t lds, S* __restrict__ dst, int64_t ldd,
                                      int64_t rows, int64_t cols) {
  // dst (rows x cols) = src^H, src is cols x rows; 32x32 tiles through shared memory
  __shared__ double2 t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    // read src rows (c0 + x), cols (r0 + y): coalesced along src rows
    const int64_t sr = c0 + threadIdx.x, sc = r0 + y;
    if (sr < cols && sc < rows) t[y][threadIdx.x] = to_c(src[sr + sc * lds]);
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t dr = r0 + threadIdx.x, dc = c0 + y;
    if (dr < rows && dc < cols) dst[dr + dc * ldd] = from_c<S>(cconj(t[threadIdx.x][y]));
  }
}

void conj_transpose(int dt, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols,
                    cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32)), block(32, 8);
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    conj_transpose_kernel<S><<<grid, block, 0, st>>>(static_cast<const S*>(src), lds, static_cast<S*>(dst), ldd, rows,
                                                     cols);
  });
  BCMG_CHECK_LAUNCH();
}

// Mirror scatter of potri's product blocks: src (rows x cols, lds) holds
// columns of logical device d's shard (local column c = global column
// ((c / T) * D + d) * T + c % T); dst(global column of c, i) = conj(src(i, c)).
template <class S>
__global__ void ct_scatter_kernel(const S* __restrict__ src, int64_t lds, int64_t rows, int64_t cols, S* dst,
                                  int64_t ldd, int64_t T, int D, int d) {
  __shared__ double2 t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, c = c0 + y;
    if (i < rows && c < cols) t[y][threadIdx.x] = to_c(src[i + c * lds]);
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + threadIdx.x, i = i0 + y;
    if (i < rows && c < cols) {
      const int64_t g = ((c / T) * D + d) * T + c % T;
      dst[g + i * ldd] = from_c<S>(cconj(t[threadIdx.x][y]));
    }
  }
}

void ct_scatter(int dt, const void* src, int64_t lds, int64_t rows, int64_t cols, void* dst, int64_t ldd, int64_t T,
                int D, int d, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32)), block(32, 8);
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    ct_scatter_kernel<S><<<grid, block, 0, st>>>(static_cast<const S*>(src), lds, rows, cols, static_cast<S*>(dst),
                                                 ldd, T, D, d);
  });
  BCMG_CHECK_LAUNCH();
}

template <class S>
__global__ void realify_diag_kernel(S* a, int64_t lda, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = to_c(a[i + i * lda]);
    a[i + i * lda] = from_c<S>(make_double2(v.x, 0.0));
  }
}

void realify_diag(int dt, void* a, int64_t lda, int64_t n, cudaStream_t st) {
  if (!dtype_complex(dt) || n <= 0) return;
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    realify_diag_kernel<S><<<ew_grid(n), 256, 0, st>>>(static_cast<S*>(a), lda, n);
  });
  BCMG_CHECK_LAUNCH();
}

template <class S>
__global__ void reduce_parts_kernel(const S* __restrict__ parts, int64_t pstride, int nparts, S* dst, int64_t ldd,
                                    int64_t rows, int64_t cols, double alpha, double beta) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % rows, c = idx / rows;
    double2 acc = make_double2(0, 0);
    for (int s = 0; s < nparts; ++s) {  // fixed order: deterministic
      double2 v = to_c(parts[s * pstride + r + c * rows]);
      acc.x += v.x;
      acc.y += v.y;
    }
    double2 o = beta != 0.0 ? to_c(dst[r + c * ldd]) : make_double2(0, 0);
    dst[r + c * ldd] = from_c<S>(make_double2(beta * o.x + alpha * acc.x, beta * o.y + alpha * acc.y));
  }
}

void reduce_parts(int dt, const void* parts, int64_t part_stride, int nparts, void* dst, int64_t ldd, int64_t rows,
                  int64_t cols, double alpha, cudaStream_t st, double beta) {
  if (rows <= 0 || cols <= 0) return;
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    reduce_parts_kernel<S><<<ew_grid(rows * cols), 256, 0, st>>>(static_cast<const S*>(parts), part_stride, nparts,
                                                                 static_cast<S*>(dst), ldd, rows, cols, alpha, beta);
  });
  BCMG_CHECK_LAUNCH();
}

// ============================================================== cycle rotation
// Each thread owns one vec-byte lane of one cycle and carries it around the
// whole cycle: new[c1] = old[c0], ..., new[c0] = old[c_{m-1}] (the rotation
// direction of layout.py:236-250).  Every address is read exactly once and
// then written once by the same thread, so there is no hazard between
// threads and no staging buffer beyond registers; loads of the next UNROLL
// members are issued before the stores (each is still read before written).
template <class W, int UNROLL>
__global__ void __launch_bounds__(256) rotate_kernel(RotateJob j) {
  for (int64_t lane = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; lane < j.total_lanes;
       lane += (int64_t)gridDim.x * blockDim.x) {
    // cycle owning this lane
    int64_t lo = 0, hi = j.n_cycles;  // lane_pref[lo] <= lane < lane_pref[hi]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(j.lane_pref + mid) <= lane) lo = mid; else hi = mid;
    }
    const int64_t c = lo;
    const int64_t off = (lane - __ldg(j.lane_pref + c)) * (int64_t)sizeof(W);
    const int64_t b = __ldg(j.offsets + c), e = __ldg(j.offsets + c + 1);
    W carry = *reinterpret_cast<const W*>(__ldg(j.addr + b) + off);
    int64_t i = b + 1;
    for (; i + UNROLL <= e; i += UNROLL) {
      W v[UNROLL];
      W* p[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        p[u] = reinterpret_cast<W*>(__ldg(j.addr + i + u) + off);
        v[u] = *p[u];
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        *p[u] = carry;
        carry = v[u];
      }
    }
    for (; i < e; ++i) {
      W* p = reinterpret_cast<W*>(__ldg(j.addr + i) + off);
      W v = *p;
      *p = carry;
      carry = v;
    }
    *reinterpret_cast<W*>(__ldg(j.addr + b) + off) = carry;
  }
  if (j.sys_fence) __threadfence_system();  // peer stores performed before the stream moves on
}

// Bulk-copy rotation (16-byte aligned segments): work item = (cycle, chunk of
// RB_CH bytes at the same offset in every member).  One thread per CTA drives
// the copy engine: cp.async.bulk loads of up to RB_G members into shared
// memory (one mbarrier transaction), then cp.async.bulk stores of each member
// into its successor.  Cycles longer than RB_G are walked in groups with the
// last member's chunk carried in a spare slot; every address is read (load
// completed) before it is written, and items touch disjoint bytes.  Three
// CTAs per SM keep ~200 KB per SM in flight.
constexpr int RB_CH = 8192, RB_G = 8;
constexpr size_t RB_SMEM = (size_t)(RB_G + 1) * RB_CH;

__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, unsigned src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(32) rotate_bulk_kernel(RotateJob j) {
  extern __shared__ __align__(128) unsigned char rb_smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x != 0) return;
  mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  const unsigned base = smem_u32(rb_smem);
  unsigned phase = 0;
  for (int64_t item = blockIdx.x; item < j.total_lanes; item += gridDim.x) {
    int64_t lo = 0, hi = j.n_cycles;  // chunk prefix: lane_pref[lo] <= item < lane_pref[hi]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(j.lane_pref + mid) <= item) lo = mid; else hi = mid;
    }
    const int64_t c = lo;
    const int64_t off = (item - __ldg(j.lane_pref + c)) * RB_CH;
    const unsigned len = (unsigned)min((int64_t)RB_CH, __ldg(j.seg_bytes + c) - off);
    const int64_t b = __ldg(j.offsets + c), m = __ldg(j.offsets + c + 1) - b;
    auto at = [&](int64_t i) { return reinterpret_cast<char*>(__ldg(j.addr + b + i)) + off; };
    int carry = -1;  // slot holding old[c_{i0-1}]
    for (int64_t i0 = 0; i0 < m; i0 += RB_G) {
      const int g = (int)min((int64_t)RB_G, m - i0);
      auto slot = [&](int k) { return (carry >= 0 && k >= carry) ? k + 1 : k; };
      mbar_expect_tx(&bar, (unsigned)g * len);
      for (int k = 0; k < g; ++k) bulk_g2s(base + slot(k) * RB_CH, at(i0 + k), len, &bar);
      mbar_wait(&bar, phase);
      phase ^= 1;
      if (carry >= 0) bulk_s2g(at(i0), base + carry * RB_CH, len);
      for (int k = 0; k + 1 < g; ++k) bulk_s2g(at(i0 + k + 1), base + slot(k) * RB_CH, len);
      carry = slot(g - 1);
      if (i0 + g == m) bulk_s2g(at(0), base + carry * RB_CH, len);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // slots reusable
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

int64_t rotate_bulk_chunk() { return RB_CH; }

void rotate_cycles(const RotateJob& j, cudaStream_t st) {
  if (j.total_lanes <= 0) return;
  if (j.bulk) {
    set_smem(rotate_bulk_kernel, RB_SMEM);
    const unsigned grid = (unsigned)std::min<int64_t>(j.total_lanes, (int64_t)num_sms() * 3);
    rotate_bulk_kernel<<<grid, 32, RB_SMEM, st>>>(j);
    BCMG_CHECK_LAUNCH();
    return;
  }
  const unsigned grid = (unsigned)std::min<int64_t>((j.total_lanes + 255) / 256, (int64_t)num_sms() * 8);
  if (j.vec == 16) rotate_kernel<uint4, 4><<<grid, 256, 0, st>>>(j);
  else if (j.vec == 8) rotate_kernel<uint2, 4><<<grid, 256, 0, st>>>(j);
  else rotate_kernel<unsigned, 4><<<grid, 256, 0, st>>>(j);
  BCMG_CHECK_LAUNCH();
}


// In-place Hermitian completion of a diagonal block: a(r,c) = conj(a(c,r))
// for r < c, diagonal made exactly real (reference solvers.py:577-583).
template <class S>
__global__ void mirror_diag_kernel(S* a, int64_t lda, int64_t n) {
  const int64_t total = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % n, c = idx / n;
    if (r < c) a[r + c * lda] = from_c<S>(cconj(to_c(a[c + r * lda])));
    else if (r == c) a[r + c * lda] = from_c<S>(make_double2(to_c(a[r + c * lda]).x, 0.0));
  }
}

void mirror_diag(int dt, void* a, int64_t lda, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    mirror_diag_kernel<S><<<ew_grid(n * n), 256, 0, st>>>(static_cast<S*>(a), lda, n);
  });
  BCMG_CHECK_LAUNCH();
}

// ============================================================== chunk copies
template <class W>
__global__ void __launch_bounds__(256) chunk_copy_kernel(const uint64_t* __restrict__ src,
                                                         const uint64_t* __restrict__ dst, int n, int64_t soff,
                                                         int64_t doff, int64_t lanes) {
  for (int i = blockIdx.y; i < n; i += gridDim.y) {
    const W* s = reinterpret_cast<const W*>(__ldg(src + i) + soff);
    W* d = reinterpret_cast<W*>(__ldg(dst + i) + doff);
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < lanes; l += (int64_t)gridDim.x * blockDim.x)
      d[l] = s[l];
  }
}

void chunk_copy(const uint64_t* src, const uint64_t* dst, int n, int64_t soff, int64_t doff, int64_t len, int vec,
                cudaStream_t st) {
  if (n <= 0 || len <= 0) return;
  const int64_t lanes = len / vec;
  const unsigned gy = (unsigned)std::min(n, 1024);
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((lanes + 255) / 256,
                                                                       (int64_t)num_sms() * 8 / gy + 1));
  dim3 grid(gx, gy);
  if (vec == 16) chunk_copy_kernel<uint4><<<grid, 256, 0, st>>>(src, dst, n, soff, doff, lanes);
  else if (vec == 8) chunk_copy_kernel<uint2><<<grid, 256, 0, st>>>(src, dst, n, soff, doff, lanes);
  else chunk_copy_kernel<unsigned><<<grid, 256, 0, st>>>(src, dst, n, soff, doff, lanes);
  BCMG_CHECK_LAUNCH();
}

// ============================================================== FP64 peak probe
// Register-resident DMMA loop (8 independent accumulators per warp, 16 warps
// per SM): the FP64 tensor roofline denominator, measured live by bench.py.
__global__ void __launch_bounds__(512) dmma_peak_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

// ============================================================== peer-memory flags
// One thread stores v to n (possibly peer, over NVLink) 32-bit words after
// everything earlier on the stream; the fence makes the stream's earlier
// peer-memory writes (fused GEMM fan-out) visible before the flag.
__global__ void signal_kernel(PtrList addrs, unsigned v) {
  __threadfence_system();
  for (int i = 0; i < addrs.n; ++i) *reinterpret_cast<volatile unsigned*>(addrs.p[i]) = v;
  __threadfence_system();
}

void stream_signal(cudaStream_t st, void* const* addrs, int n, unsigned v) {
  if (n <= 0) return;
  PtrList l{};
  l.n = std::min(n, (int)(sizeof(l.p) / sizeof(l.p[0])));
  for (int i = 0; i < l.n; ++i) l.p[i] = addrs[i];
  signal_kernel<<<1, 1, 0, st>>>(l, v);
  BCMG_CHECK_LAUNCH();
}

// ============================================================== synthetic SPD input
// A = (R + R^H)/2 + shift*I with R ~ U[-1,1) (+ i U[-1,1) for complex): the
// value of the unordered pair {i, j} is a splitmix64 hash of (seed, lo, hi),
// so any row block can be generated independently and A is exactly
// Hermitian; the diagonal is real.  Row-major row block: element (row0 + r, j)
// at p[r * ld + j].  (the BASELINE synthetic inputs.)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double unit_pm1(uint64_t h) { return (double)(h >> 11) * 0x1.0p-52 - 1.0; }

template <class S>
__global__ void gen_spd_kernel(S* p, int64_t ld, int64_t n, int64_t row0, int64_t rows, uint64_t seed,
                               double shift) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const int64_t i = row0 + r;
    const uint64_t lo = (uint64_t)(i < j ? i : j), hi = (uint64_t)(i < j ? j : i);
    const uint64_t h = mix64(seed ^ mix64(lo * 0x100000001b3ull + hi));
    double2 v = make_double2(unit_pm1(h), 0.0);
    if (Traits<S>::cplx) v.y = (i == j) ? 0.0 : (i > j ? 1.0 : -1.0) * unit_pm1(mix64(h));
    if (i == j) v.x += shift;
    p[r * ld + j] = from_c<S>(v);
  }
}

void generate_spd(int dt, void* p, int64_t ld, int64_t n, int64_t row0, int64_t rows, uint64_t seed, double shift,
                  cudaStream_t st) {
  if (rows <= 0 || n <= 0) return;
  dispatch_dtype(dt, [&](auto s) {
    using S = decltype(s);
    gen_spd_kernel<S><<<num_sms() * 8, 256, 0, st>>>(static_cast<S*>(p), ld, n, row0, rows, seed, shift);
  });
  BCMG_CHECK_LAUNCH();
}

double measure_dmma_peak(cudaStream_t st) {
  double* out = nullptr;
  BCMG_CUDA(cudaMalloc(&out, 4096 * sizeof(double)));
  cudaEvent_t e0, e1;
  BCMG_CUDA(cudaEventCreate(&e0));
  BCMG_CUDA(cudaEventCreate(&e1));
  const int grid = num_sms(), iters = 40000;
  dmma_peak_kernel<<<grid, 512, 0, st>>>(out, 1000);  // warm-up
  BCMG_CHECK_LAUNCH();
  BCMG_CUDA(cudaEventRecord(e0, st));
  dmma_peak_kernel<<<grid, 512, 0, st>>>(out, iters);
  BCMG_CHECK_LAUNCH();
  BCMG_CUDA(cudaEventRecord(e1, st));
  BCMG_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  BCMG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid * 16;
  return flops / (ms * 1e-3) / 1e12;
}
}  // namespace bcmg
