// Internal launcher interface between the drivers (solver.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

#include "gemm.cuh"

namespace bcmg {

struct PtrList {  // kernel-parameter array of device addresses
  void* p[16];
  int n;
};
long long launch_count();
double measure_dmma_peak(cudaStream_t st);  // TFLOP/s
// Synthetic Hermitian positive-definite row block (see gen_spd_kernel).
void generate_spd(int dt, void* p, int64_t ld, int64_t n, int64_t row0, int64_t rows, uint64_t seed, double shift,
                  cudaStream_t st);

// C := alpha*op(A)*op(B) + beta*C, any dtype (dt), any shape; dispatches to
// the cp.async DMMA kernel when the operands qualify, else the REG kernel.
// gemm() with a kernel choice that does not depend on N (device-count invariant bits)
void gemm_shape_fixed(int dt, int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                      const int* info, cudaStream_t st);
void gemm(int dt, int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
          const int* info, cudaStream_t st);

// Split-K GEMM into `parts` (np slabs of M x N, ld M; np <= max_parts chosen
// for >= 2 waves); returns np.  Sum the slabs with reduce_parts.
int gemm_splitk(int dt, int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, void* parts,
                int max_parts, cudaStream_t st);

// Trailing update for potrf step (see trail_kernel).
void trailing_update(int dt, const TrailParams& p, const int* info, cudaStream_t st);
// complex trailing update through the real tensor-core kernels: usable for this
// dtype / panel height?  The panel must then be expanded with expand_panel:
// P (rows x K complex, ld rows) is followed in memory by -iP, and PB receives
// the planar [Re P | Im P] (rows x 2K real, ld rows).
bool complex_embed_ok(int dt, int64_t panel_rows, int64_t T);
void expand_panel(int dt, void* P, void* PB, int64_t rows, int64_t K, cudaStream_t st);
// complex GEMM (gemm() semantics) as one real tensor-core GEMM (FP64 TMA for
// complex128, tcgen05 3xTF32 for complex64) on the embedded operands
// [Ahat | -i Ahat] and [Re Bhat | -Im Bhat], materialised in `scratch`
// (gemm_cplx_embed_bytes).  Returns false (nothing launched) when the shape or
// the operands do not qualify; the caller then uses gemm().  always: skip the
// fill-the-GPU size heuristic (callers whose N depends on the device count
// need the same arithmetic for every shape).
size_t gemm_cplx_embed_bytes(int dt, int64_t M, int64_t N, int64_t K);
bool gemm_cplx_embed(int dt, int64_t M, int64_t N, int64_t K, const Operand& A, const Operand& B, const Epilogue& ep,
                     void* scratch, size_t scratch_bytes, const int* info, cudaStream_t st, bool always = false);
// Several column groups B_i (ncols[i] columns each) against one A, outputs
// concatenated in ep.C (ld ep.ldc): A is gathered (and split) once, the
// groups' columns chunk by chunk (`chunk` columns per GEMM; scratch >=
// gemm_cplx_embed_bytes(dt, M, chunk, K)).  False: nothing launched.
bool gemm_cplx_embed_multi(int dt, int64_t M, int64_t K, const Operand& A, const Operand* Bs, const int64_t* ncols,
                           void* const* Cs, int ngroups, const Epilogue& ep, void* scratch, size_t scratch_bytes,
                           cudaStream_t st);
bool gemm_cplx_embed_grouped(int dt, int64_t M, int64_t K, const Operand& A, const Operand* Bs, const int64_t* ncols,
                             int ngroups, const Epilogue& ep, void* scratch, size_t scratch_bytes, int64_t chunk,
                             cudaStream_t st);

// tf32 hi / lo pre-split (see split_tf32_kernel) and the tcgen05 GEMM on the
// split planes.  split_ld: the K-major leading dimension for Kx columns.
int64_t split_ld(int64_t kx);
// kw: columns written per row (Kx, zero-padded; default kp); kp: row stride of the planes
void split_tf32(int mode, const void* src, int64_t ld, int64_t rows, int64_t Kx, int64_t kc, float* hi, float* lo,
                int64_t kp, cudaStream_t st, int64_t kw = -1);
// potrf on the pre-split tcgen05 path updates the trailing matrix once per
// PAIR of panels (K = 2T) when the tile is narrow (see Session::potrf)
bool pair_panels(int dt, int64_t T);
void tck_gemm(int64_t M, int64_t N, int64_t K, const float* ah, const float* al, const float* bh, const float* bl,
              int64_t kp, float* C, int64_t ldc, float alpha, float beta, const int* info, cudaStream_t st,
              const Epilogue* fan_src = nullptr);
bool tc_presplit_enabled();
void reserve_split_scratch(cudaStream_t st, size_t bytes);
size_t split_scratch_held(cudaStream_t st);  // bytes the scratch of st holds
void release_split_scratch(cudaStream_t st);  // before the stream is destroyed
size_t split_scratch_bytes(int dt, int64_t M, int64_t N, int64_t K);  // a GEMM's tf32 split planes

// Diagonal tile: in-place lower Cholesky of the n x n block at A (lda) and
// X := L^-1 (n x n, ldx, zero upper).  goff = global column of the block's
// first column; on a non-positive pivot writes the 1-based global pivot to
// *info and leaves the columns before it factored.  W is n x n scratch.
void diag_factor(int dt, void* A, int64_t lda, void* X, int64_t ldx, void* W, int64_t n, int64_t goff, int* info,
                 cudaStream_t st);

// dst(i,j) = src(i,j) (optionally conjugated), rows x cols, column-major.
void copy2d(int dt, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols, bool conj,
            const int* info, cudaStream_t st);

// In-place conjugation of a rows x cols block (complex only; no-op for real).
void conj2d(int dt, void* a, int64_t lda, int64_t rows, int64_t cols, cudaStream_t st);

// Zero the strict upper triangle (row < col + off) of a rows x cols block.
void zero_upper(int dt, void* a, int64_t lda, int64_t rows, int64_t cols, int64_t off, cudaStream_t st);

// Mirror: a(r, c) = conj(src(c, r)) for the block; diagonal forced real when diag.
void conj_transpose(int dt, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols,
                    cudaStream_t st);
// potri mirror: dst(global column of local column c of device d, i) = conj(src(i, c))
void ct_scatter(int dt, const void* src, int64_t lds, int64_t rows, int64_t cols, void* dst, int64_t ldd, int64_t T,
                int D, int d, cudaStream_t st);
void realify_diag(int dt, void* a, int64_t lda, int64_t n, cudaStream_t st);
void mirror_diag(int dt, void* a, int64_t lda, int64_t n, cudaStream_t st);

// potrs sweeps for N_RHS <= 4 (bandwidth kernels, fixed-order sums).  rows =
// n - start_k; Lk = tile k's column block from row start_k (ld ldl); xk = x +
// start_k.  parts: subst_parts_bytes(T, nrhs) (partials + a tile of z / tmp).
bool subst_gemv_ok(int dt, int64_t nrhs);
size_t subst_parts_bytes(int64_t n, int64_t T, int64_t nrhs);
void subst_fwd(int dt, int64_t rows, int64_t tc, int64_t nrhs, const void* Xkk, int64_t ldxk, const void* Lk,
               int64_t ldl, void* xk, int64_t ldx, void* tmp, cudaStream_t st);
void subst_bwd(int dt, int64_t rows, int64_t tc, int64_t nrhs, const void* Xkk, int64_t ldxk, const void* Lk,
               int64_t ldl, void* xk, int64_t ldx, void* parts, void* tmp, cudaStream_t st);

// Split-K deterministic reduction: dst = beta*dst + alpha*sum_s part[s] (fixed order).
void reduce_parts(int dt, const void* parts, int64_t part_stride, int nparts, void* dst, int64_t ldd, int64_t rows,
                  int64_t cols, double alpha, cudaStream_t st, double beta = 1.0);

// ----------------------------------------------------------------- redistribution
// Segment-level plan of the contiguous <-> cyclic permutation (layout.py:126-256).
struct SegPlan {
  int64_t seg;                        // columns per segment (T when tile-aligned, else gcd-derived, >= 1)
  std::vector<int64_t> members;       // segment positions, cycles concatenated in rotation order
  std::vector<int64_t> offsets;       // CSR offsets into members, size n_cycles + 1
  std::vector<int64_t> seg_cols;      // columns of each cycle's segments
};
// Column-level plan exactly as the reference (dest_of + cycles).
void build_dest(int64_t n_cols, int64_t tile, int ndev, int64_t* dest);
void decompose(int64_t n, const int64_t* dest, std::vector<int64_t>& members, std::vector<int64_t>& offsets);
void invert_cycles(std::vector<int64_t>& members, const std::vector<int64_t>& offsets);
SegPlan segment_plan(int64_t n_cols, int64_t tile, int ndev, bool inverse);
std::vector<int64_t> column_counts(int64_t n_cols, int64_t tile, int ndev);

// Rotate every cycle in place: members are absolute device addresses
// (segments of seg_bytes[c] bytes), data moved in vec-byte lanes.
struct RotateJob {
  const uint64_t* addr;      // device: member addresses, cycles concatenated
  const int64_t* offsets;    // device: CSR, n_cycles + 1
  const int64_t* lane_pref;  // device: prefix sum of lanes (bulk: chunks) per cycle, n_cycles + 1
  const int64_t* seg_bytes;  // device: bytes per segment of each cycle
  int64_t n_cycles, total_lanes;
  int vec;                   // 16, 8 or 4
  int bulk;                  // 1: cp.async.bulk chunks of rotate_bulk_chunk() bytes (vec == 16)
  int sys_fence = 0;         // 1: members include peer (NVLink) memory: system-scope fence at the end
};
void rotate_cycles(const RotateJob& j, cudaStream_t st);
int64_t rotate_bulk_chunk();

// n independent copies of len bytes: dst[i] + doff <- src[i] + soff (device
// address tables), vec-byte lanes.
void chunk_copy(const uint64_t* src, const uint64_t* dst, int n, int64_t soff, int64_t doff, int64_t len, int vec,
                cudaStream_t st);

}  // namespace bcmg
