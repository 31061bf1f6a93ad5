/*
 * bcmg_b200.h -- C ABI of the B200-native (sm_100a) multi-GPU Cholesky path.
 *
 * This is the drop-in boundary for the path named by BASELINE.json's north
 * star: the row-sharded -> 1D block-cyclic column redistribution and the
 * tiled potrf + potrs / potri that run on that layout.  It replaces, entry by
 * entry:
 *
 *   bcmg_open / bcmg_close      reference pkg/frontend/src/api.ts:44-62
 *                               (session = device binding + NCCL communicator
 *                               instead of a scratch directory)
 *   bcmg_last_error             api.ts:35-42; codes = errors.ts:9-23 (same
 *                               numbers, plus BCMG_ERR_CUDA)
 *   bcmg_potrs                  api.ts:137-154 -> solvers.py:931-985
 *                               (solve_positive_definite pipeline)
 *   bcmg_potri                  api.ts:157-165 -> solvers.py:988-1016
 *                               (invert_positive_definite pipeline)
 *   bcmg_syevd                  api.ts (bcmg_syevd) ->
 *                               solvers.py:1019-1043 (eigh_hermitian pipeline)
 *   bcmg_syevd_cyclic           solvers.py:862-910 (syevd on the cyclic layout)
 *   bcmg_redistribute           solvers.py:262-273 (redistribute_in/out)
 *                               -> layout.py:191-256 (execute_plan)
 *   bcmg_potrf                  solvers.py:341-406 (potrf, LAPACK info)
 *   bcmg_potrs_factored         solvers.py:430-474 (potrs on the factor)
 *   bcmg_potri_factored         solvers.py:487-594 (potri on the factor)
 *   bcmg_build_permutation      layout.py:126-145
 *   bcmg_decompose_cycles       layout.py:148-172
 *   bcmg_invert_cycles          layout.py:175-183
 *   bcmg_column_counts          layout.py:82-95
 *
 * Conventions
 *   - dtype codes follow the reference's ElementType (core.py:69-72):
 *     0 real32, 1 real64, 2 complex64, 3 complex128 (interleaved re, im).
 *   - Matrices are column-major.  A distributed matrix of order n is held as
 *     `ndev` logical-device shards, shard d being n rows x counts[d] columns
 *     (bcmg_column_counts), leading dimension n.  Each process passes the
 *     shards of ITS logical devices: ndev/world of them, devices
 *     rank*ndev/world .. (rank+1)*ndev/world-1.  With world == 1 all logical
 *     devices live on the session's GPU ("virtual devices").
 *   - All data pointers are device pointers on the session's GPU; `stream`
 *     is the caller's cudaStream_t (NULL = legacy default stream).  Work is
 *     ordered after prior work on `stream` and `stream` is ordered after it;
 *     calls returning `info` synchronise on `stream`.
 *   - A session is single-caller: a call that overlaps another call on the
 *     same session fails with BCMG_ERR_CONFIG (reference ConcurrentCallError,
 *     runtime.py:449-466).
 *   - Return value: BCMG_OK or an error code; bcmg_last_error() /
 *     bcmg_last_error_message() describe the last failure on this thread.
 */
#ifndef BCMG_B200_H
#define BCMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BCMG_OK 0
#define BCMG_ERR_NOT_POSITIVE_DEFINITE 1
#define BCMG_ERR_CONFIG 2
#define BCMG_ERR_NO_CONVERGENCE 3
#define BCMG_ERR_OUT_OF_MEMORY 4
#define BCMG_ERR_CHECK_FAILED 5
#define BCMG_ERR_STALE_SESSION 6
#define BCMG_ERR_IO 7
#define BCMG_ERR_CUDA 8

#define BCMG_R32 0
#define BCMG_R64 1
#define BCMG_C64 2
#define BCMG_C128 3

/* redistribution direction */
#define BCMG_TO_CYCLIC 0   /* contiguous -> block-cyclic (redistribute_in)  */
#define BCMG_TO_CONTIG 1   /* block-cyclic -> contiguous (redistribute_out) */

/* pipeline flags */
#define BCMG_FLAG_ROW_SHARDED 1 /* shards are row blocks of a ROW-major matrix (the
                                   JAX P("x", None) layout): for complex Hermitian
                                   input the bytes hold conj(A); handled by solving
                                   conj(A) conj(x) = conj(b). */

typedef struct bcmg_session bcmg_session;

int bcmg_version(void);
int bcmg_last_error(void);
const char* bcmg_last_error_message(void);

/* ---- layout planning (host only, no GPU needed) ---- */
int bcmg_column_counts(int64_t n_cols, int64_t tile, int ndev, int64_t* counts /* [ndev] */);
int bcmg_build_permutation(int64_t n_cols, int64_t tile, int ndev, int64_t* dest_of /* [n_cols] */);
/* members: [n] (cycles concatenated, rotation order); offsets: [n+1] CSR */
int bcmg_decompose_cycles(int64_t n, const int64_t* dest_of, int64_t* members, int64_t* offsets,
                          int64_t* n_cycles);
int bcmg_invert_cycles(int64_t n_cycles, const int64_t* offsets, int64_t* members);
/* segment width S used by the device plan (S = T at tile-aligned shapes) and
   the number of moved columns */
int bcmg_segment_plan_info(int64_t n_cols, int64_t tile, int ndev, int64_t* seg_width, int64_t* n_cycles,
                           int64_t* moved_columns);

/* Per-process operation schedule of potrf (routine 0), potrs (routine 1) or
   potri (routine 2) for `world` processes holding ndev logical devices --
   exactly the sequence the drivers execute.  Each op is 7 int64: {kind,
   stream, k, a, b, root, elems}; kinds: 1 factor tile k, 2 broadcast panel k
   (root process, elems), 3 trailing update with panel k of tiles [a, b),
   4 copy panel k back, 5 end of step k, 6 forward step k, 7 backward step k,
   8 broadcast solution rows [a, b) (root, elems); potri: 9 finalise W_k
   (owner), 10 broadcast tile k rows [start_k, n) (root, elems), 11 add
   W_k's contribution to the local tiles < k, 12 product blocks (k, j <= k)
   of the local tiles, 13 gather those blocks on the owner of k (root; elems
   this process sends) and mirror them into tile k; streams: 0 crit, 1 bulk,
   2 comm.  Host only.  Pass ops = NULL to query *count. */
int bcmg_schedule(int routine, int64_t n, int64_t tile, int ndev, int world, int rank, int64_t nrhs, int64_t* ops,
                  int64_t cap, int64_t* count);

/* Cross-process redistribution plan: every segment move {src_pos, dst_pos,
   src_rank, dst_rank} (4 int64 each, segment = *seg_width columns) in the
   global order both sides of a send/recv pair use.  Host only. */
int bcmg_redistribute_plan(int64_t n_cols, int64_t tile, int ndev, int world, int direction, int64_t* seg_width,
                           int64_t* moves, int64_t cap, int64_t* count);

/* ---- sessions ---- */
int bcmg_nccl_unique_id(unsigned char* id /* [128] */);
/* In-process loopback transport id: sessions opened with the same id in ONE
   process (one host thread per rank, each with its own streams, normally all
   on one GPU) exchange data by event-ordered device-to-device copies instead
   of NCCL -- runs the multi-process drivers on a single GPU (tests). */
int bcmg_loopback_id(unsigned char* id /* [128] */);
int bcmg_open(int cuda_device, int rank, int world, const unsigned char* nccl_id /* NULL if world==1 */,
              bcmg_session** out);
int bcmg_close(bcmg_session* s);

/* ---- pipelines (the reference's FFI routines) ---- */
/* x overwrites b (n x nrhs, ldb, replicated on every process); A's shards are
   overwritten by the factor in block-cyclic order. *info = LAPACK pivot. */
int bcmg_potrs(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t nrhs, int64_t tile, int ndev,
               void* const* shards, void* b, int64_t ldb, int flags, int* info);
/* bcmg_potrs for one process and one device with A in pinned HOST memory
   (a_host, n x n column-major -- the row-major bytes of the drop-in call): A is
   copied into a_dev (device, n x n) tile column by tile column while the
   factorisation already runs on the arrived tiles (left-looking for the first
   quarter of the tiles, then a catch-up update and the right-looking
   schedule; float64), so the upload overlaps compute.  Same result contract
   as bcmg_potrs (agreement to rounding with it). */
int bcmg_potrs_streamed(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t nrhs, int64_t tile,
                        void* a_dev, const void* a_host, void* b, int64_t ldb, int flags, int* info);
/* A's shards (contiguous layout) are overwritten by the full Hermitian inverse,
   contiguous layout. */
int bcmg_potri(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t tile, int ndev, void* const* shards,
               int flags, int* info);

/* Hermitian eigendecomposition: eigenvalues ascending into w (device, n
   elements of the real type: float for dtype 0/2, double for 1/3); A's shards
   (contiguous layout) are overwritten by the eigenvectors, column j belonging
   to w[j], each scaled so that its first largest-magnitude component is real
   and positive (solvers.py:898-909).  Across processes the matrix is gathered and
   solved on rank 0 (same bits on every rank).  *info =
   BCMG_ERR_NO_CONVERGENCE (and the same return code) when the tridiagonal QL
   exceeds 30 iterations for one eigenvalue (solvers.py:806-811). */
int bcmg_syevd(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t tile, int ndev, void* const* shards,
               void* w, int flags, int* info);

/* ---- building blocks (the reference's solvers.py routines) ---- */
int bcmg_redistribute(bcmg_session* s, void* stream, int dtype, int64_t n_rows, int64_t n_cols, int64_t tile,
                      int ndev, void* const* shards, int direction);
int bcmg_potrf(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t tile, int ndev, void* const* shards,
               int* info);
int bcmg_potrs_factored(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t nrhs, int64_t tile, int ndev,
                        void* const* shards, void* b, int64_t ldb);
int bcmg_potri_factored(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t tile, int ndev,
                        void* const* shards);
/* syevd on the block-cyclic layout: shards in, eigenvectors out (column j of
   the cyclic layout = eigenvector j), eigenvalues into w as bcmg_syevd */
int bcmg_syevd_cyclic(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t tile, int ndev,
                      void* const* shards, void* w);

/* The DMMA GEMM every contraction of the path runs on:
   C := alpha * op(A) * op(B) + beta * C, column-major, op 0 = N, 1 = C (conj-
   transpose); op(A) is m x k, op(B) is k x n.  No session needed. */
int bcmg_gemm(void* stream, int dtype, int64_t m, int64_t n, int64_t k, double alpha, const void* a, int64_t lda,
              int op_a, const void* b, int64_t ldb, int op_b, double beta, void* c, int64_t ldc);

/* ---- measurement ---- */
/* milliseconds of the last pipeline call: [0] redistribute_in, [1] potrf,
   [2] potrs/potri(+redistribute_out), [3] total (CUDA events on `stream`) */
int bcmg_last_timings(bcmg_session* s, float* ms /* [4] */);
/* algorithmic bytes (read + write) moved by the last redistribution */
int64_t bcmg_last_moved_bytes(bcmg_session* s);

/* MPMD / isolated-namespace handle exchange (reference runtime.py:170-233
   HandleRegistry / _TokenChannel, publish_handle / open_handle :390-406):
   export any device address of this process as a 72-byte token (CUDA IPC
   handle of its allocation + the offset inside it); another process on the
   node opens the token into its own address space (NVLink peer memory on
   another GPU).  Opening is cached per allocation; a process cannot open its
   own tokens (CONFIG).  bcmg_ipc_close_all unmaps every opened token. */
#define BCMG_IPC_TOKEN_BYTES 72
int bcmg_ipc_export(const void* ptr, unsigned char* token /* [72] */);
int bcmg_ipc_open(const unsigned char* token /* [72] */, void** ptr);
int bcmg_ipc_close_all(void);
/* The stream-ordered flags of the peer hand-offs (cuStreamWriteValue32 /
   cuStreamWaitValue32 on a device word, e.g. an opened token): write v after
   everything earlier on `stream` (CONFIG if the driver refuses the address),
   or make `stream` wait until the word is >= v. */
int bcmg_stream_write_flag(void* stream, void* addr, unsigned v);
int bcmg_stream_wait_flag(void* stream, const void* addr, unsigned v);

/* Device workspace of one process for a pipeline (routine 1: potrs, 2:
   potri), excluding the shards: the exact bytes bcmg_potrs / bcmg_potri
   reserve before moving any data (reference solvers.py:279-308
   workspace_nbytes; the OUT_OF_MEMORY-before-movement contract of
   test_solvers.py:344-352).  Needs no GPU (148 SMs assumed without one). */
int bcmg_workspace_nbytes(int routine, int dtype, int64_t n, int64_t tile, int ndev, int world, int64_t nrhs,
                          int64_t* bytes);
/* device bytes the session's workspace holds now (grow-only buffers) */
int bcmg_session_workspace_bytes(bcmg_session* s, int64_t* bytes);

/* Per-kernel timing: when on, every launch of a kernel kind is bracketed by
   CUDA events on the stream it is launched on.  kind: 0 trailing update
   (DMMA GEMM), 1 panel TRSM, 2 diagonal factor+inverse, 3 cycle rotation.
   stats[4] = {launches, total ms, algorithmic work (flops; bytes for kind 3),
   max ms}; reading clears the record. */
int bcmg_set_profiling(bcmg_session* s, int on);
int bcmg_kernel_stats(bcmg_session* s, int kind, double* stats /* [4] */);
/* kernels launched by this library in this process so far */
int64_t bcmg_launch_count(void);
/* FP64 tensor-core (DMMA) throughput of a register-resident mma.sync loop on
   all SMs, TFLOP/s: the roofline denominator of the FP64 kernels */
int bcmg_measure_fp64_peak(int cuda_device, double* tflops);
/* Synthetic input: rows [row0, row0+rows) of the n x n
   Hermitian positive-definite A = (R + R^H)/2 + shift*I, R ~ U[-1,1)
   (+ i U[-1,1) for complex dtypes), written row-major: element (row0+r, j)
   at a[r*lda + j] (device).  Element {i,j} is a hash of (seed, min, max),
   so row blocks generated on different GPUs form one exact Hermitian A.
   Stream-ordered on `stream`. */
int bcmg_generate_spd(void* stream, int dtype, int64_t n, int64_t row0, int64_t rows, void* a, int64_t lda,
                      uint64_t seed, double shift);

#ifdef __cplusplus
}
#endif
#endif /* BCMG_B200_H */
