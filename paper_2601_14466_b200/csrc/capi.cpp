// extern "C" surface of libbcmg_b200.so (declared in include/bcmg_b200.h).
// Every entry point converts exceptions into the reference's stable error
// codes (pkg/frontend/src/errors.ts:9-23) and records a per-thread message.
#include <nccl.h>

#include <cstring>
#include <string>

#include "../../include/bcmg_b200.h"
#include "ops.h"
#include "comm.h"
#include "solver.h"

struct bcmg_session {
  bcmg::Session* impl;
};

namespace {
thread_local int g_err = BCMG_OK;
thread_local std::string g_msg;

int fail(int code, const std::string& msg) {
  g_err = code;
  g_msg = msg;
  return code;
}
int ok() {
  g_err = BCMG_OK;
  g_msg.clear();
  return BCMG_OK;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return ok();
  } catch (const bcmg::Error& e) {
    return fail(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return fail(BCMG_ERR_OUT_OF_MEMORY, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(BCMG_ERR_CONFIG, e.what());
  }
}

bcmg::Session* live(bcmg_session* s) {
  if (!s || !s->impl) throw bcmg::Error(BCMG_ERR_STALE_SESSION, "no open session");
  return s->impl;
}

// Single-caller contract (reference runtime.py:449-466).
struct Entry {
  bcmg::Session* s;
  explicit Entry(bcmg::Session* s_, void* stream) : s(s_) {
    bool expected = false;
    if (!s->busy.compare_exchange_strong(expected, true))
      throw bcmg::Error(BCMG_ERR_CONFIG, "concurrent call on a single-caller session");
    s->begin(static_cast<cudaStream_t>(stream));
  }
  ~Entry() { s->busy.store(false); }
};

void check_common(int dtype, int ndev, void* const* shards) {
  if (bcmg::dtype_size(dtype) == 0) throw bcmg::Error(BCMG_ERR_CONFIG, "unknown element-type code " + std::to_string(dtype));
  if (ndev < 1) throw bcmg::Error(BCMG_ERR_CONFIG, "need at least one device");
  if (!shards) throw bcmg::Error(BCMG_ERR_CONFIG, "null shard table");
}

// Conjugates a complex right-hand side for the row-sharded pipeline and
// restores it if the call fails before the solve completes, so the caller's b
// is never left conjugated on an error path.
struct ConjGuard {
  int dt;
  void* b;
  int64_t ldb, n, nrhs;
  cudaStream_t st;
  bool armed = false;
  ConjGuard(bool on, int dt_, void* b_, int64_t ldb_, int64_t n_, int64_t nrhs_, cudaStream_t st_)
      : dt(dt_), b(b_), ldb(ldb_), n(n_), nrhs(nrhs_), st(st_), armed(on) {
    if (armed) bcmg::conj2d(dt, b, ldb, n, nrhs, st);
  }
  void finish() {  // the solution is conjugated back as part of the result
    if (armed) bcmg::conj2d(dt, b, ldb, n, nrhs, st);
    armed = false;
  }
  ~ConjGuard() {
    if (!armed) return;
    try {
      bcmg::conj2d(dt, b, ldb, n, nrhs, st);
      cudaStreamSynchronize(st);
    } catch (...) {
    }
  }
};

void finish_timings(bcmg::Session* s, bool has_redist_out) {
  (void)has_redist_out;
  BCMG_CUDA(cudaEventSynchronize(s->ev_time[bcmg::T_SOLVE]));
  float a = 0, b = 0, c = 0;
  BCMG_CUDA(cudaEventElapsedTime(&a, s->ev_time[bcmg::T_BEGIN], s->ev_time[bcmg::T_REDIST]));
  BCMG_CUDA(cudaEventElapsedTime(&b, s->ev_time[bcmg::T_REDIST], s->ev_time[bcmg::T_POTRF]));
  BCMG_CUDA(cudaEventElapsedTime(&c, s->ev_time[bcmg::T_POTRF], s->ev_time[bcmg::T_SOLVE]));
  s->phase_ms[0] = a;
  s->phase_ms[1] = b;
  s->phase_ms[2] = c;
  s->phase_ms[3] = a + b + c;
}
}  // namespace

extern "C" {

int bcmg_version(void) { return 1; }
int bcmg_last_error(void) { return g_err; }
const char* bcmg_last_error_message(void) { return g_msg.c_str(); }

int bcmg_column_counts(int64_t n_cols, int64_t tile, int ndev, int64_t* counts) {
  return guarded([&] {
    auto c = bcmg::column_counts(n_cols, tile, ndev);
    std::memcpy(counts, c.data(), c.size() * sizeof(int64_t));
  });
}

int bcmg_build_permutation(int64_t n_cols, int64_t tile, int ndev, int64_t* dest_of) {
  return guarded([&] {
    bcmg::column_counts(n_cols, tile, ndev);  // validates
    bcmg::build_dest(n_cols, tile, ndev, dest_of);
  });
}

int bcmg_decompose_cycles(int64_t n, const int64_t* dest_of, int64_t* members, int64_t* offsets, int64_t* n_cycles) {
  return guarded([&] {
    if (n < 0) throw bcmg::Error(BCMG_ERR_CONFIG, "negative size");
    std::vector<int64_t> m, o;
    bcmg::decompose(n, dest_of, m, o);
    std::memcpy(members, m.data(), m.size() * sizeof(int64_t));
    std::memcpy(offsets, o.data(), o.size() * sizeof(int64_t));
    *n_cycles = (int64_t)o.size() - 1;
  });
}

int bcmg_invert_cycles(int64_t n_cycles, const int64_t* offsets, int64_t* members) {
  return guarded([&] {
    std::vector<int64_t> o(offsets, offsets + n_cycles + 1);
    std::vector<int64_t> m(members, members + o.back());
    bcmg::invert_cycles(m, o);
    std::memcpy(members, m.data(), m.size() * sizeof(int64_t));
  });
}

int bcmg_segment_plan_info(int64_t n_cols, int64_t tile, int ndev, int64_t* seg_width, int64_t* n_cycles,
                           int64_t* moved_columns) {
  return guarded([&] {
    auto p = bcmg::segment_plan(n_cols, tile, ndev, false);
    *seg_width = p.seg;
    *n_cycles = (int64_t)p.offsets.size() - 1;
    *moved_columns = (int64_t)p.members.size() * p.seg;
  });
}

int bcmg_schedule(int routine, int64_t n, int64_t tile, int ndev, int world, int rank, int64_t nrhs, int64_t* ops,
                  int64_t cap, int64_t* count) {
  return guarded([&] {
    std::vector<bcmg::SchedOp> v;
    if (routine == 0) v = bcmg::potrf_schedule(n, tile, ndev, world, rank);
    else if (routine == 1) v = bcmg::potrs_schedule(n, tile, ndev, world, rank, nrhs);
    else if (routine == 2) v = bcmg::potri_schedule(n, tile, ndev, world, rank);
    else throw bcmg::Error(BCMG_ERR_CONFIG, "unknown routine");
    *count = (int64_t)v.size();
    if (ops) {
      if ((int64_t)v.size() > cap) throw bcmg::Error(BCMG_ERR_CONFIG, "schedule buffer too small");
      for (size_t i = 0; i < v.size(); ++i) {
        const auto& o = v[i];
        const int64_t row[7] = {o.kind, o.stream, o.k, o.a, o.b, o.root, o.elems};
        std::memcpy(ops + 7 * i, row, sizeof(row));
      }
    }
  });
}

int bcmg_redistribute_plan(int64_t n_cols, int64_t tile, int ndev, int world, int direction, int64_t* seg_width,
                           int64_t* moves, int64_t cap, int64_t* count) {
  return guarded([&] {
    if (direction != BCMG_TO_CYCLIC && direction != BCMG_TO_CONTIG)
      throw bcmg::Error(BCMG_ERR_CONFIG, "unknown redistribution direction");
    const auto rp = bcmg::redist_plan(n_cols, tile, ndev, world, direction == BCMG_TO_CONTIG);
    *seg_width = rp.seg;
    *count = (int64_t)rp.moves.size();
    if (moves) {
      if (*count > cap) throw bcmg::Error(BCMG_ERR_CONFIG, "move buffer too small");
      for (size_t i = 0; i < rp.moves.size(); ++i) {
        moves[4 * i + 0] = rp.moves[i].src_pos;
        moves[4 * i + 1] = rp.moves[i].dst_pos;
        moves[4 * i + 2] = rp.moves[i].src_rank;
        moves[4 * i + 3] = rp.moves[i].dst_rank;
      }
    }
  });
}

int bcmg_nccl_unique_id(unsigned char* id) {
  return guarded([&] {
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) throw bcmg::Error(BCMG_ERR_CUDA, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(u) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(id, &u, sizeof(u));
  });
}

int bcmg_loopback_id(unsigned char* id) {
  return guarded([&] {
    if (!id) throw bcmg::Error(BCMG_ERR_CONFIG, "null id");
    bcmg::make_loopback_id(id);
  });
}

int bcmg_open(int cuda_device, int rank, int world, const unsigned char* nccl_id, bcmg_session** out) {
  return guarded([&] {
    if (!out) throw bcmg::Error(BCMG_ERR_CONFIG, "null output handle");
    *out = nullptr;
    auto* s = new bcmg_session{nullptr};
    try {
      s->impl = new bcmg::Session(cuda_device, rank, world, nccl_id);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int bcmg_close(bcmg_session* s) {
  return guarded([&] {
    if (!s || !s->impl) throw bcmg::Error(BCMG_ERR_STALE_SESSION, "no open session");
    delete s->impl;
    s->impl = nullptr;
    delete s;
  });
}

int bcmg_redistribute(bcmg_session* s, void* stream, int dtype, int64_t n_rows, int64_t n_cols, int64_t tile, int ndev,
                      void* const* shards, int direction) {
  return guarded([&] {
    auto* S = live(s);
    check_common(dtype, ndev, shards);
    if (direction != BCMG_TO_CYCLIC && direction != BCMG_TO_CONTIG)
      throw bcmg::Error(BCMG_ERR_CONFIG, "unknown redistribution direction");
    Entry e(S, stream);
    S->redistribute(dtype, n_rows, n_cols, tile, ndev, shards, direction == BCMG_TO_CONTIG);
  });
}

int bcmg_potrf(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t tile, int ndev, void* const* shards,
               int* info) {
  return guarded([&] {
    auto* S = live(s);
    check_common(dtype, ndev, shards);
    Entry e(S, stream);
    *info = S->potrf(dtype, n, tile, ndev, shards);
  });
}

int bcmg_potrs_factored(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t nrhs, int64_t tile, int ndev,
                        void* const* shards, void* b, int64_t ldb) {
  return guarded([&] {
    auto* S = live(s);
    check_common(dtype, ndev, shards);
    Entry e(S, stream);
    S->potrs(dtype, n, nrhs, tile, ndev, shards, b, ldb);
  });
}

int bcmg_potri_factored(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t tile, int ndev,
                        void* const* shards) {
  return guarded([&] {
    auto* S = live(s);
    check_common(dtype, ndev, shards);
    Entry e(S, stream);
    S->potri(dtype, n, tile, ndev, shards);
  });
}

int bcmg_potrs(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t nrhs, int64_t tile, int ndev,
               void* const* shards, void* b, int64_t ldb, int flags, int* info) {
  int rc = guarded([&] {
    auto* S = live(s);
    check_common(dtype, ndev, shards);
    if (nrhs < 1) throw bcmg::Error(BCMG_ERR_CONFIG, "right-hand side must be non-empty");
    if (ldb < n) throw bcmg::Error(BCMG_ERR_CONFIG, "ldb < n");
    if (tile < 1 || tile > n) throw bcmg::Error(BCMG_ERR_CONFIG, "tile width out of range");
    Entry e(S, stream);
    S->reserve_workspace(1, dtype, n, tile, ndev, nrhs);
    const bool conj = (flags & BCMG_FLAG_ROW_SHARDED) && bcmg::dtype_complex(dtype);
    S->mark(bcmg::T_BEGIN);
    ConjGuard cg(conj, dtype, b, ldb, n, nrhs, S->user);
    S->redistribute(dtype, n, n, tile, ndev, shards, false);
    S->mark(bcmg::T_REDIST);
    *info = S->potrf(dtype, n, tile, ndev, shards);
    S->mark(bcmg::T_POTRF);
    if (*info) {
      S->mark(bcmg::T_SOLVE);
      finish_timings(S, false);
      throw bcmg::Error(BCMG_ERR_NOT_POSITIVE_DEFINITE,
                        "matrix is not positive definite: leading minor of order " + std::to_string(*info) +
                            " (pivot=" + std::to_string(*info) + ")");
    }
    S->begin(S->user);
    S->potrs(dtype, n, nrhs, tile, ndev, shards, b, ldb);
    cg.finish();
    S->mark(bcmg::T_SOLVE);
    finish_timings(S, false);
  });
  return rc;
}

int bcmg_potrs_streamed(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t nrhs, int64_t tile,
                        void* a_dev, const void* a_host, void* b, int64_t ldb, int flags, int* info) {
  int rc = guarded([&] {
    auto* S = live(s);
    if (bcmg::dtype_size(dtype) == 0) throw bcmg::Error(BCMG_ERR_CONFIG, "unknown element-type code");
    if (!a_dev || !a_host) throw bcmg::Error(BCMG_ERR_CONFIG, "null matrix pointer");
    if (S->world != 1) throw bcmg::Error(BCMG_ERR_CONFIG, "streamed input is single-process");
    if (nrhs < 1) throw bcmg::Error(BCMG_ERR_CONFIG, "right-hand side must be non-empty");
    if (ldb < n) throw bcmg::Error(BCMG_ERR_CONFIG, "ldb < n");
    if (tile < 1 || tile > n) throw bcmg::Error(BCMG_ERR_CONFIG, "tile width out of range");
    Entry e(S, stream);
    S->reserve_workspace(1, dtype, n, tile, 1, nrhs);
    const bool conj = (flags & BCMG_FLAG_ROW_SHARDED) && bcmg::dtype_complex(dtype);
    S->mark(bcmg::T_BEGIN);
    ConjGuard cg(conj, dtype, b, ldb, n, nrhs, S->user);
    S->mark(bcmg::T_REDIST);  // one device: the block-cyclic layout is the contiguous one
    void* shards[1] = {a_dev};
    *info = S->potrf(dtype, n, tile, 1, shards, a_host);
    S->mark(bcmg::T_POTRF);
    if (*info) {
      S->mark(bcmg::T_SOLVE);
      finish_timings(S, false);
      throw bcmg::Error(BCMG_ERR_NOT_POSITIVE_DEFINITE,
                        "matrix is not positive definite: leading minor of order " + std::to_string(*info) +
                            " (pivot=" + std::to_string(*info) + ")");
    }
    S->begin(S->user);
    S->potrs(dtype, n, nrhs, tile, 1, shards, b, ldb);
    cg.finish();
    S->mark(bcmg::T_SOLVE);
    finish_timings(S, false);
  });
  return rc;
}

int bcmg_potri(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t tile, int ndev, void* const* shards,
               int flags, int* info) {
  (void)flags;  // inv(conj(A)) = conj(inv(A)) is the row-major view of inv(A): no fix-up needed
  return guarded([&] {
    auto* S = live(s);
    check_common(dtype, ndev, shards);
    if (tile < 1 || tile > n) throw bcmg::Error(BCMG_ERR_CONFIG, "tile width out of range");
    Entry e(S, stream);
    S->reserve_workspace(2, dtype, n, tile, ndev, 1);
    S->mark(bcmg::T_BEGIN);
    S->redistribute(dtype, n, n, tile, ndev, shards, false);
    S->mark(bcmg::T_REDIST);
    *info = S->potrf(dtype, n, tile, ndev, shards);
    S->mark(bcmg::T_POTRF);
    if (*info) {
      S->mark(bcmg::T_SOLVE);
      finish_timings(S, true);
      throw bcmg::Error(BCMG_ERR_NOT_POSITIVE_DEFINITE,
                        "matrix is not positive definite: leading minor of order " + std::to_string(*info) +
                            " (pivot=" + std::to_string(*info) + ")");
    }
    S->begin(S->user);
    S->potri(dtype, n, tile, ndev, shards);
    S->redistribute(dtype, n, n, tile, ndev, shards, true);
    S->mark(bcmg::T_SOLVE);
    finish_timings(S, true);
  });
}

static void check_syevd(int dtype, int64_t n, int64_t tile, int ndev, void* const* shards, void* w, int* info) {
  check_common(dtype, ndev, shards);
  if (n < 1) throw bcmg::Error(BCMG_ERR_CONFIG, "matrix order must be positive");
  if (tile < 1 || tile > n) throw bcmg::Error(BCMG_ERR_CONFIG, "tile width out of range");
  if (!w || !info) throw bcmg::Error(BCMG_ERR_CONFIG, "null eigenvalue / info pointer");
}

int bcmg_syevd(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t tile, int ndev, void* const* shards,
               void* w, int flags, int* info) {
  (void)flags;
  return guarded([&] {
    auto* S = live(s);
    check_syevd(dtype, n, tile, ndev, shards, w, info);
    *info = 0;
    Entry e(S, stream);
    S->mark(bcmg::T_BEGIN);
    // the dense working copy is gathered straight from the contiguous layout
    // and the eigenvectors scattered straight back: redistribute_in / _out
    // (solvers.py:1035-1037) are pure data movement and fold into the gather
    S->mark(bcmg::T_REDIST);
    try {
      S->syevd(dtype, n, tile, ndev, shards, false, w);
    } catch (const bcmg::Error& err) {
      if (err.code == BCMG_ERR_NO_CONVERGENCE) *info = BCMG_ERR_NO_CONVERGENCE;
      throw;
    }
    S->mark(bcmg::T_POTRF);
    S->mark(bcmg::T_SOLVE);
    finish_timings(S, true);
  });
}

int bcmg_syevd_cyclic(bcmg_session* s, void* stream, int dtype, int64_t n, int64_t tile, int ndev,
                      void* const* shards, void* w) {
  return guarded([&] {
    auto* S = live(s);
    int info = 0;
    check_syevd(dtype, n, tile, ndev, shards, w, &info);
    Entry e(S, stream);
    S->syevd(dtype, n, tile, ndev, shards, true, w);
  });
}

int bcmg_gemm(void* stream, int dtype, int64_t m, int64_t n, int64_t k, double alpha, const void* a, int64_t lda,
              int op_a, const void* b, int64_t ldb, int op_b, double beta, void* c, int64_t ldc) {
  return guarded([&] {
    if (bcmg::dtype_size(dtype) == 0) throw bcmg::Error(BCMG_ERR_CONFIG, "unknown element-type code");
    if ((op_a != 0 && op_a != 1) || (op_b != 0 && op_b != 1)) throw bcmg::Error(BCMG_ERR_CONFIG, "op must be 0 or 1");
    if (m < 0 || n < 0 || k < 0) throw bcmg::Error(BCMG_ERR_CONFIG, "negative dimension");
    bcmg::gemm(dtype, m, n, k, bcmg::opA(a, lda, op_a), bcmg::opB(b, ldb, op_b),
               bcmg::Epilogue{c, ldc, alpha, beta, 0, 0}, nullptr, static_cast<cudaStream_t>(stream));
  });
}

int bcmg_last_timings(bcmg_session* s, float* ms) {
  return guarded([&] {
    auto* S = live(s);
    for (int i = 0; i < 4; ++i) ms[i] = S->phase_ms[i];
  });
}

int64_t bcmg_last_moved_bytes(bcmg_session* s) { return (s && s->impl) ? s->impl->last_moved_bytes : -1; }

int bcmg_workspace_nbytes(int routine, int dtype, int64_t n, int64_t tile, int ndev, int world, int64_t nrhs,
                          int64_t* bytes) {
  return guarded([&] {
    if (!bytes) throw bcmg::Error(BCMG_ERR_CONFIG, "null output");
    if (nrhs < 1) throw bcmg::Error(BCMG_ERR_CONFIG, "right-hand side must be non-empty");
    int nsm = 148, dev = 0, cnt = 0;
    if (cudaGetDeviceCount(&cnt) == cudaSuccess && cnt > 0 && cudaGetDevice(&dev) == cudaSuccess) {
      int v = 0;
      if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) nsm = v;
    }
    cudaGetLastError();
    *bytes = (int64_t)bcmg::workspace_plan(routine, dtype, n, tile, ndev, world, nrhs, nsm).total();
  });
}

int bcmg_ipc_export(const void* ptr, unsigned char* token) {
  return guarded([&] {
    if (!ptr || !token) throw bcmg::Error(BCMG_ERR_CONFIG, "null pointer");
    static_assert(sizeof(bcmg::IpcHandle) == BCMG_IPC_TOKEN_BYTES, "token layout");
    const bcmg::IpcHandle h = bcmg::ipc_export(ptr);
    std::memcpy(token, &h, sizeof(h));
  });
}

int bcmg_ipc_open(const unsigned char* token, void** ptr) {
  return guarded([&] {
    if (!ptr || !token) throw bcmg::Error(BCMG_ERR_CONFIG, "null pointer");
    bcmg::IpcHandle h;
    std::memcpy(&h, token, sizeof(h));
    try {
      *ptr = bcmg::ipc_import(h);
    } catch (const bcmg::Error& e) {
      // cudaIpcOpenMemHandle refuses this process's own allocations and stale handles
      throw bcmg::Error(BCMG_ERR_CONFIG, std::string("cannot open handle token: ") + e.what());
    }
  });
}

int bcmg_ipc_close_all(void) {
  return guarded([&] { bcmg::ipc_close_all(); });
}

int bcmg_stream_write_flag(void* stream, void* addr, unsigned v) {
  return guarded([&] {
    if (!addr) throw bcmg::Error(BCMG_ERR_CONFIG, "null flag address");
    if (!bcmg::stream_write_value(static_cast<cudaStream_t>(stream), addr, v))
      throw bcmg::Error(BCMG_ERR_CONFIG, "cuStreamWriteValue32 refused the address");
  });
}

int bcmg_stream_wait_flag(void* stream, const void* addr, unsigned v) {
  return guarded([&] {
    if (!addr) throw bcmg::Error(BCMG_ERR_CONFIG, "null flag address");
    if (!bcmg::stream_wait_supported()) throw bcmg::Error(BCMG_ERR_CONFIG, "cuStreamWaitValue32 unavailable");
    bcmg::stream_wait_geq(static_cast<cudaStream_t>(stream), addr, v);
  });
}

int bcmg_session_workspace_bytes(bcmg_session* s, int64_t* bytes) {
  return guarded([&] { *bytes = (int64_t)live(s)->held_workspace_bytes(); });
}

int bcmg_set_profiling(bcmg_session* s, int on) {
  return guarded([&] { live(s)->profiling = on != 0; });
}

int bcmg_kernel_stats(bcmg_session* s, int kind, double* stats) {
  return guarded([&] { live(s)->kernel_stats(kind, stats); });
}

int64_t bcmg_launch_count(void) { return (int64_t)bcmg::launch_count(); }

int bcmg_generate_spd(void* stream, int dtype, int64_t n, int64_t row0, int64_t rows, void* a, int64_t lda,
                      uint64_t seed, double shift) {
  return guarded([&] {
    if (bcmg::dtype_size(dtype) == 0) throw bcmg::Error(BCMG_ERR_CONFIG, "unknown element-type code");
    if (n < 0 || rows < 0 || row0 < 0 || row0 + rows > n || lda < n)
      throw bcmg::Error(BCMG_ERR_CONFIG, "bad row block");
    bcmg::generate_spd(dtype, a, lda, n, row0, rows, seed, shift, static_cast<cudaStream_t>(stream));
  });
}

int bcmg_measure_fp64_peak(int cuda_device, double* tflops) {
  return guarded([&] {
    BCMG_CUDA(cudaSetDevice(cuda_device));
    *tflops = bcmg::measure_dmma_peak(nullptr);
  });
}

}  // extern "C"
