// Session object behind the C-ABI handle (include/bcmg_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <memory>
#include <cstdint>
#include <vector>

#include "comm.h"
#include "common.cuh"

namespace bcmg {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n);  // grow-only; throws Error(OUT_OF_MEMORY)
  void release();
};

// One operation of a process's potrf / potrs schedule (solver.cu).
enum SchedKind : int { S_FACTOR = 1, S_BCAST = 2, S_UPDATE = 3, S_COPYBACK = 4, S_STEP_END = 5, S_FWD = 6,
                       S_BWD = 7, S_SHARE = 8,
                       // potri
                       S_WFINAL = 9, S_TILE_BCAST = 10, S_WACC = 11, S_PGEMM = 12, S_PGATHER = 13 };
enum SchedStream : int { STREAM_CRIT = 0, STREAM_BULK = 1, STREAM_COMM = 2 };
struct SchedOp {
  int64_t kind, stream, k;
  int64_t a, b;      // S_UPDATE: tile range [a, b); S_SHARE: row range [a, b); S_STEP_END: a = lookahead flag
  int64_t root;      // S_BCAST / S_SHARE / S_TILE_BCAST / S_PGATHER: source (gather: destination) process;
                     // S_UPDATE (bulk): 1 = grid capped
  int64_t elems;     // S_BCAST / S_SHARE / S_TILE_BCAST: elements moved; S_PGATHER: elements this process sends
};
std::vector<SchedOp> potrf_schedule(int64_t n, int64_t T, int ndev, int world, int rank);
std::vector<SchedOp> potrs_schedule(int64_t n, int64_t T, int ndev, int world, int rank, int64_t nrhs);
std::vector<SchedOp> potri_schedule(int64_t n, int64_t T, int ndev, int world, int rank);

// Cross-process redistribution: every segment move of the cycle plan
// (cycles in order, c_i -> c_{i+1} within a cycle) with the processes that
// own its source and destination segments.
struct RedistMove {
  int64_t src_pos, dst_pos;  // segment indices (column = index * seg)
  int src_rank, dst_rank;
};
struct RedistPlan {
  int64_t seg = 1;
  std::vector<RedistMove> moves;
};
RedistPlan redist_plan(int64_t n_cols, int64_t T, int ndev, int world, bool inverse);

// Every device buffer a pipeline needs: Session::reserve_workspace allocates
// exactly these before moving any data (so OUT_OF_MEMORY leaves the shards
// untouched), bcmg_workspace_nbytes reports them, and the drivers never grow
// a buffer past them.
struct WsPlan {
  size_t panel = 0, panel_pb = 0, split = 0, embed = 0, dinv = 0, wdiag = 0, info = 0, tmp = 0, acc = 0;
  size_t split_scratch = 0;  // tf32 hi / lo planes of the generic tensor-core GEMMs (crit stream)
  size_t total() const {
    return 2 * panel + 2 * panel_pb + 2 * split + embed + dinv + wdiag + info + tmp + acc + split_scratch;
  }
};
// routine: 1 potrs pipeline, 2 potri pipeline; nsm: the GPU's SM count
WsPlan workspace_plan(int routine, int dt, int64_t n, int64_t T, int ndev, int world, int64_t nrhs, int nsm);

// Phase timing slots (CUDA events on the critical stream).
enum Phase : int { T_BEGIN = 0, T_REDIST = 1, T_POTRF = 2, T_SOLVE = 3, T_END = 4 };

struct Session {
  int device, rank, world;
  std::unique_ptr<Comm> net;  // world > 1: NCCL or in-process loopback transport
  cudaStream_t crit = nullptr, bulk = nullptr, comm = nullptr, user = nullptr;
  cudaStream_t side = nullptr;  // copy-engine work off the critical path (potrf copy-back)
  static constexpr int kEvents = 64, kJoin = 56, kTimeEvents = 5;
  cudaEvent_t ev_pool[kEvents];
  cudaEvent_t ev_time[kTimeEvents];
  DevBuf panel[2], panel_pb[2], split_buf[2], dinv, wdiag, info_dev, tmp, acc, plan_buf, embed_buf;
  // peer-memory mode of potrf: every process's panel buffers and flag words
  std::vector<void*> peer_panel[2];
  uint32_t panel_seq = 0, free_seq[2] = {0, 0};
  std::vector<char> plan_host;
  int* info_host = nullptr;
  // Which factorization the diagonal-block inverses in `dinv` belong to:
  // potrs / potri read X_kk from there, so they only accept the shards, shape,
  // type and tiling of the last successful potrf of this session.
  struct FactorKey {
    bool valid = false;
    int dt = -1, ndev = 0;
    int64_t n = 0, T = 0;
    std::vector<uintptr_t> shards;
    bool matches(int dt_, int64_t n_, int64_t T_, int ndev_, void* const* sh, int nloc) const {
      if (!valid || dt != dt_ || n != n_ || T != T_ || ndev != ndev_ || (int)shards.size() != nloc) return false;
      for (int i = 0; i < nloc; ++i)
        if (shards[i] != reinterpret_cast<uintptr_t>(sh[i])) return false;
      return true;
    }
  } fkey;
  int64_t last_moved_bytes = 0;
  std::atomic<bool> busy{false};
  float phase_ms[kTimeEvents] = {0, 0, 0, 0, 0};

  // Optional per-kernel timing (bcmg_set_profiling): CUDA events around each
  // launch of a kind on the stream it is launched on, plus its algorithmic flops/bytes.
  enum Kind : int { K_TRAIL = 0, K_TRSM = 1, K_DIAG = 2, K_ROTATE = 3, K_SUBST = 4, K_KINDS = 5 };
  bool profiling = false;
  struct KStat {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    double work = 0;
    std::vector<double> works;  // per launch
  } kstat[K_KINDS];
  std::vector<cudaEvent_t> ev_spare;
  cudaEvent_t take_event();
  template <class F>
  void timed(int kind, cudaStream_t st, double work, F&& f) {
    if (!profiling) {
      f();
      return;
    }
    cudaEvent_t a = take_event(), b = take_event();
    BCMG_CUDA(cudaEventRecord(a, st));
    f();
    BCMG_CUDA(cudaEventRecord(b, st));
    kstat[kind].ev.emplace_back(a, b);
    kstat[kind].work += work;
    kstat[kind].works.push_back(work);
  }
  // launches, total ms, work (flops or bytes), max ms; clears the record
  void kernel_stats(int kind, double* out);

  Session(int device, int rank, int world, const unsigned char* nccl_id);
  ~Session();

  cudaEvent_t ev(int i);
  void begin(cudaStream_t user_stream);  // internal streams wait on the caller's stream
  void join();                           // caller's stream waits on internal streams
  void sync_streams(cudaStream_t waiter, cudaStream_t on);
  void mark(int phase);
  void bcast(void* buf, size_t bytes, int root, cudaStream_t st);
  int reduce_info(int local);

  // drivers (see solver.cu); shards are this process's logical-device shards
  void redistribute(int dt, int64_t n_rows, int64_t n_cols, int64_t T, int ndev, void* const* shards, bool inverse);
  void redistribute_multi(int dt, int64_t n_rows, int64_t n_cols, int64_t T, int ndev, void* const* shards,
                          bool inverse);
  // world > 1: in-place rotation over peer-mapped shards (false: peers not mappable, nothing done)
  bool redistribute_p2p(int dt, int64_t n_rows, int64_t n_cols, int64_t T, int ndev, void* const* shards,
                        bool inverse);
  int last_redist_path = 0;  // 0 single process, 1 P2P rotation, 2 NCCL pack/exchange/unpack
  int last_bcast_mode = 0;   // potrf panel broadcast: 0 NCCL (or none), 1 copy engines, 2 fused fan-out
  DevBuf stage_buf, desc_buf;
  // host != nullptr: shards[0] (one device) is filled from pinned host memory
  // (same layout) while the factorisation starts (see solver.cu)
  int potrf(int dt, int64_t n, int64_t T, int ndev, void* const* shards, const void* host = nullptr);
  // routine: 1 potrs pipeline, 2 potri pipeline (throws OUT_OF_MEMORY before any data moves)
  void reserve_workspace(int routine, int dt, int64_t n, int64_t T, int ndev, int64_t nrhs);
  size_t held_workspace_bytes() const;  // device bytes this session's workspace holds now
  int nsm = 148;
  void potrs(int dt, int64_t n, int64_t nrhs, int64_t T, int ndev, void* const* shards, void* x, int64_t ldx);
  void potri(int dt, int64_t n, int64_t T, int ndev, void* const* shards);
  // Hermitian eigendecomposition (eigen.cu): eigenvalues ascending into w
  // (device, real type of dt), eigenvectors over the shards (cyclic or
  // contiguous layout); throws NO_CONVERGENCE
  DevBuf eig[7];
  void* eig_host = nullptr;  // pinned staging of the QL rotation ring (grow-only)
  size_t eig_host_bytes = 0;
  void syevd(int dt, int64_t n, int64_t T, int ndev, void* const* shards, bool cyclic, void* w);
};

}  // namespace bcmg
