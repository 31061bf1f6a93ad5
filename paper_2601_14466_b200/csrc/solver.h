// Session object behind the C-ABI handle (include/bcmg_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace bcmg {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n);  // grow-only; throws Error(OUT_OF_MEMORY)
  void release();
};

// Phase timing slots (CUDA events on the critical stream).
enum Phase : int { T_BEGIN = 0, T_REDIST = 1, T_POTRF = 2, T_SOLVE = 3, T_END = 4 };

struct Session {
  int device, rank, world;
  void* nccl = nullptr;  // ncclComm_t when world > 1
  cudaStream_t crit = nullptr, bulk = nullptr, comm = nullptr, user = nullptr;
  static constexpr int kEvents = 64, kJoin = 56, kTimeEvents = 5;
  cudaEvent_t ev_pool[kEvents];
  cudaEvent_t ev_time[kTimeEvents];
  DevBuf panel[2], dinv, wdiag, info_dev, tmp, acc, plan_buf;
  std::vector<char> plan_host;
  int* info_host = nullptr;
  int64_t last_dinv_T = 0;
  int64_t last_moved_bytes = 0;
  std::atomic<bool> busy{false};
  float phase_ms[kTimeEvents] = {0, 0, 0, 0, 0};

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
  int potrf(int dt, int64_t n, int64_t T, int ndev, void* const* shards);
  void potrs(int dt, int64_t n, int64_t nrhs, int64_t T, int ndev, void* const* shards, void* x, int64_t ldx);
  void potri(int dt, int64_t n, int64_t T, int ndev, void* const* shards);
};

}  // namespace bcmg
