// Transport between the processes ("ranks") of a session.
//
//   * NcclComm     -- one process per GPU: ncclBroadcast / grouped
//                     ncclSend+ncclRecv / ncclAllReduce on the caller's stream.
//   * LoopbackComm -- several sessions of ONE process act as the ranks, each on
//                     its own host thread and streams (normally on one GPU):
//                     every transfer is a device-to-device copy ordered by
//                     CUDA events, matched on the host exactly as NCCL matches
//                     collectives (same call order on every rank) and
//                     point-to-point messages (FIFO per sender/receiver pair).
//                     No kernel ever waits on another rank, so ranks sharing
//                     one GPU cannot deadlock it.  This runs the multi-process
//                     drivers (schedules, events, buffers) on a single GPU.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

namespace bcmg {

class Comm {
 public:
  virtual ~Comm() = default;
  // bytes of buf from `root` to every rank (stream-ordered on st)
  virtual void bcast(void* buf, size_t bytes, int root, cudaStream_t st) = 0;
  // grouped point-to-point exchange: sends and receives between group_start
  // and group_end are matched per (sender, receiver) pair in issue order
  virtual void group_start() = 0;
  virtual void send(const void* buf, size_t bytes, int peer, cudaStream_t st) = 0;
  virtual void recv(void* buf, size_t bytes, int peer, cudaStream_t st) = 0;
  virtual void group_end() = 0;
  // host value in, minimum over ranks out (synchronous); scratch: 4 device bytes
  virtual int allreduce_min(int v, void* scratch, cudaStream_t st) = 0;
  // stream-ordered barrier: work enqueued on st after it starts only once every
  // rank's stream has reached its barrier (no kernel waits on another rank
  // in the loopback transport; across GPUs it is one 4-byte NCCL all-reduce)
  virtual void barrier(cudaStream_t st) = 0;
  // Peer memory (NVLink P2P through CUDA IPC handles; the shared address space
  // of loopback ranks): every rank contributes one device address (any
  // address inside a cudaMalloc allocation) and gets every rank's address
  // mapped into its own address space (collective, same call order on every
  // rank; mappings are cached per allocation and closed with the transport).
  // Empty if unsupported on any rank (all ranks agree).
  virtual std::vector<void*> exchange_pointers(void* local) = 0;
  virtual void release_pointers(std::vector<void*>& ptrs) = 0;
  // Stream-ordered flags of the peer-memory hand-offs: per rank kFlagSlots
  // monotone 32-bit counters.  post_flag: once everything earlier on st is
  // done (and visible to the peer), rank `peer`'s counter `slot` becomes v.
  // wait_flag: work enqueued on st afterwards starts once this rank's counter
  // `slot` is >= v.  Across GPUs these are stream memory operations on
  // CUDA-IPC-mapped words (cuStreamWriteValue32 / cuStreamWaitValue32: no
  // kernel, no SM, no stream of one rank parked inside another rank's
  // context); loopback ranks match them on the host and order the streams
  // with CUDA events (no stream ever parks in the shared context).
  static constexpr int kFlagSlots = 64;
  virtual bool flags_supported() const = 0;
  virtual void post_flag(int peer, int slot, uint32_t v, cudaStream_t st) = 0;
  virtual void wait_flag(int slot, uint32_t v, cudaStream_t st) = 0;
};

// CUDA IPC export / import of any device address (the allocation's handle plus
// the offset inside it; reference runtime.py HandleRegistry publish / open).
struct IpcHandle {
  unsigned char bytes[64];
  uint64_t offset;
};
IpcHandle ipc_export(const void* ptr);
void* ipc_import(const IpcHandle& h);  // cached per allocation; owner process may not import its own
void ipc_close_all();                  // closes every imported mapping

// Stream-ordered flags for peer-memory hand-offs: `signal` stores v to a
// (possibly peer) 32-bit word from a one-thread kernel; `wait_geq` blocks the
// stream until a LOCAL word reaches v (no kernel waits on another rank).
bool stream_wait_supported();
void stream_wait_geq(cudaStream_t st, const void* addr, unsigned v);
void stream_signal(cudaStream_t st, void* const* addrs, int n, unsigned v);
// the same store as a stream memory operation (no kernel, no SM: issued by
// the stream front end after everything earlier on st, with a memory
// barrier); false if the driver refused it (nothing enqueued)
bool stream_write_value(cudaStream_t st, void* addr, unsigned v);

int nccl_max_ctas();  // CTA limit of the NCCL communicators (BCMG_NCCL_MAX_CTAS, default 8)

constexpr size_t kCommIdBytes = 128;
// id: kCommIdBytes from bcmg_nccl_unique_id (NCCL) or bcmg_loopback_id (loopback)
std::unique_ptr<Comm> make_comm(int rank, int world, const unsigned char* id);
void make_loopback_id(unsigned char* id);

}  // namespace bcmg
