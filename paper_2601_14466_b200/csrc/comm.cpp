// Transports of comm.h.
#include "comm.h"

#include <cuda.h>
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <climits>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace bcmg {

#define BCMG_NCCL_CALL(call)                                                                          \
  do {                                                                                                \
    ncclResult_t r_ = (call);                                                                         \
    if (r_ != ncclSuccess) throw Error(CUDA, std::string(#call) + ": " + ncclGetErrorString(r_));     \
  } while (0)

// ------------------------------------------------------------------ CUDA IPC
namespace {
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
  static const AddrRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (AddrRangeFn) nullptr;
    }
    return reinterpret_cast<AddrRangeFn>(f);
  }();
  return fn;
}
}  // namespace

IpcHandle ipc_export(const void* ptr) {
  IpcHandle h{};
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!addr_range_fn()) throw Error(CUDA, "cuMemGetAddressRange unavailable");
  const CUresult r = addr_range_fn()(&base, &size, reinterpret_cast<CUdeviceptr>(ptr));
  if (r != CUDA_SUCCESS) throw Error(CONFIG, "address is not inside a device allocation (" + std::to_string((int)r) + ")");
  cudaIpcMemHandle_t mh;
  BCMG_CUDA(cudaIpcGetMemHandle(&mh, reinterpret_cast<void*>(base)));
  static_assert(sizeof(mh) == sizeof(h.bytes), "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(h.bytes, &mh, sizeof(mh));
  h.offset = reinterpret_cast<uint64_t>(ptr) - (uint64_t)base;
  return h;
}

// Imported allocations, one mapping per exporter allocation (opening the same
// handle twice in a process is not allowed).
// At most kMaxOpen mappings are kept (least recently used closed first): a
// mapping keeps the exporter's allocation alive, and callers that pass new
// buffers on every call would otherwise accumulate them.  Only mappings used
// by earlier calls are evicted -- a call's own mappings are its most recent.
class IpcCache {
 public:
  static constexpr size_t kMaxOpen = 32;
  // pin: never evicted (mappings whose addresses live for the whole transport)
  void* import(const IpcHandle& h, bool pin = false) {
    std::lock_guard<std::mutex> lk(mu_);
    const std::string key(reinterpret_cast<const char*>(h.bytes), sizeof(h.bytes));
    auto it = map_.find(key);
    void* base = nullptr;
    const uint64_t stamp = pin ? UINT64_MAX : ++tick_;
    if (it != map_.end()) {
      base = it->second.first;
      it->second.second = std::max(it->second.second == UINT64_MAX ? UINT64_MAX : 0, stamp);
    } else {
      if (map_.size() >= kMaxOpen) {
        auto old = map_.end();
        for (auto e = map_.begin(); e != map_.end(); ++e)
          if (e->second.second != UINT64_MAX && (old == map_.end() || e->second.second < old->second.second)) old = e;
        if (old != map_.end()) {
          cudaIpcCloseMemHandle(old->second.first);
          map_.erase(old);
        }
      }
      cudaIpcMemHandle_t mh;
      std::memcpy(&mh, h.bytes, sizeof(mh));
      BCMG_CUDA(cudaIpcOpenMemHandle(&base, mh, cudaIpcMemLazyEnablePeerAccess));
      map_[key] = {base, stamp};
    }
    return static_cast<char*>(base) + h.offset;
  }
  void close_all() {
    std::lock_guard<std::mutex> lk(mu_);
    for (auto& e : map_) cudaIpcCloseMemHandle(e.second.first);
    map_.clear();
  }
  ~IpcCache() { close_all(); }

 private:
  std::mutex mu_;
  uint64_t tick_ = 0;
  std::map<std::string, std::pair<void*, uint64_t>> map_;
};

namespace {
IpcCache& global_ipc() {
  static IpcCache* c = new IpcCache();  // process lifetime (closed explicitly by ipc_close_all)
  return *c;
}
}  // namespace
void* ipc_import(const IpcHandle& h) { return global_ipc().import(h); }
void ipc_close_all() { global_ipc().close_all(); }

int nccl_max_ctas() {
  static const int v = [] {
    const char* e = getenv("BCMG_NCCL_MAX_CTAS");
    return e && *e ? std::max(1, atoi(e)) : 8;
  }();
  return v;
}

// ------------------------------------------------------------------ NCCL
class NcclComm final : public Comm {
 public:
  NcclComm(int rank, int world, const unsigned char* id) {
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    // at most nccl_max_ctas() CTAs per collective: the trailing-update grid
    // leaves that many SMs free while an NCCL panel broadcast may be in flight
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.maxCTAs = nccl_max_ctas();
    cfg.minCTAs = 1;
    BCMG_NCCL_CALL(ncclCommInitRankConfig(&c_, world, u, rank, &cfg));
    world_ = world;
    me_ = rank;
    // scratch: the barrier word and the all-gather of exchange_pointers (no
    // allocation -- cudaFree synchronises the device -- on the hot path)
    scratch_bytes_ = 4096 + 128 * (size_t)(world + 1);
    BCMG_CUDA(cudaMalloc(&scratch_, scratch_bytes_));
    BCMG_CUDA(cudaMemset(scratch_, 0, scratch_bytes_));
    BCMG_CUDA(cudaStreamCreateWithFlags(&xstream_, cudaStreamNonBlocking));
    // flag words of this rank, mapped into every peer (collective, like the init)
    BCMG_CUDA(cudaMalloc(&flags_, kFlagSlots * sizeof(uint32_t)));
    BCMG_CUDA(cudaMemset(flags_, 0, kFlagSlots * sizeof(uint32_t)));
    BCMG_CUDA(cudaDeviceSynchronize());
    if (stream_wait_supported()) peer_flags_ = exchange(flags_, true);  // pinned: used for the comm's lifetime
  }
  bool flags_supported() const override { return (int)peer_flags_.size() == world_; }
  void post_flag(int peer, int slot, uint32_t v, cudaStream_t st) override {
    void* w = static_cast<uint32_t*>(peer_flags_.at(peer)) + slot;
    if (!stream_write_value(st, w, v)) stream_signal(st, &w, 1, v);  // a one-thread kernel if refused
  }
  void wait_flag(int slot, uint32_t v, cudaStream_t st) override {
    stream_wait_geq(st, static_cast<uint32_t*>(flags_) + slot, v);
  }
  ~NcclComm() override {
    ipc_.close_all();
    if (c_) ncclCommDestroy(c_);
    if (scratch_) cudaFree(scratch_);
    if (flags_) cudaFree(flags_);
    if (xstream_) cudaStreamDestroy(xstream_);
  }
  void barrier(cudaStream_t st) override {
    BCMG_NCCL_CALL(ncclAllReduce(scratch_, scratch_, 1, ncclInt32, ncclSum, c_, st));
  }
  void bcast(void* buf, size_t bytes, int root, cudaStream_t st) override {
    BCMG_NCCL_CALL(ncclBroadcast(buf, buf, bytes, ncclUint8, root, c_, st));
  }
  void group_start() override { BCMG_NCCL_CALL(ncclGroupStart()); }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t st) override {
    BCMG_NCCL_CALL(ncclSend(buf, bytes, ncclUint8, peer, c_, st));
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t st) override {
    BCMG_NCCL_CALL(ncclRecv(buf, bytes, ncclUint8, peer, c_, st));
  }
  void group_end() override { BCMG_NCCL_CALL(ncclGroupEnd()); }
  std::vector<void*> exchange_pointers(void* local) override { return exchange(local, false); }
  // every rank's (IPC handle, offset, ok) all-gathered over NCCL, then opened
  std::vector<void*> exchange(void* local, bool pin) {
    struct Rec {
      IpcHandle h;
      int32_t ok, pad;
    };
    Rec mine{};
    try {
      mine.h = ipc_export(local);
      mine.ok = 1;
    } catch (const Error&) {
      cudaGetLastError();
      mine.ok = 0;
    }
    static_assert(sizeof(Rec) <= 128, "exchange record fits its scratch slot");
    std::vector<Rec> all(world_);
    cudaStream_t st = xstream_;
    char* d = static_cast<char*>(scratch_) + 4096;
    BCMG_CUDA(cudaMemcpyAsync(d + sizeof(Rec) * world_, &mine, sizeof(Rec), cudaMemcpyHostToDevice, st));
    BCMG_NCCL_CALL(ncclAllGather(d + sizeof(Rec) * world_, d, sizeof(Rec), ncclUint8, c_, st));
    BCMG_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(Rec) * world_, cudaMemcpyDeviceToHost, st));
    BCMG_CUDA(cudaStreamSynchronize(st));
    std::vector<void*> out(world_, nullptr);
    int ok = 1;
    for (int r = 0; r < world_; ++r) ok &= all[r].ok;
    if (ok) {
      for (int r = 0; r < world_ && ok; ++r) {
        if (r == me_) {
          out[r] = local;
          continue;
        }
        try {
          out[r] = ipc_.import(all[r].h, pin);
        } catch (const Error&) {
          cudaGetLastError();
          ok = 0;
        }
      }
    }
    // every rank must agree (an import can fail on one rank only)
    int* flag = reinterpret_cast<int*>(d);
    BCMG_CUDA(cudaMemcpyAsync(flag, &ok, sizeof(int), cudaMemcpyHostToDevice, st));
    BCMG_NCCL_CALL(ncclAllReduce(flag, flag, 1, ncclInt32, ncclMin, c_, st));
    BCMG_CUDA(cudaMemcpyAsync(&ok, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    BCMG_CUDA(cudaStreamSynchronize(st));
    if (!ok) return {};
    return out;
  }
  // mappings stay cached (per exporter allocation) until the transport closes
  void release_pointers(std::vector<void*>& ptrs) override { ptrs.clear(); }
  int allreduce_min(int v, void* scratch, cudaStream_t st) override {
    int* d = static_cast<int*>(scratch);
    BCMG_CUDA(cudaMemcpyAsync(d, &v, sizeof(int), cudaMemcpyHostToDevice, st));
    BCMG_NCCL_CALL(ncclAllReduce(d, d, 1, ncclInt32, ncclMin, c_, st));
    int out = 0;
    BCMG_CUDA(cudaMemcpyAsync(&out, d, sizeof(int), cudaMemcpyDeviceToHost, st));
    BCMG_CUDA(cudaStreamSynchronize(st));
    return out;
  }


 private:
  ncclComm_t c_ = nullptr;
  int me_ = 0, world_ = 1;
  void* scratch_ = nullptr;
  size_t scratch_bytes_ = 0;
  cudaStream_t xstream_ = nullptr;
  void* flags_ = nullptr;
  std::vector<void*> peer_flags_;
  IpcCache ipc_;
};

// ------------------------------------------------------------------ loopback
namespace {

cudaEvent_t new_event() {
  cudaEvent_t e;
  BCMG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return e;
}

struct Hub {
  explicit Hub(int w) : world(w) {}
  const int world;
  std::mutex mu;
  std::condition_variable cv;
  struct Bcast {
    const void* src = nullptr;
    cudaEvent_t ready = nullptr;
    std::vector<cudaEvent_t> done;
    bool posted = false;
  };
  std::map<uint64_t, Bcast> bcasts;  // by collective sequence number
  struct Msg {
    const void* src;
    size_t bytes;
    cudaEvent_t ready;
    cudaEvent_t done = nullptr;
    bool acked = false;
  };
  std::map<std::pair<int, int>, std::deque<std::shared_ptr<Msg>>> queues;  // (sender, receiver) FIFO
  struct Reduce {
    int count = 0, value = INT_MAX, reads = 0;
  };
  std::map<uint64_t, Reduce> reduces;
  struct Gather {
    std::vector<void*> ptrs;
    int count = 0, reads = 0;
  };
  std::map<uint64_t, Gather> gathers;
  struct Barrier {
    std::vector<cudaEvent_t> ev;
    int count = 0, reads = 0;
  };
  std::map<uint64_t, Barrier> barriers;
  // (rank, slot) -> posted (value, event), increasing values
  std::map<std::pair<int, int>, std::deque<std::pair<uint32_t, cudaEvent_t>>> flags;
  ~Hub() {
    for (auto& kv : flags)
      for (auto& e : kv.second) cudaEventDestroy(e.second);
  }
};

std::mutex g_hubs_mu;
std::map<uint64_t, std::weak_ptr<Hub>> g_hubs;
std::atomic<uint64_t> g_next_key{1};
constexpr char kMagic[] = "bcmg-loopback-v1";

std::shared_ptr<Hub> join_hub(uint64_t key, int world) {
  std::lock_guard<std::mutex> lk(g_hubs_mu);
  auto it = g_hubs.find(key);
  if (it != g_hubs.end())
    if (auto h = it->second.lock()) {
      if (h->world != world) throw Error(CONFIG, "loopback id reused with a different world size");
      return h;
    }
  auto h = std::make_shared<Hub>(world);
  g_hubs[key] = h;
  return h;
}

}  // namespace

class LoopbackComm final : public Comm {
  // a rank that never arrives (a schedule mismatch or a crashed peer thread)
  // becomes an error instead of a hang
  template <class Pred>
  void hub_wait(std::unique_lock<std::mutex>& lk, Pred pred) {
    if (!hub_->cv.wait_for(lk, std::chrono::seconds(300), pred))
      throw Error(CUDA, "loopback transport: peer rank did not arrive within 300 s");
  }

 public:
  LoopbackComm(int rank, int world, uint64_t key) : rank_(rank), hub_(join_hub(key, world)) {}

  void bcast(void* buf, size_t bytes, int root, cudaStream_t st) override {
    const uint64_t seq = bc_seq_++;
    std::unique_lock<std::mutex> lk(hub_->mu);
    auto& b = hub_->bcasts[seq];
    if (rank_ == root) {
      cudaEvent_t ready = new_event();
      BCMG_CUDA(cudaEventRecord(ready, st));
      b.src = buf;
      b.ready = ready;
      b.posted = true;
      hub_->cv.notify_all();
      // the source buffer stays untouched until every receiver's copy has run
      hub_wait(lk, [&] { return (int)hub_->bcasts[seq].done.size() == hub_->world - 1; });
      auto& bb = hub_->bcasts[seq];
      for (cudaEvent_t e : bb.done) {
        BCMG_CUDA(cudaStreamWaitEvent(st, e, 0));
        cudaEventDestroy(e);
      }
      cudaEventDestroy(bb.ready);
      hub_->bcasts.erase(seq);
      return;
    }
    hub_wait(lk, [&] { return hub_->bcasts[seq].posted; });
    const void* src = hub_->bcasts[seq].src;
    cudaEvent_t ready = hub_->bcasts[seq].ready;
    lk.unlock();
    BCMG_CUDA(cudaStreamWaitEvent(st, ready, 0));
    if (bytes) BCMG_CUDA(cudaMemcpyAsync(buf, src, bytes, cudaMemcpyDeviceToDevice, st));
    cudaEvent_t done = new_event();
    BCMG_CUDA(cudaEventRecord(done, st));
    lk.lock();
    hub_->bcasts[seq].done.push_back(done);
    hub_->cv.notify_all();
  }

  void group_start() override {
    sends_.clear();
    recvs_.clear();
  }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t st) override {
    auto m = std::make_shared<Hub::Msg>();
    m->src = buf;
    m->bytes = bytes;
    m->ready = new_event();
    BCMG_CUDA(cudaEventRecord(m->ready, st));
    {
      std::lock_guard<std::mutex> lk(hub_->mu);
      hub_->queues[{rank_, peer}].push_back(m);
    }
    hub_->cv.notify_all();
    sends_.push_back({m, st});
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t st) override { recvs_.push_back({buf, bytes, peer, st}); }
  void group_end() override {
    // receives first (every send of the group is already posted), then wait for
    // the receivers of our sends so that the send buffers can be reused
    for (const auto& r : recvs_) {
      std::shared_ptr<Hub::Msg> m;
      {
        std::unique_lock<std::mutex> lk(hub_->mu);
        auto& q = hub_->queues[{r.peer, rank_}];
        hub_wait(lk, [&] { return !q.empty(); });
        m = q.front();
        q.pop_front();
      }
      if (m->bytes != r.bytes) throw Error(CONFIG, "loopback: send/recv size mismatch");
      BCMG_CUDA(cudaStreamWaitEvent(r.st, m->ready, 0));
      if (r.bytes) BCMG_CUDA(cudaMemcpyAsync(r.buf, m->src, r.bytes, cudaMemcpyDeviceToDevice, r.st));
      cudaEvent_t done = new_event();
      BCMG_CUDA(cudaEventRecord(done, r.st));
      {
        std::lock_guard<std::mutex> lk(hub_->mu);
        m->done = done;
        m->acked = true;
      }
      hub_->cv.notify_all();
    }
    for (auto& s : sends_) {
      std::unique_lock<std::mutex> lk(hub_->mu);
      hub_wait(lk, [&] { return s.m->acked; });
      lk.unlock();
      BCMG_CUDA(cudaStreamWaitEvent(s.st, s.m->done, 0));
      cudaEventDestroy(s.m->done);
      cudaEventDestroy(s.m->ready);
    }
    sends_.clear();
    recvs_.clear();
  }

  std::vector<void*> exchange_pointers(void* local) override {
    // one address space: the other ranks' allocations are directly usable
    const uint64_t seq = gather_seq_++;
    std::unique_lock<std::mutex> lk(hub_->mu);
    auto& gth = hub_->gathers[seq];
    if (gth.ptrs.empty()) gth.ptrs.assign(hub_->world, nullptr);
    gth.ptrs[rank_] = local;
    gth.count++;
    hub_->cv.notify_all();
    hub_wait(lk, [&] { return hub_->gathers[seq].count == hub_->world; });
    auto& g2 = hub_->gathers[seq];
    std::vector<void*> out = g2.ptrs;
    if (++g2.reads == hub_->world) hub_->gathers.erase(seq);
    return out;
  }
  void release_pointers(std::vector<void*>& ptrs) override { ptrs.clear(); }

  bool flags_supported() const override { return true; }
  void post_flag(int peer, int slot, uint32_t v, cudaStream_t st) override {
    cudaEvent_t e = new_event();
    BCMG_CUDA(cudaEventRecord(e, st));
    std::lock_guard<std::mutex> lk(hub_->mu);
    hub_->flags[{peer, slot}].push_back({v, e});
    hub_->cv.notify_all();
  }
  void wait_flag(int slot, uint32_t v, cudaStream_t st) override {
    std::unique_lock<std::mutex> lk(hub_->mu);
    auto& q = hub_->flags[{rank_, slot}];
    auto found = [&] {
      for (size_t i = 0; i < q.size(); ++i)
        if (q[i].first >= v) return (int)i;
      return -1;
    };
    hub_wait(lk, [&] { return found() >= 0; });
    const int i = found();
    BCMG_CUDA(cudaStreamWaitEvent(st, q[i].second, 0));
    // waits on a slot ask for increasing values: older posts are never needed again
    for (int j = 0; j < i; ++j) cudaEventDestroy(q[j].second);
    q.erase(q.begin(), q.begin() + i);
  }

  void barrier(cudaStream_t st) override {
    const uint64_t seq = bar_seq_++;
    cudaEvent_t mine = new_event();
    BCMG_CUDA(cudaEventRecord(mine, st));
    std::vector<cudaEvent_t> others;
    {
      std::unique_lock<std::mutex> lk(hub_->mu);
      auto& b = hub_->barriers[seq];
      if (b.ev.empty()) b.ev.assign(hub_->world, nullptr);
      b.ev[rank_] = mine;
      b.count++;
      hub_->cv.notify_all();
      hub_wait(lk, [&] { return hub_->barriers[seq].count == hub_->world; });
      others = hub_->barriers[seq].ev;
    }
    for (int r = 0; r < (int)others.size(); ++r)
      if (r != rank_) BCMG_CUDA(cudaStreamWaitEvent(st, others[r], 0));
    std::unique_lock<std::mutex> lk(hub_->mu);
    auto& b = hub_->barriers[seq];
    if (++b.reads == hub_->world) {  // everyone has enqueued its waits: the events may go
      for (cudaEvent_t e : b.ev) cudaEventDestroy(e);
      hub_->barriers.erase(seq);
    }
  }

  int allreduce_min(int v, void*, cudaStream_t) override {
    const uint64_t seq = red_seq_++;
    std::unique_lock<std::mutex> lk(hub_->mu);
    auto& r = hub_->reduces[seq];
    r.count++;
    r.value = std::min(r.value, v);
    hub_->cv.notify_all();
    hub_wait(lk, [&] { return hub_->reduces[seq].count == hub_->world; });
    auto& rr = hub_->reduces[seq];
    const int out = rr.value;
    if (++rr.reads == hub_->world) hub_->reduces.erase(seq);
    return out;
  }

 private:
  struct PendingSend {
    std::shared_ptr<Hub::Msg> m;
    cudaStream_t st;
  };
  struct PendingRecv {
    void* buf;
    size_t bytes;
    int peer;
    cudaStream_t st;
  };
  const int rank_;
  std::shared_ptr<Hub> hub_;
  uint64_t bc_seq_ = 0, red_seq_ = 0, gather_seq_ = 0, bar_seq_ = 0;
  std::vector<PendingSend> sends_;
  std::vector<PendingRecv> recvs_;
};

// ------------------------------------------------------------------ stream flags
namespace {
typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValueFn wait_fn() {
  static WaitValueFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (WaitValueFn) nullptr;
    }
    return reinterpret_cast<WaitValueFn>(f);
  }();
  return fn;
}
}  // namespace

bool stream_wait_supported() { return wait_fn() != nullptr; }

void stream_wait_geq(cudaStream_t st, const void* addr, unsigned v) {
  const CUresult r = wait_fn()(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v,
                               CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) throw Error(CUDA, "cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")");
}

namespace {
typedef CUresult (*WriteValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValueFn write_fn() {
  static const WriteValueFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (WriteValueFn) nullptr;
    }
    return reinterpret_cast<WriteValueFn>(f);
  }();
  return fn;
}
}  // namespace

bool stream_write_value(cudaStream_t st, void* addr, unsigned v) {
  if (!write_fn()) return false;
  // default flags: the write is ordered after (and made visible after) every
  // earlier memory operation of the stream, copies included
  return write_fn()(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v,
                    CU_STREAM_WRITE_VALUE_DEFAULT) == CUDA_SUCCESS;
}

void make_loopback_id(unsigned char* id) {
  std::memset(id, 0, kCommIdBytes);
  std::memcpy(id, kMagic, sizeof(kMagic));
  const uint64_t key = g_next_key.fetch_add(1);
  std::memcpy(id + 32, &key, sizeof(key));
}

std::unique_ptr<Comm> make_comm(int rank, int world, const unsigned char* id) {
  if (!id) throw Error(CONFIG, "world > 1 needs a communicator id (bcmg_nccl_unique_id / bcmg_loopback_id)");
  if (std::memcmp(id, kMagic, sizeof(kMagic)) == 0) {
    uint64_t key;
    std::memcpy(&key, id + 32, sizeof(key));
    return std::make_unique<LoopbackComm>(rank, world, key);
  }
  return std::make_unique<NcclComm>(rank, world, id);
}

}  // namespace bcmg
