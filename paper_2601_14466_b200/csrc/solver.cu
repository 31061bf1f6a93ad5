// Session + drivers of the multi-GPU Cholesky path (B200, sm_100a).
//
// Process model: one process per GPU (torchrun), each process owning
// ndev/world consecutive LOGICAL devices of the 1D block-cyclic layout
// (tile k -> logical device k mod ndev, reference solvers.py:373).  With
// world == 1 all logical devices are "virtual devices" sharing one GPU,
// which keeps the reference's multi-device arithmetic testable on one B200.
// Cross-process traffic is NCCL (panel broadcast per potrf step, solution
// blocks in potrs); intra-process "peer copies" of the reference are plain
// device memory accesses.
//
// Drivers:
//   redistribute : segment-level cycle plan + in-place rotation kernel
//                  (reference layout.py:191-256)
//   potrf        : right-looking tiled Cholesky with depth-1 lookahead on a
//                  high-priority stream (reference solvers.py:341-406)
//   potrs        : forward/backward substitution over the tiles using the
//                  diagonal-block inverses kept by potrf (solvers.py:430-474)
//   potri        : W = L^-1 sweep, A^-1 = W^H W sweep, Hermitian mirror
//                  (solvers.py:487-594)
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "ops.h"
#include "solver.h"

namespace bcmg {

// ------------------------------------------------------------------ buffers
void DevBuf::ensure(size_t n) {
  if (n <= bytes) return;
  release();
  if (n == 0) return;
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(OUT_OF_MEMORY, "device workspace of " + std::to_string(n) + " bytes: " + cudaGetErrorString(e));
  }
  p = q;
  bytes = n;
}
void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

// ------------------------------------------------------------------ session
Session::Session(int device_, int rank_, int world_, const unsigned char* nccl_id) : device(device_), rank(rank_), world(world_) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(CONFIG, "bad rank/world");
  BCMG_CUDA(cudaSetDevice(device));
  int lo = 0, hi = 0;
  BCMG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  BCMG_CUDA(cudaStreamCreateWithPriority(&crit, cudaStreamNonBlocking, hi));
  BCMG_CUDA(cudaStreamCreateWithPriority(&bulk, cudaStreamNonBlocking, lo));
  BCMG_CUDA(cudaStreamCreateWithPriority(&comm, cudaStreamNonBlocking, hi));
  BCMG_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo));
  for (auto& e : ev_pool) BCMG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : ev_time) BCMG_CUDA(cudaEventCreate(&e));
  BCMG_CUDA(cudaMallocHost(&info_host, sizeof(int)));
  BCMG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  if (world > 1) net = make_comm(rank, world, nccl_id);
}

Session::~Session() {
  cudaSetDevice(device);
  cudaDeviceSynchronize();
  if (net) {
    net->release_pointers(peer_panel[0]);
    net->release_pointers(peer_panel[1]);
  }
  net.reset();
  for (auto* b : {&panel[0], &panel[1], &panel_pb[0], &panel_pb[1], &dinv, &wdiag, &info_dev, &tmp, &acc, &plan_buf,
                  &stage_buf, &desc_buf, &embed_buf, &split_buf[0], &split_buf[1]})
    b->release();
  for (auto& b : eig) b.release();
  if (eig_host) cudaFreeHost(eig_host);
  for (auto& e : ev_pool) cudaEventDestroy(e);
  for (auto& e : ev_time) cudaEventDestroy(e);
  for (auto& k : kstat)
    for (auto& pr : k.ev) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  for (auto& e : ev_spare) cudaEventDestroy(e);
  if (info_host) cudaFreeHost(info_host);
  for (cudaStream_t st : {crit, bulk, comm, side}) {
    release_split_scratch(st);
    cudaStreamDestroy(st);
  }
}

cudaEvent_t Session::ev(int i) { return ev_pool[i % kEvents]; }

cudaEvent_t Session::take_event() {
  if (!ev_spare.empty()) {
    cudaEvent_t e = ev_spare.back();
    ev_spare.pop_back();
    return e;
  }
  cudaEvent_t e;
  BCMG_CUDA(cudaEventCreate(&e));
  return e;
}

void Session::kernel_stats(int kind, double* out) {
  if (kind < 0 || kind >= K_KINDS) throw Error(CONFIG, "unknown kernel kind");
  KStat& k = kstat[kind];
  double tot = 0, mx = 0;
  FILE* dump = nullptr;
  if (const char* path = getenv("BCMG_PROFILE_DUMP")) dump = fopen(path, "a");
  for (size_t i = 0; i < k.ev.size(); ++i) {
    auto& pr = k.ev[i];
    BCMG_CUDA(cudaEventSynchronize(pr.second));
    float ms = 0;
    BCMG_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
    if (dump) fprintf(dump, "%d %zu %.6f %.6e\n", kind, i, ms, i < k.works.size() ? k.works[i] : 0.0);
    tot += ms;
    mx = std::max(mx, (double)ms);
    ev_spare.push_back(pr.first);
    ev_spare.push_back(pr.second);
  }
  out[0] = (double)k.ev.size();
  out[1] = tot;
  out[2] = k.work;
  out[3] = mx;
  if (dump) fclose(dump);
  k.ev.clear();
  k.works.clear();
  k.work = 0;
}

void Session::begin(cudaStream_t user_stream) {
  user = user_stream;
  BCMG_CUDA(cudaSetDevice(device));
  BCMG_CUDA(cudaEventRecord(ev(kJoin + 4), user));
  for (cudaStream_t s : {crit, bulk, comm, side}) BCMG_CUDA(cudaStreamWaitEvent(s, ev(kJoin + 4), 0));
}

void Session::join() {
  // user stream waits for every internal stream
  int i = 0;
  for (cudaStream_t s : {crit, bulk, comm, side}) {
    BCMG_CUDA(cudaEventRecord(ev(kJoin + (i < 3 ? i : 5)), s));
    BCMG_CUDA(cudaStreamWaitEvent(user, ev(kJoin + (i < 3 ? i : 5)), 0));
    ++i;
  }
}

void Session::sync_streams(cudaStream_t waiter, cudaStream_t on) {
  BCMG_CUDA(cudaEventRecord(ev(kJoin + 3), on));
  BCMG_CUDA(cudaStreamWaitEvent(waiter, ev(kJoin + 3), 0));
}

void Session::mark(int phase) {
  if (phase >= 0 && phase < kTimeEvents) BCMG_CUDA(cudaEventRecord(ev_time[phase], user));
}

void Session::bcast(void* buf, size_t bytes, int root, cudaStream_t st) {
  if (world == 1 || bytes == 0) return;
  net->bcast(buf, bytes, root, st);
}

int Session::reduce_info(int local) {
  if (world == 1) return local;
  // smallest nonzero pivot over ranks (later tiles can only fail at larger pivots)
  const int out = net->allreduce_min(local ? local : 0x7fffffff, tmp.p, comm);
  return out == 0x7fffffff ? 0 : out;
}

// ------------------------------------------------------------------ geometry
struct Geo {
  int64_t n, T, nt;
  int D, nloc, dev0;
  int esz;
  bool owns(int64_t k) const {
    const int d = (int)(k % D);
    return d >= dev0 && d < dev0 + nloc;
  }
  int owner_rank(int64_t k) const { return (int)((k % D) / nloc); }
  int64_t start(int64_t k) const { return k * T; }
  int64_t stop(int64_t k) const { return std::min(n, (k + 1) * T); }
  int64_t loc(int64_t k) const { return (k / D) * T; }  // local first column of tile k on its device
};

static Geo make_geo(const Session& s, int dt, int64_t n, int64_t T, int ndev) {
  if (n < 1) throw Error(CONFIG, "matrix order must be positive");
  if (T < 1 || T > n) throw Error(CONFIG, "tile width " + std::to_string(T) + " out of range for " + std::to_string(n) + " columns");
  if (ndev < 1) throw Error(CONFIG, "need at least one device");
  if (ndev % s.world) throw Error(CONFIG, "logical device count must be a multiple of the process count");
  Geo g;
  g.n = n;
  g.T = T;
  g.nt = (n + T - 1) / T;
  g.D = ndev;
  g.nloc = ndev / s.world;
  g.dev0 = s.rank * g.nloc;
  g.esz = dtype_size(dt);
  if (!g.esz) throw Error(CONFIG, "unknown element-type code");
  if (g.nloc > MAX_LOCAL_DEV) throw Error(CONFIG, "too many logical devices per process");
  return g;
}

static char* colp(void* shard, const Geo& g, int64_t row, int64_t col) {
  return static_cast<char*>(shard) + (row + col * g.n) * g.esz;
}

// ------------------------------------------------------------------ redistribution
void Session::redistribute(int dt, int64_t n_rows, int64_t n_cols, int64_t T, int ndev, void* const* shards,
                           bool inverse) {
  if (n_rows < 1 || n_cols < 1) throw Error(CONFIG, "matrix dimensions must be positive");
  if (T < 1 || T > n_cols) throw Error(CONFIG, "tile width out of range");
  if (ndev < 1) throw Error(CONFIG, "need at least one device");
  const int esz = dtype_size(dt);
  if (!esz) throw Error(CONFIG, "unknown element-type code");
  // BCMG_STAGED_REDIST=1 routes a single process through the staged
  // (cross-process) algorithm too, so one GPU exercises its pack/unpack path.
  const char* staged = getenv("BCMG_STAGED_REDIST");
  const char* nccl_env = getenv("BCMG_REDIST_NCCL");
  if (world > 1 && !(nccl_env && atoi(nccl_env)) && redistribute_p2p(dt, n_rows, n_cols, T, ndev, shards, inverse)) {
    last_redist_path = 1;
    return;
  }
  if (world > 1 || (staged && atoi(staged))) {
    last_redist_path = 2;
    return redistribute_multi(dt, n_rows, n_cols, T, ndev, shards, inverse);
  }
  last_redist_path = 0;
  last_moved_bytes = 0;
  SegPlan plan = segment_plan(n_cols, T, ndev, inverse);
  const int64_t nc = (int64_t)plan.offsets.size() - 1;
  if (nc == 0) return;
  const auto counts = column_counts(n_cols, T, ndev);
  std::vector<int64_t> off(ndev, 0);
  for (int d = 1; d < ndev; ++d) off[d] = off[d - 1] + counts[d - 1];
  const int64_t col_bytes = n_rows * esz;
  int vec = (col_bytes % 16 == 0) ? 16 : (col_bytes % 8 == 0 ? 8 : 4);
  for (int d = 0; d < ndev; ++d)
    if (reinterpret_cast<uintptr_t>(shards[d]) % vec) vec = (reinterpret_cast<uintptr_t>(shards[d]) % 8) ? 4 : 8;
  // host tables: member addresses, CSR offsets, lane prefix, segment bytes
  const size_t nm = plan.members.size();
  std::vector<uint64_t> addr(nm);
  for (size_t i = 0; i < nm; ++i) {
    const int64_t pos = plan.members[i] * plan.seg;
    int d = (int)(std::upper_bound(off.begin(), off.end(), pos) - off.begin()) - 1;
    addr[i] = reinterpret_cast<uint64_t>(shards[d]) + (uint64_t)((pos - off[d]) * col_bytes);
  }
  // 16-byte aligned segments go through the bulk-copy engine in chunks
  const char* lanes_env = getenv("BCMG_ROTATE_LANES");
  const bool bulk = vec == 16 && !(lanes_env && atoi(lanes_env));
  const int64_t unit = bulk ? rotate_bulk_chunk() : vec;
  std::vector<int64_t> lane_pref(nc + 1, 0), seg_bytes(nc);
  for (int64_t c = 0; c < nc; ++c) {
    seg_bytes[c] = plan.seg_cols[c] * col_bytes;
    lane_pref[c + 1] = lane_pref[c] + (seg_bytes[c] + unit - 1) / unit;
  }
  const size_t bytes = nm * 8 + (nc + 1) * 8 * 2 + nc * 8;
  plan_host.resize(bytes);
  char* h = plan_host.data();
  std::memcpy(h, addr.data(), nm * 8);
  std::memcpy(h + nm * 8, plan.offsets.data(), (nc + 1) * 8);
  std::memcpy(h + nm * 8 + (nc + 1) * 8, lane_pref.data(), (nc + 1) * 8);
  std::memcpy(h + nm * 8 + (nc + 1) * 16, seg_bytes.data(), nc * 8);
  plan_buf.ensure(bytes);
  char* dptr = static_cast<char*>(plan_buf.p);
  BCMG_CUDA(cudaMemcpyAsync(dptr, h, bytes, cudaMemcpyHostToDevice, crit));
  RotateJob j;
  j.addr = reinterpret_cast<const uint64_t*>(dptr);
  j.offsets = reinterpret_cast<const int64_t*>(dptr + nm * 8);
  j.lane_pref = reinterpret_cast<const int64_t*>(dptr + nm * 8 + (nc + 1) * 8);
  j.seg_bytes = reinterpret_cast<const int64_t*>(dptr + nm * 8 + (nc + 1) * 16);
  j.n_cycles = nc;
  j.total_lanes = lane_pref[nc];
  j.vec = vec;
  j.bulk = bulk ? 1 : 0;
  timed(K_ROTATE, crit, 2.0 * (double)nm * plan.seg * col_bytes, [&] { rotate_cycles(j, crit); });
  // (cudaMemcpyAsync from pageable memory returns once the source is consumed)
  last_moved_bytes = 2 * (int64_t)nm * plan.seg * col_bytes;
  sync_streams(user, crit);
}

// ------------------------------------------------------------------ cross-process redistribution (P2P)
// The reference rotates every cycle in place with peer copies and two staging
// columns (layout.py:191-256).  Across processes the shards
// of every rank are mapped into each rank's address space (CUDA IPC over
// NVLink; the shared address space of loopback ranks) and the SAME in-place
// rotation kernel runs over them: every cycle's bytes are split into `world`
// equal lane ranges and rank r rotates range r of every cycle -- each lane is
// read from all its members into registers and written to the successors by
// one thread, so no staging buffer and no pack/unpack passes: HBM traffic is
// the algorithmic 2 s N per moved column, and a rank's NVLink traffic is the
// members of its ranges that live on other ranks (read once, written once;
// for 1D block-cyclic shapes this equals the point-to-point minimum on
// average).  Stream-ordered barriers before (every rank's shards final) and
// after (every peer store performed) -- no kernel waits on another rank.
bool Session::redistribute_p2p(int dt, int64_t n_rows, int64_t n_cols, int64_t T, int ndev, void* const* shards,
                               bool inverse) {
  const int esz = dtype_size(dt);
  const int nloc = ndev / world;
  // every rank's i-th local shard, in this process's address space
  std::vector<std::vector<void*>> peer(nloc);
  for (int i = 0; i < nloc; ++i) {
    peer[i] = net->exchange_pointers(shards[i]);
    if ((int)peer[i].size() != world) return false;  // collective outcome: all ranks fall back together
  }
  last_moved_bytes = 0;
  const SegPlan plan = segment_plan(n_cols, T, ndev, inverse);
  const int64_t nc = (int64_t)plan.offsets.size() - 1;
  if (nc == 0) return true;
  const auto counts = column_counts(n_cols, T, ndev);
  std::vector<int64_t> off(ndev, 0);
  for (int d = 1; d < ndev; ++d) off[d] = off[d - 1] + counts[d - 1];
  const int64_t col_bytes = n_rows * esz;
  auto member_addr = [&](int64_t seg_pos) {
    const int64_t pos = seg_pos * plan.seg;
    const int d = (int)(std::upper_bound(off.begin(), off.end(), pos) - off.begin()) - 1;
    return reinterpret_cast<uint64_t>(peer[d % nloc][d / nloc]) + (uint64_t)((pos - off[d]) * col_bytes);
  };
  int vec = (col_bytes % 16 == 0) ? 16 : (col_bytes % 8 == 0 ? 8 : 4);
  for (const auto& pv : peer)
    for (void* q : pv) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(q);
      while (vec > 4 && a % vec) vec /= 2;
    }
  // this rank's lane range of every cycle
  std::vector<uint64_t> addr;
  std::vector<int64_t> offs{0}, lane_pref{0}, seg_bytes;
  double my_bytes = 0;
  for (int64_t c = 0; c < nc; ++c) {
    const int64_t sb = plan.seg_cols[c] * col_bytes, lanes = sb / vec;
    const int64_t lo = lanes * rank / world, hi = lanes * (rank + 1) / world;
    const int64_t m = plan.offsets[c + 1] - plan.offsets[c];
    last_moved_bytes += 2 * m * sb;
    if (hi <= lo) continue;
    for (int64_t i = plan.offsets[c]; i < plan.offsets[c + 1]; ++i)
      addr.push_back(member_addr(plan.members[i]) + (uint64_t)(lo * vec));
    offs.push_back((int64_t)addr.size());
    lane_pref.push_back(lane_pref.back() + (hi - lo));
    seg_bytes.push_back((hi - lo) * vec);
    my_bytes += 2.0 * (double)m * (double)((hi - lo) * vec);
  }
  const int64_t np = (int64_t)seg_bytes.size();
  const size_t bytes = addr.size() * 8 + (np + 1) * 8 * 2 + np * 8;
  plan_host.resize(std::max<size_t>(bytes, 8));
  char* h = plan_host.data();
  std::memcpy(h, addr.data(), addr.size() * 8);
  std::memcpy(h + addr.size() * 8, offs.data(), (np + 1) * 8);
  std::memcpy(h + addr.size() * 8 + (np + 1) * 8, lane_pref.data(), (np + 1) * 8);
  std::memcpy(h + addr.size() * 8 + (np + 1) * 16, seg_bytes.data(), np * 8);
  plan_buf.ensure(std::max<size_t>(bytes, 8));
  char* dptr = static_cast<char*>(plan_buf.p);
  if (np) BCMG_CUDA(cudaMemcpyAsync(dptr, h, bytes, cudaMemcpyHostToDevice, crit));
  RotateJob j;
  j.addr = reinterpret_cast<const uint64_t*>(dptr);
  j.offsets = reinterpret_cast<const int64_t*>(dptr + addr.size() * 8);
  j.lane_pref = reinterpret_cast<const int64_t*>(dptr + addr.size() * 8 + (np + 1) * 8);
  j.seg_bytes = reinterpret_cast<const int64_t*>(dptr + addr.size() * 8 + (np + 1) * 16);
  j.n_cycles = np;
  j.total_lanes = lane_pref.back();
  j.vec = vec;
  j.bulk = 0;
  j.sys_fence = 1;
  net->barrier(crit);  // every rank's shards hold their final contiguous data
  timed(K_ROTATE, crit, my_bytes, [&] { rotate_cycles(j, crit); });
  net->barrier(crit);  // every rank's peer stores have landed
  // (cudaMemcpyAsync from pageable memory returns once the source is consumed)
  sync_streams(user, crit);
  return true;
}

// ------------------------------------------------------------------ cross-process redistribution (staged NCCL)
// Fallback (BCMG_REDIST_NCCL=1, or shards that cannot be peer-mapped).
// Same segment-level cycle plan on every process.  A move c_i -> c_{i+1}
// between processes becomes an NCCL send/recv pair; a move inside a process a
// device copy.  In place with bounded staging: the segments are processed in
// byte chunks of CH; per chunk every process first PACKS (reads) the chunk of
// each segment it owns that moves -- so every slot that is about to be
// overwritten has already been read -- then exchanges (one ncclGroup of
// sends/recvs, paired in the global move order on both sides), then UNPACKS
// into the destination slots.  Algorithmic traffic is the reference's
// (each moved segment read once and written once, layout.py:234-250).
RedistPlan redist_plan(int64_t n_cols, int64_t T, int ndev, int world, bool inverse) {
  if (world < 1 || ndev % world) throw Error(CONFIG, "logical devices must be a multiple of the processes");
  const SegPlan sp = segment_plan(n_cols, T, ndev, inverse);
  const auto counts = column_counts(n_cols, T, ndev);
  std::vector<int64_t> off(ndev, 0);
  for (int d = 1; d < ndev; ++d) off[d] = off[d - 1] + counts[d - 1];
  const int nloc = ndev / world;
  auto rank_of = [&](int64_t seg_pos) {
    const int64_t col = seg_pos * sp.seg;
    const int d = (int)(std::upper_bound(off.begin(), off.end(), col) - off.begin()) - 1;
    return d / nloc;
  };
  RedistPlan rp;
  rp.seg = sp.seg;
  for (size_t c = 0; c + 1 < sp.offsets.size(); ++c) {
    const int64_t b = sp.offsets[c], e = sp.offsets[c + 1], m = e - b;
    for (int64_t i = 0; i < m; ++i) {
      const int64_t src = sp.members[b + i], dst = sp.members[b + (i + 1) % m];
      rp.moves.push_back(RedistMove{src, dst, rank_of(src), rank_of(dst)});
    }
  }
  return rp;
}

void Session::redistribute_multi(int dt, int64_t n_rows, int64_t n_cols, int64_t T, int ndev, void* const* shards,
                                 bool inverse) {
  const int esz = dtype_size(dt);
  const RedistPlan rp = redist_plan(n_cols, T, ndev, world, inverse);
  const auto counts = column_counts(n_cols, T, ndev);
  std::vector<int64_t> off(ndev, 0);
  for (int d = 1; d < ndev; ++d) off[d] = off[d - 1] + counts[d - 1];
  const int nloc = ndev / world, dev0 = rank * nloc;
  const int64_t col_bytes = n_rows * esz, seg_bytes = rp.seg * col_bytes;
  auto addr = [&](int64_t seg_pos) {
    const int64_t col = seg_pos * rp.seg;
    const int d = (int)(std::upper_bound(off.begin(), off.end(), col) - off.begin()) - 1;
    return reinterpret_cast<uint64_t>(shards[d - dev0]) + (uint64_t)((col - off[d]) * col_bytes);
  };
  std::vector<const RedistMove*> sends, recvs, locals;
  for (const auto& mv : rp.moves) {
    if (mv.src_rank == rank && mv.dst_rank == rank) locals.push_back(&mv);
    else if (mv.src_rank == rank) sends.push_back(&mv);
    else if (mv.dst_rank == rank) recvs.push_back(&mv);
  }
  last_moved_bytes = 2 * (int64_t)rp.moves.size() * seg_bytes;  // whole-job algorithmic bytes
  const int64_t slots = (int64_t)(sends.size() + locals.size() + recvs.size());
  // every process takes part in the exchange rounds even with nothing to move,
  // so all processes agree on the chunk size (it depends on global counts only)
  int64_t max_slots = 0;
  for (int r = 0; r < world; ++r) {
    int64_t s = 0;
    for (const auto& mv : rp.moves) s += (mv.src_rank == r) + (mv.dst_rank == r && mv.src_rank != r);
    max_slots = std::max(max_slots, s);
  }
  if (max_slots == 0) return;
  int64_t budget = (int64_t)1 << 30;
  if (const char* e = getenv("BCMG_REDIST_STAGING")) budget = std::max<int64_t>(4096, atoll(e));
  int64_t CH = std::min<int64_t>(seg_bytes, std::max<int64_t>(budget < (1 << 20) ? 256 : (1 << 20), budget / max_slots));
  if (CH < seg_bytes) CH = std::max<int64_t>(256, CH / 256 * 256);
  const int vec = (col_bytes % 16 == 0) ? 16 : (col_bytes % 8 == 0 ? 8 : 4);
  // staging: [sends | locals] pack slots, then recv slots
  stage_buf.ensure((size_t)std::max<int64_t>(slots, 1) * CH);
  char* pack = static_cast<char*>(stage_buf.p);
  char* recv = pack + (sends.size() + locals.size()) * CH;
  // descriptor tables: pack (src = segment, dst = slot), unpack (src = slot, dst = segment)
  const size_t npk = sends.size() + locals.size(), nup = locals.size() + recvs.size();
  std::vector<uint64_t> h(2 * npk + 2 * nup);
  for (size_t j = 0; j < sends.size(); ++j) {
    h[j] = addr(sends[j]->src_pos);
    h[npk + j] = reinterpret_cast<uint64_t>(pack + j * CH);
  }
  for (size_t j = 0; j < locals.size(); ++j) {
    const size_t s = sends.size() + j;
    h[s] = addr(locals[j]->src_pos);
    h[npk + s] = reinterpret_cast<uint64_t>(pack + s * CH);
    h[2 * npk + j] = reinterpret_cast<uint64_t>(pack + s * CH);
    h[2 * npk + nup + j] = addr(locals[j]->dst_pos);
  }
  for (size_t j = 0; j < recvs.size(); ++j) {
    const size_t u = locals.size() + j;
    h[2 * npk + u] = reinterpret_cast<uint64_t>(recv + j * CH);
    h[2 * npk + nup + u] = addr(recvs[j]->dst_pos);
  }
  desc_buf.ensure(std::max<size_t>(8, h.size() * 8));
  const uint64_t* d = static_cast<const uint64_t*>(desc_buf.p);
  if (!h.empty()) BCMG_CUDA(cudaMemcpyAsync(desc_buf.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, crit));
  for (int64_t o = 0; o < seg_bytes; o += CH) {
    const int64_t len = std::min(CH, seg_bytes - o);
    timed(K_ROTATE, crit, 2.0 * (double)len * (npk), [&] {
      chunk_copy(d, d + npk, (int)npk, o, 0, len, vec, crit);
    });
    if (world > 1) {
      net->group_start();
      for (size_t j = 0; j < sends.size(); ++j) net->send(pack + j * CH, (size_t)len, sends[j]->dst_rank, crit);
      for (size_t j = 0; j < recvs.size(); ++j) net->recv(recv + j * CH, (size_t)len, recvs[j]->src_rank, crit);
      net->group_end();
    }
    chunk_copy(d + 2 * npk, d + 2 * npk + nup, (int)nup, 0, o, len, vec, crit);
  }
  sync_streams(user, crit);
}

// ------------------------------------------------------------------ schedules
// The per-process operation sequence of potrf / potrs.  The drivers below
// execute it on CUDA streams; bcmg_schedule() exposes it so the multi-process
// logic (ownership, broadcast roots / sizes / order, update ranges) is tested
// on CPU ranks without GPUs (tests/test_multirank_schedule.py).
static Geo geo_only(int64_t n, int64_t T, int ndev, int world, int rank) {
  if (n < 1 || T < 1 || T > n) throw Error(CONFIG, "bad matrix order / tile width");
  if (ndev < 1 || world < 1 || ndev % world || rank < 0 || rank >= world) throw Error(CONFIG, "bad device grid");
  Geo g;
  g.n = n;
  g.T = T;
  g.nt = (n + T - 1) / T;
  g.D = ndev;
  g.nloc = ndev / world;
  g.dev0 = rank * g.nloc;
  g.esz = 1;
  return g;
}

std::vector<SchedOp> potrf_schedule(int64_t n, int64_t T, int ndev, int world, int rank) {
  const Geo g = geo_only(n, T, ndev, world, rank);
  std::vector<SchedOp> ops;
  auto push = [&](int kind, int stream, int64_t k, int64_t a, int64_t b, int64_t root, int64_t elems) {
    ops.push_back(SchedOp{kind, stream, k, a, b, root, elems});
  };
  if (g.owns(0)) push(S_FACTOR, STREAM_CRIT, 0, 0, 0, 0, 0);
  for (int64_t k = 0; k < g.nt; ++k) {
    const int64_t s0 = g.start(k), s1 = g.stop(k);
    if (s1 >= n) break;  // last tile: nothing below it
    // panel rows [stop_k, n) x tile width, from the owner of tile k
    if (world > 1) push(S_BCAST, STREAM_COMM, k, 0, 0, g.owner_rank(k), (n - s1) * (s1 - s0));
    const bool look = g.owns(k + 1);
    if (look) push(S_UPDATE, STREAM_CRIT, k, k + 1, k + 2, 0, 0);
    // world > 1, owner of k+1: factor k+1 right after its lookahead update, on
    // the whole GPU, and start the bulk update after it (root field = 2) --
    // the others need panel k+1 as soon as they finish step k
    const bool first = look && world > 1;
    if (first) push(S_FACTOR, STREAM_CRIT, k + 1, 0, 0, 0, 0);
    // bulk: root field = 1 when the grid is capped to leave SMs to the lookahead path
    push(S_UPDATE, STREAM_BULK, k, look ? k + 2 : k + 1, g.nt, first ? 2 : look ? 1 : 0, 0);
    if (g.owns(k)) push(S_COPYBACK, STREAM_BULK, k, 0, 0, 0, 0);
    push(S_STEP_END, STREAM_BULK, k, look ? 1 : 0, 0, 0, 0);
    if (look && !first) push(S_FACTOR, STREAM_CRIT, k + 1, 0, 0, 0, 0);
  }
  return ops;
}

std::vector<SchedOp> potrs_schedule(int64_t n, int64_t T, int ndev, int world, int rank, int64_t nrhs) {
  const Geo g = geo_only(n, T, ndev, world, rank);
  std::vector<SchedOp> ops;
  for (int64_t k = 0; k < g.nt; ++k) {
    if (g.owns(k)) ops.push_back(SchedOp{S_FWD, STREAM_CRIT, k, 0, 0, 0, 0});
    if (world > 1)  // updated x[start_k:] from the owner
      ops.push_back(SchedOp{S_SHARE, STREAM_CRIT, k, g.start(k), n, g.owner_rank(k), (n - g.start(k)) * nrhs});
  }
  for (int64_t k = g.nt - 1; k >= 0; --k) {
    if (g.owns(k)) ops.push_back(SchedOp{S_BWD, STREAM_CRIT, k, 0, 0, 0, 0});
    if (world > 1)  // solved x_k from the owner
      ops.push_back(SchedOp{S_SHARE, STREAM_CRIT, k, g.start(k), g.stop(k), g.owner_rank(k),
                            (g.stop(k) - g.start(k)) * nrhs});
  }
  return ops;
}

// ------------------------------------------------------------------ workspace
// Every buffer a pipeline will need, allocated BEFORE it moves any data, so an
// out-of-memory failure leaves the caller's shards untouched (the reference
// raises before any data movement, test_solvers.py:344-352).  The drivers'
// own ensure() calls then find the buffers large enough (grow-only).
static int64_t cols_below(const Geo& g, int d, int64_t s);
static int64_t cols_upto(const Geo& g, int d, int64_t s);

// potri's complex real-embedding scratch: column chunks of whole waves of
// output tiles for the product sweep (2*tcs real rows in 128-row blocks; 2 CTAs
// per SM of 64-wide tiles for complex128 on the FP64 TMA kernel, 1 CTA per SM
// of 256-wide tiles for complex64 on tcgen05)
static int64_t potri_wave_cols(int dt, int64_t tcs, int nsm) {
  const int64_t rb = (2 * tcs + 127) / 128;
  return dt == C64 ? std::max<int64_t>(1, nsm / rb) * 256 : std::max<int64_t>(1, 2 * nsm / rb) * 64;
}
// (T and n even: every column count is even, so the choice is the same for any
// device count; complex64: the tcgen05 tile minimums hold for every D)
static bool potri_embeds(int dt, int64_t n, int64_t T) {
  if (getenv("BCMG_NO_CPLX_EMBED")) return false;
  return (dt == C128 && T % 2 == 0 && n % 2 == 0) || (dt == C64 && T % 64 == 0 && n % 4 == 0);
}
static size_t potri_embed_bytes(int dt, int64_t n, int64_t T, int nsm) {
  const size_t esz = dtype_size(dt);
  return std::max(gemm_cplx_embed_bytes(dt, n, n, T), (size_t)(2 * T + 2 * potri_wave_cols(dt, T, nsm)) * n * esz);
}
// columns per product-sweep chunk of the embedded GEMM for a W tile starting at ss
static int64_t potri_chunk_cols(int dt, int64_t n, int64_t ss, int64_t tcs, size_t emb_bytes, int nsm) {
  const int64_t wave = potri_wave_cols(dt, tcs, nsm);
  int64_t nc = (int64_t)(emb_bytes / ((size_t)(n - ss) * dtype_size(dt))) - 2 * tcs;
  return nc >= wave ? nc / wave * wave : nc / 64 * 64;
}
// the tf32 split planes gemm() (float32, tcgen05) requests for an M x N x K product, 0 if it stays off tcgen05
static size_t f32_gemm_split(int64_t M, int64_t N, int64_t K) {
  if (!tc_presplit_enabled() || M < 256 || N < 64 || K < 32) return 0;
  return split_scratch_bytes(R32, M, N, K);
}

WsPlan workspace_plan(int routine, int dt, int64_t n, int64_t T, int ndev, int world, int64_t nrhs, int nsm) {
  if (routine != 1 && routine != 2) throw Error(CONFIG, "unknown routine");
  if (n < 1 || T < 1 || T > n || ndev < 1 || world < 1 || ndev % world)
    throw Error(CONFIG, "bad matrix order / tile width / device grid");
  const size_t esz = dtype_size(dt);
  if (!esz) throw Error(CONFIG, "unknown element-type code");
  const int64_t nt = (n + T - 1) / T;
  WsPlan w;
  const size_t panel_bytes = (size_t)n * T * esz;
  const bool presplit = (dt == R32 || dt == C64) && tc_presplit_enabled();
  if (presplit) {
    const int64_t kx = dt == C64 ? 2 * T : T;
    const size_t plane = (size_t)n * (pair_panels(dt, T) ? 2 * kx : split_ld(kx)) * 4;
    w.split = dt == C64 ? 6 * plane : 2 * plane;
    w.split_scratch = split_scratch_bytes(dt, n, T, T);  // the panel solves
  }
  const bool embed = !presplit && complex_embed_ok(dt, 0, T);
  w.panel = embed ? 2 * panel_bytes : panel_bytes;
  if (embed) w.panel_pb = panel_bytes;
  if (dt == C128 || dt == C64) w.embed = gemm_cplx_embed_bytes(dt, n, T, T);
  w.dinv = (size_t)nt * T * T * esz;
  w.wdiag = (size_t)T * T * esz;
  w.info = sizeof(int);
  if (routine == 1) {  // potrs: split-K slabs + (multi-process) the solution hand-off buffer
    const size_t parts_bytes = std::max((size_t)64 * T * nrhs * esz, subst_gemv_ok(dt, nrhs) ? subst_parts_bytes(n, T, nrhs) : 0);
    w.tmp = std::max<size_t>(4096, parts_bytes + (world > 1 ? (size_t)n * nrhs * esz : 0));
    if (dt == R32)  // forward substitution x[stop:] -= L x_k when the split-K slabs do not fit
      for (int64_t k = 0; k < nt; ++k) {
        const int64_t s1 = std::min(n, (k + 1) * T);
        if (s1 < n && (int64_t)(parts_bytes / ((size_t)(n - s1) * nrhs * esz)) < 2)
          w.split_scratch = std::max(w.split_scratch, f32_gemm_split(n - s1, nrhs, s1 - k * T));
      }
    return w;
  }
  // potri: the W-tile / block buffers and the GEMMs of both sweeps
  w.tmp = 4096;
  w.panel = std::max(w.panel, panel_bytes);
  w.acc = panel_bytes;
  const bool emb = potri_embeds(dt, n, T);
  if (emb) w.embed = std::max(w.embed, potri_embed_bytes(dt, n, T, nsm));
  if (dt == R32 || (dt == C64 && emb && presplit)) {
    Geo g{};
    g.n = n;
    g.T = T;
    g.nt = nt;
    g.D = ndev;
    g.nloc = ndev / world;
    for (int r = 0; r < world; ++r)
      for (int64_t s = 0; s < nt; ++s) {
        const int64_t ss = s * T, se = std::min(n, ss + T), tcs = se - ss;
        if (dt == R32 && se < n) w.split_scratch = std::max(w.split_scratch, f32_gemm_split(n - se, tcs, tcs));
        for (int d = r * g.nloc; d < (r + 1) * g.nloc; ++d) {
          const int64_t cb = cols_below(g, d, s), cu = cols_upto(g, d, s);
          if (dt == R32) {
            if (cb) w.split_scratch = std::max(w.split_scratch, f32_gemm_split(n - ss, cb, tcs));
            if (cu) w.split_scratch = std::max(w.split_scratch, f32_gemm_split(tcs, cu, n - ss));
            continue;
          }
          // complex64 through the embedded tcgen05 GEMM (gemm_cplx_embed's shape rules)
          auto emb_split = [&](int64_t M, int64_t N, int64_t K) -> size_t {
            if (N % 4 || (2 * M) % 4 || 2 * M < 256 || N < 64 || K <= 0) return 0;
            if (w.embed < gemm_cplx_embed_bytes(dt, M, N, K)) return 0;
            return split_scratch_bytes(C64, M, N, K);
          };
          if (cb) w.split_scratch = std::max(w.split_scratch, emb_split(n - ss, cb, tcs));
          if (cu) {
            const int64_t nc = potri_chunk_cols(dt, n, ss, tcs, w.embed, nsm);
            if (nc >= 64)
              for (int64_t c0 = 0; c0 < cu; c0 += nc)
                w.split_scratch = std::max(w.split_scratch, emb_split(tcs, std::min(nc, cu - c0), n - ss));
          }
        }
        // the grouped product GEMM over all local devices (gemm_cplx_embed_grouped) splits whole chunks
        if (dt == C64 && g.nloc > 1 && 2 * tcs >= 256) {
          int64_t tot = 0;
          for (int d = r * g.nloc; d < (r + 1) * g.nloc; ++d) tot += cols_upto(g, d, s);
          const int64_t nc = potri_chunk_cols(dt, n, ss, tcs, w.embed, nsm);
          if (tot && nc >= 64) w.split_scratch = std::max(w.split_scratch, split_scratch_bytes(C64, tcs, nc, n - ss));
        }
      }
  }
  return w;
}

void Session::reserve_workspace(int routine, int dt, int64_t n, int64_t T, int ndev, int64_t nrhs) {
  make_geo(*this, dt, n, T, ndev);  // validates
  const WsPlan w = workspace_plan(routine, dt, n, T, ndev, world, nrhs, nsm);
  if (w.split) {
    split_buf[0].ensure(w.split);
    split_buf[1].ensure(w.split);
  }
  if (w.split_scratch) reserve_split_scratch(crit, w.split_scratch);
  panel[0].ensure(w.panel);
  panel[1].ensure(w.panel);
  if (w.panel_pb) {
    panel_pb[0].ensure(w.panel_pb);
    panel_pb[1].ensure(w.panel_pb);
  }
  if (w.embed) embed_buf.ensure(w.embed);
  dinv.ensure(w.dinv);
  wdiag.ensure(w.wdiag);
  info_dev.ensure(w.info);
  tmp.ensure(w.tmp);
  if (w.acc) acc.ensure(w.acc);
}

size_t Session::held_workspace_bytes() const {
  size_t b = split_scratch_held(crit);
  for (const DevBuf* d : {&panel[0], &panel[1], &panel_pb[0], &panel_pb[1], &split_buf[0], &split_buf[1], &embed_buf,
                          &dinv, &wdiag, &info_dev, &tmp, &acc})
    b += d->bytes;
  return b;
}

// ------------------------------------------------------------------ potrf
// Panel k lives in panel[k % 2] with rows [stop_k, n) (ld = n - stop_k): only
// the rows the trailing update reads (the reference copies the full-height
// panel, solvers.py:389-394).  X_kk = L_kk^-1 is kept in dinv for potrs/potri.
int Session::potrf(int dt, int64_t n, int64_t T, int ndev, void* const* shards, const void* host) {
  const Geo g = make_geo(*this, dt, n, T, ndev);
  if (host && (world != 1 || ndev != 1)) throw Error(CONFIG, "streamed host input needs one process and one device");
  const size_t panel_bytes = (size_t)n * T * g.esz;
  // complex128: the panel is followed by -iP, plus a planar copy (TrailParams::cplx)
  // float32 / complex64 on tcgen05: the panel is split once per step into tf32
  // hi / lo K-major planes (split_buf[k % 2]) that every trailing tile reads
  const bool presplit = (dt == R32 || dt == C64) && tc_presplit_enabled();
  const int64_t kx = dt == C64 ? 2 * T : T, kp = split_ld(kx);
  // Paired panels (pair_panels: tcgen05 path, T <= 256): panels 2j and 2j+1
  // share split buffer split_buf[j % 2] -- K-major rows of width 2 kx starting
  // at row stop(2j), panel 2j in columns [0, kx), panel 2j+1 in [kx, 2 kx)
  // from row stop(2j+1) = stop(2j) + T.  Step 2j updates only its lookahead
  // tile (K = T); step 2j+1 updates tile 2j+2 and the bulk with both panels at
  // once (K = 2T): every trailing tile is read and written once per pair
  // instead of once per panel.  The pairing is global, so the arithmetic (and
  // the bits) do not depend on the device or process count.
  const bool pair = presplit && pair_panels(dt, T);
  const int64_t kpp = pair ? 2 * kx : kp;
  if (presplit) {
    const size_t plane = (size_t)n * kpp * 4;  // rows x kpp floats (A rows: 2n for complex64)
    const size_t bytes = dt == C64 ? 2 * (2 * plane) + 2 * plane : 2 * plane;
    split_buf[0].ensure(bytes);
    split_buf[1].ensure(bytes);
  }
  // split buffer of panel k, the rows of its first panel (stride of the planes) and
  // the row / column offset of panel k inside it
  struct SplitAt {
    float* base;
    int64_t rows0, roff, coff, ld;
  };
  auto split_at = [&](int64_t k) {
    if (!pair) return SplitAt{static_cast<float*>(split_buf[k % 2].p), n - g.stop(k), 0, 0, 0};
    const int64_t k0 = k - (k % 2);
    return SplitAt{static_cast<float*>(split_buf[(k0 / 2) % 2].p), n - g.stop(k0), k % 2 ? T : 0, k % 2 ? kx : 0,
                   kpp};
  };
  auto split_panel = [&](int64_t k, cudaStream_t st) {
    const int64_t rows = n - g.stop(k), tck = g.stop(k) - g.start(k);
    if (!presplit || rows <= 0) return;
    const SplitAt sa = split_at(k);
    const int64_t kpk = pair ? kpp : split_ld(dt == C64 ? 2 * tck : tck);
    const int64_t kw = pair ? kx : -1;
    float* b = sa.base;
    if (dt == R32) {
      float* hi = b + sa.roff * kpk + sa.coff;
      split_tf32(0, panel[k % 2].p, rows, rows, tck, tck, hi, hi + sa.rows0 * kpk, kpk, st, kw);
    } else {
      const int64_t r0 = pair ? sa.rows0 : rows;
      float* ah = b + 2 * sa.roff * kpk + sa.coff;
      float* bh = b + 2 * (2 * r0) * kpk + sa.roff * kpk + sa.coff;  // B planes after the two A planes
      split_tf32(1, panel[k % 2].p, rows, 2 * rows, 2 * tck, tck, ah, ah + 2 * r0 * kpk, kpk, st, kw);
      split_tf32(2, panel[k % 2].p, rows, rows, 2 * tck, tck, bh, bh + r0 * kpk, kpk, st, kw);
    }
  };
  const bool embed = !presplit && complex_embed_ok(dt, 0, T);
  panel[0].ensure(embed ? 2 * panel_bytes : panel_bytes);
  panel[1].ensure(embed ? 2 * panel_bytes : panel_bytes);
  if (embed) {
    panel_pb[0].ensure(panel_bytes);
    panel_pb[1].ensure(panel_bytes);
  }
  const bool cplx_dt = dt == C128 || dt == C64;
  if (cplx_dt) embed_buf.ensure(gemm_cplx_embed_bytes(dt, n, T, T));  // panel solve by real embedding
  auto embed_k = [&](int64_t k) { return embed && complex_embed_ok(dt, n - g.stop(k), T); };
  // Panel broadcast (world > 1), BCMG_PANEL_BCAST = ce | fan | nccl:
  //   ce   (default) the owner pushes panel k into every process's panel
  //        buffer with copy-engine peer copies (cudaMemcpyAsync over NVLink
  //        between CUDA-IPC-mapped buffers) and raises the receivers' ready
  //        flags with stream memory operations: no SM takes part, so the
  //        hand-off never queues behind a persistent trailing-update grid;
  //   fan  the panel solve's epilogue writes every element also into each
  //        peer's buffer (the GEMM fused with its broadcast);
  //   nccl ncclBroadcast (the fallback when peers cannot be mapped).
  // sig words (uint32): [b] panel in buffer b ready (written by the owner),
  // [2 + 16 b + r] process r done with buffer b (written by r).  Receivers
  // park a stream on cuStreamWaitValue32; no kernel waits on another rank.
  enum { BC_NCCL = 0, BC_CE = 1, BC_FAN = 2 };
  int bc_mode = BC_NCCL;
  if (world > 1) {
    const char* m = getenv("BCMG_PANEL_BCAST");
    const char* legacy = getenv("BCMG_P2P");  // round-1 name of the fan-out mode
    bc_mode = m ? (!strcmp(m, "fan") ? BC_FAN : !strcmp(m, "nccl") ? BC_NCCL : BC_CE)
                : (legacy ? (atoi(legacy) ? BC_FAN : BC_NCCL) : BC_CE);
    if (!net->flags_supported() || (bc_mode == BC_FAN && world > MAX_FAN + 1)) bc_mode = BC_NCCL;
  }
  bool p2p = bc_mode != BC_NCCL;
  std::vector<void*> fan_panel[2];
  uint32_t seq0 = 0;
  if ((dt == R32 || dt == C64) && tc_presplit_enabled())  // the panel solves' split planes, sized up front
    reserve_split_scratch(crit, split_scratch_bytes(dt, n, T, T));
  if (p2p) {
    for (int b2 = 0; b2 < 2; ++b2) {
      net->release_pointers(peer_panel[b2]);
      peer_panel[b2] = net->exchange_pointers(panel[b2].p);
      for (int r = 0; r < (int)peer_panel[b2].size(); ++r)
        if (r != rank) fan_panel[b2].push_back(peer_panel[b2][r]);
    }
    // every rank sees the same exchange outcome (collective agreement in exchange_pointers)
    if (peer_panel[0].empty() || peer_panel[1].empty()) {
      p2p = false;
      bc_mode = BC_NCCL;
      fan_panel[0].clear();
      fan_panel[1].clear();
    }
  }
  if (p2p) {
    seq0 = panel_seq;
    panel_seq += (uint32_t)g.nt + 4;
  }
  last_bcast_mode = bc_mode;
  // flag slots (Comm::post_flag / wait_flag): [b] panel in buffer b ready,
  // [2 + 16 b + r] process r done with buffer b
  auto post_all = [&](cudaStream_t st, int slot_base, bool per_rank, uint32_t v) {
    for (int r = 0; r < world; ++r)
      if (r != rank) net->post_flag(r, slot_base + (per_rank ? rank : 0), v, st);
  };
  auto seq_of = [&](int64_t k) { return seq0 + (uint32_t)k + 1; };
  // peers done with buffer b before panel k is written into it: their last use
  // was panel k - 2 (or the last panel in b of the previous call)
  auto wait_peers_free = [&](int64_t k, cudaStream_t st) {
    const int bb = (int)(k % 2);
    const uint32_t need = k >= 2 ? seq_of(k - 2) : free_seq[bb];
    if (!need) return;
    for (int r = 0; r < world; ++r)
      if (r != rank) net->wait_flag(2 + 16 * bb + r, need, st);
  };
  dinv.ensure((size_t)g.nt * T * T * g.esz);
  wdiag.ensure((size_t)T * T * g.esz);
  info_dev.ensure(sizeof(int));
  tmp.ensure(4096);
  int* info = static_cast<int*>(info_dev.p);
  BCMG_CUDA(cudaMemsetAsync(info, 0, sizeof(int), crit));
  sync_streams(bulk, crit);
  sync_streams(comm, crit);
  fkey.valid = false;  // dinv is being overwritten

  auto dinv_k = [&](int64_t k) { return static_cast<char*>(dinv.p) + (size_t)k * T * T * g.esz; };
  auto shard_of = [&](int64_t k) { return shards[(k % g.D) - g.dev0]; };

  // F(k): factor diagonal block + inverse, panel solve into panel[k%2]
  auto factor = [&](int64_t k) {
    const int64_t s0 = g.start(k), s1 = g.stop(k), tc = s1 - s0;
    void* sh = shard_of(k);
    void* Akk = colp(sh, g, s0, g.loc(k));
    const double cf = dtype_complex(dt) ? 4.0 : 1.0;
    timed(K_DIAG, crit, cf * (double)tc * tc * tc / 3.0,
          [&] { diag_factor(dt, Akk, n, dinv_k(k), T, wdiag.p, tc, s0, info, crit); });
    if (s1 < n) {
      timed(K_TRSM, crit, cf * 2.0 * (double)(n - s1) * tc * tc, [&] {
        const Operand a21 = opA(colp(sh, g, s1, g.loc(k)), n, OP_N), xh = opB(dinv_k(k), T, OP_C);
        Epilogue ep{panel[k % 2].p, n - s1, 1.0, 0.0, 0, 0};
        if (bc_mode == BC_FAN) {  // the panel solve's epilogue also writes every peer's copy of the panel
          ep.nfan = (int)fan_panel[k % 2].size();
          for (int e = 0; e < ep.nfan; ++e) ep.fan[e] = fan_panel[k % 2][e];
        }
        if (!(cplx_dt && gemm_cplx_embed(dt, n - s1, tc, tc, a21, xh, ep, embed_buf.p, embed_buf.bytes, info, crit)))
          gemm(dt, n - s1, tc, tc, a21, xh, ep, info, crit);
      });
      if (embed_k(k)) expand_panel(dt, panel[k % 2].p, panel_pb[k % 2].p, n - s1, tc, crit);
      split_panel(k, crit);
    }
  };
  // While the lookahead path (diag factor + panel solve of tile k+1) runs on the
  // crit stream, the bulk update is a persistent grid capped at (SMs - reserve)
  // CTAs: its CTAs fill an SM's shared memory, so the cap is what leaves SMs
  // on which the latency-bound critical path can overlap the bulk GEMM.
  // Per step: while the trailing matrix is at least 32 tiles wide the DMMA
  // bulk update dwarfs the critical path and gets every SM; below that, 2 SMs
  // stay free for it (measured, f64 T=1024: N=131072 reserve 0/1/2 -> 34.3/
  // 34.2/33.9 TFLOP/s; N=32768 reserve 2/4/8 -> 28.9/27.7/28.2).  The tcgen05
  // bulk update (float32 / complex64) finishes a step so much sooner that the
  // critical path needs its 2 SMs throughout (N=65536 T=1024 reserve 0/2/4:
  // f32 165/177/177, c64 184/190/191 TFLOP/s; T=128 unchanged).
  int reserve_fixed = -1;
  if (const char* e = getenv("BCMG_RESERVE_SMS"); e && *e) reserve_fixed = std::max(0, atoi(e));
  auto reserve_at = [&](int64_t k) {
    if (reserve_fixed >= 0) return reserve_fixed;
    // complex64 at T_A >= 2048: the diagonal factor (7.4 ms per 2048 tile) needs more
    // than 2 SMs to hide (N=65536, 8 devices, reserve 2 / 8 / 12: 189.4, 187.5 / 196.2,
    // 197.4 / 193.1, 194.0 TFLOP/s; float32 flat, complex64 T_A=1024 -1 % at 8)
    if (presplit) return dt == C64 && T >= 2048 ? 8 : 2;
    return (n - g.stop(k)) / T >= 32 ? 0 : 2;
  };
  // world > 1 with the NCCL broadcast: the NCCL kernels need SMs on every
  // rank while the bulk grid runs, so the grid leaves the communicator's CTA
  // limit free (NcclComm caps its CTAs at BCMG_NCCL_MAX_CTAS, default 8)
  int bulk_cap = 0;
  if (world > 1 && bc_mode == BC_NCCL) bulk_cap = std::max(1, nsm - nccl_max_ctas());
  auto trail = [&](int64_t k, int64_t m_first, int64_t m_last, cudaStream_t st, int cap = 0) {
    TrailParams p{};
    p.max_ctas = cap;
    p.P = panel[k % 2].p;
    if (embed_k(k)) {
      p.cplx = 1;
      p.PB = panel_pb[k % 2].p;
    }
    int64_t K = g.stop(k) - g.start(k);
    if (presplit) {
      const int64_t rows = n - g.stop(k);
      const SplitAt sa = split_at(k);
      const int64_t kpk = pair ? kpp : split_ld(dt == C64 ? 2 * K : K);
      const int64_t r0 = pair ? sa.rows0 : rows;  // rows of the planes
      float* b = sa.base;
      if (pair && k % 2) K += T;  // both panels of the pair (columns [0, 2 kx), zero-padded)
      if (dt == R32) {
        p.split[0] = p.split[2] = b + sa.roff * kpk;
        p.split[1] = p.split[3] = b + r0 * kpk + sa.roff * kpk;
      } else {
        p.cplx = 1;
        p.split[0] = b + 2 * sa.roff * kpk;
        p.split[1] = b + 2 * r0 * kpk + 2 * sa.roff * kpk;
        p.split[2] = b + 4 * r0 * kpk + sa.roff * kpk;
        p.split[3] = b + 5 * r0 * kpk + sa.roff * kpk;
      }
      p.split_ld[0] = p.split_ld[1] = kpk;
    }
    p.prow0 = g.stop(k);
    p.ldp = n - p.prow0;
    p.N = n;
    p.T = T;
    p.K = K;
    p.D = g.D;
    p.dev0 = g.dev0;
    p.nloc = g.nloc;
    for (int i = 0; i < g.nloc; ++i) p.shards[i] = shards[i];
    p.m_first = m_first;
    p.m_last = m_last;
    double flops = 0;  // algorithmic: lower trapezoid of every updated local tile
    for (int64_t m = m_first; m < m_last; ++m) {
      if (!g.owns(m)) continue;
      const double rows = (double)(n - m * T), tcm = (double)std::min<int64_t>(T, n - m * T);
      flops += 2.0 * (double)p.K * (rows * tcm - tcm * (tcm - 1) / 2);
    }
    if (dtype_complex(dt)) flops *= 4.0;
    static const int dbg = [] {
      const char* e = getenv("BCMG_PAIR_DEBUG");
      return e ? atoi(e) : 0;
    }();
    if (dbg & 1) BCMG_CUDA(cudaDeviceSynchronize());
    if (flops > 0) timed(K_TRAIL, st, flops, [&] { trailing_update(dt, p, info, st); });
    if (dbg & 2) BCMG_CUDA(cudaDeviceSynchronize());
  };

  // Streamed host input (one device): the tile columns are copied from pinned
  // host memory on the comm stream in order; while they arrive, tiles [0, j)
  // are factored LEFT-looking (tile m -= L[:, 0:m] L[m rows, 0:m]^H, one GEMM
  // with K = m T, then its diagonal factor and panel solve), so the GPU works
  // during the upload; once everything is resident the trailing tiles receive
  // the update of panels [0, j) in one trailing-update launch (K = j T) and the
  // right-looking schedule continues from step j.  (float64; other types
  // upload first.)  The summation order of those first updates differs from
  // the device-input path, so results agree to rounding, not bit for bit.
  int64_t k0 = 0;
  if (host) {
    std::vector<cudaEvent_t> up(g.nt);
    char* dev = static_cast<char*>(shards[0]);
    const char* src = static_cast<const char*>(host);
    BCMG_CUDA(cudaStreamWaitEvent(comm, ev(kJoin + 4), 0));
    for (int64_t m = 0; m < g.nt; ++m) {
      const size_t off = (size_t)g.start(m) * n * g.esz, bytes = (size_t)(g.stop(m) - g.start(m)) * n * g.esz;
      BCMG_CUDA(cudaMemcpyAsync(dev + off, src + off, bytes, cudaMemcpyHostToDevice, comm));
      BCMG_CUDA(cudaEventCreateWithFlags(&up[m], cudaEventDisableTiming));
      BCMG_CUDA(cudaEventRecord(up[m], comm));
    }
    const int64_t j = (dt == R64 && g.nt >= 8 && !getenv("BCMG_NO_STREAMED_LEFT")) ? g.nt / 4 : 0;
    for (int64_t m = 0; m < j; ++m) {
      const int64_t ms = g.start(m), me = g.stop(m), tc = me - ms;
      BCMG_CUDA(cudaStreamWaitEvent(crit, up[m], 0));
      if (m > 0) {
        char* A = static_cast<char*>(shards[0]);
        gemm(dt, n - ms, tc, ms, opA(A + ms * g.esz, n, OP_N), opB(A + ms * g.esz, n, OP_C),
             Epilogue{A + (ms + ms * n) * g.esz, n, -1.0, 1.0, 0, 0}, info, crit);
      }
      factor(m);
      if (me < n) copy2d(dt, panel[m % 2].p, n - me, colp(shards[0], g, me, g.loc(m)), n, n - me, tc, false, info,
                         crit);
    }
    BCMG_CUDA(cudaStreamWaitEvent(crit, up[g.nt - 1], 0));
    if (j > 0 && j < g.nt) {  // catch-up: tiles [j, nt) -= L[:, 0:jT] L[tile rows, 0:jT]^H
      TrailParams p{};
      p.P = static_cast<char*>(shards[0]) + g.start(j) * g.esz;
      p.ldp = n;
      p.prow0 = g.start(j);
      p.N = n;
      p.T = T;
      p.K = g.start(j);
      p.D = 1;
      p.dev0 = 0;
      p.nloc = 1;
      p.shards[0] = shards[0];
      p.m_first = j;
      p.m_last = g.nt;
      double flops = 0;
      for (int64_t m = j; m < g.nt; ++m) {
        const double rows = (double)(n - m * T), tcm = (double)std::min<int64_t>(T, n - m * T);
        flops += 2.0 * (double)p.K * (rows * tcm - tcm * (tcm - 1) / 2);
      }
      timed(K_TRAIL, crit, flops, [&] { trailing_update(dt, p, info, crit); });
    }
    for (cudaEvent_t e : up) cudaEventDestroy(e);
    sync_streams(bulk, crit);
    sync_streams(comm, crit);
    k0 = j;
  }

  // Execute this process's schedule (potrf_schedule).  Event slots:
  // type*8 + k%8 (dependencies reach back at most two steps).
  //   R[k]    panel k usable on this process     C[k] broadcast of panel k done
  //   B[k]    bulk update + copy-back of step k  U[k] lookahead update of step k
  //   FREE[k] panel buffer k%2 reusable
  //   CB[k]   copy-back of panel k into A done (side stream, copy engine)
  enum { R = 0, C = 1, B = 2, U = 3, FREE = 4, CB = 5 };
  auto E = [&](int type, int64_t k) { return ev(type * 8 + (int)(k % 8)); };
  for (const SchedOp& op : potrf_schedule(n, T, ndev, world, rank)) {
    if (op.k < k0) continue;  // factored left-looking during a streamed upload
    const int64_t k = op.k, s1 = g.stop(k);
    const bool mine = g.owns(k);
    const int b = (int)(k % 2);
    switch (op.kind) {
      case S_FACTOR:  // F(k) overwrites panel buffer k%2, last used by panel k-2 (and its copy-back)
        if (k >= 2) BCMG_CUDA(cudaStreamWaitEvent(crit, E(FREE, k - 2), 0));
        if (k >= 2 && g.owns(k - 2) && k - 2 >= k0) BCMG_CUDA(cudaStreamWaitEvent(crit, E(CB, k - 2), 0));
        if (bc_mode == BC_FAN && s1 < n) wait_peers_free(k, crit);
        factor(k);
        if (bc_mode == BC_FAN && s1 < n) {  // panel k is in every peer's buffer: raise their ready flags
          post_all(crit, b, false, seq_of(k));
          BCMG_CUDA(cudaEventRecord(E(C, k), crit));
        }
        BCMG_CUDA(cudaEventRecord(E(R, k), crit));
        break;
      case S_BCAST:  // panel k reaches every process
        if (bc_mode == BC_CE && mine) {  // copy-engine push into every peer's buffer b, then the ready flags
          const size_t bytes = (size_t)op.elems * g.esz;
          BCMG_CUDA(cudaStreamWaitEvent(comm, E(R, k), 0));
          wait_peers_free(k, comm);
          for (void* dst : fan_panel[b])
            if (bytes) BCMG_CUDA(cudaMemcpyAsync(dst, panel[b].p, bytes, cudaMemcpyDeviceToDevice, comm));
          post_all(comm, b, false, seq_of(k));
          BCMG_CUDA(cudaEventRecord(E(C, k), comm));
          break;
        }
        if (p2p) {
          if (mine) break;
          net->wait_flag(b, seq_of(k), comm);  // raised by the owner after its copies / fused solve
          BCMG_CUDA(cudaEventRecord(E(C, k), comm));
          if (embed_k(k)) expand_panel(dt, panel[b].p, panel_pb[b].p, n - s1, s1 - g.start(k), comm);
          split_panel(k, comm);
          BCMG_CUDA(cudaEventRecord(E(R, k), comm));
          break;
        }
        if (mine) BCMG_CUDA(cudaStreamWaitEvent(comm, E(R, k), 0));
        else if (k >= 2) BCMG_CUDA(cudaStreamWaitEvent(comm, E(FREE, k - 2), 0));
        bcast(panel[b].p, (size_t)op.elems * g.esz, (int)op.root, comm);
        BCMG_CUDA(cudaEventRecord(E(C, k), comm));
        if (!mine && embed_k(k)) expand_panel(dt, panel[b].p, panel_pb[b].p, n - s1, s1 - g.start(k), comm);
        if (!mine) split_panel(k, comm);
        if (!mine) BCMG_CUDA(cudaEventRecord(E(R, k), comm));
        break;
      case S_UPDATE:
        if (op.stream == STREAM_CRIT) {  // lookahead: tile k+1 first, full grid
          if (!mine) BCMG_CUDA(cudaStreamWaitEvent(crit, E(R, k), 0));
          if (pair && k % 2) BCMG_CUDA(cudaStreamWaitEvent(crit, E(R, k - 1), 0));  // the pair's first split
          if (k >= 1) BCMG_CUDA(cudaStreamWaitEvent(crit, E(B, k - 1), 0));
          trail(k, op.a, op.b, crit);
          BCMG_CUDA(cudaEventRecord(E(U, k), crit));
        } else {
          BCMG_CUDA(cudaStreamWaitEvent(bulk, E(R, k), 0));  // (also orders the copy-back of panel k)
          // paired panels: the bulk of step 2j waits for step 2j+1 (both panels at once)
          if (pair && k % 2 == 0 && k + 2 < g.nt) break;
          if (pair && k % 2) BCMG_CUDA(cudaStreamWaitEvent(bulk, E(R, k - 1), 0));
          // with a lookahead this step, the full-grid update of tile k+1 goes
          // first; otherwise both persistent grids would race for the SMs and
          // the critical path could be queued behind the whole bulk update
          if (op.root) BCMG_CUDA(cudaStreamWaitEvent(bulk, E(U, k), 0));
          if (op.root == 2) {
            // owner first (world > 1): panel k+1 is factored and solved on the
            // whole GPU before this process's bulk update, so the other
            // processes receive it while they are still busy with step k
            BCMG_CUDA(cudaStreamWaitEvent(bulk, E(R, k + 1), 0));
            trail(k, op.a, op.b, bulk, bulk_cap);
          } else {
            trail(k, op.a, op.b, bulk, op.root ? std::max(1, nsm - reserve_at(k)) : 0);
          }
        }
        break;
      case S_COPYBACK:  // factor below the diagonal back into A (potrs/potri read it there)
        // on the copy engines, off the bulk stream: nothing in potrf reads it, and
        // between two bulk launches it was part of the gap the critical path sees
        BCMG_CUDA(cudaStreamWaitEvent(side, E(R, k), 0));
        if (s1 < n)
          BCMG_CUDA(cudaMemcpy2DAsync(colp(shard_of(k), g, s1, g.loc(k)), (size_t)n * g.esz, panel[b].p,
                                      (size_t)(n - s1) * g.esz, (size_t)(n - s1) * g.esz, (size_t)(s1 - g.start(k)),
                                      cudaMemcpyDeviceToDevice, side));
        BCMG_CUDA(cudaEventRecord(E(CB, k), side));
        break;
      case S_STEP_END:  // panel buffer k%2 reusable once bulk(k), U(k) and the broadcast are done
        BCMG_CUDA(cudaEventRecord(E(B, k), bulk));
        if (op.a) BCMG_CUDA(cudaStreamWaitEvent(bulk, E(U, k), 0));
        if (world > 1) BCMG_CUDA(cudaStreamWaitEvent(bulk, E(C, k), 0));
        BCMG_CUDA(cudaEventRecord(E(FREE, k), bulk));
        if (p2p && s1 < n) {  // tell every process that buffer b may take panel k + 2
          post_all(bulk, 2 + 16 * b, true, seq_of(k));
          free_seq[b] = seq_of(k);
        }
        break;
      default:
        throw Error(CONFIG, "bad potrf schedule op");
    }
  }
  join();
  BCMG_CUDA(cudaMemcpyAsync(info_host, info, sizeof(int), cudaMemcpyDeviceToHost, user));
  BCMG_CUDA(cudaStreamSynchronize(user));
  const int out = reduce_info(*info_host);
  if (out == 0) {
    fkey.valid = true;
    fkey.dt = dt;
    fkey.n = n;
    fkey.T = T;
    fkey.ndev = ndev;
    fkey.shards.assign(g.nloc, 0);
    for (int i = 0; i < g.nloc; ++i) fkey.shards[i] = reinterpret_cast<uintptr_t>(shards[i]);
  }
  return out;
}


// ------------------------------------------------------------------ potrs
// Substitution on the owners of each tile (no panel movement, unlike the
// reference's _fetch_panel, solvers.py:412-427).  x (n x nrhs, ldx) is
// replicated on every process; each step's arithmetic happens on the tile
// owner only, in tile order, so the bits do not depend on the device count.
//   forward : x_k <- X_kk x_k ; x[stop:] -= L[stop:, k] x_k      (solvers.py:455-461)
//   backward: x_k -= L[stop:, k]^H x[stop:] ; x_k <- X_kk^H x_k   (solvers.py:462-469)
// With world > 1 the owner broadcasts x[start:] (forward) / x_k (backward).
void Session::potrs(int dt, int64_t n, int64_t nrhs, int64_t T, int ndev, void* const* shards, void* x, int64_t ldx) {
  const Geo g = make_geo(*this, dt, n, T, ndev);
  if (nrhs < 1) throw Error(CONFIG, "right-hand side must be non-empty");
  if (ldx < n) throw Error(CONFIG, "ldx < n");
  if (!fkey.matches(dt, n, T, ndev, shards, g.nloc) || dinv.bytes < (size_t)g.nt * T * T * g.esz)
    throw Error(CONFIG, "potrs needs the factorization of the last successful potrf of this session "
                        "(same shards, order, element type, tile width and device count)");
  // split-K slabs (fixed count per shape: bits independent of the device count)
  const int64_t max_parts = 64;
  const bool fast = subst_gemv_ok(dt, nrhs);  // bandwidth kernels for narrow right-hand sides
  const size_t parts_bytes = std::max((size_t)max_parts * T * nrhs * g.esz, fast ? subst_parts_bytes(n, T, nrhs) : 0);
  const size_t pack_bytes = world > 1 ? (size_t)n * nrhs * g.esz : 0;
  tmp.ensure(std::max<size_t>(4096, parts_bytes + pack_bytes));
  char* parts = static_cast<char*>(tmp.p);
  char* pack = parts + parts_bytes;
  char* xb = static_cast<char*>(x);
  auto xrow = [&](int64_t r) { return xb + r * g.esz; };
  auto dinv_k = [&](int64_t k) { return static_cast<char*>(dinv.p) + (size_t)k * T * T * g.esz; };
  cudaStream_t st = crit;
  auto share = [&](int64_t r0, int64_t rows, int root) {  // broadcast x[r0:r0+rows, :]
    if (world == 1 || rows <= 0) return;
    if (rank == root) copy2d(dt, xrow(r0), ldx, pack, rows, rows, nrhs, false, nullptr, st);
    bcast(pack, (size_t)rows * nrhs * g.esz, root, st);
    if (rank != root) copy2d(dt, pack, rows, xrow(r0), ldx, rows, nrhs, false, nullptr, st);
  };
  for (const SchedOp& op : potrs_schedule(n, T, ndev, world, rank, nrhs)) {
    const int64_t k = op.k, s0 = g.start(k), s1 = g.stop(k), tc = s1 - s0;
    if (op.kind == S_SHARE) {
      share(op.a, op.b - op.a, (int)op.root);
      continue;
    }
    void* sh = shards[(k % g.D) - g.dev0];
    if (fast) {
      char* tmpz = parts + subst_parts_bytes(n, T, nrhs) - (size_t)T * nrhs * 16;
      if (op.kind == S_FWD)
        subst_fwd(dt, n - s0, tc, nrhs, dinv_k(k), T, colp(sh, g, s0, g.loc(k)), n, xrow(s0), ldx, tmpz, st);
      else
        subst_bwd(dt, n - s0, tc, nrhs, dinv_k(k), T, colp(sh, g, s0, g.loc(k)), n, xrow(s0), ldx, parts, tmpz, st);
      continue;
    }
    if (op.kind == S_FWD) {
      // x_k <- X_kk x_k: split-K straight into x_k (the slabs hold the product)
      const int npd = gemm_splitk(dt, tc, nrhs, tc, opA(dinv_k(k), T, OP_N), opB(xrow(s0), ldx, OP_N), parts,
                                  (int)max_parts, st);
      reduce_parts(dt, parts, tc * nrhs, npd, xrow(s0), ldx, tc, nrhs, 1.0, st, 0.0);
      if (s1 < n) {
        // x[stop:] -= L[stop:, k] x_k, split-K when the row blocks alone are under two waves
        const int64_t cap = (int64_t)(parts_bytes / ((size_t)(n - s1) * nrhs * g.esz));
        if (cap >= 2) {
          const int np = gemm_splitk(dt, n - s1, nrhs, tc, opA(colp(sh, g, s1, g.loc(k)), n, OP_N),
                                     opB(xrow(s0), ldx, OP_N), parts, (int)std::min(cap, max_parts), st);
          reduce_parts(dt, parts, (n - s1) * nrhs, np, xrow(s1), ldx, n - s1, nrhs, -1.0, st);
        } else {
          gemm(dt, n - s1, nrhs, tc, opA(colp(sh, g, s1, g.loc(k)), n, OP_N), opB(xrow(s0), ldx, OP_N),
               Epilogue{xrow(s1), ldx, -1.0, 1.0, 0, 0}, nullptr, st);
        }
      }
      continue;
    }
    {
      if (s1 < n) {
        // split-K over the rows below the tile (fixed slabs, fixed-order sum:
        // the bits depend on n and T only, not on the device count)
        const int np = gemm_splitk(dt, tc, nrhs, n - s1, opA(colp(sh, g, s1, g.loc(k)), n, OP_C),
                                   opB(xrow(s1), ldx, OP_N), parts, (int)max_parts, st);
        reduce_parts(dt, parts, tc * nrhs, np, xrow(s0), ldx, tc, nrhs, -1.0, st);
      }
      const int npd = gemm_splitk(dt, tc, nrhs, tc, opA(dinv_k(k), T, OP_C), opB(xrow(s0), ldx, OP_N), parts,
                                  (int)max_parts, st);
      reduce_parts(dt, parts, tc * nrhs, npd, xrow(s0), ldx, tc, nrhs, 1.0, st, 0.0);
    }
  }
  sync_streams(user, crit);
}

// ------------------------------------------------------------------ potri
// In place on the cyclic shards, restructured so that every W tile crosses
// the processes exactly once per sweep (the reference fetches W_s once per
// (k, s) pair, solvers.py:513-571):
//
//   W sweep (s = nt-1 .. 0), W = L^-1:
//     WFINAL(s)  owner: W21_s = -acc_s X_ss (acc_s accumulated in tile s rows
//                [stop_s, n) -- those rows of L21_s are dead by then); W_ss = X_ss
//     BCAST(s)   W_s rows [start_s, n) to every process
//     WACC(s)    every process, for all its tiles k < s at once (contiguous
//                local columns): acc_k[start_s:] += W_s L21_k[start_s:stop_s]
//                (the L21 rows are staged first: acc and L21 share storage)
//   product sweep (s = 0 .. nt-1), A^-1 = W^H W:
//     BCAST(s)   W_s rows [start_s, n)
//     PGEMM(s)   every process: block (s, j) = W_s^H W_j[start_s:] for all its
//                tiles j <= s in one GEMM; written to tile j rows [start_s, stop_s)
//     PGATHER(s) blocks gathered on the owner of s and mirrored (conjugate
//                transpose) into tile s rows [start_j, stop_j); diagonal block
//                made exactly Hermitian with a real diagonal (solvers.py:577-583)
//
// acc_k receives W_s in descending s on every process and each product block
// is one GEMM, so the bits do not depend on the device or process count.
static int64_t cols_below(const Geo& g, int d, int64_t s) {  // local columns of device d's tiles < s
  return s > d ? ((s - d + g.D - 1) / g.D) * g.T : 0;
}
static int64_t cols_upto(const Geo& g, int d, int64_t s) {  // ... tiles <= s
  return cols_below(g, d, s) + (s % g.D == d ? g.stop(s) - g.start(s) : 0);
}

std::vector<SchedOp> potri_schedule(int64_t n, int64_t T, int ndev, int world, int rank) {
  const Geo g = geo_only(n, T, ndev, world, rank);
  std::vector<SchedOp> ops;
  auto tile_elems = [&](int64_t s) { return (n - g.start(s)) * (g.stop(s) - g.start(s)); };
  for (int64_t s = g.nt - 1; s >= 0; --s) {
    if (g.owns(s)) ops.push_back(SchedOp{S_WFINAL, STREAM_CRIT, s, 0, 0, 0, 0});
    if (s == 0) break;  // nothing below tile 0 accumulates
    ops.push_back(SchedOp{S_TILE_BCAST, STREAM_CRIT, s, 0, 0, g.owner_rank(s), tile_elems(s)});
    ops.push_back(SchedOp{S_WACC, STREAM_CRIT, s, 0, 0, 0, 0});
  }
  for (int64_t s = 0; s < g.nt; ++s) {
    const int64_t tcs = g.stop(s) - g.start(s);
    int64_t mine = 0;
    for (int d = g.dev0; d < g.dev0 + g.nloc; ++d) mine += cols_upto(g, d, s);
    ops.push_back(SchedOp{S_TILE_BCAST, STREAM_CRIT, s, 0, 0, g.owner_rank(s), tile_elems(s)});
    ops.push_back(SchedOp{S_PGEMM, STREAM_CRIT, s, 0, 0, 0, 0});
    ops.push_back(SchedOp{S_PGATHER, STREAM_CRIT, s, 0, 0, g.owner_rank(s), tcs * mine});
  }
  return ops;
}

void Session::potri(int dt, int64_t n, int64_t T, int ndev, void* const* shards) {
  const Geo g = make_geo(*this, dt, n, T, ndev);
  if (!fkey.matches(dt, n, T, ndev, shards, g.nloc) || dinv.bytes < (size_t)g.nt * T * T * g.esz)
    throw Error(CONFIG, "potri needs the factorization of the last successful potrf of this session "
                        "(same shards, order, element type, tile width and device count)");
  fkey.valid = false;  // the shards are overwritten with the inverse
  const size_t nt_bytes = (size_t)n * T * g.esz;
  panel[0].ensure(nt_bytes);  // broadcast W tile
  panel[1].ensure(nt_bytes);  // staged L21 rows / finalisation product
  acc.ensure(nt_bytes);       // product blocks of every device (gather buffer)
  // complex128: scratch of the real-embedding GEMMs (W sweep: (2(n-s)+c) x T; product
  // sweep: column chunks of (2T + chunk) x (n-s))
  // columns of one full wave of embedded output tiles for a product sweep GEMM
  // with tcs rows: 2*tcs real rows in 128-row blocks, 2 CTAs per SM of 64-wide
  // tiles (complex128, FP64 TMA kernel) or 1 CTA per SM of 256-wide tiles
  // (complex64, tcgen05)
  const bool emb = potri_embeds(dt, n, T);
  // the planned size, not embed_buf.bytes (grow-only: a larger earlier call
  // would change the chunking and the scratch it requests)
  const size_t emb_bytes = emb ? std::max(gemm_cplx_embed_bytes(dt, n, T, T), potri_embed_bytes(dt, n, T, nsm)) : 0;
  if (emb) embed_buf.ensure(emb_bytes);
  cudaStream_t st = crit;
  char* pan = static_cast<char*>(panel[0].p);
  char* stage = static_cast<char*>(panel[1].p);
  char* blocks = static_cast<char*>(acc.p);
  auto shard_of = [&](int64_t k) { return shards[(k % g.D) - g.dev0]; };
  auto dinv_k = [&](int64_t k) { return static_cast<char*>(dinv.p) + (size_t)k * T * T * g.esz; };
  // W_s rows [start_s, n): the owner's tile itself in one process, else the broadcast copy
  auto w_of = [&](int64_t s, int64_t* ld) -> const void* {
    if (world == 1) {
      *ld = n;
      return colp(shard_of(s), g, g.start(s), g.loc(s));
    }
    *ld = n - g.start(s);
    return pan;
  };
  // offset (elements) of device d's product block in the gather buffer
  auto block_off = [&](int64_t s, int d) {
    int64_t o = 0;
    for (int e = 0; e < d; ++e) o += cols_upto(g, e, s);
    return o * (g.stop(s) - g.start(s));
  };
  for (const SchedOp& op : potri_schedule(n, T, ndev, world, rank)) {
    const int64_t s = op.k, ss = g.start(s), se = g.stop(s), tcs = se - ss;
    switch (op.kind) {
      case S_WFINAL: {
        char* Ws = colp(shard_of(s), g, 0, g.loc(s));
        if (se < n) {  // W21 = -acc X_ss, through the staging buffer (in place otherwise)
          gemm(dt, n - se, tcs, tcs, opA(Ws + se * g.esz, n, OP_N), opB(dinv_k(s), T, OP_N),
               Epilogue{stage, n - se, -1.0, 0.0, 0, 0}, nullptr, st);
          copy2d(dt, stage, n - se, Ws + se * g.esz, n, n - se, tcs, false, nullptr, st);
        }
        copy2d(dt, dinv_k(s), T, Ws + ss * g.esz, n, tcs, tcs, false, nullptr, st);
        break;
      }
      case S_TILE_BCAST:
        if (world == 1) break;
        if (rank == op.root) copy2d(dt, colp(shard_of(s), g, ss, g.loc(s)), n, pan, n - ss, n - ss, tcs, false,
                                    nullptr, st);
        bcast(pan, (size_t)op.elems * g.esz, (int)op.root, st);
        break;
      case S_WACC: {
        int64_t ldw = 0;
        const void* W = w_of(s, &ldw);
        const Operand wa = opA(W, ldw, OP_N);
        // L21_k rows [ss, se) of all k < s, staged per device as (L21 rows)^H (c x tcs, one
        // region each) so that the GEMM's B operand is in natural orientation (TMA-eligible)
        std::vector<Operand> bs;
        std::vector<int64_t> nc_d;
        std::vector<void*> cs;
        int64_t soff = 0;
        for (int d = g.dev0; d < g.dev0 + g.nloc; ++d) {
          const int64_t c = cols_below(g, d, s);
          if (c == 0) continue;
          char* sh = colp(shards[d - g.dev0], g, ss, 0);
          char* sd = stage + soff * g.esz;
          conj_transpose(dt, sh, n, sd, c, c, tcs, st);
          BCMG_CUDA(cudaMemset2DAsync(sh, n * g.esz, 0, tcs * g.esz, c, st));  // first touch of acc rows [ss, se)
          bs.push_back(opB(sd, c, OP_C));
          nc_d.push_back(c);
          cs.push_back(sh);
          soff += c * tcs;
        }
        const Epilogue ep{nullptr, n, 1.0, 1.0, 0, 0};
        // complex128: W embedded once, one launch over every local device's columns (also the
        // faster loop with one device)
        if (emb && !bs.empty() &&
            gemm_cplx_embed_multi(dt, n - ss, tcs, wa, bs.data(), nc_d.data(), cs.data(), (int)bs.size(), ep,
                                  embed_buf.p, emb_bytes, st))
          break;
        for (size_t i = 0; i < bs.size(); ++i) {
          Epilogue e = ep;
          e.C = cs[i];
          if (!(emb && gemm_cplx_embed(dt, n - ss, nc_d[i], tcs, wa, bs[i], e, embed_buf.p, emb_bytes, nullptr, st, true)))
            gemm_shape_fixed(dt, n - ss, nc_d[i], tcs, wa, bs[i], e, nullptr, st);
        }
        break;
      }
      case S_PGEMM: {
        int64_t ldw = 0;
        const void* W = w_of(s, &ldw);
        // all local devices at once: one embedded GEMM over the concatenated
        // columns (their product blocks are contiguous in `blocks`), W_s
        // gathered once -- per-device GEMMs would be 1/nloc as wide
        bool grouped = false;
        if (emb && g.nloc > 1) {
          std::vector<Operand> bs;
          std::vector<int64_t> nc_d;
          for (int d = g.dev0; d < g.dev0 + g.nloc; ++d) {
            const int64_t c = cols_upto(g, d, s);
            if (!c) continue;
            bs.push_back(opB(colp(shards[d - g.dev0], g, ss, 0), n, OP_N));
            nc_d.push_back(c);
          }
          const int64_t nc = potri_chunk_cols(dt, n, ss, tcs, emb_bytes, nsm);
          grouped = !bs.empty() &&
                    gemm_cplx_embed_grouped(dt, tcs, n - ss, opA(W, ldw, OP_C), bs.data(), nc_d.data(), (int)bs.size(),
                                            Epilogue{blocks + block_off(s, g.dev0) * g.esz, tcs, 1.0, 0.0, 0, 0},
                                            embed_buf.p, emb_bytes, nc, st);
        }
        for (int d = g.dev0; !grouped && d < g.dev0 + g.nloc; ++d) {
          const int64_t c = cols_upto(g, d, s);
          if (c == 0) continue;
          const Operand wh = opA(W, ldw, OP_C);
          char* sh = colp(shards[d - g.dev0], g, ss, 0);
          char* blk = blocks + block_off(s, d) * g.esz;
          if (emb) {
            // real embedding in column chunks of whole waves of output tiles
            // (both operands are gathered into the scratch, which bounds the chunk)
            const int64_t nc = potri_chunk_cols(dt, n, ss, tcs, emb_bytes, nsm);
            bool done = nc >= 64;
            for (int64_t c0 = 0; done && c0 < c; c0 += nc) {
              const int64_t cn = std::min(nc, c - c0);
              done = gemm_cplx_embed(dt, tcs, cn, n - ss, wh, opB(sh + c0 * n * g.esz, n, OP_N),
                                     Epilogue{blk + c0 * tcs * g.esz, tcs, 1.0, 0.0, 0, 0}, embed_buf.p,
                                     emb_bytes, nullptr, st, true);
              if (!done && c0 > 0) {  // finish the remaining columns on the complex kernels
                gemm_shape_fixed(dt, tcs, c - c0, n - ss, wh, opB(sh + c0 * n * g.esz, n, OP_N),
                                 Epilogue{blk + c0 * tcs * g.esz, tcs, 1.0, 0.0, 0, 0}, nullptr, st);
                done = true;
                break;
              }
            }
            if (done) continue;
          }
          gemm_shape_fixed(dt, tcs, c, n - ss, wh, opB(sh, n, OP_N), Epilogue{blk, tcs, 1.0, 0.0, 0, 0}, nullptr, st);
        }
        // written back only after every GEMM: with one process W_s is read from tile s itself
        for (int d = g.dev0; d < g.dev0 + g.nloc; ++d) {
          const int64_t c = cols_upto(g, d, s);
          if (c) copy2d(dt, blocks + block_off(s, d) * g.esz, tcs, colp(shards[d - g.dev0], g, ss, 0), n, tcs, c,
                        false, nullptr, st);
        }
        break;
      }
      case S_PGATHER: {
        const int root = (int)op.root;
        if (world > 1) {
          const size_t off = (size_t)block_off(s, g.dev0) * g.esz;
          net->group_start();
          if (rank != root) {
            if (op.elems) net->send(blocks + off, (size_t)op.elems * g.esz, root, st);
          } else {
            for (int r = 0; r < world; ++r) {
              if (r == root) continue;
              const int d0 = r * g.nloc;
              const size_t bytes = (size_t)(block_off(s, d0 + g.nloc) - block_off(s, d0)) * g.esz;
              if (bytes)
                net->recv(blocks + (size_t)block_off(s, d0) * g.esz, bytes, r, st);
            }
          }
          net->group_end();
        }
        if (rank != root) break;
        // mirror: tile s rows [start_j, stop_j) = (block (s, j))^H for every j < s, any device
        char* Ts = colp(shard_of(s), g, 0, g.loc(s));
        for (int d = 0; d < g.D; ++d) {
          const int64_t c = cols_below(g, d, s);
          if (c) ct_scatter(dt, blocks + block_off(s, d) * g.esz, tcs, tcs, c, Ts, n, T, g.D, d, st);
        }
        mirror_diag(dt, Ts + ss * g.esz, n, tcs, st);
        break;
      }
      default:
        throw Error(CONFIG, "bad potri schedule op");
    }
  }
  sync_streams(user, crit);
}
}  // namespace bcmg
