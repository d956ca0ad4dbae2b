// Rank runtime: exchange over the in-process (local) backend or NCCL.
#include "runtime.h"

#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdlib>

#include "nccl_loader.h"

namespace qtnhb {

std::atomic<int64_t> g_kernel_launches{0};

void RankCtx::activate() const { QTNH_CUDA(cudaSetDevice(device)); }

void ensure_max_dynamic_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> size set
  int dev = 0;
  QTNH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{kernel, dev}];
  if (have >= bytes) return;
  QTNH_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

cudaStream_t RankCtx::side_stream(int i) {
  if (!side[i]) QTNH_CUDA(cudaStreamCreateWithFlags(&side[i], cudaStreamNonBlocking));
  return side[i];
}

RankCtx::~RankCtx() {
  for (auto& st : side)
    if (st) cudaStreamDestroy(st);
}

// Tensors come from the device's stream-ordered pool. The default release
// threshold (0) hands freed pages back to the driver at every synchronisation,
// so the next same-sized tensor pays a fresh mapping; a world keeps its pool
// warm for its lifetime and trims it when destroyed.
std::atomic<double> g_pool_reserve_gb{0.0};
void set_pool_reserve_gb(double gb) { g_pool_reserve_gb.store(gb); }

namespace {
std::mutex g_pool_mu;
std::map<int, int> g_pool_users;  // live worlds per device
}  // namespace

void keep_pool(int device) {
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (g_pool_users[device]++ > 0) return;
  }
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  uint64_t keep = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  // Optional up-front reservation (option "pool_reserve_gb" / QTNH_POOL_RESERVE_GB):
  // map the pool's memory once so tensors allocated later in a long sequence of
  // varying sizes (a network contraction) never wait on new physical mappings --
  // measured: C3 1.3-1.9 s with on-demand growth, 1.16 s reserved.
  {
    double gb = g_pool_reserve_gb.load();
    if (const char* e = std::getenv("QTNH_POOL_RESERVE_GB")) gb = std::max(gb, std::atof(e));
    if (gb > 0) {
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(device);
      void* p = nullptr;
      size_t bytes = static_cast<size_t>(gb * (1ull << 30));
      if (cudaMallocAsync(&p, bytes, 0) == cudaSuccess) {
        cudaFreeAsync(p, 0);
        cudaStreamSynchronize(0);
      } else {
        cudaGetLastError();
      }
      cudaSetDevice(prev);
    }
  }
}

void trim_pool(int device) {
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (--g_pool_users[device] > 0) return;
  }
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  // Keep a bounded warm reserve (QTNH_POOL_WARM_GB, default 8) mapped after the last
  // world on the device goes away: programs (and test suites) that create worlds
  // one after another then reuse mapped blocks instead of paying fresh physical
  // mappings for every allocation of the next world; everything above it is
  // returned to the driver.
  static const uint64_t warm = [] {
    const char* e = std::getenv("QTNH_POOL_WARM_GB");
    const double gb = e ? std::atof(e) : 8.0;
    return static_cast<uint64_t>(std::max(0.0, gb) * double(1ull << 30));
  }();
  uint64_t thr = warm;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  cudaMemPoolTrimTo(pool, warm);
}

size_t ipc_legacy_min_bytes() {
  static const size_t v = [] {
    const char* e = std::getenv("QTNH_IPC_LEGACY_MIN");
    return e ? static_cast<size_t>(std::atoll(e)) : (size_t(2) << 30);
  }();
  return v;
}

DevBuf::DevBuf(size_t b, const RankCtx& r) : bytes(b), device(r.device), stream(r.stream) {
  if (b == 0) b = 16;
  if (r.world && r.world->kind == World::kIpc && b >= ipc_legacy_min_bytes()) {
    QTNH_CUDA(cudaStreamSynchronize(stream));  // cudaMalloc is not stream-ordered
    QTNH_CUDA(cudaMalloc(&ptr, b));
    legacy_ipc = true;
    return;
  }
  QTNH_CUDA(cudaMallocAsync(&ptr, b, stream));
}

DevBuf::~DevBuf() {
  if (ptr) {
    cudaSetDevice(device);
    if (legacy_ipc) cudaFree(ptr);  // synchronises the device: no pending reader remains
    else cudaFreeAsync(ptr, stream);
  }
}

std::shared_ptr<TensorImpl> make_tensor(RankCtx& r, Shape shape, Dist dist, bool alloc) {
  shape.validate();
  dist.validate();
  auto t = std::make_shared<TensorImpl>();
  t->rank = &r;
  t->shape = std::move(shape);
  t->dist = dist;
  Dim need = dist.offset + dist.span(t->shape.dist_size());
  if (need > r.world->size) throw_resource("tensor span exceeds world size", need);
  t->in_span = dist.locate(r.rank, t->shape.dist_size(), &t->block, &t->cycle, &t->slot);
  if (t->in_span && alloc)
    t->buf = std::make_shared<DevBuf>(static_cast<size_t>(t->shape.local_size()) * 16, r);
  return t;
}

std::vector<int> span_ranks(const TensorImpl& t) {
  std::vector<int> out;
  for (Dim i = 0; i < t.span(); ++i) out.push_back(static_cast<int>(t.dist.offset + i));
  return out;
}

std::vector<int> union_members(const std::vector<std::pair<Dim, Dim>>& spans) {
  std::vector<int> out;
  for (auto [off, span] : spans)
    for (Dim r = off; r < off + span; ++r) out.push_back(static_cast<int>(r));
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

namespace {

// ---- local backend -----------------------------------------------------------
// Two-phase rendezvous per collective: (1) every member posts its send buffer,
// send list and a "packed" event; receivers then pull their chunks with
// stream-ordered device/peer copies on their own stream; (2) every member posts a
// "pulled" event and senders make their stream wait on the receivers' events, so
// a send buffer is never released before the copies that read it complete.
void local_exchange(RankCtx& r, const std::vector<int>& members, const void* send_buf,
                    const std::vector<Xfer>& sends, void* recv_buf, const std::vector<Xfer>& recvs) {
  World& w = *r.world;
  uint64_t seq = r.seq[members]++;
  auto key = std::make_pair(members, seq);
  int n = static_cast<int>(members.size());
  int me = static_cast<int>(std::find(members.begin(), members.end(), r.rank) - members.begin());
  if (me >= n) throw_invalid("rank is not a member of its own collective");
  cudaEvent_t packed, pulled;
  QTNH_CUDA(cudaEventCreateWithFlags(&packed, cudaEventDisableTiming));
  QTNH_CUDA(cudaEventCreateWithFlags(&pulled, cudaEventDisableTiming));
  QTNH_CUDA(cudaEventRecord(packed, r.stream));

  auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(w.timeout_ms);
  auto wait_for = [&](std::unique_lock<std::mutex>& lk, auto pred) {
    while (!pred()) {
      if (w.aborted) throw Status(QTNH_E_ABORTED, "world aborted");
      if (w.timeout_ms > 0) {
        if (w.cv.wait_until(lk, deadline) == std::cv_status::timeout && !pred() && !w.aborted)
          throw Status(QTNH_E_PROTOCOL, "collective timed out (possible deadlock)");
      } else {
        w.cv.wait(lk);
      }
    }
  };

  std::unique_lock<std::mutex> lk(w.mu);
  World::Slot& slot = w.slots[key];
  if (slot.posts.empty()) slot.posts.resize(n);
  World::Post& mine = slot.posts[me];
  mine.posted = true;
  mine.send_buf = send_buf;
  mine.sends = sends;
  mine.packed = packed;
  if (++slot.arrived == n) w.cv.notify_all();
  wait_for(lk, [&] { return slot.arrived == n || !slot.error.empty(); });
  if (!slot.error.empty()) throw Status(QTNH_E_PROTOCOL, slot.error);

  // Match my receives against the senders' lists, in order per peer.
  struct Pull {
    const Xfer* rv;
    const Xfer* sx;
    const World::Post* sp;
  };
  std::vector<Pull> pulls;
  std::map<int, int> used;
  for (const Xfer& rv : recvs) {
    int si = static_cast<int>(std::find(members.begin(), members.end(), rv.peer) - members.begin());
    if (si >= n) throw_invalid("exchange peer outside the member set");
    const World::Post& sp = slot.posts[si];
    int& u = used[rv.peer];
    const Xfer* sx = nullptr;
    for (int j = 0, seen = 0; j < static_cast<int>(sp.sends.size()); ++j)
      if (sp.sends[j].peer == r.rank && seen++ == u) {
        sx = &sp.sends[j];
        break;
      }
    ++u;
    if (!sx || sx->count != rv.count) {
      Dim got = 0;
      for (const Xfer& x : sp.sends)
        if (x.peer == r.rank) got += x.count;
      slot.error = "exchange count mismatch for pair (" + std::to_string(rv.peer) + " -> " +
                   std::to_string(r.rank) + "): got " + std::to_string(got) + ", expected " +
                   std::to_string(rv.count);
      w.cv.notify_all();
      throw Status(QTNH_E_PROTOCOL, slot.error);
    }
    pulls.push_back({&rv, sx, &sp});
  }
  lk.unlock();
  for (const Pull& p : pulls) {
    if (p.rv->count == 0) continue;
    if (p.rv->peer != r.rank) QTNH_CUDA(cudaStreamWaitEvent(r.stream, p.sp->packed, 0));
    QTNH_CUDA(cudaMemcpyAsync(static_cast<char*>(recv_buf) + p.rv->offset * 16,
                              static_cast<const char*>(p.sp->send_buf) + p.sx->offset * 16,
                              static_cast<size_t>(p.rv->count) * 16, cudaMemcpyDefault, r.stream));
  }
  QTNH_CUDA(cudaEventRecord(pulled, r.stream));

  lk.lock();
  mine.pulled = pulled;
  mine.done_posted = true;
  if (++slot.done == n) w.cv.notify_all();
  wait_for(lk, [&] { return slot.done == n || !slot.error.empty(); });
  if (!slot.error.empty()) throw Status(QTNH_E_PROTOCOL, slot.error);
  // My send buffer may be read by any receiver: order my stream after their pulls.
  for (int j = 0; j < n; ++j) {
    if (j == me) continue;
    bool reads_me = false;
    for (const Xfer& sx : sends)
      if (sx.peer == members[j] && sx.count > 0) reads_me = true;
    if (reads_me) QTNH_CUDA(cudaStreamWaitEvent(r.stream, slot.posts[j].pulled, 0));
  }
  if (++slot.left == n) {
    for (auto& p : slot.posts) {
      cudaEventDestroy(p.packed);
      cudaEventDestroy(p.pulled);
    }
    w.slots.erase(key);
  }
}

// ---- NCCL backend --------------------------------------------------------------
// Failure semantics of the simulated runtime carried over to NCCL:
//  * counts: every member pair swaps (elements I send you, elements I expect from
//    you) before the payload, so a mismatch is seen on BOTH sides of the pair and
//    raised as ProtocolError "(src -> dst)" (runtime.hpp:464-471) instead of a hang;
//  * timeout: completion is awaited by polling the stream and
//    ncclCommGetAsyncError; past QTNH_COLLECTIVE_TIMEOUT_MS the communicator is
//    aborted (ncclCommAbort) and ProtocolError "collective timed out" raised
//    (runtime.hpp:335-345);
//  * abort: qtnh_world_abort aborts the communicator; later calls raise
//    AbortedError (runtime.hpp:276-298).
void nccl_abort_comm(World& w) {
  std::lock_guard<std::mutex> lk(w.mu);
  if (w.nccl_comm && !w.aborted) nccl().CommAbort(static_cast<ncclComm_t>(w.nccl_comm));
  if (w.nccl_comm) w.nccl_comm = nullptr;
  w.aborted = true;
  w.cv.notify_all();
}

void nccl_wait_impl(RankCtx& r) {
  World& w = *r.world;
  const Nccl& N = nccl();
  cudaEvent_t ev;
  QTNH_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  QTNH_CUDA(cudaEventRecord(ev, r.stream));
  auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(w.timeout_ms > 0 ? w.timeout_ms : 1L << 40);
  for (int spin = 0;; ++spin) {
    cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) {
      cudaEventDestroy(ev);
      QTNH_CUDA(q);
    }
    if (w.aborted) {
      cudaEventDestroy(ev);
      throw Status(QTNH_E_ABORTED, "world aborted");
    }
    ncclResult_t ae = ncclSuccess;
    if (w.nccl_comm) N.CommGetAsyncError(static_cast<ncclComm_t>(w.nccl_comm), &ae);
    if (ae != ncclSuccess && ae != ncclInProgress) {
      cudaEventDestroy(ev);
      nccl_abort_comm(w);
      throw Status(QTNH_E_RUNTIME, std::string("NCCL asynchronous error: ") + N.GetErrorString(ae));
    }
    if (std::chrono::steady_clock::now() > deadline) {
      cudaEventDestroy(ev);
      nccl_abort_comm(w);
      throw Status(QTNH_E_PROTOCOL, "collective timed out (possible deadlock)");
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  cudaEventDestroy(ev);
}

ncclComm_t nccl_comm_of(RankCtx& r) {
  if (r.world->aborted || !r.world->nccl_comm) throw Status(QTNH_E_ABORTED, "world aborted");
  return static_cast<ncclComm_t>(r.world->nccl_comm);
}

void nccl_check_counts(RankCtx& r, const std::vector<int>& members, const std::vector<Xfer>& sends,
                       const std::vector<Xfer>& recvs) {
  const Nccl& N = nccl();
  ncclComm_t comm = nccl_comm_of(r);
  const int n = static_cast<int>(members.size());
  std::vector<int64_t> out(2 * n, 0), in(2 * n, 0);
  for (int i = 0; i < n; ++i) {
    for (const Xfer& x : sends)
      if (x.peer == members[i]) out[2 * i] += x.count;
    for (const Xfer& x : recvs)
      if (x.peer == members[i]) out[2 * i + 1] += x.count;
  }
  DevBuf ob(16 * n, r), ib(16 * n, r);
  QTNH_CUDA(cudaMemcpyAsync(ob.ptr, out.data(), 16 * n, cudaMemcpyHostToDevice, r.stream));
  nccl_check(N.GroupStart(), "group start");
  for (int i = 0; i < n; ++i) {
    if (members[i] == r.rank) continue;
    nccl_check(N.Send(static_cast<char*>(ob.ptr) + 16 * i, 16, ncclUint8, members[i], comm, r.stream), "send");
    nccl_check(N.Recv(static_cast<char*>(ib.ptr) + 16 * i, 16, ncclUint8, members[i], comm, r.stream), "recv");
  }
  nccl_check(N.GroupEnd(), "group end");
  QTNH_CUDA(cudaMemcpyAsync(in.data(), ib.ptr, 16 * n, cudaMemcpyDeviceToHost, r.stream));
  nccl_wait_impl(r);
  for (int i = 0; i < n; ++i) {
    if (members[i] == r.rank) continue;
    // in[2i] = what member i sends me; in[2i+1] = what member i expects from me
    if (in[2 * i] != out[2 * i + 1])
      throw Status(QTNH_E_PROTOCOL, "exchange count mismatch for pair (" + std::to_string(members[i]) + " -> " +
                                        std::to_string(r.rank) + "): got " + std::to_string(in[2 * i]) +
                                        ", expected " + std::to_string(out[2 * i + 1]));
    if (in[2 * i + 1] != out[2 * i])
      throw Status(QTNH_E_PROTOCOL, "exchange count mismatch for pair (" + std::to_string(r.rank) + " -> " +
                                        std::to_string(members[i]) + "): got " + std::to_string(out[2 * i]) +
                                        ", expected " + std::to_string(in[2 * i + 1]));
  }
}

void nccl_exchange(RankCtx& r, const std::vector<int>& members, const void* send_buf, const std::vector<Xfer>& sends,
                   void* recv_buf, const std::vector<Xfer>& recvs, bool checked, bool wait) {
  const Nccl& N = nccl();
  ncclComm_t comm = nccl_comm_of(r);
  if (checked && members.size() > 1) nccl_check_counts(r, members, sends, recvs);
  // Self chunks: direct device copies, matched in order.
  std::vector<const Xfer*> self_s, self_r;
  for (const Xfer& s : sends)
    if (s.peer == r.rank) self_s.push_back(&s);
  for (const Xfer& v : recvs)
    if (v.peer == r.rank) self_r.push_back(&v);
  if (self_s.size() != self_r.size())
    throw Status(QTNH_E_PROTOCOL, "exchange count mismatch for pair (" + std::to_string(r.rank) +
                                      " -> " + std::to_string(r.rank) + ")");
  for (size_t i = 0; i < self_s.size(); ++i) {
    if (self_s[i]->count != self_r[i]->count)
      throw Status(QTNH_E_PROTOCOL, "exchange count mismatch for pair (" + std::to_string(r.rank) +
                                        " -> " + std::to_string(r.rank) + ")");
    if (self_s[i]->count)
      QTNH_CUDA(cudaMemcpyAsync(static_cast<char*>(recv_buf) + self_r[i]->offset * 16,
                                static_cast<const char*>(send_buf) + self_s[i]->offset * 16,
                                self_s[i]->count * 16, cudaMemcpyDeviceToDevice, r.stream));
  }
  nccl_check(N.GroupStart(), "group start");
  for (const Xfer& s : sends)
    if (s.peer != r.rank && s.count)
      nccl_check(N.Send(static_cast<const char*>(send_buf) + s.offset * 16, s.count * 16, ncclUint8,
                        s.peer, comm, r.stream),
                 "send");
  for (const Xfer& v : recvs)
    if (v.peer != r.rank && v.count)
      nccl_check(N.Recv(static_cast<char*>(recv_buf) + v.offset * 16, v.count * 16, ncclUint8,
                        v.peer, comm, r.stream),
                 "recv");
  nccl_check(N.GroupEnd(), "group end");
  if (wait) nccl_wait_impl(r);
}

}  // namespace

namespace {
std::atomic<bool> g_peer_direct{[] {
  const char* e = std::getenv("QTNH_PEER_DIRECT");
  return !(e && e[0] == '0');
}()};
}  // namespace

void set_peer_direct(bool on) { g_peer_direct.store(on); }

bool peer_direct(const RankCtx& r) {
  return (r.world->kind == World::kLocal || r.world->kind == World::kIpc) && r.world->peer_ok && g_peer_direct.load();
}

std::vector<void*> peer_pointers(RankCtx& r, const std::vector<int>& members, void* mine) {
  if (r.world->kind == World::kIpc) return ipc_peer_pointers(r, members, mine);
  World& w = *r.world;
  int n = static_cast<int>(members.size());
  int me = static_cast<int>(std::find(members.begin(), members.end(), r.rank) - members.begin());
  if (me >= n) throw_invalid("rank is not a member of its own collective");
  if (n == 1) return {mine};
  uint64_t seq = r.seq[members]++;
  auto key = std::make_pair(members, seq);
  cudaEvent_t ready;
  QTNH_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  QTNH_CUDA(cudaEventRecord(ready, r.stream));
  auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(w.timeout_ms);
  std::unique_lock<std::mutex> lk(w.mu);
  World::Slot& slot = w.slots[key];
  if (slot.posts.empty()) slot.posts.resize(n);
  slot.posts[me].posted = true;
  slot.posts[me].send_buf = mine;
  slot.posts[me].packed = ready;
  if (++slot.arrived == n) w.cv.notify_all();
  while (slot.arrived != n) {
    if (w.aborted) throw Status(QTNH_E_ABORTED, "world aborted");
    if (w.timeout_ms > 0) {
      if (w.cv.wait_until(lk, deadline) == std::cv_status::timeout && slot.arrived != n && !w.aborted)
        throw Status(QTNH_E_PROTOCOL, "collective timed out (possible deadlock)");
    } else {
      w.cv.wait(lk);
    }
  }
  std::vector<void*> out(n);
  for (int j = 0; j < n; ++j) {
    out[j] = const_cast<void*>(slot.posts[j].send_buf);
    if (j != me) QTNH_CUDA(cudaStreamWaitEvent(r.stream, slot.posts[j].packed, 0));
  }
  if (++slot.left == n) {
    for (auto& p : slot.posts) cudaEventDestroy(p.packed);
    w.slots.erase(key);
  }
  return out;
}

void exchange(RankCtx& r, const std::vector<int>& members, const void* send_buf,
              const std::vector<Xfer>& sends, void* recv_buf, const std::vector<Xfer>& recvs, bool checked,
              bool wait) {
  QTNH_RANGE("qtnh::exchange");
  if (r.world->kind == World::kLocal) {
    local_exchange(r, members, send_buf, sends, recv_buf, recvs);
  } else if (r.world->kind == World::kIpc) {
    ipc_exchange(r, members, send_buf, sends, recv_buf, recvs);
  } else {
    nccl_exchange(r, members, send_buf, sends, recv_buf, recvs, checked, wait);
  }
}

void nccl_wait(RankCtx& r) {
  if (r.world->kind == World::kNccl) nccl_wait_impl(r);
}

void nccl_abort(World& w) { nccl_abort_comm(w); }

void barrier(RankCtx& r, const std::vector<int>& members) {
  if (members.size() <= 1) return;
  if (r.world->kind == World::kIpc) {
    QTNH_CUDA(cudaStreamSynchronize(r.stream));
    ipc_allgather(r, members, std::string());
    return;
  }
  if (r.world->kind == World::kLocal) {
    local_exchange(r, members, nullptr, {}, nullptr, {});
    QTNH_CUDA(cudaStreamSynchronize(r.stream));
    return;
  }
  // NCCL: a one-element all-to-all among members, then drain the stream.
  DevBuf sb(16 * members.size(), r), rb(16 * members.size(), r);
  std::vector<Xfer> s, v;
  for (size_t i = 0; i < members.size(); ++i) {
    s.push_back({members[i], static_cast<Dim>(i), 1});
    v.push_back({members[i], static_cast<Dim>(i), 1});
  }
  QTNH_CUDA(cudaMemsetAsync(sb.ptr, 0, sb.bytes, r.stream));
  nccl_exchange(r, members, sb.ptr, s, rb.ptr, v, false, true);
}

}  // namespace qtnhb
