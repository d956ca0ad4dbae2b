// Process-per-GPU world without NCCL: CUDA IPC over NVLink / peer memory.
//
// One process per GPU (torchrun), like the NCCL world, but every collective is a
// peer-memory operation: each process allocates its tensors from an EXPORTABLE
// stream-ordered pool (POSIX-fd handles, cudaDeviceSetMemPool), the pools are
// shared once at world creation over Unix-domain sockets (SCM_RIGHTS), and per
// collective a member ships 64-byte pointer-export records plus the index of an
// interprocess event in its ring; peers import the pointers, order their streams
// on the events and then load / store each other's HBM directly -- the same
// kernels (push remap, pairwise swap, fused distributed gate / QFT) and the same
// pull-copy exchange as the thread-per-GPU world. The sockets carry only these
// small records: the payload never leaves device memory.
//
// Ordering and lifetime rules (CUDA IPC pools): an imported pointer is released
// (cudaFreeAsync in the importer, stream-ordered after its last use) before the
// importer records the event of the collective's completion phase, so the owner,
// which frees only after waiting on those events, never frees under a live
// import. The event ring is reused only after two further collectives with the
// same peers, by which time every peer has enqueued its waits.
#include <fcntl.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/stat.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "runtime.h"

namespace qtnhb {

namespace {

constexpr int kRing = 256;

std::string sock_path(const std::string& dir, int rank) { return dir + "/qtnh_ipc_" + std::to_string(rank) + ".sock"; }

void io_all(int fd, void* buf, size_t n, bool send, long timeout_ms) {
  char* p = static_cast<char*>(buf);
  auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms > 0 ? timeout_ms : 1L << 40);
  while (n) {
    pollfd pf{fd, static_cast<short>(send ? POLLOUT : POLLIN), 0};
    long left = std::chrono::duration_cast<std::chrono::milliseconds>(deadline - std::chrono::steady_clock::now()).count();
    if (left <= 0) throw Status(QTNH_E_PROTOCOL, "collective timed out (possible deadlock)");
    int rc = ::poll(&pf, 1, static_cast<int>(std::min<long>(left, 1 << 30)));
    if (rc < 0 && errno == EINTR) continue;
    if (rc <= 0) continue;
    ssize_t k = send ? ::send(fd, p, n, MSG_NOSIGNAL) : ::recv(fd, p, n, 0);
    if (k < 0 && (errno == EINTR || errno == EAGAIN)) continue;
    if (k <= 0) throw Status(QTNH_E_ABORTED, "IPC peer connection lost");
    p += k;
    n -= static_cast<size_t>(k);
  }
}

void send_msg(int fd, const std::string& s, long t) {
  uint64_t n = s.size();
  io_all(fd, &n, 8, true, t);
  if (n) io_all(fd, const_cast<char*>(s.data()), n, true, t);
}

std::string recv_msg(int fd, long t) {
  uint64_t n = 0;
  io_all(fd, &n, 8, false, t);
  std::string s(n, '\0');
  if (n) io_all(fd, s.data(), n, false, t);
  return s;
}

void send_fd(int sock, int fd) {
  char dummy = 'F';
  iovec iov{&dummy, 1};
  char ctrl[CMSG_SPACE(sizeof(int))];
  std::memset(ctrl, 0, sizeof(ctrl));
  msghdr msg{};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  msg.msg_control = ctrl;
  msg.msg_controllen = sizeof(ctrl);
  cmsghdr* c = CMSG_FIRSTHDR(&msg);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int));
  std::memcpy(CMSG_DATA(c), &fd, sizeof(int));
  if (::sendmsg(sock, &msg, 0) != 1) throw Status(QTNH_E_RUNTIME, "IPC: sending the pool handle failed");
}

int recv_fd(int sock) {
  char dummy;
  iovec iov{&dummy, 1};
  char ctrl[CMSG_SPACE(sizeof(int))];
  msghdr msg{};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  msg.msg_control = ctrl;
  msg.msg_controllen = sizeof(ctrl);
  if (::recvmsg(sock, &msg, 0) != 1) throw Status(QTNH_E_RUNTIME, "IPC: receiving a pool handle failed");
  cmsghdr* c = CMSG_FIRSTHDR(&msg);
  if (!c || c->cmsg_type != SCM_RIGHTS) throw Status(QTNH_E_RUNTIME, "IPC: no pool handle in message");
  int fd;
  std::memcpy(&fd, CMSG_DATA(c), sizeof(int));
  return fd;
}

}  // namespace

void ipc_init(World& w, int rank, int size, int device, const std::string& dir) {
  auto st = std::make_unique<IpcState>();
  IpcState& S = *st;
  S.fd.assign(size, -1);
  // exportable pool, made the device's current pool for cudaMallocAsync
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypePosixFileDescriptor;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  QTNH_CUDA(cudaMemPoolCreate(&S.pool, &props));
  uint64_t keep = UINT64_MAX;
  QTNH_CUDA(cudaMemPoolSetAttribute(S.pool, cudaMemPoolAttrReleaseThreshold, &keep));
  QTNH_CUDA(cudaDeviceSetMemPool(device, S.pool));
  // full socket mesh: connect to lower ranks, accept higher ones
  ::mkdir(dir.c_str(), 0700);
  int lfd = ::socket(AF_UNIX, SOCK_STREAM, 0);
  sockaddr_un addr{};
  addr.sun_family = AF_UNIX;
  std::string me = sock_path(dir, rank);
  if (me.size() >= sizeof(addr.sun_path)) throw_invalid("IPC rendezvous path too long");
  std::strcpy(addr.sun_path, me.c_str());
  ::unlink(me.c_str());
  if (::bind(lfd, reinterpret_cast<sockaddr*>(&addr), sizeof(addr)) != 0 || ::listen(lfd, size) != 0)
    throw Status(QTNH_E_RUNTIME, "IPC: cannot listen on " + me);
  const long t = w.timeout_ms;
  auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(t > 0 ? t : 600000);
  for (int j = 0; j < rank; ++j) {
    std::string p = sock_path(dir, j);
    for (;;) {
      int fd = ::socket(AF_UNIX, SOCK_STREAM, 0);
      sockaddr_un a{};
      a.sun_family = AF_UNIX;
      std::strcpy(a.sun_path, p.c_str());
      if (::connect(fd, reinterpret_cast<sockaddr*>(&a), sizeof(a)) == 0) {
        int32_t r = rank;
        io_all(fd, &r, 4, true, t);
        S.fd[j] = fd;
        break;
      }
      ::close(fd);
      if (std::chrono::steady_clock::now() > deadline) throw Status(QTNH_E_PROTOCOL, "IPC: rank " + std::to_string(j) + " never listened");
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
  }
  for (int n_acc = 0; n_acc < size - 1 - rank; ++n_acc) {
    pollfd pf{lfd, POLLIN, 0};
    long left = std::chrono::duration_cast<std::chrono::milliseconds>(deadline - std::chrono::steady_clock::now()).count();
    if (left <= 0 || ::poll(&pf, 1, static_cast<int>(left)) <= 0) throw Status(QTNH_E_PROTOCOL, "IPC: peers never connected");
    int fd = ::accept(lfd, nullptr, nullptr);
    int32_t r = -1;
    io_all(fd, &r, 4, false, t);
    if (r <= rank || r >= size) throw Status(QTNH_E_PROTOCOL, "IPC: unexpected peer id");
    S.fd[r] = fd;
  }
  ::close(lfd);
  ::unlink(me.c_str());
  // pools: send mine to every peer, import theirs
  int my_pool_fd = -1;
  QTNH_CUDA(cudaMemPoolExportToShareableHandle(&my_pool_fd, S.pool, cudaMemHandleTypePosixFileDescriptor, 0));
  S.peer_pool.assign(size, nullptr);
  S.peer_dev.assign(size, device);
  for (int j = 0; j < size; ++j) {
    if (j == rank) continue;
    // lower rank sends first to keep the pairwise order deterministic
    auto exchange_pool = [&](bool send_first) {
      if (send_first) {
        send_fd(S.fd[j], my_pool_fd);
        int32_t d = device;
        io_all(S.fd[j], &d, 4, true, t);
      }
      int pfd = recv_fd(S.fd[j]);
      int32_t pd = 0;
      io_all(S.fd[j], &pd, 4, false, t);
      S.peer_dev[j] = pd;
      QTNH_CUDA(cudaMemPoolImportFromShareableHandle(&S.peer_pool[j], reinterpret_cast<void*>(static_cast<intptr_t>(pfd)),
                                                     cudaMemHandleTypePosixFileDescriptor, 0));
      ::close(pfd);
      if (pd != device) {
        cudaMemAccessDesc acc{};
        acc.location.type = cudaMemLocationTypeDevice;
        acc.location.id = device;
        acc.flags = cudaMemAccessFlagsProtReadWrite;
        QTNH_CUDA(cudaMemPoolSetAccess(S.peer_pool[j], &acc, 1));
      }
      if (!send_first) {
        send_fd(S.fd[j], my_pool_fd);
        int32_t d = device;
        io_all(S.fd[j], &d, 4, true, t);
      }
    };
    exchange_pool(rank < j);
  }
  ::close(my_pool_fd);
  // interprocess event rings
  S.my_ev.resize(kRing);
  std::string handles(kRing * sizeof(cudaIpcEventHandle_t), '\0');
  for (int k = 0; k < kRing; ++k) {
    QTNH_CUDA(cudaEventCreateWithFlags(&S.my_ev[k], cudaEventDisableTiming | cudaEventInterprocess));
    QTNH_CUDA(cudaIpcGetEventHandle(reinterpret_cast<cudaIpcEventHandle_t*>(&handles[k * sizeof(cudaIpcEventHandle_t)]),
                                    S.my_ev[k]));
  }
  S.peer_ev.assign(size, {});
  for (int j = 0; j < size; ++j)
    if (j != rank) send_msg(S.fd[j], handles, t);
  for (int j = 0; j < size; ++j) {
    if (j == rank) continue;
    std::string h = recv_msg(S.fd[j], t);
    if (h.size() != handles.size()) throw Status(QTNH_E_PROTOCOL, "IPC: bad event handle block");
    S.peer_ev[j].resize(kRing);
    for (int k = 0; k < kRing; ++k) {
      cudaIpcEventHandle_t eh;
      std::memcpy(&eh, &h[k * sizeof(cudaIpcEventHandle_t)], sizeof(eh));
      QTNH_CUDA(cudaIpcOpenEventHandle(&S.peer_ev[j][k], eh));
    }
  }
  w.ipc = std::move(st);
}

void ipc_destroy(World& w) {
  if (!w.ipc) return;
  IpcState& S = *w.ipc;
  for (auto& v : S.peer_ev)
    for (auto e : v) cudaEventDestroy(e);
  for (auto e : S.my_ev) cudaEventDestroy(e);
  for (int fd : S.fd)
    if (fd >= 0) ::close(fd);
  for (auto p : S.peer_pool)
    if (p) cudaMemPoolDestroy(p);
  // the device's current pool goes back to the default one before ours dies
  cudaMemPool_t def;
  if (w.proc_rank && cudaDeviceGetDefaultMemPool(&def, w.proc_rank->device) == cudaSuccess)
    cudaDeviceSetMemPool(w.proc_rank->device, def);
  cudaMemPoolDestroy(S.pool);
  w.ipc.reset();
}

std::vector<std::string> ipc_allgather(RankCtx& r, const std::vector<int>& members, const std::string& mine) {
  World& w = *r.world;
  IpcState& S = *w.ipc;
  std::vector<std::string> out(members.size());
  for (size_t i = 0; i < members.size(); ++i)
    if (members[i] != r.rank) send_msg(S.fd[members[i]], mine, w.timeout_ms);
  for (size_t i = 0; i < members.size(); ++i)
    out[i] = members[i] == r.rank ? mine : recv_msg(S.fd[members[i]], w.timeout_ms);
  return out;
}

int ipc_record(RankCtx& r) {
  IpcState& S = *r.world->ipc;
  int k = static_cast<int>(S.ev_next++ % kRing);
  QTNH_CUDA(cudaEventRecord(S.my_ev[k], r.stream));
  return k;
}

void ipc_wait(RankCtx& r, int peer, int k) {
  QTNH_CUDA(cudaStreamWaitEvent(r.stream, r.world->ipc->peer_ev[peer][k], 0));
}

// Export record: kind byte (0 none, 1 pool pointer, 2 legacy IPC handle) + data.
constexpr size_t kExportData = sizeof(cudaMemPoolPtrExportData) > sizeof(cudaIpcMemHandle_t)
                                   ? sizeof(cudaMemPoolPtrExportData)
                                   : sizeof(cudaIpcMemHandle_t);

std::string ipc_export(const void* p) {
  std::string s(1 + kExportData, '\0');
  if (!p) return s;
  cudaMemPoolPtrExportData d;
  if (cudaMemPoolExportPointer(&d, const_cast<void*>(p)) == cudaSuccess) {
    s[0] = 1;
    std::memcpy(&s[1], &d, sizeof(d));
    return s;
  }
  cudaGetLastError();  // not a pool block: a large cudaMalloc block (kIpcLegacyMinBytes)
  cudaIpcMemHandle_t h;
  QTNH_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(p)));
  s[0] = 2;
  std::memcpy(&s[1], &h, sizeof(h));
  return s;
}

std::pair<void*, int> ipc_import(RankCtx& r, int peer, const char* rec) {
  if (!rec[0]) return {nullptr, 0};
  void* p = nullptr;
  if (rec[0] == 1) {
    cudaMemPoolPtrExportData d;
    std::memcpy(&d, rec + 1, sizeof(d));
    QTNH_CUDA(cudaMemPoolImportPointer(&p, r.world->ipc->peer_pool[peer], &d));
    return {p, 1};
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, rec + 1, sizeof(h));
  QTNH_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  return {p, 2};
}

// Release imports after the stream work that used them: pool imports are freed
// stream-ordered; legacy mappings are closed after the stream drains.
void ipc_release(RankCtx& r, std::vector<std::pair<void*, int>>& v) {
  bool legacy = false;
  for (auto& pi : v) {
    if (pi.second == 1) QTNH_CUDA(cudaFreeAsync(pi.first, r.stream));
    legacy |= pi.second == 2;
  }
  if (legacy) {
    QTNH_CUDA(cudaStreamSynchronize(r.stream));
    for (auto& pi : v)
      if (pi.second == 2) QTNH_CUDA(cudaIpcCloseMemHandle(pi.first));
  }
  v.clear();
}

constexpr size_t kExportLen = 1 + kExportData;

// peer_pointers for the IPC world: the second call of a pair (the fence) first
// releases the imports of the first, stream-ordered after the peer kernels.
std::vector<void*> ipc_peer_pointers(RankCtx& r, const std::vector<int>& members, void* mine) {
  IpcState& S = *r.world->ipc;
  static const bool dbg = std::getenv("QTNH_IPC_DEBUG") != nullptr;
  if (dbg) std::fprintf(stderr, "[ipc %d] peer_pointers mine=%p releasing %zu\n", r.rank, mine, S.imports.size());
  ipc_release(r, S.imports);
  int k = ipc_record(r);
  std::string rec = ipc_export(mine);
  rec.append(reinterpret_cast<const char*>(&k), sizeof(k));
  auto all = ipc_allgather(r, members, rec);
  if (dbg) std::fprintf(stderr, "[ipc %d] gathered\n", r.rank);
  std::vector<void*> out(members.size());
  for (size_t i = 0; i < members.size(); ++i) {
    if (members[i] == r.rank) {
      out[i] = mine;
      continue;
    }
    const std::string& m = all[i];
    int pk;
    std::memcpy(&pk, m.data() + kExportLen, sizeof(pk));
    ipc_wait(r, members[i], pk);
    auto im = ipc_import(r, members[i], m.data());
    out[i] = im.first;
    if (dbg) std::fprintf(stderr, "[ipc %d] imported %p (kind %d) from %d\n", r.rank, out[i], im.second, members[i]);
    if (out[i]) S.imports.push_back(im);
  }
  return out;
}

// Two-phase exchange (as the local world): post send buffer + send list + packed
// event; receivers import and pull; post pulled events; senders order after them.
void ipc_exchange(RankCtx& r, const std::vector<int>& members, const void* send_buf, const std::vector<Xfer>& sends,
                  void* recv_buf, const std::vector<Xfer>& recvs) {
  int k = ipc_record(r);
  std::string rec = ipc_export(send_buf);
  rec.append(reinterpret_cast<const char*>(&k), sizeof(k));
  uint64_t ns = sends.size();
  rec.append(reinterpret_cast<const char*>(&ns), 8);
  for (const Xfer& x : sends) rec.append(reinterpret_cast<const char*>(&x), sizeof(Xfer));
  auto all = ipc_allgather(r, members, rec);
  std::map<int, size_t> idx;
  for (size_t i = 0; i < members.size(); ++i) idx[members[i]] = i;
  std::map<int, void*> imported;
  std::vector<std::pair<void*, int>> held;
  std::map<int, int> used;
  for (const Xfer& rv : recvs) {
    auto it = idx.find(rv.peer);
    if (it == idx.end()) throw_invalid("exchange peer outside the member set");
    const std::string& m = all[it->second];
    int pk;
    std::memcpy(&pk, m.data() + kExportLen, sizeof(pk));
    uint64_t n;
    std::memcpy(&n, m.data() + kExportLen + sizeof(int), 8);
    const Xfer* xs = reinterpret_cast<const Xfer*>(m.data() + kExportLen + sizeof(int) + 8);
    const Xfer* sx = nullptr;
    int& u = used[rv.peer];
    for (uint64_t j = 0, seen = 0; j < n; ++j)
      if (xs[j].peer == r.rank && seen++ == static_cast<uint64_t>(u)) {
        sx = &xs[j];
        break;
      }
    ++u;
    if (!sx || sx->count != rv.count)
      throw Status(QTNH_E_PROTOCOL, "exchange count mismatch for pair (" + std::to_string(rv.peer) + " -> " +
                                        std::to_string(r.rank) + ")");
    if (rv.count == 0) continue;
    const void* src;
    if (rv.peer == r.rank) {
      src = send_buf;
    } else {
      auto im = imported.find(rv.peer);
      if (im == imported.end()) {
        ipc_wait(r, rv.peer, pk);
        auto got = ipc_import(r, rv.peer, m.data());
        held.push_back(got);
        im = imported.emplace(rv.peer, got.first).first;
      }
      src = im->second;
    }
    QTNH_CUDA(cudaMemcpyAsync(static_cast<char*>(recv_buf) + rv.offset * 16,
                              static_cast<const char*>(src) + sx->offset * 16, rv.count * 16, cudaMemcpyDefault,
                              r.stream));
  }
  ipc_release(r, held);
  int k2 = ipc_record(r);
  std::string rec2(reinterpret_cast<const char*>(&k2), sizeof(k2));
  auto all2 = ipc_allgather(r, members, rec2);
  for (size_t i = 0; i < members.size(); ++i) {
    if (members[i] == r.rank) continue;
    bool reads_me = false;
    for (const Xfer& sx : sends)
      if (sx.peer == members[i] && sx.count > 0) reads_me = true;
    if (!reads_me) continue;
    int pk2;
    std::memcpy(&pk2, all2[i].data(), sizeof(pk2));
    ipc_wait(r, members[i], pk2);
  }
}

}  // namespace qtnhb
