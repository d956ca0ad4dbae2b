// Rank runtime of libqtnh_b200: worlds, ranks, device tensors and the exchange
// primitive every redistribution goes through.
//
// Reference: the simulated SPMD runtime (runtime.hpp) -- one host thread per
// rank, collectives as rendezvous over a global mutex, member-only groups
// (runtime.hpp:191-223), abort propagation (:276-298) and a collective timeout
// (QTNH_COLLECTIVE_TIMEOUT_MS, :116, :255-257). Here a rank owns a GPU, a CUDA
// stream and (process-per-GPU) an NCCL communicator; the host rendezvous only
// orders stream work -- data never leaves HBM/NVLink.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"

namespace qtnhb {

struct World;

struct RankCtx {
  World* world = nullptr;
  int rank = 0;
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;  // current launch stream
  std::map<std::vector<int>, uint64_t> seq;  // per member-set collective sequence
  cudaStream_t side[2] = {nullptr, nullptr}; // pipeline streams (pack / unpack), created on first use
  void activate() const;                     // cudaSetDevice(device)
  cudaStream_t side_stream(int i);
  ~RankCtx();
};

// One transfer of `count` complex elements at element `offset` of a buffer,
// to (send) or from (recv) world rank `peer`.
struct Xfer {
  int peer;
  Dim offset;
  Dim count;
};

// Process-per-GPU world over CUDA IPC (ipc.cpp): sockets to every peer, this
// process's exportable pool and the peers' imported pools, interprocess event rings.
struct IpcState {
  std::vector<int> fd;
  cudaMemPool_t pool = nullptr;
  std::vector<cudaMemPool_t> peer_pool;
  std::vector<int> peer_dev;
  std::vector<cudaEvent_t> my_ev;
  std::vector<std::vector<cudaEvent_t>> peer_ev;
  uint64_t ev_next = 0;
  std::vector<std::pair<void*, int>> imports;  // (pointer, kind 1 pool / 2 legacy) of the last peer_pointers call
};

struct World {
  enum Kind { kLocal, kNccl, kIpc } kind = kLocal;
  int size = 1;
  std::vector<int> devices;  // local: device of each rank
  bool peer_ok = false;      // local: every rank can load/store every other rank's HBM
  // process-per-GPU backends (NCCL or IPC): this process's rank
  int my_rank = 0;
  void* nccl_comm = nullptr;
  std::unique_ptr<RankCtx> proc_rank;
  std::unique_ptr<IpcState> ipc;

  // local backend rendezvous
  std::mutex mu;
  std::condition_variable cv;
  bool aborted = false;
  long timeout_ms = 120000;
  struct Post {
    bool posted = false, done_posted = false;
    const void* send_buf = nullptr;
    std::vector<Xfer> sends;
    cudaEvent_t packed = nullptr;
    cudaEvent_t pulled = nullptr;
  };
  struct Slot {
    std::vector<Post> posts;
    int arrived = 0, done = 0, left = 0;
    std::string error;
  };
  std::map<std::pair<std::vector<int>, uint64_t>, Slot> slots;
};

// Collective over the sorted world ranks `members` (must include r.rank).
// Moves the listed chunks from send_buf to the peers' recv_bufs. Self transfers
// are allowed. Stream-ordered on every member's stream; returns when all copies
// are enqueued. Count mismatches raise ProtocolError naming "(src -> dst)"
// (runtime.hpp:464-471).
// NCCL world: `checked` = exchange the pairwise counts first (a mismatch raises
// ProtocolError on both sides of the pair); `wait` = block until the transfer
// completes, with the collective timeout (ncclCommAbort + ProtocolError) --
// a pipelined caller verifies once and waits once (nccl_wait) at the end.
void exchange(RankCtx& r, const std::vector<int>& members, const void* send_buf,
              const std::vector<Xfer>& sends, void* recv_buf, const std::vector<Xfer>& recvs, bool checked = true,
              bool wait = true);
// NCCL world: wait for the rank stream with the collective timeout and async-error
// polling; no-op for the other backends.
void nccl_wait(RankCtx& r);
// Abort the NCCL communicator of a process-per-GPU world (qtnh_world_abort).
void nccl_abort(World& w);
void barrier(RankCtx& r, const std::vector<int>& members);

// Peer-memory collectives (local world with peer_ok): kernels read and write
// the other members' device buffers directly over NVLink instead of staging
// through pack/exchange/unpack.
bool peer_direct(const RankCtx& r);
void set_peer_direct(bool on);  // option "peer_direct" / QTNH_PEER_DIRECT=0
// All-gather of one device pointer per member (in member order). Stream-ordered:
// on return my stream waits for the work every member enqueued before its call,
// so a second call after the peer kernels acts as the completion fence. The
// returned peer pointers are valid until this rank's next peer_pointers call.
std::vector<void*> peer_pointers(RankCtx& r, const std::vector<int>& members, void* mine);

// IPC backend (ipc.cpp)
void ipc_init(World& w, int rank, int size, int device, const std::string& dir);
void ipc_destroy(World& w);
std::vector<std::string> ipc_allgather(RankCtx& r, const std::vector<int>& members, const std::string& mine);
std::vector<void*> ipc_peer_pointers(RankCtx& r, const std::vector<int>& members, void* mine);
void ipc_exchange(RankCtx& r, const std::vector<int>& members, const void* send_buf, const std::vector<Xfer>& sends,
                  void* recv_buf, const std::vector<Xfer>& recvs);

// ---- device tensors -----------------------------------------------------------
void keep_pool(int device);  // stream-ordered pool keeps freed blocks (world lifetime)
void set_pool_reserve_gb(double gb);  // reserve (map) this much at the next world creation
void trim_pool(int device);  // return unused pool memory to the driver
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool legacy_ipc = false;  // IPC world, large block: cudaMalloc (legacy IPC handle), not the pool
  DevBuf(size_t b, const RankCtx& r);
  ~DevBuf();
};
// Blocks at least this large in an IPC world are shared through legacy CUDA IPC
// handles: importing multi-GiB stream-ordered-pool allocations crashed the driver.
// Default 2 GiB; QTNH_IPC_LEGACY_MIN (bytes) overrides it (tests force 0).
size_t ipc_legacy_min_bytes();

struct TensorImpl {
  RankCtx* rank = nullptr;
  Shape shape;
  Dist dist;
  bool in_span = false;
  Dim block = 0, cycle = 0, slot = 0;
  std::shared_ptr<DevBuf> buf;
  // tensor.hpp:28 storage variant: 0 dense, 1 symmetric (dense storage, half-split
  // layout), 2 diagonal (buf = this block's slice of the diagonal, only on blocks
  // whose input and output distributed coordinates agree), 3 identity / 4 swap
  // (no storage; pair_in / pair_out as constructed). Everything outside
  // variants.cpp and io.cpp sees dense tensors only (capi.cpp's impl_of
  // materialises the compact ones on demand).
  int variant = 0;
  std::vector<int> pair_in, pair_out;
  bool canonical() const { return in_span && cycle == 0 && slot == 0; }
  Dim span() const { return dist.span(shape.dist_size()); }
  void* data() const { return buf ? buf->ptr : nullptr; }
};

// Tensor::make (tensor.hpp:458-477): validates, raises ResourceError when the
// span exceeds the world, locates this rank; allocates the local block when
// `alloc` (uninitialised).
std::shared_ptr<TensorImpl> make_tensor(RankCtx& r, Shape shape, Dist dist, bool alloc);
std::vector<int> span_ranks(const TensorImpl& t);

// ---- tensor variants (variants.cpp; tensor.hpp:95-164, :209-337, ops.hpp:54-161) ----
enum { kDense = 0, kSymmetric = 1, kDiagonal = 2, kIdentity = 3, kSwap = 4 };
void check_symmetric_shape(const Shape& s);                       // tensor.hpp:479-489
Dim diag_local_count(const Shape& s);                             // elements of one block's diagonal slice
bool diag_block_on_diagonal(const Shape& s, Dim block, Dim* in_block = nullptr);
Dim stored_count(const TensorImpl& t);                            // elements buf holds (local_data().size())
std::shared_ptr<TensorImpl> make_diagonal(RankCtx& r, Shape s, Dist d, const double* diag_global_host, Dim count);
std::shared_ptr<TensorImpl> make_paired(RankCtx& r, Shape s, Dist d, const std::vector<int>& in_pos,
                                        const std::vector<int>& out_pos, bool crossed);
std::shared_ptr<TensorImpl> variant_to_dense(const std::shared_ptr<TensorImpl>& t);       // tensor.hpp:282-296
std::shared_ptr<TensorImpl> variant_rebcast(const std::shared_ptr<TensorImpl>& t, Dist d); // ops.hpp:54-112
std::shared_ptr<TensorImpl> variant_scale(const std::shared_ptr<TensorImpl>& t, double re, double im,
                                          bool conj);                                      // ops.hpp:147-161
// Tensor::local_element (tensor.hpp:209-247): value at global coordinates from this
// rank's storage; InvalidArgument when a stored variant's block lives elsewhere.
void variant_local_element(const TensorImpl& t, const std::vector<Dim>& coords, double* out2);
std::vector<int> union_members(const std::vector<std::pair<Dim, Dim>>& spans);

}  // namespace qtnhb

struct qtnh_world_s {
  std::unique_ptr<qtnhb::World> w;
};
struct qtnh_rank_s {
  qtnhb::World* world;
  std::unique_ptr<qtnhb::RankCtx> owned;  // local backend
  qtnhb::RankCtx* ctx;
};
struct qtnh_tensor_s {
  std::shared_ptr<qtnhb::TensorImpl> impl;
  std::shared_ptr<qtnhb::TensorImpl> dense;  // dense view of a non-dense variant, built on first use
  std::atomic<int> refs{1};
};
