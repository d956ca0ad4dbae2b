// extern "C" boundary of libqtnh_b200.so (declared in include/qtnh_b200.h).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <chrono>

#include "nccl_loader.h"
#include "ops.h"
#include "strided_copy.h"

using namespace qtnhb;

namespace {

thread_local std::string t_err;
thread_local int64_t t_info = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    return QTNH_OK;
  } catch (const Status& s) {
    t_err = s.what();
    t_info = s.info;
    return s.code;
  } catch (const std::bad_alloc&) {
    t_err = "host allocation failed";
    t_info = 0;
    return QTNH_E_RUNTIME;
  } catch (const std::exception& e) {
    t_err = e.what();
    t_info = 0;
    return QTNH_E_RUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw_invalid(std::string("null ") + what);
}

RankCtx& ctx_of(qtnh_rank_t r) {
  need(r, "rank");
  r->ctx->activate();
  return *r->ctx;
}

// The tensor as constructed (any storage variant).
TP& raw_of(qtnh_tensor_t t) {
  need(t, "tensor");
  t->impl->rank->activate();
  return t->impl;
}

// The tensor as the structural ops, contraction and factorisation see it: dense.
// The reference's ops call to_dense() on the other variants (ops.hpp:128, :143,
// :178, ...; remap.hpp:75-95 visits their non-zeros); here the dense block is
// materialised on the device on first use and kept with the handle.
TP& impl_of(qtnh_tensor_t t) {
  TP& p = raw_of(t);
  if (p->variant == kDense) return p;
  if (!t->dense) t->dense = variant_to_dense(p);
  return t->dense;
}

// Before an in-place update: the handle becomes its dense value.
TP& dense_in_place(qtnh_tensor_t t) {
  TP& p = raw_of(t);
  if (p->variant != kDense) {
    TP d = t->dense ? t->dense : variant_to_dense(p);
    t->dense.reset();
    if (p->variant == kSymmetric) d = std::make_shared<TensorImpl>(*d);  // own tag, shared block
    d->variant = kDense;
    p = d;
  }
  return p;
}

qtnh_tensor_t wrap(TP p) {
  auto* h = new qtnh_tensor_s;
  h->impl = std::move(p);
  return h;
}

Shape shape_from(int n, const int64_t* dims, int split) {
  if (n < 0) throw_invalid("negative tensor rank");
  if (n > 0) need(dims, "dims");
  return Shape(std::vector<Dim>(dims, dims + n), split);
}

// Copy-on-write before an in-place update: other handles must not see it.
void make_exclusive(TP& p) {
  if (p->in_span && (p.use_count() > 1 || (p->buf && p->buf.use_count() > 1))) {
    TP c = make_tensor(*p->rank, p->shape, p->dist, true);
    QTNH_CUDA(cudaMemcpyAsync(c->data(), p->data(), p->shape.local_size() * 16, cudaMemcpyDeviceToDevice,
                              p->rank->stream));
    p = c;
  } else if (!p->in_span && p.use_count() > 1) {
    p = make_tensor(*p->rank, p->shape, p->dist, false);
  }
}

long env_timeout() {
  const char* t = std::getenv("QTNH_COLLECTIVE_TIMEOUT_MS");
  return t ? std::strtol(t, nullptr, 10) : 120000;
}

}  // namespace

extern "C" {

int qtnh_last_error(char* buf, size_t len) {
  if (buf && len) {
    std::strncpy(buf, t_err.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return static_cast<int>(t_err.size());
}
int64_t qtnh_last_error_info(void) { return t_info; }
const char* qtnh_version(void) { return "qtnh_b200 0.1.0 (sm_100a)"; }
int64_t qtnh_kernel_launch_count(void) { return g_kernel_launches.load(); }
int64_t qtnh_svd_split_count(void) { return svd_split_count(); }

// ---- worlds -----------------------------------------------------------------
int qtnh_world_create_local(int n, const int* devices, qtnh_world_t* out) {
  return guard([&] {
    need(out, "out");
    if (n < 1) throw_invalid("world size must be >= 1, got " + std::to_string(n));
    auto w = std::make_unique<World>();
    w->kind = World::kLocal;
    w->size = n;
    w->timeout_ms = env_timeout();
    for (int i = 0; i < n; ++i) w->devices.push_back(devices ? devices[i] : 0);
    {  // one keep per distinct device (qtnh_world_destroy trims each distinct device once)
      std::vector<int> uniq = w->devices;
      std::sort(uniq.begin(), uniq.end());
      uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
      for (int d : uniq) keep_pool(d);
    }
    // Peer access between distinct devices (NVLink) for the exchange copies and
    // the peer-memory kernels (remap push, in-place swaps).
    w->peer_ok = true;
    for (int a : w->devices)
      for (int b : w->devices)
        if (a != b) {
          int can = 0;
          cudaDeviceCanAccessPeer(&can, a, b);
          if (!can) w->peer_ok = false;
          if (can) {
            cudaSetDevice(a);
            cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            // tensors come from b's stream-ordered pool: map it for a as well
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, b) == cudaSuccess) {
              cudaMemAccessDesc acc{};
              acc.location.type = cudaMemLocationTypeDevice;
              acc.location.id = a;
              acc.flags = cudaMemAccessFlagsProtReadWrite;
              if (cudaMemPoolSetAccess(pool, &acc, 1) != cudaSuccess) {
                cudaGetLastError();
                w->peer_ok = false;
              }
            }
          }
        }
    auto* h = new qtnh_world_s;
    h->w = std::move(w);
    *out = h;
  });
}

int qtnh_nccl_unique_id(void* uid128) {
  return guard([&] {
    need(uid128, "uid");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "get unique id");
    std::memcpy(uid128, &id, sizeof(id));
  });
}

int qtnh_world_create_nccl(int rank, int size, int device, const void* uid128, qtnh_world_t* out) {
  return guard([&] {
    need(out, "out");
    need(uid128, "uid");
    if (size < 1 || rank < 0 || rank >= size) throw_invalid("invalid rank/size");
    auto w = std::make_unique<World>();
    w->kind = World::kNccl;
    w->size = size;
    w->my_rank = rank;
    w->timeout_ms = env_timeout();
    QTNH_CUDA(cudaSetDevice(device));
    keep_pool(device);
    ncclUniqueId id;
    std::memcpy(&id, uid128, sizeof(id));
    ncclComm_t comm = nullptr;
    const Nccl& N = nccl();
    if (N.CommInitRankConfig) {
      // Non-blocking initialisation polled against the collective timeout: a
      // missing peer aborts the communicator and raises ProtocolError instead of
      // blocking forever (runtime.hpp:335-345). Blocking mode is restored after
      // init so every later NCCL call completes its enqueue before returning.
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      cfg.blocking = 0;
      ncclResult_t rc = N.CommInitRankConfig(&comm, size, id, rank, &cfg);
      if (rc != ncclSuccess && rc != ncclInProgress) nccl_check(rc, "comm init");
      auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(w->timeout_ms > 0 ? w->timeout_ms : 1L << 40);
      ncclResult_t st = ncclInProgress;
      while (true) {
        N.CommGetAsyncError(comm, &st);
        if (st != ncclInProgress) break;
        if (std::chrono::steady_clock::now() > deadline) {
          N.CommAbort(comm);
          throw Status(QTNH_E_PROTOCOL, "NCCL communicator initialisation timed out (rank " + std::to_string(rank) +
                                            " of " + std::to_string(size) + "; missing peers?)");
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
      if (st != ncclSuccess) {
        N.CommAbort(comm);
        nccl_check(st, "comm init");
      }
    } else {
      nccl_check(N.CommInitRank(&comm, size, id, rank), "comm init");
    }
    w->nccl_comm = comm;
    auto rc = std::make_unique<RankCtx>();
    rc->world = w.get();
    rc->rank = rank;
    rc->device = device;
    QTNH_CUDA(cudaStreamCreateWithFlags(&rc->own_stream, cudaStreamNonBlocking));
    rc->stream = rc->own_stream;
    w->proc_rank = std::move(rc);
    auto* h = new qtnh_world_s;
    h->w = std::move(w);
    *out = h;
  });
}

int qtnh_world_create_ipc(int rank, int size, int device, const char* dir, qtnh_world_t* out) {
  return guard([&] {
    need(out, "out");
    need(dir, "dir");
    if (size < 1 || rank < 0 || rank >= size) throw_invalid("invalid rank/size");
    auto w = std::make_unique<World>();
    w->kind = World::kIpc;
    w->size = size;
    w->my_rank = rank;
    w->timeout_ms = env_timeout();
    w->peer_ok = true;
    QTNH_CUDA(cudaSetDevice(device));
    auto rc = std::make_unique<RankCtx>();
    rc->world = w.get();
    rc->rank = rank;
    rc->device = device;
    QTNH_CUDA(cudaStreamCreateWithFlags(&rc->own_stream, cudaStreamNonBlocking));
    rc->stream = rc->own_stream;
    w->proc_rank = std::move(rc);
    ipc_init(*w, rank, size, device, dir);
    auto* h = new qtnh_world_s;
    h->w = std::move(w);
    *out = h;
  });
}

int qtnh_world_destroy(qtnh_world_t w) {
  return guard([&] {
    if (!w) return;
    if (w->w->kind == World::kIpc) {
      cudaSetDevice(w->w->proc_rank->device);
      cudaStreamSynchronize(w->w->proc_rank->stream);
      ipc_destroy(*w->w);
      cudaStreamDestroy(w->w->proc_rank->own_stream);
      delete w;
      return;
    }
    if (w->w->kind == World::kNccl) {
      cudaSetDevice(w->w->proc_rank->device);
      cudaStreamSynchronize(w->w->proc_rank->stream);
      if (w->w->nccl_comm) nccl().CommDestroy(static_cast<ncclComm_t>(w->w->nccl_comm));
      cudaStreamDestroy(w->w->proc_rank->own_stream);
    }
    std::vector<int> devs = w->w->kind == World::kNccl ? std::vector<int>{w->w->proc_rank->device} : w->w->devices;
    delete w;
    std::sort(devs.begin(), devs.end());
    devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
    for (int d : devs) trim_pool(d);
  });
}

int qtnh_world_size(qtnh_world_t w) { return w ? w->w->size : 0; }

int qtnh_world_abort(qtnh_world_t w) {
  return guard([&] {
    need(w, "world");
    if (w->w->kind == World::kNccl) {  // ncclCommAbort: peers blocked in NCCL fail instead of hanging
      nccl_abort(*w->w);
      return;
    }
    std::lock_guard<std::mutex> lk(w->w->mu);
    w->w->aborted = true;
    w->w->cv.notify_all();
  });
}

int qtnh_rank_bind(qtnh_world_t w, int rank, qtnh_rank_t* out) {
  return guard([&] {
    need(w, "world");
    need(out, "out");
    World& W = *w->w;
    auto* h = new qtnh_rank_s;
    h->world = &W;
    if (W.kind == World::kNccl || W.kind == World::kIpc) {
      if (rank != W.my_rank) {
        delete h;
        throw_invalid("process-per-GPU world: this process is rank " + std::to_string(W.my_rank));
      }
      h->ctx = W.proc_rank.get();
    } else {
      if (rank < 0 || rank >= W.size) {
        delete h;
        throw_invalid("rank out of range");
      }
      h->owned = std::make_unique<RankCtx>();
      h->ctx = h->owned.get();
      h->ctx->world = &W;
      h->ctx->rank = rank;
      h->ctx->device = W.devices[rank];
      QTNH_CUDA(cudaSetDevice(h->ctx->device));
      QTNH_CUDA(cudaStreamCreateWithFlags(&h->ctx->own_stream, cudaStreamNonBlocking));
      h->ctx->stream = h->ctx->own_stream;
    }
    // Keep freed blocks in the stream-ordered pool (no OS round trips per op).
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, h->ctx->device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = h;
  });
}

int qtnh_rank_release(qtnh_rank_t r) {
  return guard([&] {
    if (!r) return;
    if (r->owned) {
      cudaSetDevice(r->ctx->device);
      cudaStreamSynchronize(r->ctx->own_stream);
      cudaStreamDestroy(r->ctx->own_stream);
    }
    delete r;
  });
}

int qtnh_rank_id(qtnh_rank_t r) { return r ? r->ctx->rank : -1; }

int qtnh_rank_set_stream(qtnh_rank_t r, void* stream) {
  return guard([&] {
    RankCtx& c = ctx_of(r);
    c.stream = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream
  });
}

int qtnh_rank_reset_stream(qtnh_rank_t r) {
  return guard([&] {
    RankCtx& c = ctx_of(r);
    c.stream = c.own_stream;
  });
}

void* qtnh_rank_stream(qtnh_rank_t r) { return r ? static_cast<void*>(r->ctx->stream) : nullptr; }

struct qtnh_graph_s {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

int qtnh_rank_capture_begin(qtnh_rank_t r) {
  return guard([&] {
    RankCtx& c = ctx_of(r);
    if (c.stream == nullptr) throw_invalid("stream capture needs a non-default rank stream");
    QTNH_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  });
}

int qtnh_rank_capture_end(qtnh_rank_t r, qtnh_graph_t* out) {
  return guard([&] {
    need(out, "out");
    RankCtx& c = ctx_of(r);
    auto* g = new qtnh_graph_s;
    cudaError_t e = cudaStreamEndCapture(c.stream, &g->graph);
    if (e != cudaSuccess) {
      delete g;
      QTNH_CUDA(e);
    }
    e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(g->graph);
      delete g;
      QTNH_CUDA(e);
    }
    *out = g;
  });
}

int qtnh_graph_launch(qtnh_rank_t r, qtnh_graph_t g) {
  return guard([&] {
    need(g, "graph");
    QTNH_CUDA(cudaGraphLaunch(g->exec, ctx_of(r).stream));
    g_kernel_launches.fetch_add(1);
  });
}

int qtnh_graph_destroy(qtnh_graph_t g) {
  return guard([&] {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
  });
}

int qtnh_rank_synchronize(qtnh_rank_t r) {
  return guard([&] { QTNH_CUDA(cudaStreamSynchronize(ctx_of(r).stream)); });
}

int qtnh_barrier(qtnh_rank_t r) {
  return guard([&] {
    RankCtx& c = ctx_of(r);
    std::vector<int> all(c.world->size);
    std::iota(all.begin(), all.end(), 0);
    barrier(c, all);
  });
}

// ---- tensors --------------------------------------------------------------------
int qtnh_tensor_dense(qtnh_rank_t r, int n, const int64_t* dims, int split, const int64_t* dist,
                      const double* local, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    RankCtx& c = ctx_of(r);
    TP t = make_tensor(c, shape_from(n, dims, split), dist_from(dist), true);
    if (t->in_span) {
      Dim nl = t->shape.local_size();
      if (local) QTNH_CUDA(cudaMemcpyAsync(t->data(), local, nl * 16, cudaMemcpyHostToDevice, c.stream));
      else fill_zero(t->data(), nl, c.stream);
      if (local) QTNH_CUDA(cudaStreamSynchronize(c.stream));  // host buffer may be pageable/temporary
    }
    *out = wrap(t);
  });
}

int qtnh_tensor_from_global(qtnh_rank_t r, int n, const int64_t* dims, int split, const int64_t* dist,
                            const double* global, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    need(global, "global");
    RankCtx& c = ctx_of(r);
    TP t = make_tensor(c, shape_from(n, dims, split), dist_from(dist), true);
    if (t->in_span) {
      Dim nl = t->shape.local_size();
      QTNH_CUDA(cudaMemcpyAsync(t->data(), global + 2 * t->block * nl, nl * 16, cudaMemcpyHostToDevice,
                                c.stream));
      QTNH_CUDA(cudaStreamSynchronize(c.stream));
    }
    *out = wrap(t);
  });
}

int qtnh_tensor_from_device(qtnh_rank_t r, int n, const int64_t* dims, int split, const int64_t* dist,
                            const void* dev, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    RankCtx& c = ctx_of(r);
    TP t = make_tensor(c, shape_from(n, dims, split), dist_from(dist), true);
    if (t->in_span) {
      need(dev, "device pointer");
      QTNH_CUDA(cudaMemcpyAsync(t->data(), dev, t->shape.local_size() * 16, cudaMemcpyDeviceToDevice, c.stream));
    }
    *out = wrap(t);
  });
}

int qtnh_tensor_retain(qtnh_tensor_t t) {
  return guard([&] {
    need(t, "tensor");
    t->refs.fetch_add(1);
  });
}

int qtnh_tensor_free(qtnh_tensor_t t) {
  return guard([&] {
    if (!t) return;
    if (t->refs.fetch_sub(1) == 1) {
      t->impl->rank->activate();
      delete t;
    }
  });
}

int qtnh_tensor_rank(qtnh_tensor_t t) { return t ? t->impl->shape.n_idx() : -1; }
int qtnh_tensor_dims(qtnh_tensor_t t, int64_t* dims) {
  return guard([&] {
    need(t, "tensor");
    if (t->impl->shape.n_idx() > 0) need(dims, "dims");  // a rank-0 scalar has none
    for (int i = 0; i < t->impl->shape.n_idx(); ++i) dims[i] = t->impl->shape.dims[i];
  });
}
int qtnh_tensor_split(qtnh_tensor_t t) { return t ? t->impl->shape.split : -1; }
int qtnh_tensor_dist(qtnh_tensor_t t, int64_t* d) {
  return guard([&] {
    need(t, "tensor");
    need(d, "dist");
    d[0] = t->impl->dist.stretch;
    d[1] = t->impl->dist.cycles;
    d[2] = t->impl->dist.offset;
  });
}
int64_t qtnh_tensor_local_size(qtnh_tensor_t t) { return t ? t->impl->shape.local_size() : -1; }
int64_t qtnh_tensor_span(qtnh_tensor_t t) { return t ? t->impl->span() : -1; }
int qtnh_tensor_in_span(qtnh_tensor_t t) { return t ? t->impl->in_span : 0; }
int64_t qtnh_tensor_my_block(qtnh_tensor_t t) { return t ? t->impl->block : -1; }
int qtnh_tensor_is_canonical(qtnh_tensor_t t) { return t ? t->impl->canonical() : 0; }
void* qtnh_tensor_device_ptr(qtnh_tensor_t t) { return t ? t->impl->data() : nullptr; }

int qtnh_tensor_download_local(qtnh_tensor_t t, double* host) {
  return guard([&] {
    TP& p = raw_of(t);
    const Dim n = stored_count(*p);
    if (n == 0) return;
    need(host, "host");
    QTNH_CUDA(cudaMemcpyAsync(host, p->data(), n * 16, cudaMemcpyDeviceToHost, p->rank->stream));
    QTNH_CUDA(cudaStreamSynchronize(p->rank->stream));
  });
}

int qtnh_tensor_download_local_async(qtnh_tensor_t t, double* host) {
  return guard([&] {
    TP& p = raw_of(t);
    const Dim n = stored_count(*p);
    if (n == 0) return;
    need(host, "host");
    QTNH_CUDA(cudaMemcpyAsync(host, p->data(), n * 16, cudaMemcpyDeviceToHost, p->rank->stream));
  });
}

int qtnh_tensor_upload_local(qtnh_tensor_t t, const double* host) {
  return guard([&] {
    TP& p = raw_of(t);
    const Dim n = stored_count(*p);
    if (n == 0) return;
    need(host, "host");
    t->dense.reset();
    QTNH_CUDA(cudaMemcpyAsync(p->data(), host, n * 16, cudaMemcpyHostToDevice, p->rank->stream));
  });
}

int qtnh_tensor_to_global(qtnh_tensor_t t, double* host) {
  return guard([&] {
    TP& p = impl_of(t);
    if (p->in_span) need(host, "host");
    op_to_global(*p, host);
  });
}

int qtnh_tensor_paired(qtnh_rank_t r, int n, const int64_t* dims, int split, const int64_t* dist, int n_pairs,
                       const int* in_pos, const int* out_pos, int crossed, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    RankCtx& x = ctx_of(r);
    Shape s = shape_from(n, dims, split);
    if (n_pairs) {
      need(in_pos, "in_pos");
      need(out_pos, "out_pos");
    }
    *out = wrap(make_paired(x, s, dist ? dist_from(dist) : Dist{}, std::vector<int>(in_pos, in_pos + n_pairs),
                            std::vector<int>(out_pos, out_pos + n_pairs), crossed != 0));
  });
}

int qtnh_tensor_diagonal(qtnh_rank_t r, int n, const int64_t* dims, int split, const int64_t* dist,
                         const double* diag_global, int64_t count, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    RankCtx& x = ctx_of(r);
    Shape s = shape_from(n, dims, split);
    check_symmetric_shape(s);
    if (count < 0 && !diag_global) {  // zero diagonal of the right length (Tensor::adopt)
      count = diag_local_count(s);
      for (int i = 0; i < s.split / 2; ++i) count *= s.dims[i];
    }
    *out = wrap(make_diagonal(x, s, dist ? dist_from(dist) : Dist{}, diag_global, count));
  });
}

int qtnh_tensor_symmetric(qtnh_rank_t r, int n, const int64_t* dims, int split, const int64_t* dist,
                          const double* data, int64_t count, int is_global, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    RankCtx& x = ctx_of(r);
    Shape s = shape_from(n, dims, split);
    check_symmetric_shape(s);  // tensor.hpp:99, :107: the layout is validated first
    if (data && is_global && count != s.total_size()) throw_invalid("global element count mismatch");
    TP t = make_tensor(x, s, dist_from(dist), true);
    t->variant = kSymmetric;
    if (t->in_span) {
      const Dim nl = t->shape.local_size();
      if (!data) {  // zero block (Tensor::adopt)
        fill_zero(t->data(), nl, x.stream);
      } else if (!is_global && count != nl) {
        throw_invalid("dense local data has " + std::to_string(count) + " elements, expected " + std::to_string(nl));
      } else if (nl > 0) {
        QTNH_CUDA(cudaMemcpyAsync(t->data(), data + (is_global ? 2 * t->block * nl : 0), nl * 16,
                                  cudaMemcpyHostToDevice, x.stream));
        QTNH_CUDA(cudaStreamSynchronize(x.stream));
      }
    }
    *out = wrap(t);
  });
}

int qtnh_tensor_variant(qtnh_tensor_t t) { return t ? t->impl->variant : -1; }
int64_t qtnh_tensor_stored_size(qtnh_tensor_t t) { return t ? stored_count(*t->impl) : -1; }

int qtnh_tensor_pairs(qtnh_tensor_t t, int* in_pos, int* out_pos) {
  return guard([&] {
    TP& p = raw_of(t);
    for (size_t i = 0; i < p->pair_in.size(); ++i) {
      if (in_pos) in_pos[i] = p->pair_in[i];
      if (out_pos) out_pos[i] = p->pair_out[i];
    }
  });
}

int qtnh_tensor_to_dense(qtnh_tensor_t t, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    TP d = impl_of(t);
    if (d->variant != kDense) {  // never the case; keep the tag honest
      d = std::make_shared<TensorImpl>(*d);
      d->variant = kDense;
    }
    *out = wrap(d);
  });
}

int qtnh_tensor_local_element(qtnh_tensor_t t, const int64_t* coords, double* out2) {
  return guard([&] {
    need(out2, "out");
    TP& p = raw_of(t);
    const int n = p->shape.n_idx();
    if (n) need(coords, "coords");
    variant_local_element(*p, std::vector<Dim>(coords, coords + n), out2);
  });
}

int qtnh_squeeze(qtnh_tensor_t t, int pos, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    const Shape& rs = raw_of(t)->shape;
    if (pos < 0 || pos >= rs.n_idx() || rs.dims[pos] != 1) throw_invalid("squeeze needs a size-1 index");
    TP& p = impl_of(t);
    std::vector<Dim> dims = p->shape.dims;
    dims.erase(dims.begin() + pos);
    auto q = std::make_shared<TensorImpl>(*p);  // flat layouts ignore unit dimensions (ops.hpp:234-244)
    q->shape = Shape(dims, p->shape.split - (pos < p->shape.split ? 1 : 0));
    *out = wrap(q);
  });
}

int qtnh_unsqueeze(qtnh_tensor_t t, int pos, int as_dist, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    const Shape& rs = raw_of(t)->shape;
    if (pos < 0 || pos > rs.n_idx()) throw_invalid("unsqueeze position out of range");
    if (as_dist && pos > rs.split) throw_invalid("distributed index must precede the split");
    if (!as_dist && pos < rs.split) throw_invalid("local index must follow the split");
    TP& p = impl_of(t);
    std::vector<Dim> dims = p->shape.dims;
    dims.insert(dims.begin() + pos, 1);
    auto q = std::make_shared<TensorImpl>(*p);
    q->shape = Shape(dims, p->shape.split + (as_dist ? 1 : 0));
    *out = wrap(q);
  });
}

int qtnh_tensor_save(qtnh_tensor_t t, const char* path) {
  return guard([&] {
    need(path, "path");
    op_save(*raw_of(t), path);
  });
}

int qtnh_tensor_load(qtnh_rank_t r, const char* path, qtnh_tensor_t* out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    *out = wrap(op_load(ctx_of(r), path));
  });
}

int qtnh_plan_order(int n_tensors, const int* label_offsets, const int* labels, int n_labels,
                    const double* label_log2, uint64_t seed, int trials, int* order_out) {
  return qtnh_plan_order_capped(n_tensors, label_offsets, labels, n_labels, label_log2, seed, trials, 0.0, order_out);
}

int qtnh_plan_order_capped(int n_tensors, const int* label_offsets, const int* labels, int n_labels,
                           const double* label_log2, uint64_t seed, int trials, double log2_cap, int* order_out) {
  return guard([&] {
    if (n_tensors < 1) throw_invalid("empty network");
    need(label_offsets, "label_offsets");
    need(order_out, "order_out");
    std::vector<std::vector<int>> lab(n_tensors);
    for (int t = 0; t < n_tensors; ++t)
      for (int j = label_offsets[t]; j < label_offsets[t + 1]; ++j) {
        if (labels[j] < 0 || labels[j] >= n_labels) throw_invalid("label id out of range");
        lab[t].push_back(labels[j]);
      }
    std::vector<double> lg(label_log2, label_log2 + n_labels);
    auto order = plan_order(lab, lg, seed, trials, log2_cap);
    for (size_t i = 0; i < order.size(); ++i) {
      order_out[2 * i] = order[i].first;
      order_out[2 * i + 1] = order[i].second;
    }
  });
}

// ---- ops --------------------------------------------------------------------------
int qtnh_permute(qtnh_tensor_t t, const int* perm, int new_split, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    TP& p = impl_of(t);
    int n = p->shape.n_idx();
    if (n) need(perm, "perm");
    *out = wrap(op_permute(p, std::vector<int>(perm, perm + n), new_split));
  });
}

int qtnh_rebcast(qtnh_tensor_t t, const int64_t* nd, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    *out = wrap(variant_rebcast(raw_of(t), dist_from(nd)));
  });
}

int qtnh_remap(qtnh_tensor_t t, const int* axis_map, int n_dst, const int64_t* dst_dims, int dst_split,
               const int64_t* dst_dist, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    TP& p = impl_of(t);
    const Shape& ss = p->shape;
    const int n = ss.n_idx();
    if (n) need(axis_map, "axis_map");
    if (n_dst != n) throw_invalid("axis map is not a bijection");
    Shape ds = shape_from(n_dst, dst_dims, dst_split);
    std::vector<int> am(axis_map, axis_map + n);
    std::vector<char> seen(n, 0);
    bool embed = false;
    for (int i = 0; i < n; ++i) {
      int q = am[i];
      if (q < 0 || q >= n || seen[q]) throw_invalid("axis map is not a bijection");
      seen[q] = 1;
      if (ds.dims[q] < ss.dims[i]) throw_invalid("destination dimension smaller than source");
      if (ds.dims[q] > ss.dims[i]) {
        if (q < dst_split) throw_invalid("zero-embedding into a larger distributed index is not supported");
        embed = true;
      }
    }
    Dist dd = dst_dist ? dist_from(dst_dist) : p->dist;
    if (!embed) {
      *out = wrap(remap(p, ds, dd, am));
      return;
    }
    // remap onto the source dimensions, then zero-embed the local ones
    std::vector<Dim> eq(n);
    for (int i = 0; i < n; ++i) eq[am[i]] = ss.dims[i];
    TP mid = remap(p, Shape(eq, dst_split), dd, am);
    *out = wrap(op_pad_local(mid, ds.local_dims()));
  });
}

int qtnh_scatter_index(qtnh_tensor_t t, int pos, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    *out = wrap(op_scatter_index(impl_of(t), pos));
  });
}

int qtnh_gather_index(qtnh_tensor_t t, int pos, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    *out = wrap(op_gather_index(impl_of(t), pos));
  });
}

int qtnh_slice_local_dims(qtnh_tensor_t t, const int64_t* nl, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    TP& p = impl_of(t);
    int k = p->shape.n_local();
    if (k) need(nl, "new_local_dims");
    *out = wrap(op_slice_local(p, std::vector<Dim>(nl, nl + k)));
  });
}

int qtnh_pad_local_dims(qtnh_tensor_t t, const int64_t* nl, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    TP& p = impl_of(t);
    int k = p->shape.n_local();
    if (k) need(nl, "new_local_dims");
    *out = wrap(op_pad_local(p, std::vector<Dim>(nl, nl + k)));
  });
}

int qtnh_conj(qtnh_tensor_t t, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    *out = wrap(variant_scale(raw_of(t), 1.0, 0.0, true));
  });
}

int qtnh_scale(qtnh_tensor_t t, double re, double im, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    *out = wrap(variant_scale(raw_of(t), re, im, false));
  });
}

int qtnh_scale_index(qtnh_tensor_t t, int pos, const double* factors, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    need(factors, "factors");
    TP& p = impl_of(t);
    if (pos < 0 || pos >= p->shape.n_idx()) throw_invalid("scale_index position out of range");
    std::vector<double> f(factors, factors + p->shape.dims[pos]);
    *out = wrap(op_scale_index(p, pos, f));
  });
}

int qtnh_tensor_clone(qtnh_tensor_t t, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    *out = wrap(raw_of(t));
  });
}

int qtnh_tensor_reshape(qtnh_tensor_t t, int n, const int64_t* dims, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    TP& p = impl_of(t);
    Shape ns = shape_from(n, dims, 0);
    if (p->shape.split != 0) throw_invalid("reshape needs a tensor without distributed indices");
    if (ns.total_size() != p->shape.total_size()) throw_invalid("reshape must keep the element count");
    auto q = std::make_shared<TensorImpl>(*p);  // same value (row-major block), new index tuple
    q->shape = ns;
    *out = wrap(q);
  });
}

int qtnh_contract_chain(int n_inputs, const qtnh_tensor_t* inputs, int n_steps, const int* step_ab,
                        const int* step_npairs, const int* a_pos, const int* b_pos, qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    if (n_inputs < 1 || n_steps < 0) throw_invalid("invalid chain sizes");
    need(inputs, "inputs");
    if (n_steps) {
      need(step_ab, "step_ab");
      need(step_npairs, "step_npairs");
    }
    std::vector<TP> live(n_inputs + n_steps);
    for (int i = 0; i < n_inputs; ++i) live[i] = impl_of(inputs[i]);
    size_t off = 0;
    int last = n_inputs - 1;
    for (int s = 0; s < n_steps; ++s) {
      const int a = step_ab[2 * s], b = step_ab[2 * s + 1], k = step_npairs[s];
      if (a < 0 || b < 0 || a >= n_inputs + s || b >= n_inputs + s || a == b || !live[a] || !live[b])
        throw_invalid("chain step " + std::to_string(s) + " references a consumed or unknown tensor");
      if (k && (!a_pos || !b_pos)) throw_invalid("missing contracted positions");
      live[n_inputs + s] = op_contract(live[a], live[b], std::vector<int>(a_pos + off, a_pos + off + k),
                                       std::vector<int>(b_pos + off, b_pos + off + k));
      off += static_cast<size_t>(k);
      live[a].reset();  // intermediates die as soon as they are consumed
      live[b].reset();
      last = n_inputs + s;
    }
    *out = wrap(live[last]);
  });
}

int qtnh_contract(qtnh_tensor_t a, qtnh_tensor_t b, int n_pairs, const int* a_pos, const int* b_pos,
                  qtnh_tensor_t* out) {
  return guard([&] {
    need(out, "out");
    if (n_pairs < 0) throw_invalid("negative pair count");
    if (n_pairs) {
      need(a_pos, "a_pos");
      need(b_pos, "b_pos");
    }
    TP& pa = impl_of(a);
    TP& pb = impl_of(b);
    *out = wrap(op_contract(pa, pb, std::vector<int>(a_pos, a_pos + n_pairs),
                            std::vector<int>(b_pos, b_pos + n_pairs)));
  });
}

int qtnh_gate_apply(qtnh_tensor_t state, int n_targets, const int* targets, const double* gate, int diagonal) {
  return guard([&] {
    TP& p = dense_in_place(state);
    if (n_targets < 1) throw_invalid("gate needs at least one target");
    need(targets, "targets");
    need(gate, "gate");
    // Copy-on-write: other handles (or views) must not observe the update.
    if (p->in_span && (p.use_count() > 1 || (p->buf && p->buf.use_count() > 1))) {
      TP c = make_tensor(*p->rank, p->shape, p->dist, true);
      QTNH_CUDA(cudaMemcpyAsync(c->data(), p->data(), p->shape.local_size() * 16, cudaMemcpyDeviceToDevice,
                                p->rank->stream));
      p = c;
    } else if (!p->in_span && p.use_count() > 1) {
      p = make_tensor(*p->rank, p->shape, p->dist, false);
    }
    op_gate_apply(p, std::vector<int>(targets, targets + n_targets), gate, diagonal != 0);
  });
}

int qtnh_gate_apply_tensor(qtnh_tensor_t state, int n_targets, const int* targets, qtnh_tensor_t gate) {
  return guard([&] {
    TP& g = raw_of(gate);
    TP& st = raw_of(state);
    if (n_targets < 1) throw_invalid("gate needs at least one target");
    need(targets, "targets");
    const Shape& gs = g->shape;
    if (gs.split != 0 || g->dist.stretch * g->dist.cycles != st->rank->world->size || g->dist.offset != 0)
      throw_invalid("gate tensors are replicated on every rank (split 0, DistParams{1, P, 0})");
    if (gs.n_idx() != 2 * n_targets) throw_invalid("gate tensor needs one output and one input index per target");
    Dim D = 1;
    for (int i = 0; i < n_targets; ++i) {
      if (targets[i] < 0 || targets[i] >= st->shape.n_idx()) throw_invalid("gate target out of range");
      const Dim d = st->shape.dims[targets[i]];
      if (gs.dims[i] != d || gs.dims[n_targets + i] != d) throw_invalid("gate dimensions do not match the targets");
      D *= d;
    }
    if (g->variant == kIdentity || g->variant == kSwap) {
      // element = 1 iff the paired coordinates agree: with (outputs; inputs) pairs the
      // identity leaves the state alone and the swap exchanges the two targets.
      bool plain = n_targets == static_cast<int>(g->pair_in.size());
      for (int i = 0; plain && i < n_targets; ++i) {
        const int a = std::min(g->pair_in[i], g->pair_out[i]), b = std::max(g->pair_in[i], g->pair_out[i]);
        plain = a < n_targets && b == a + n_targets;
      }
      if (plain && g->variant == kIdentity) return;
      if (plain && n_targets == 2) {
        TP& p = dense_in_place(state);
        make_exclusive(p);
        op_swap_indices(p, targets[0], targets[1]);
        return;
      }
    }
    const bool diag = g->variant == kDiagonal;
    const Dim n = diag ? D : D * D;
    std::vector<double> host(static_cast<size_t>(2 * n));
    TP& src = diag ? g : impl_of(gate);
    QTNH_CUDA(cudaMemcpyAsync(host.data(), src->data(), n * 16, cudaMemcpyDeviceToHost, src->rank->stream));
    QTNH_CUDA(cudaStreamSynchronize(src->rank->stream));
    TP& p = dense_in_place(state);
    make_exclusive(p);
    op_gate_apply(p, std::vector<int>(targets, targets + n_targets), host.data(), diag);
  });
}

int qtnh_tensor_make_mutable(qtnh_tensor_t t) {
  return guard([&] {
    TP& p = raw_of(t);  // the stored elements of any variant (tensor.hpp:178)
    t->dense.reset();
    if (p->variant == kDiagonal) {
      if (p.use_count() > 1 || (p->buf && p->buf.use_count() > 1)) p = variant_scale(p, 1.0, 0.0, false);
    } else if (p->variant == kIdentity || p->variant == kSwap) {
      if (p.use_count() > 1) p = std::make_shared<TensorImpl>(*p);
    } else {
      const int var = p->variant;
      make_exclusive(p);
      p->variant = var;
    }
    QTNH_CUDA(cudaStreamSynchronize(p->rank->stream));
  });
}

// Host-data all-to-all among `members` in group order (the Group collectives of
// runtime.hpp:122-163): receive sizes travel first, so a count mismatch against
// expected_counts is seen -- and raised as ProtocolError naming the first
// "(src -> dst)" pair in member order -- by EVERY member (runtime.hpp:464-471
// poisons the shared slot); then the payload moves through device staging with
// the world's exchange (NVLink / NCCL / IPC).
int qtnh_group_all_to_all_v_host(qtnh_rank_t r, int n_members, const int* members, size_t elem_size,
                                 const void* const* send_lists, const int64_t* send_counts,
                                 const int64_t* expected_counts, void** recv_data, int64_t* recv_counts) {
  return guard([&] {
    RankCtx& x = ctx_of(r);
    need(recv_data, "recv_data");
    need(recv_counts, "recv_counts");
    if (n_members < 1) throw_invalid("group members must be non-empty");
    if (elem_size < 1) throw_invalid("element size must be positive");
    need(members, "members");
    std::vector<int> mem(members, members + n_members), sorted = mem;
    std::sort(sorted.begin(), sorted.end());
    if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end()) throw_invalid("duplicate group member");
    for (int m : mem)
      if (m < 0 || m >= x.world->size) throw_invalid("group member " + std::to_string(m) + " out of range");
    const int me = static_cast<int>(std::find(mem.begin(), mem.end(), x.rank) - mem.begin());
    if (me >= n_members)
      throw_invalid("rank " + std::to_string(x.rank) + " cannot open a group it is not a member of");
    const Dim n = n_members;
    // phase 1: counts (one 16-byte element per member pair)
    std::vector<int64_t> cnt_out(2 * n, 0), cnt_in(2 * n, 0);
    for (Dim i = 0; i < n; ++i) cnt_out[2 * i] = send_counts ? send_counts[i] : 0;
    DevBuf cs(16 * n, x), cr(16 * n, x);
    std::vector<Xfer> s1, r1;
    for (Dim i = 0; i < n; ++i) {
      s1.push_back({mem[i], i, 1});
      r1.push_back({mem[i], i, 1});
    }
    QTNH_CUDA(cudaMemcpyAsync(cs.ptr, cnt_out.data(), 16 * n, cudaMemcpyHostToDevice, x.stream));
    exchange(x, sorted, cs.ptr, s1, cr.ptr, r1);
    QTNH_CUDA(cudaMemcpyAsync(cnt_in.data(), cr.ptr, 16 * n, cudaMemcpyDeviceToHost, x.stream));
    QTNH_CUDA(cudaStreamSynchronize(x.stream));
    // phase 2: every member learns the first mismatch (src member, got, expected)
    int64_t bad[4] = {-1, 0, 0, 0};
    if (expected_counts)
      for (Dim i = 0; i < n; ++i)
        if (cnt_in[2 * i] != expected_counts[i]) {
          bad[0] = i;
          bad[1] = cnt_in[2 * i];
          bad[2] = expected_counts[i];
          break;
        }
    std::vector<int64_t> flags_out(4 * n), flags_in(4 * n);
    for (Dim i = 0; i < n; ++i) std::copy(bad, bad + 4, flags_out.begin() + 4 * i);
    DevBuf fs(32 * n, x), fr(32 * n, x);
    std::vector<Xfer> s2, r2;
    for (Dim i = 0; i < n; ++i) {
      s2.push_back({mem[i], 2 * i, 2});
      r2.push_back({mem[i], 2 * i, 2});
    }
    QTNH_CUDA(cudaMemcpyAsync(fs.ptr, flags_out.data(), 32 * n, cudaMemcpyHostToDevice, x.stream));
    exchange(x, sorted, fs.ptr, s2, fr.ptr, r2);
    QTNH_CUDA(cudaMemcpyAsync(flags_in.data(), fr.ptr, 32 * n, cudaMemcpyDeviceToHost, x.stream));
    QTNH_CUDA(cudaStreamSynchronize(x.stream));
    for (Dim j = 0; j < n; ++j)
      if (flags_in[4 * j] >= 0)
        throw Status(QTNH_E_PROTOCOL, "all_to_all_v count mismatch for pair (" +
                                          std::to_string(mem[flags_in[4 * j]]) + " -> " + std::to_string(mem[j]) +
                                          "): got " + std::to_string(flags_in[4 * j + 1]) + ", expected " +
                                          std::to_string(flags_in[4 * j + 2]));
    // phase 3: payload in 16-byte units
    auto units = [&](int64_t c) { return static_cast<Dim>((c * static_cast<int64_t>(elem_size) + 15) / 16); };
    Dim so = 0, ro = 0;
    std::vector<Xfer> s3, r3;
    std::vector<Dim> soff(n), roff(n);
    for (Dim i = 0; i < n; ++i) {
      soff[i] = so;
      roff[i] = ro;
      if (cnt_out[2 * i]) s3.push_back({mem[i], so, units(cnt_out[2 * i])});
      if (cnt_in[2 * i]) r3.push_back({mem[i], ro, units(cnt_in[2 * i])});
      so += units(cnt_out[2 * i]);
      ro += units(cnt_in[2 * i]);
    }
    std::vector<char> sh(static_cast<size_t>(so) * 16, 0), rh(static_cast<size_t>(ro) * 16);
    for (Dim i = 0; i < n; ++i)
      if (cnt_out[2 * i]) {
        if (!send_lists || !send_lists[i]) throw_invalid("null send list");
        std::memcpy(sh.data() + soff[i] * 16, send_lists[i], cnt_out[2 * i] * elem_size);
      }
    DevBuf ds(16 * std::max<Dim>(so, 1), x), dr(16 * std::max<Dim>(ro, 1), x);
    if (so) QTNH_CUDA(cudaMemcpyAsync(ds.ptr, sh.data(), so * 16, cudaMemcpyHostToDevice, x.stream));
    exchange(x, sorted, ds.ptr, s3, dr.ptr, r3);
    if (ro) QTNH_CUDA(cudaMemcpyAsync(rh.data(), dr.ptr, ro * 16, cudaMemcpyDeviceToHost, x.stream));
    QTNH_CUDA(cudaStreamSynchronize(x.stream));
    int64_t total = 0;
    for (Dim i = 0; i < n; ++i) total += cnt_in[2 * i];
    char* out = static_cast<char*>(std::malloc(std::max<size_t>(1, total * elem_size)));
    if (!out) throw std::bad_alloc();
    size_t at = 0;
    for (Dim i = 0; i < n; ++i) {
      std::memcpy(out + at, rh.data() + roff[i] * 16, cnt_in[2 * i] * elem_size);
      at += cnt_in[2 * i] * elem_size;
      recv_counts[i] = cnt_in[2 * i];
    }
    *recv_data = out;
  });
}

void qtnh_free_host(void* p) { std::free(p); }

int qtnh_contract_host(qtnh_rank_t r, int na, const int64_t* dims_a, const double* a, int nb,
                       const int64_t* dims_b, const double* b, int n_pairs, const int* a_pos, const int* b_pos,
                       double* c, int64_t* c_dims) {
  return guard([&] {
    RankCtx& x = ctx_of(r);
    need(a, "a");
    need(b, "b");
    need(c, "c");
    if (na > 0) need(dims_a, "dims_a");
    if (nb > 0) need(dims_b, "dims_b");
    std::vector<Dim> da(dims_a, dims_a + na), db(dims_b, dims_b + nb), cd;
    for (Dim d : da)
      if (d < 1) throw_invalid("index dimensions must be positive");
    for (Dim d : db)
      if (d < 1) throw_invalid("index dimensions must be positive");
    static const int chunks = [] {
      const char* e = std::getenv("QTNH_HOST_CHUNKS");
      return e ? std::max(1, std::atoi(e)) : 16;
    }();
    contract_host(x, da, a, db, b, std::vector<int>(a_pos, a_pos + n_pairs), std::vector<int>(b_pos, b_pos + n_pairs),
                  c, &cd, chunks);
    if (c_dims)
      for (size_t i = 0; i < cd.size(); ++i) c_dims[i] = cd[i];
  });
}

int qtnh_swap_indices(qtnh_tensor_t t, int a, int b) {
  return guard([&] {
    TP& p = dense_in_place(t);
    make_exclusive(p);
    op_swap_indices(p, a, b);
  });
}

int qtnh_qft_layer(qtnh_tensor_t t, int j) {
  return guard([&] {
    TP& p = dense_in_place(t);
    make_exclusive(p);
    op_qft_layer(p, j);
  });
}

int qtnh_all_to_all_v(qtnh_rank_t r, int n_members, const int* members, const void* send_buf,
                      const int64_t* send_counts, const int64_t* send_displs, void* recv_buf,
                      const int64_t* recv_counts, const int64_t* recv_displs) {
  return guard([&] {
    RankCtx& x = ctx_of(r);
    if (n_members < 1) throw_invalid("group members must be non-empty");
    need(members, "members");
    std::vector<int> mem(members, members + n_members);
    std::vector<int> sorted = mem;
    std::sort(sorted.begin(), sorted.end());
    if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end()) throw_invalid("duplicate group member");
    for (int m : mem)
      if (m < 0 || m >= x.world->size) throw_invalid("group member " + std::to_string(m) + " out of range");
    if (!std::binary_search(sorted.begin(), sorted.end(), x.rank))
      throw_invalid("rank " + std::to_string(x.rank) + " cannot open a group it is not a member of");
    std::vector<Xfer> sends, recvs;
    for (int i = 0; i < n_members; ++i) {
      if (send_counts && send_counts[i] > 0) sends.push_back({mem[i], send_displs ? send_displs[i] : 0, send_counts[i]});
      if (recv_counts && recv_counts[i] > 0) recvs.push_back({mem[i], recv_displs ? recv_displs[i] : 0, recv_counts[i]});
    }
    exchange(x, sorted, send_buf, sends, recv_buf, recvs);
  });
}

int qtnh_set_option(const char* name, double value) {
  return guard([&] {
    need(name, "name");
    std::string n(name);
    if (n == "swap_chunk_bytes") set_swap_chunk_bytes(static_cast<Dim>(value));
    else if (n == "peer_direct") set_peer_direct(value != 0);
    else if (n == "pool_reserve_gb") set_pool_reserve_gb(value);
    else throw_invalid("unknown option " + n);
  });
}

int qtnh_qft(qtnh_tensor_t t, int swaps) {
  return guard([&] {
    TP& p = dense_in_place(t);
    make_exclusive(p);
    op_qft(p, swaps != 0);
  });
}

int qtnh_svd_device(qtnh_rank_t r, int64_t batch, int64_t m, int64_t n, const void* a, int64_t chi, int absorb,
                    void* u, void* s, void* vh) {
  return guard([&] {
    RankCtx& x = ctx_of(r);
    need(a, "a");
    need(u, "u");
    need(s, "s");
    need(vh, "vh");
    int sweeps = 0;
    svd_batched(x, batch, m, n, a, chi, absorb, u, s, vh, &sweeps);
    t_info = sweeps;
    const Dim c = chi > 0 ? chi : std::min(m, n);
    std::vector<void*> up(batch), vp(batch);
    for (int64_t b = 0; b < batch; ++b) {
      up[b] = static_cast<char*>(u) + static_cast<size_t>(b * m * c) * 16;
      vp[b] = static_cast<char*>(vh) + static_cast<size_t>(b * c * n) * 16;
    }
    svd_complete_null(x, batch, m, n, c, absorb, up.data(), s, vp.data());
  });
}

int qtnh_mps_apply_layer(int n_pairs, const qtnh_tensor_t* left, const qtnh_tensor_t* right, const double* gate,
                         int64_t chi, qtnh_tensor_t* new_left, qtnh_tensor_t* new_right, double* s_out,
                         int64_t* keep_out, double* norm2_out) {
  return guard([&] {
    if (n_pairs < 0) throw_invalid("negative pair count");
    if (n_pairs == 0) return;
    need(left, "left");
    need(right, "right");
    need(gate, "gate");
    need(new_left, "new_left");
    need(new_right, "new_right");
    std::vector<TP> l(n_pairs), r(n_pairs), nl, nr;
    for (int i = 0; i < n_pairs; ++i) {
      l[i] = impl_of(left[i]);
      r[i] = impl_of(right[i]);
    }
    mps_apply_layer(l, r, gate, chi, nl, nr, s_out, keep_out, norm2_out);
    for (int i = 0; i < n_pairs; ++i) {
      new_left[i] = wrap(nl[i]);
      new_right[i] = wrap(nr[i]);
    }
  });
}

int qtnh_svd(qtnh_tensor_t t, int n_row, const int* row_pos, int n_col, const int* col_pos, int64_t chi,
             int absorb, qtnh_tensor_t* u_out, qtnh_tensor_t* vh_out, double* s_host) {
  return guard([&] {
    need(u_out, "u");
    need(vh_out, "vh");
    TP p = impl_of(t);
    // A distributed theta is gathered onto its root copy first (linalg::psvd gathers
    // the block-cyclic matrix onto the group root, linalg.hpp:441-462); S then goes
    // back to every rank of the original span (:464).
    std::vector<int> span_members;
    if (p->shape.split != 0) {
      span_members = span_ranks(*p);
      std::vector<int> id(p->shape.n_idx());
      std::iota(id.begin(), id.end(), 0);
      p = op_permute(p, id, 0);
    }
    const Shape& sh = p->shape;
    if (n_row + n_col != sh.n_idx()) throw_invalid("row/col index sets must partition the tensor indices");
    std::vector<int> perm, seen(sh.n_idx(), 0);
    for (int i = 0; i < n_row; ++i) perm.push_back(row_pos[i]);
    for (int i = 0; i < n_col; ++i) perm.push_back(col_pos[i]);
    for (int q : perm) {
      if (q < 0 || q >= sh.n_idx() || seen[q]) throw_invalid("row/col index sets must partition the tensor indices");
      seen[q] = 1;
    }
    Dim m = 1, n = 1;
    std::vector<Dim> udims, vdims;
    for (int i = 0; i < n_row; ++i) {
      m *= sh.dims[row_pos[i]];
      udims.push_back(sh.dims[row_pos[i]]);
    }
    for (int i = 0; i < n_col; ++i) {
      n *= sh.dims[col_pos[i]];
      vdims.push_back(sh.dims[col_pos[i]]);
    }
    Dim k = std::min(m, n);
    if (chi <= 0) chi = k;
    udims.push_back(chi);
    vdims.insert(vdims.begin(), chi);
    RankCtx& r = *p->rank;
    TP mat = op_permute(p, perm, 0);
    TP u = make_tensor(r, Shape(udims, 0), p->dist, true);
    TP vh = make_tensor(r, Shape(vdims, 0), p->dist, true);
    const Dim s_units = (chi + 1) / 2;  // S as 16-byte elements for the broadcast
    DevBuf s(static_cast<size_t>(s_units) * 16, r);
    if (p->in_span) {
      int sweeps = 0;
      svd_batched(r, 1, m, n, mat->data(), chi, absorb, u->data(), s.ptr, vh->data(), &sweeps);
      t_info = sweeps;
      void* up = u->data();
      void* vp = vh->data();
      svd_complete_null(r, 1, m, n, chi, absorb, &up, s.ptr, &vp);
    }
    if (!span_members.empty() &&
        std::find(span_members.begin(), span_members.end(), r.rank) != span_members.end()) {
      const int root = static_cast<int>(p->dist.canonical(0));
      std::vector<Xfer> sends, recvs;
      if (r.rank == root)
        for (int mbr : span_members) sends.push_back({mbr, 0, s_units});
      DevBuf got(static_cast<size_t>(s_units) * 16, r);
      recvs.push_back({root, 0, s_units});
      exchange(r, span_members, s.ptr, sends, got.ptr, recvs);
      if (s_host) {
        QTNH_CUDA(cudaMemcpyAsync(s_host, got.ptr, chi * sizeof(double), cudaMemcpyDeviceToHost, r.stream));
        QTNH_CUDA(cudaStreamSynchronize(r.stream));
      }
    } else if (p->in_span && s_host) {
      QTNH_CUDA(cudaMemcpyAsync(s_host, s.ptr, chi * sizeof(double), cudaMemcpyDeviceToHost, r.stream));
      QTNH_CUDA(cudaStreamSynchronize(r.stream));
    }
    *u_out = wrap(u);
    *vh_out = wrap(vh);
  });
}

int qtnh_remap_plan_json(int n, const int64_t* dims, int split, const int64_t* dist, const int* perm,
                         int new_split, const int64_t* new_dist, int rank, int world_size, char* buf, size_t len) {
  return guard([&] {
    need(buf, "buf");
    Shape ss = shape_from(n, dims, split);
    std::vector<int> pv(perm, perm + n), inv(n, -1);
    for (int p = 0; p < n; ++p) {
      if (pv[p] < 0 || pv[p] >= n || inv[pv[p]] != -1) throw_invalid("invalid index permutation");
      inv[pv[p]] = p;
    }
    std::vector<Dim> nd(n);
    for (int p = 0; p < n; ++p) nd[p] = ss.dims[pv[p]];
    Dist sd = dist_from(dist), dd = new_dist ? dist_from(new_dist) : sd;
    RemapPlan P = plan_remap(ss, sd, Shape(nd, new_split), dd, inv, rank, world_size);
    auto vec = [](const std::vector<Dim>& v) {
      std::string s = "[";
      for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
      return s + "]";
    };
    auto box = [&](const CopyBox& b) {
      return "{\"dims\":" + vec(b.dims) + ",\"in_stride\":" + vec(b.in_stride) + ",\"out_stride\":" +
             vec(b.out_stride) + "}";
    };
    auto xf = [](const std::vector<Xfer>& v) {
      std::string s = "[";
      for (size_t i = 0; i < v.size(); ++i)
        s += (i ? "," : "") + std::string("[") + std::to_string(v[i].peer) + "," + std::to_string(v[i].offset) +
             "," + std::to_string(v[i].count) + "]";
      return s + "]";
    };
    std::vector<Dim> mem(P.members.begin(), P.members.end());
    std::string j = "{\"members\":" + vec(mem) + ",\"member\":" + std::to_string(P.member) +
                    ",\"local_only\":" + std::to_string(P.local_only) + ",\"direct_layout\":" +
                    std::to_string(P.direct_layout) + ",\"src_canonical\":" + std::to_string(P.src_canonical) +
                    ",\"dst_in_span\":" + std::to_string(P.dst_in_span) + ",\"pack_to_dst\":" +
                    std::to_string(P.pack_to_dst) + ",\"recv_into_dst\":" + std::to_string(P.recv_into_dst) +
                    ",\"unpack\":" + std::to_string(P.unpack) + ",\"pack\":" + box(P.pack) +
                    ",\"unpack_box\":" + box(P.unpack_box) + ",\"pack_elems\":" + std::to_string(P.pack_elems) +
                    ",\"recv_elems\":" + std::to_string(P.recv_elems) + ",\"sends\":" + xf(P.sends) +
                    ",\"recvs\":" + xf(P.recvs) + ",\"push_box\":" + box(P.push_box) + ",\"pushes\":[";
    for (size_t i = 0; i < P.pushes.size(); ++i)
      j += (i ? ",[" : "[") + std::to_string(P.pushes[i].peer) + "," + std::to_string(P.pushes[i].src_off) + "," +
           std::to_string(P.pushes[i].dst_off) + "]";
    j += "]}";
    if (j.size() + 1 > len) throw_invalid("plan buffer too small: need " + std::to_string(j.size() + 1));
    std::memcpy(buf, j.c_str(), j.size() + 1);
  });
}

int qtnh_zgemm_device(qtnh_rank_t r, int64_t m, int64_t n, int64_t k, const void* a, const void* b, void* c) {
  return guard([&] {
    RankCtx& x = ctx_of(r);
    zgemm(a, b, c, m, n, k, x.stream);
  });
}

int qtnh_permute_device(qtnh_rank_t r, int n, const int64_t* dims, const int* perm, const void* in, void* out) {
  return guard([&] {
    RankCtx& x = ctx_of(r);
    std::vector<Dim> d(dims, dims + n);
    std::vector<int> p(perm, perm + n);
    std::vector<char> seen(n, 0);
    for (int v : p) {
      if (v < 0 || v >= n || seen[v]) throw_invalid("invalid index permutation");
      seen[v] = 1;
    }
    strided_copy(in, out, permute_box(d, p), true, x.stream);
  });
}

}  // extern "C"
