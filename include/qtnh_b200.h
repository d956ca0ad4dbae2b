/*
 * qtnh_b200.h -- C ABI of libqtnh_b200.so, the B200-native (sm_100a) hot path of
 * the QTNH distributed tensor-network library (arXiv 2505.06119).
 *
 * The reference (/root/reference/proj/include/qtnh, header-only C++20) exposes the
 * path as C++ functions, not an FFI; each entry point below replaces one of them
 * and keeps its argument meaning, result layout and error class:
 *
 *   qtnh_world_create_local / qtnh_rank_bind  <- World(n) + World::run  runtime.hpp:245, :263-299
 *   qtnh_world_create_nccl                    <- Backend::external_message_passing  runtime.hpp:248-251
 *   qtnh_tensor_dense / _from_global          <- Tensor::dense / from_global  tensor.hpp:61, :83
 *   qtnh_tensor_download_local / _global      <- Tensor::local_data / to_global_vector  tensor.hpp:177, :341
 *   qtnh_permute                              <- ops::permute  ops.hpp:27-49
 *   qtnh_rebcast                              <- ops::rebcast (dense)  ops.hpp:54, :104-109
 *   qtnh_scatter_index / qtnh_gather_index    <- ops::scatter_index / gather_index  ops.hpp:118, :133
 *   qtnh_slice_local_dims / _pad_local_dims   <- ops::slice_local_dims / pad_local_dims  ops.hpp:166, :201
 *   qtnh_conj / qtnh_scale                    <- ops::conj / ops::scale  ops.hpp:147-161
 *   qtnh_contract                             <- tensor_to_matrix -> pgemm -> matrix_to_tensor
 *                                                linalg.hpp:208, :347, :273 with the SPEC.md:408 order
 *   qtnh_gate_apply                           <- contract(state, gate) + permute back (same values,
 *                                                index order kept, in place)
 *   qtnh_svd                                  <- psvd + truncate_svd + absorb_singular_*  linalg.hpp:441-523
 *
 * Conventions
 *   - Elements are complex128 stored as interleaved (re, im) doubles, row-major,
 *     rightmost index fastest (indexing.hpp:106-134).
 *   - perm[new_pos] = old_pos (ops.hpp:21-23).
 *   - dist[3] = {stretch, cycles, offset} (indexing.hpp:84-101); NULL means {1,1,0}.
 *   - Every tensor operation is collective over the union of the involved spans and
 *     must be called by each member rank with equal arguments; ranks
 *     outside every span return immediately with a metadata-only handle.
 *   - Elements whose real and imaginary parts are both zero come out as (+0, +0),
 *     exactly like the reference's zero-skipping remap (remap.hpp:69-70, :125-127).
 *   - Every function returns a status: 0 on success, else one QTNH_E_* code.
 *     qtnh_last_error() returns the thread-local message; qtnh_last_error_info()
 *     the required rank count (QTNH_E_RESOURCE) or solver info (QTNH_E_NUMERICAL).
 */
#ifndef QTNH_B200_H_
#define QTNH_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error classes, one per qtnh::Error subclass (common.hpp:31-74). */
enum {
  QTNH_OK = 0,
  QTNH_E_INVALID_ARGUMENT = 1, /* InvalidArgument */
  QTNH_E_RESOURCE = 2,         /* ResourceError(required_ranks) */
  QTNH_E_PROTOCOL = 3,         /* ProtocolError */
  QTNH_E_NUMERICAL = 4,        /* NumericalError(info) */
  QTNH_E_PRECONDITION = 5,     /* PreconditionError */
  QTNH_E_DEGENERATE = 6,       /* DegenerateStateError */
  QTNH_E_ABORTED = 7,          /* AbortedError */
  QTNH_E_RUNTIME = 8           /* Error: CUDA / NCCL / allocation failure */
};

typedef struct qtnh_world_s* qtnh_world_t;
typedef struct qtnh_rank_s* qtnh_rank_t;
typedef struct qtnh_tensor_s* qtnh_tensor_t;

/* ---- errors / build info ------------------------------------------------- */
int qtnh_last_error(char* buf, size_t len);
int64_t qtnh_last_error_info(void);
const char* qtnh_version(void);
/* Tunables: "swap_chunk_bytes" = staging size of the in-place distributed swap;
   "peer_direct" (1 default) = in a local world whose ranks can address each
   other's HBM, redistribute by peer-memory kernels (push remap, pairwise
   in-place swap) instead of pack -> exchange -> unpack;
   "pool_reserve_gb" (0 default) = GiB of the device's stream-ordered pool to map
   when the next world is created (long sequences of varying tensor sizes then
   never wait on new mappings). */
int qtnh_set_option(const char* name, double value);
/* Number of this library's kernels launched so far by the calling process. */
int64_t qtnh_kernel_launch_count(void);

/* ---- worlds and ranks ---------------------------------------------------- */
/* In-process world of n ranks; rank r runs on device devices[r] (NULL: all on
 * device 0). Each rank is driven by its own host thread that calls
 * qtnh_rank_bind(world, r, &rank) -- the B200 analogue of World::run. Exchanges
 * are stream-ordered device (or NVLink peer) copies coordinated by a host
 * rendezvous; no kernel ever waits on another rank. */
int qtnh_world_create_local(int n_ranks, const int* devices, qtnh_world_t* out);
/* One process per GPU (torchrun): this process is rank `rank` of `size` and owns
 * `device`. uid is the 128-byte NCCL unique id produced by qtnh_nccl_unique_id on
 * rank 0 and shared out of band. NCCL is loaded lazily (dlopen). */
int qtnh_nccl_unique_id(void* uid128);
int qtnh_world_create_nccl(int rank, int size, int device, const void* uid128, qtnh_world_t* out);
/* Process-per-GPU world without NCCL (one process per GPU, one node): every
 * collective is a CUDA-IPC peer-memory operation -- exportable stream-ordered
 * pools shared once over Unix sockets under `dir`, interprocess events for
 * stream ordering, pointer-export records per collective; the fused peer kernels
 * (push remap, pairwise swap, distributed gate / QFT) run across processes. */
int qtnh_world_create_ipc(int rank, int size, int device, const char* dir, qtnh_world_t* out);
int qtnh_world_destroy(qtnh_world_t w);
int qtnh_world_size(qtnh_world_t w);
/* Abort all pending and future collectives of the world (AbortedError on peers). */
int qtnh_world_abort(qtnh_world_t w);

int qtnh_rank_bind(qtnh_world_t w, int rank, qtnh_rank_t* out);
int qtnh_rank_release(qtnh_rank_t r);
int qtnh_rank_id(qtnh_rank_t r);
/* Stream the rank launches on (cudaStream_t as void*; NULL = the legacy default
 * stream, e.g. torch's default stream). qtnh_rank_reset_stream restores the
 * rank's own non-blocking stream. */
int qtnh_rank_set_stream(qtnh_rank_t r, void* stream);
int qtnh_rank_reset_stream(qtnh_rank_t r);
void* qtnh_rank_stream(qtnh_rank_t r);
int qtnh_rank_synchronize(qtnh_rank_t r);
/* CUDA-graph capture of a launch-bound sequence of in-place, rank-local ops on
 * existing tensors (gate applications, qubit swaps, QFT layers): everything the
 * rank launches between begin and end is recorded on its stream (thread-local
 * capture mode) and replayed with one qtnh_graph_launch. Collectives, host
 * copies and ops that allocate result tensors must stay outside a capture. */
typedef struct qtnh_graph_s* qtnh_graph_t;
int qtnh_rank_capture_begin(qtnh_rank_t r);
int qtnh_rank_capture_end(qtnh_rank_t r, qtnh_graph_t* out);
int qtnh_graph_launch(qtnh_rank_t r, qtnh_graph_t g);
int qtnh_graph_destroy(qtnh_graph_t g);
int qtnh_barrier(qtnh_rank_t r);

/* Group::all_to_all_v (runtime.hpp:448-475) on device buffers of complex128
 * elements: member i receives send_counts[i] elements from send_buf+send_displs[i];
 * this rank receives recv_counts[i] elements from member i into
 * recv_buf+recv_displs[i]. Collective over `members` (world ranks; member-only,
 * runtime.hpp:191-223). Each sender's count must equal the receiver's expected
 * count, else QTNH_E_PROTOCOL naming the "(src -> dst)" pair (runtime.hpp:464-471);
 * a zero count means "nothing to/from that member". Stream-ordered. */
int qtnh_all_to_all_v(qtnh_rank_t r, int n_members, const int* members, const void* send_buf,
                      const int64_t* send_counts, const int64_t* send_displs, void* recv_buf,
                      const int64_t* recv_counts, const int64_t* recv_displs);
/* Group::all_to_all_v on HOST data (runtime.hpp:448-475; the building block of the
 * C++ layer's Group broadcast / gather / scatter / all_reduce_sum / barrier):
 * members in group order; send_lists[i] holds send_counts[i] elements of
 * elem_size bytes for member i. Receive counts are exchanged first; with
 * expected_counts (may be NULL) a mismatch raises QTNH_E_PROTOCOL "all_to_all_v
 * count mismatch for pair (src -> dst): got G, expected E" on every member.
 * *recv_data = one malloc'ed buffer (release with qtnh_free_host) holding what
 * each member sent here, concatenated in member order; recv_counts[i] = its
 * element count. */
int qtnh_group_all_to_all_v_host(qtnh_rank_t r, int n_members, const int* members, size_t elem_size,
                                 const void* const* send_lists, const int64_t* send_counts,
                                 const int64_t* expected_counts, void** recv_data, int64_t* recv_counts);
void qtnh_free_host(void* p);

/* ---- tensors ------------------------------------------------------------- */
/* Dense tensor; `local` holds local_size complex numbers of this rank's block
 * (host memory, NULL = zeros). Ranks outside the span ignore `local`. */
int qtnh_tensor_dense(qtnh_rank_t r, int n_idx, const int64_t* dims, int split,
                      const int64_t* dist, const double* local, qtnh_tensor_t* out);
/* Dense tensor from a replicated global host vector (tensor.hpp:83-94). */
int qtnh_tensor_from_global(qtnh_rank_t r, int n_idx, const int64_t* dims, int split,
                            const int64_t* dist, const double* global, qtnh_tensor_t* out);
/* Dense tensor adopting this rank's block from device memory (copied, stream-ordered). */
int qtnh_tensor_from_device(qtnh_rank_t r, int n_idx, const int64_t* dims, int split,
                            const int64_t* dist, const void* dev_local, qtnh_tensor_t* out);
int qtnh_tensor_retain(qtnh_tensor_t t);
int qtnh_tensor_free(qtnh_tensor_t t);

int qtnh_tensor_rank(qtnh_tensor_t t);                 /* number of indices */
int qtnh_tensor_dims(qtnh_tensor_t t, int64_t* dims);  /* n_idx entries */
int qtnh_tensor_split(qtnh_tensor_t t);
int qtnh_tensor_dist(qtnh_tensor_t t, int64_t* dist3);
int64_t qtnh_tensor_local_size(qtnh_tensor_t t);
int64_t qtnh_tensor_span(qtnh_tensor_t t);
int qtnh_tensor_in_span(qtnh_tensor_t t);
int64_t qtnh_tensor_my_block(qtnh_tensor_t t);
int qtnh_tensor_is_canonical(qtnh_tensor_t t);
/* Device pointer of this rank's block (interleaved complex128), NULL outside the span. */
void* qtnh_tensor_device_ptr(qtnh_tensor_t t);
/* Copy this rank's block to host (local_size complex). Synchronises the rank stream. */
int qtnh_tensor_download_local(qtnh_tensor_t t, double* host);
/* Async variant into caller-provided (pinned) host memory; completes on the rank stream. */
int qtnh_tensor_download_local_async(qtnh_tensor_t t, double* host);
int qtnh_tensor_upload_local(qtnh_tensor_t t, const double* host);
/* Span-collective gather of the full global vector into `host` (total_size complex)
 * on every span rank (tensor.hpp:341-371). */
int qtnh_tensor_to_global(qtnh_tensor_t t, double* host);
/* ---- storage variants (tensor.hpp:28: dense 0, symmetric 1, diagonal 2, identity 3,
 * swap 4) ---------------------------------------------------------------------
 * The compact variants keep the reference's storage contract in HBM: a diagonal
 * tensor holds its block's slice of the diagonal (only on blocks whose input and
 * output distributed coordinates agree), identity and swap hold nothing. rebcast,
 * conj, scale, clone, save and load keep the variant (ops.hpp:54-161, tensor.hpp:
 * 373-446); every other operation reads the tensor through its dense value
 * (to_dense, materialised on the device on first use), as the reference's ops do. */
enum { QTNH_DENSE = 0, QTNH_SYMMETRIC = 1, QTNH_DIAGONAL = 2, QTNH_IDENTITY = 3, QTNH_SWAP = 4 };
/* Tensor::identity / Tensor::swap_tensor (tensor.hpp:144-164): element = 1 iff
 * coords[in_pos[k]] == coords[out_pos[k]] for every pair (crossed != 0: swap, the
 * two outputs exchanged; exactly two pairs). No storage. */
int qtnh_tensor_paired(qtnh_rank_t r, int n, const int64_t* dims, int split, const int64_t* dist, int n_pairs,
                       const int* in_pos, const int* out_pos, int crossed, qtnh_tensor_t* out);
/* Tensor::diagonal (tensor.hpp:114-142) over the symmetric half-split layout
 * (in_dist, out_dist; in_local, out_local): `count` complex values, the diagonal in
 * row-major order of the input coordinates; each on-diagonal block keeps its slice.
 * diag_global == NULL with count < 0: a zero diagonal (filled later by upload_local). */
int qtnh_tensor_diagonal(qtnh_rank_t r, int n, const int64_t* dims, int split, const int64_t* dist,
                         const double* diag_global, int64_t count, qtnh_tensor_t* out);
/* Tensor::symmetric / symmetric_from_global (tensor.hpp:97-112): dense storage, the
 * half-split layout validated first; data = this rank's block (is_global == 0,
 * `count` must equal the local size) or the global vector (is_global != 0);
 * data == NULL: a zero block. */
int qtnh_tensor_symmetric(qtnh_rank_t r, int n, const int64_t* dims, int split, const int64_t* dist,
                          const double* data, int64_t count, int is_global, qtnh_tensor_t* out);
int qtnh_tensor_variant(qtnh_tensor_t t);          /* Tensor::variant(), tensor.hpp:174 */
int64_t qtnh_tensor_stored_size(qtnh_tensor_t t);  /* local_data().size(): complex elements this rank stores */
/* equality_in() / equality_out() (tensor.hpp:193-194): the rank/2 pairs as constructed. */
int qtnh_tensor_pairs(qtnh_tensor_t t, int* in_pos, int* out_pos);
/* Tensor::to_dense (tensor.hpp:282-296): same shape, distribution and values. */
int qtnh_tensor_to_dense(qtnh_tensor_t t, qtnh_tensor_t* out);
/* Tensor::local_element (tensor.hpp:209-247): value at global coordinates from this
 * rank's storage (computed for identity / swap, 0 off the diagonal of a diagonal
 * tensor); QTNH_E_INVALID_ARGUMENT when the hosting block lives on another rank. */
int qtnh_tensor_local_element(qtnh_tensor_t t, const int64_t* coords, double* out_re_im);
/* ops::squeeze / unsqueeze (ops.hpp:234-262): remove / insert a size-1 index;
 * metadata only, the result shares the block. */
int qtnh_squeeze(qtnh_tensor_t t, int pos, qtnh_tensor_t* out);
int qtnh_unsqueeze(qtnh_tensor_t t, int pos, int as_dist, qtnh_tensor_t* out);
/* QTNHTEN1 files (tensor.hpp:373-446), byte-identical to the reference's, every
 * variant (a diagonal tensor stores its diagonal, identity and swap their pair
 * list). Save is span-collective (Tensor::save(path), tensor.hpp:388-397): the first
 * span rank writes the header, every canonical holder writes its own block (or
 * diagonal slice) at its offset straight from HBM (no gather). Load
 * (Tensor::load(Rank&, path), tensor.hpp:399-446) reads only this rank's part. */
int qtnh_tensor_save(qtnh_tensor_t t, const char* path);
int qtnh_tensor_load(qtnh_rank_t r, const char* path, qtnh_tensor_t* out);

/* ---- structural ops (ops.hpp) --------------------------------------------- */
int qtnh_permute(qtnh_tensor_t t, const int* perm, int new_split, qtnh_tensor_t* out);
int qtnh_rebcast(qtnh_tensor_t t, const int64_t* new_dist, qtnh_tensor_t* out);
/* remap::tensor_to_tensor (remap.hpp:106-161), dense: axis_map[src_pos] = dst_pos,
 * destination dims >= the mapped source dims (larger local dims zero-embed;
 * larger distributed dims are rejected), new split and DistParams (NULL: keep).
 * One redistribution pass (plus a local pad when embedding). */
int qtnh_remap(qtnh_tensor_t t, const int* axis_map, int n_dst, const int64_t* dst_dims, int dst_split,
               const int64_t* dst_dist, qtnh_tensor_t* out);
int qtnh_scatter_index(qtnh_tensor_t t, int pos, qtnh_tensor_t* out);
int qtnh_gather_index(qtnh_tensor_t t, int pos, qtnh_tensor_t* out);
int qtnh_slice_local_dims(qtnh_tensor_t t, const int64_t* new_local_dims, qtnh_tensor_t* out);
int qtnh_pad_local_dims(qtnh_tensor_t t, const int64_t* new_local_dims, qtnh_tensor_t* out);
int qtnh_conj(qtnh_tensor_t t, qtnh_tensor_t* out);
/* Real factor factors[c] on every element whose coordinate at index `pos` is c
 * (replaces absorb_singular_left / _right(..., power), linalg.hpp:508-523, on the
 * tensor form of U / Vh: factors = s^power). `factors` has dims[pos] entries. */
int qtnh_scale_index(qtnh_tensor_t t, int pos, const double* factors, qtnh_tensor_t* out);
/* A new handle on the same immutable value (tensor.hpp:41-43 value semantics:
 * copies share storage until one is mutated, see qtnh_tensor_make_mutable). */
int qtnh_tensor_clone(qtnh_tensor_t t, qtnh_tensor_t* out);
/* Copy-on-write for Tensor::mutable_local_data (tensor.hpp:177-178): after this
 * call the handle's local block is not shared with any other handle, so
 * qtnh_tensor_upload_local writes only this value. */
int qtnh_tensor_make_mutable(qtnh_tensor_t t);
/* Same local row-major block under new dims (no distributed indices before or
 * after; equal element count); shares the value. Used to regroup matrix digits
 * in matrix_to_tensor / pgemm when the row or column factorisation changes. */
int qtnh_tensor_reshape(qtnh_tensor_t t, int n_idx, const int64_t* dims, qtnh_tensor_t* out);
int qtnh_scale(qtnh_tensor_t t, double re, double im, qtnh_tensor_t* out);

/* Contraction order of a labelled network (SPEC network::contract_order,
 * SPEC.md:391-399): tensor t has labels[label_offsets[t] .. label_offsets[t+1]),
 * label l has log2 dimension label_log2[l]; a label shared by two tensors is a bond.
 * Seeded randomised greedy (trial 0: smallest result first, ties by hash), best of
 * `trials` by (largest intermediate, flops). order_out receives n_tensors - 1
 * pairs; the result of step s gets id n_tensors + s. */
int qtnh_plan_order(int n_tensors, const int* label_offsets, const int* labels, int n_labels,
                    const double* label_log2, uint64_t seed, int trials, int* order_out);
/* The same search under a memory budget: orders whose largest intermediate has at
 * most 2^log2_cap elements compete on flops (then size) and beat every order that
 * does not fit; log2_cap <= 0 is qtnh_plan_order. */
int qtnh_plan_order_capped(int n_tensors, const int* label_offsets, const int* labels, int n_labels,
                           const double* label_log2, uint64_t seed, int trials, double log2_cap, int* order_out);

/* ---- contraction ----------------------------------------------------------- */
/* Contract a[a_pos[i]] with b[b_pos[i]] for i < n_pairs. Result indices: open
 * indices of a, then open indices of b, each in operand order;
 * DistParams of a; split = number of a's distributed indices left
 * open. complex128 GEMM on the FP64 tensor cores (DMMA). */
int qtnh_contract(qtnh_tensor_t a, qtnh_tensor_t b, int n_pairs, const int* a_pos,
                  const int* b_pos, qtnh_tensor_t* out);

/* A whole contraction order in one call (network::contract_order):
 * ids 0..n_inputs-1 are `inputs`, step s contracts step_ab[2s] with step_ab[2s+1]
 * over step_npairs[s] position pairs (consecutive in a_pos / b_pos) and its result
 * gets id n_inputs + s; intermediates are released as soon as they are consumed.
 * `out` receives the last result (the inputs' handles stay valid). */
int qtnh_contract_chain(int n_inputs, const qtnh_tensor_t* inputs, int n_steps, const int* step_ab,
                        const int* step_npairs, const int* a_pos, const int* b_pos, qtnh_tensor_t* out);

/* Contraction with both operands and the result in HOST memory (the reference's
 * contract takes host-resident std::vector tensors): A is streamed through the GPU
 * in chunks of its leading open indices; H2D of chunk i+1, the GEMM of chunk i and
 * the D2H of chunk i-1 overlap on three streams (use pinned memory for overlap).
 * Result order/values as qtnh_contract on undistributed tensors; c_dims receives
 * the result dims (may be NULL). Completes on the rank's stream. */
int qtnh_contract_host(qtnh_rank_t r, int na, const int64_t* dims_a, const double* a, int nb,
                       const int64_t* dims_b, const double* b, int n_pairs, const int* a_pos, const int* b_pos,
                       double* c, int64_t* c_dims);

/* In-place gate application on a state whose indices all have the same role as
 * in contract(state, gate) followed by a permute that puts the gate outputs back
 * at `targets`. gate: host row-major D x D complex matrix, D = prod dims[targets],
 * row index = gate output (targets[0] most significant). `diagonal` != 0 means the
 * matrix is diagonal and only its D diagonal entries are passed. Copy-on-write:
 * if the state handle is shared, it is duplicated first. */
int qtnh_gate_apply(qtnh_tensor_t state, int n_targets, const int* targets,
                    const double* gate, int diagonal);
/* The same with the gate as a replicated tensor (outputs; inputs) of any variant
 * (split 0, DistParams{1, P, 0}): a diagonal-variant gate runs the diagonal kernel
 * from its stored diagonal and needs no exchange even on distributed targets
 * (tensor.hpp:114-142), an identity does nothing, a two-target swap
 * is an index exchange, dense / symmetric gates take the dense path. */
int qtnh_gate_apply_tensor(qtnh_tensor_t state, int n_targets, const int* targets, qtnh_tensor_t gate);

/* In-place exchange of two equal-size indices (values of ops::permute with the
 * two positions swapped -- a contraction with a swap tensor, tensor.hpp:157-164);
 * a distributed index goes through the exchange path. */
int qtnh_swap_indices(qtnh_tensor_t t, int a, int b);
/* Fused QFT layer j on a qubit tensor (all dims 2, qubit j = index j, index 0 most
 * significant): H on qubit j and every CP(2 pi / 2^m) between j and qubit j+m-1
 * (Fig. 1) in one pass over the state. */
int qtnh_qft_layer(qtnh_tensor_t t, int j);

/* The whole QFT circuit of PAPER.md Fig. 1 on a qubit tensor, in place: layers on
 * distributed qubits one by one, local layers cache-blocked (the lowest 11 in
 * shared memory, upper ones in register groups), final SWAP network as one
 * in-place bit reversal when nothing is distributed. */
int qtnh_qft(qtnh_tensor_t t, int swaps);

/* ---- factorisation --------------------------------------------------------- */
enum { QTNH_ABSORB_NONE = 0, QTNH_ABSORB_LEFT = 1, QTNH_ABSORB_RIGHT = 2, QTNH_ABSORB_SPLIT = 3 };
/* Batched thin SVD of `batch` row-major m x n matrices stored back to back in
 * device memory a (not modified), truncated/zero-padded to chi columns
 * (linalg.hpp:476-505), singular values absorbed per `absorb` (linalg.hpp:508-523).
 * Outputs (device, row-major): u [batch][m][chi], s [batch][chi] (doubles,
 * descending), vh [batch][chi][n]. chi <= 0 means min(m, n). Runs on the rank's
 * stream. NumericalError if Jacobi sweeps fail to converge. Like zgesdd's, the
 * non-absorbed factors are isometries whatever the rank of a: null directions
 * (sigma <= max(m, n) eps sigma_0) get an orthonormal completion; columns past
 * min(m, n) stay zero (truncate_svd's padding). */
int qtnh_svd_device(qtnh_rank_t r, int64_t batch, int64_t m, int64_t n, const void* a,
                    int64_t chi, int absorb, void* u, void* s, void* vh);

/* ---- seeded inputs (common.hpp:83-146) ------------------------------------- */
/* hash_counter(seed, k0, k1, k2) of the reference (common.hpp:93-100). */
uint64_t qtnh_hash_counter(uint64_t seed, uint64_t k0, uint64_t k1, uint64_t k2);
/* `count` values of one sequential Rng(seed).next_complex_normal() stream (host,
 * bit-identical to the reference). */
void qtnh_rng_complex_normals(uint64_t seed, int64_t count, double* out);
/* Counter-based complex normals for elements start..start+count-1 (host, glibc
 * Box-Muller, bit-identical across shards and runs); `threads` host threads. */
void qtnh_counter_complex_normals(uint64_t seed, int64_t start, int64_t count, double* out, int threads);
/* Same stream generated on the device (CUDA log/sincos: ~1 ulp from glibc). */
int qtnh_counter_complex_normals_device(void* stream, uint64_t seed, int64_t start, int64_t count, void* out);

/* ---- host-only planning ----------------------------------------------------- */
/* The exchange plan of rank `rank` (of `world_size`) for ops::permute(t, perm,
 * new_split) followed by a move to `new_dist` (NULL: keep t's dist), as JSON:
 * pack box, send/recv lists (peer, element offset, count), unpack box. No device
 * state is touched -- this is what the multi-process CPU tests execute. */
int qtnh_remap_plan_json(int n_idx, const int64_t* dims, int split, const int64_t* dist, const int* perm,
                         int new_split, const int64_t* new_dist, int rank, int world_size, char* buf, size_t len);

/* Tensor-level split (SPEC network::decompose / linalg psvd + truncate_svd +
 * absorb_singular_*): rows = indices row_pos (in order), cols = col_pos. Outputs
 * u with dims [row dims..., chi], vh with dims [chi, col dims...] (same DistParams
 * as t), s_host (chi doubles, descending, zero-padded; may be NULL).
 * A t with distributed indices is first gathered onto its root copy (linalg::psvd
 * gathers to the group root, linalg.hpp:441-462): u and vh live there, and S is
 * sent back to every rank of t's span (:464). qtnh_last_error_info() afterwards
 * = Jacobi sweeps (on the ranks that ran the SVD). Null directions are completed
 * to orthonormal vectors as in qtnh_svd_device. */
int qtnh_svd(qtnh_tensor_t t, int n_row, const int* row_pos, int n_col, const int* col_pos, int64_t chi,
             int absorb, qtnh_tensor_t* u, qtnh_tensor_t* vh, double* s_host);

/* One brickwork layer of MPS two-site updates (config 4; SPEC apply_raw_gate,
 * SPEC.md:371-379 / :475-483, composed in the reference from contract ->
 * gate -> psvd -> truncate_svd -> absorb_singular_left, linalg.hpp:208-523).
 * Pair i: left[i] (l, d, c) and right[i] (c, d, r), both held by the calling
 * rank without distributed indices; gate = 4 x 4 complex128 (interleaved re/im,
 * row-major (out1 out2, in1 in2)). Thetas of equal shape are factorised by one
 * batched SVD; U S and Vh are written straight into the new site tensors
 * new_left[i] (l, d, keep), new_right[i] (keep, d, r), keep = min(chi, l d, d r).
 * s_out[i * chi ...] = the kept singular values (descending, zero-padded to chi;
 * may be NULL), keep_out[i] = keep, norm2_out[i] = ||theta_i||_F^2 (the kept
 * weight is sum(s^2) / norm2). The inputs are not consumed. */
int qtnh_mps_apply_layer(int n_pairs, const qtnh_tensor_t* left, const qtnh_tensor_t* right, const double* gate,
                         int64_t chi, qtnh_tensor_t* new_left, qtnh_tensor_t* new_right, double* s_out,
                         int64_t* keep_out, double* norm2_out);

/* ---- raw kernels on device buffers (bench / integration) ------------------ */
/* out = a(M x K) * b(K x N), row-major complex128 on the rank's stream. */
int qtnh_zgemm_device(qtnh_rank_t r, int64_t m, int64_t n, int64_t k, const void* a,
                      const void* b, void* c);
/* Local strided permutation of a dense block: out (row-major over permuted dims)
 * <- in (row-major over dims), perm[new] = old; zero canonicalisation applied. */
int qtnh_permute_device(qtnh_rank_t r, int n_idx, const int64_t* dims, const int* perm,
                        const void* in, void* out);

/* Matrices the truncated SVD has factorised through its spectral-split path
 * (svd_split.cu) since the library loaded -- the rest took the full Jacobi SVD. */
int64_t qtnh_svd_split_count(void);

/* FP64 tensor-pipe (DMMA) peak measured on the current device, TFLOP/s. */
int qtnh_probe_fp64_peak(void* stream, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* QTNH_B200_H_ */
