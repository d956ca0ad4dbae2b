// Structural operations, contraction and gate application on device tensors.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "runtime.h"
#include "strided_copy.h"

namespace qtnhb {

using TP = std::shared_ptr<TensorImpl>;

// Host-only plan of one rank's part of a redistribution (no device state): the
// pack box, the exchange lists and the unpack box. Shared by the device executor
// (remap) and the CPU executor of the multi-process tests.
struct RemapPlan {
  std::vector<int> members;
  bool member = false, local_only = false, direct_layout = false;
  bool src_canonical = false, dst_in_span = false;
  bool pack_to_dst = false, recv_into_dst = false, unpack = false;
  CopyBox pack, unpack_box;
  Dim pack_elems = 0, recv_elems = 0;
  std::vector<Xfer> sends, recvs;
  // Peer-memory form (local world): this rank writes each chunk straight into
  // the destination block of every home: dst(peer) + dst_off <- src + src_off
  // over push_box (W indices), zero canonicalised.
  struct Push {
    int peer;
    Dim src_off, dst_off;
  };
  std::vector<Push> pushes;
  CopyBox push_box;
};
RemapPlan plan_remap(const Shape& ss, const Dist& sd, const Shape& ds, const Dist& dd, const std::vector<int>& am,
                     int rank, int world_size);

// remap::tensor_to_tensor (remap.hpp:106-161) restricted to equal dimensions:
// axis_map[src_pos] = dst_pos.
TP remap(const TP& src, Shape dst_shape, Dist dst_dist, const std::vector<int>& axis_map);

TP op_permute(const TP& t, const std::vector<int>& perm, int new_split);  // ops.hpp:27
TP op_rebcast(const TP& t, Dist d);                                        // ops.hpp:54
TP op_scatter_index(const TP& t, int pos);                                 // ops.hpp:118
TP op_gather_index(const TP& t, int pos);                                  // ops.hpp:133
TP op_slice_local(const TP& t, const std::vector<Dim>& nl);                // ops.hpp:166
TP op_pad_local(const TP& t, const std::vector<Dim>& nl);                  // ops.hpp:201
TP op_scale(const TP& t, double re, double im, bool conj);                 // ops.hpp:147-161
// Real factor f[c] on every element whose coordinate at index pos is c
// (absorb_singular_left/right(..., power), linalg.hpp:508-523).
TP op_scale_index(const TP& t, int pos, const std::vector<double>& f);
void op_to_global(const TensorImpl& t, double* host);                      // tensor.hpp:341
// Contraction order of a labelled network (plan.cpp); ids of results continue
// after the n input tensors in step order.
std::vector<std::pair<int, int>> plan_order(const std::vector<std::vector<int>>& labels, const std::vector<double>& lg,
                                            uint64_t seed, int trials, double log2_cap = 0.0);
void op_save(const TensorImpl& t, const std::string& path);                // tensor.hpp:388-397
TP op_load(RankCtx& r, const std::string& path);                           // tensor.hpp:399-446 (dense)

// Contraction with SPEC.md:408 result order (see qtnh_b200.h).
TP op_contract(const TP& a, const TP& b, const std::vector<int>& apos, const std::vector<int>& bpos);
// In-place gate on t (caller guarantees exclusive ownership).
void op_gate_apply(TP& t, const std::vector<int>& targets, const double* gate, bool diagonal);

// In-place exchange of a distributed index a with a local index b (equal size),
// pairwise NVLink/NCCL exchange through a staging buffer of ~chunk_bytes.
void op_swap_dist_local_inplace(TP& t, int a, int b, Dim chunk_bytes);
void set_swap_chunk_bytes(Dim v);
// In-place (local) / remapped (distributed) exchange of two equal-size indices.
void op_swap_indices(TP& t, int a, int b);
// Fused QFT layer j on a qubit tensor (see gate.cu k_qft_layer).
void op_qft_layer(TP& t, int j);
// Whole QFT: distributed layers one by one, local layers cache-blocked, final
// SWAP network as an in-place bit reversal (undistributed) or index swaps.
void op_qft(TP& t, bool swaps);

// Contraction with host operands/result, pipelined H2D / GEMM / D2H (single rank).
void contract_host(RankCtx& r, const std::vector<Dim>& da, const double* a, const std::vector<Dim>& db,
                   const double* b, const std::vector<int>& apos, const std::vector<int>& bpos, double* c,
                   std::vector<Dim>* c_dims, int target_chunks);

// Kernels (zgemm.cu, gate.cu)
void zgemm(const void* a, const void* b, void* c, Dim m, Dim n, Dim k, cudaStream_t st);
// zgemm with A(m, k) gathered from a + rowoff[m] + coloff[k] (elements): the
// contraction's layout permutation fused into the operand loads.
void zgemm_gather_a(const void* a, const int64_t* rowoff, const int64_t* coloff, bool rows_fastest,
                    const void* b, void* c, Dim m, Dim n, Dim k, cudaStream_t st, const int64_t* cohi = nullptr,
                    int co_sh = 0, const int64_t* rohi = nullptr, int ro_sh = 0);
// out[i] = sum_d digit_d(i) * strides[d], digits row-major over dims.
void index_offsets(int64_t* out, Dim count, const std::vector<Dim>& dims, const std::vector<Dim>& strides,
                   cudaStream_t st);
// Batched thin SVD (blocked one-sided Jacobi), truncated / zero-padded to chi,
// singular values absorbed per QTNH_ABSORB_*; device row-major in/out.
void svd_batched(RankCtx& r, Dim batch, Dim m, Dim n, const void* a, Dim chi, int absorb, void* u, void* s,
                 void* vh, int* sweeps_out);
// The same with one output pointer per matrix (U: m x chi, Vh: chi x n each).
// Truncating calls (chi < min(m, n)) try the spectral-split path first
// (svd_split.cu); everything else, and every matrix the split cannot certify,
// runs the blocked one-sided Jacobi (svd_jacobi_ptrs).
void svd_batched_ptrs(RankCtx& r, Dim batch, Dim m, Dim n, const void* a, Dim chi, int absorb, void* const* u_ptrs,
                      void* s, void* const* vh_ptrs, int* sweeps_out);
int64_t svd_split_count();  // matrices factorised by the split path so far
// Null singular directions (sigma <= max(m, n) eps sigma_0) of svd outputs
// replaced by an orthonormal completion (svd_null.cu): U and Vh stay isometries
// on their non-absorbed side like zgesdd's (linalg.hpp:441-471).
void svd_complete_null(RankCtx& r, Dim batch, Dim m, Dim n, Dim chi, int absorb, void* const* u_ptrs, const void* s,
                       void* const* vh_ptrs);
// out (cols x rows) = conj(in (rows x cols))^T, complex128 row-major.
void conj_transpose(const void* in, void* out, Dim rows, Dim cols, cudaStream_t st);
void svd_jacobi_ptrs(RankCtx& r, Dim batch, Dim m, Dim n, const void* a, Dim chi, int absorb, void* const* u_ptrs,
                     void* s, void* const* vh_ptrs, int* sweeps_out);
// One layer of MPS two-site updates (mps.cu): pair i = (left[i], right[i]),
// sites (l, d, c) and (c, d, r) held by this rank; gate = 4x4 complex row-major
// (out1 out2, in1 in2). New sites U S (l, d, keep) and Vh (keep, d, r), keep =
// min(chi, l d, d r); s_out[i*chi ..] = kept singular values (zero-padded),
// keep_out[i], norm2_out[i] = ||theta_i||_F^2.
void mps_apply_layer(const std::vector<TP>& left, const std::vector<TP>& right, const double* gate, Dim chi,
                     std::vector<TP>& new_left, std::vector<TP>& new_right, double* s_out, int64_t* keep_out,
                     double* norm2_out);
// Fused QFT layer on a local qubit block (all dims 2): H on bit t + the layer's
// controlled phases; phase-only variant for a distributed target with x_j = 1.
void qft_layer_local(void* data, int local_bits, int t, cudaStream_t st);
void qft_phase_local(void* data, int local_bits, int64_t v_off, int t, cudaStream_t st);
// Cache-blocked QFT layers on a local block of nb qubits: layers whose target
// bits are first_layer_bit..0 (the low bits staged in shared memory, upper bits
// in register groups of 5); in-place bit reversal (the final SWAP network).
void qft_local_fused(void* data, int nb, int first_layer_bit, cudaStream_t st);
void bitrev_local(void* data, int nb, cudaStream_t st);
// Reverse the top nh bits of the local index, holding the low k bits.
void bitrev_hi_local(void* data, int nh, int k, cudaStream_t st);
// Peer-memory distributed QFT pieces; ptrs = the 2^k group members' blocks by
// distributed coordinate (see gate.cu).
void qft_dist_layers(void* const* ptrs, int k, int nb, Dim i0, Dim i1, cudaStream_t st);
void dist_bitrev(void* const* ptrs, int k, Dim m0, Dim m1, cudaStream_t st);
// In-place exchange of two equal-size local indices.
void swap_indices_local(void* data, const std::vector<Dim>& dims, int ia, int ib, cudaStream_t st);
// Gate on a dense local block: dims = local dims, targets = local positions.
void gate_local(void* data, const std::vector<Dim>& dims, const std::vector<int>& targets,
                const double* gate_host, bool diagonal, cudaStream_t st);
// gate_local over explicit element strides, fibers [f_begin, f_end) only
// (f_end < 0: all); strides may span buffers (peer pointers).
void gate_strided(void* data, const std::vector<Dim>& dims, const std::vector<Dim>& strides,
                  const std::vector<int>& targets, const double* gh, bool diagonal, cudaStream_t st, Dim f_begin,
                  Dim f_end);

}  // namespace qtnhb
