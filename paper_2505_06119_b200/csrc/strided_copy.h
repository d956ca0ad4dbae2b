// Strided-copy engine: every structural operation of the remap path
// (permutation, pack into per-destination chunks, unpack into the destination
// block) is one launch of this engine. It replaces the per-element
// (address, value) Item packing of remap::pack_sends (remap.hpp:56-101) and the
// scatter loop of tensor_to_tensor (remap.hpp:155-159).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "common.h"

namespace qtnhb {

// out[sum_i c_i*out_stride_i] = f(in[sum_i c_i*in_stride_i]) for every coordinate
// tuple c of the box; strides in complex128 elements. With `canon` set, elements
// whose two parts are both zero are written as (+0, +0) (remap.hpp:69-70 skips
// them and the destination starts zeroed, remap.hpp:125-127).
struct CopyBox {
  std::vector<Dim> dims, in_stride, out_stride;
};

void strided_copy(const void* in, void* out, const CopyBox& box, bool canon, cudaStream_t st);

// Box of a row-major permutation: out = permute(in over dims, perm[new] = old).
CopyBox permute_box(const std::vector<Dim>& dims, const std::vector<int>& perm);

// Elementwise y = alpha * conj?(x) over n complex numbers.
void scale_conj(const void* in, void* out, Dim n, double re, double im, bool conj, cudaStream_t st);
// out[i] = in[i] * f_dev[(i / inner) % dim] (real factors, device array of dim)
void scale_index(const void* in, void* out, Dim n, Dim inner, Dim dim, const double* f_dev, cudaStream_t st);
void fill_zero(void* out, Dim n, cudaStream_t st);
// Dense materialisation of an identity / swap tensor's local block (1 where every
// pairing eq_in[k] == eq_out[k] holds on the global coordinates).
void fill_paired(void* out, Dim nl, Dim block, const std::vector<Dim>& dims, int split, const std::vector<int>& eq_in,
                 const std::vector<int>& eq_out, cudaStream_t st);

// In-place exchange of two equally shaped strided regions (elements [begin, end)
// of the row-major enumeration of `dims`): a[off] <-> b[off], zero canonicalised.
// a and b may live on different devices (NVLink peer pointers). keep_a / keep_b
// (optional) are canonicalised in place at the same offsets.
void swap_regions(void* a, void* b, const std::vector<Dim>& dims, const std::vector<Dim>& strides, Dim begin,
                  Dim end, cudaStream_t st, void* keep_a = nullptr, void* keep_b = nullptr);
// Zero canonicalisation of a strided region in place (writes only non-canonical zeros).
void canon_region(void* p, const std::vector<Dim>& dims, const std::vector<Dim>& strides, cudaStream_t st);

}  // namespace qtnhb
