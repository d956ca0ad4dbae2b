"""ctypes binding of libqtnh_b200.so (C ABI in include/qtnh_b200.h).

The product path has no fallback: if the shared library is missing or fails to
load, importing the package raises. Build it with ``__graft_entry__.build()``
(or ``make -C paper_2505_06119_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqtnh_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()')")

lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

i32, i64, f64, vp, sz = C.c_int, C.c_int64, C.c_double, C.c_void_p, C.c_size_t
P_i32 = C.POINTER(C.c_int)
P_i64 = C.POINTER(C.c_int64)
P_f64 = C.POINTER(C.c_double)

# name: (restype, argtypes)
_SIGS = {
    "qtnh_last_error": (i32, [C.c_char_p, sz]),
    "qtnh_last_error_info": (i64, []),
    "qtnh_version": (C.c_char_p, []),
    "qtnh_kernel_launch_count": (i64, []),
    "qtnh_set_option": (i32, [C.c_char_p, f64]),
    "qtnh_world_create_local": (i32, [i32, P_i32, C.POINTER(vp)]),
    "qtnh_nccl_unique_id": (i32, [vp]),
    "qtnh_world_create_nccl": (i32, [i32, i32, i32, vp, C.POINTER(vp)]),
    "qtnh_world_create_ipc": (i32, [i32, i32, i32, C.c_char_p, C.POINTER(vp)]),
    "qtnh_world_destroy": (i32, [vp]),
    "qtnh_world_size": (i32, [vp]),
    "qtnh_world_abort": (i32, [vp]),
    "qtnh_rank_bind": (i32, [vp, i32, C.POINTER(vp)]),
    "qtnh_rank_release": (i32, [vp]),
    "qtnh_rank_id": (i32, [vp]),
    "qtnh_rank_set_stream": (i32, [vp, vp]),
    "qtnh_rank_reset_stream": (i32, [vp]),
    "qtnh_rank_stream": (vp, [vp]),
    "qtnh_rank_capture_begin": (i32, [vp]),
    "qtnh_rank_capture_end": (i32, [vp, C.POINTER(vp)]),
    "qtnh_graph_launch": (i32, [vp, vp]),
    "qtnh_graph_destroy": (i32, [vp]),
    "qtnh_rank_synchronize": (i32, [vp]),
    "qtnh_barrier": (i32, [vp]),
    "qtnh_all_to_all_v": (i32, [vp, i32, P_i32, vp, P_i64, P_i64, vp, P_i64, P_i64]),
    "qtnh_tensor_dense": (i32, [vp, i32, P_i64, i32, P_i64, vp, C.POINTER(vp)]),
    "qtnh_tensor_from_global": (i32, [vp, i32, P_i64, i32, P_i64, vp, C.POINTER(vp)]),
    "qtnh_tensor_from_device": (i32, [vp, i32, P_i64, i32, P_i64, vp, C.POINTER(vp)]),
    "qtnh_tensor_retain": (i32, [vp]),
    "qtnh_tensor_free": (i32, [vp]),
    "qtnh_tensor_rank": (i32, [vp]),
    "qtnh_tensor_dims": (i32, [vp, P_i64]),
    "qtnh_tensor_split": (i32, [vp]),
    "qtnh_tensor_dist": (i32, [vp, P_i64]),
    "qtnh_tensor_local_size": (i64, [vp]),
    "qtnh_tensor_span": (i64, [vp]),
    "qtnh_tensor_in_span": (i32, [vp]),
    "qtnh_tensor_my_block": (i64, [vp]),
    "qtnh_tensor_is_canonical": (i32, [vp]),
    "qtnh_tensor_device_ptr": (vp, [vp]),
    "qtnh_tensor_download_local": (i32, [vp, vp]),
    "qtnh_tensor_download_local_async": (i32, [vp, vp]),
    "qtnh_tensor_upload_local": (i32, [vp, vp]),
    "qtnh_tensor_to_global": (i32, [vp, vp]),
    "qtnh_tensor_paired": (i32, [vp, i32, P_i64, i32, P_i64, i32, P_i32, P_i32, i32, C.POINTER(vp)]),
    "qtnh_tensor_diagonal": (i32, [vp, i32, P_i64, i32, P_i64, vp, i64, C.POINTER(vp)]),
    "qtnh_tensor_symmetric": (i32, [vp, i32, P_i64, i32, P_i64, vp, i64, i32, C.POINTER(vp)]),
    "qtnh_tensor_variant": (i32, [vp]),
    "qtnh_tensor_stored_size": (i64, [vp]),
    "qtnh_tensor_pairs": (i32, [vp, P_i32, P_i32]),
    "qtnh_tensor_to_dense": (i32, [vp, C.POINTER(vp)]),
    "qtnh_tensor_local_element": (i32, [vp, P_i64, vp]),
    "qtnh_squeeze": (i32, [vp, i32, C.POINTER(vp)]),
    "qtnh_unsqueeze": (i32, [vp, i32, i32, C.POINTER(vp)]),
    "qtnh_gate_apply_tensor": (i32, [vp, i32, P_i32, vp]),
    "qtnh_tensor_save": (i32, [vp, C.c_char_p]),
    "qtnh_tensor_load": (i32, [vp, C.c_char_p, C.POINTER(vp)]),
    "qtnh_permute": (i32, [vp, P_i32, i32, C.POINTER(vp)]),
    "qtnh_rebcast": (i32, [vp, P_i64, C.POINTER(vp)]),
    "qtnh_remap": (i32, [vp, P_i32, i32, P_i64, i32, P_i64, C.POINTER(vp)]),
    "qtnh_scatter_index": (i32, [vp, i32, C.POINTER(vp)]),
    "qtnh_gather_index": (i32, [vp, i32, C.POINTER(vp)]),
    "qtnh_slice_local_dims": (i32, [vp, P_i64, C.POINTER(vp)]),
    "qtnh_pad_local_dims": (i32, [vp, P_i64, C.POINTER(vp)]),
    "qtnh_conj": (i32, [vp, C.POINTER(vp)]),
    "qtnh_scale": (i32, [vp, f64, f64, C.POINTER(vp)]),
    "qtnh_plan_order": (i32, [i32, P_i32, P_i32, i32, vp, C.c_uint64, i32, P_i32]),
    "qtnh_plan_order_capped": (i32, [i32, P_i32, P_i32, i32, vp, C.c_uint64, i32, C.c_double, P_i32]),
    "qtnh_contract_chain": (i32, [i32, C.POINTER(vp), i32, P_i32, P_i32, P_i32, P_i32, C.POINTER(vp)]),
    "qtnh_contract": (i32, [vp, vp, i32, P_i32, P_i32, C.POINTER(vp)]),
    "qtnh_gate_apply": (i32, [vp, i32, P_i32, vp, i32]),
    "qtnh_swap_indices": (i32, [vp, i32, i32]),
    "qtnh_contract_host": (i32, [vp, i32, P_i64, vp, i32, P_i64, vp, i32, P_i32, P_i32, vp, P_i64]),
    "qtnh_qft_layer": (i32, [vp, i32]),
    "qtnh_qft": (i32, [vp, i32]),
    "qtnh_svd_device": (i32, [vp, i64, i64, i64, vp, i64, i32, vp, vp, vp]),
    "qtnh_scale_index": (i32, [vp, i32, vp, C.POINTER(vp)]),
    "qtnh_tensor_clone": (i32, [vp, C.POINTER(vp)]),
    "qtnh_tensor_make_mutable": (i32, [vp]),
    "qtnh_tensor_reshape": (i32, [vp, i32, P_i64, C.POINTER(vp)]),
    "qtnh_group_all_to_all_v_host": (i32, [vp, i32, P_i32, sz, C.POINTER(vp), P_i64, vp, C.POINTER(vp), P_i64]),
    "qtnh_free_host": (None, [vp]),
    "qtnh_svd_split_count": (i64, []),
    "qtnh_mps_apply_layer": (i32, [i32, C.POINTER(vp), C.POINTER(vp), vp, i64, C.POINTER(vp), C.POINTER(vp), vp, vp,
                                   vp]),
    "qtnh_svd": (i32, [vp, i32, P_i32, i32, P_i32, i64, i32, C.POINTER(vp), C.POINTER(vp), vp]),
    "qtnh_zgemm_device": (i32, [vp, i64, i64, i64, vp, vp, vp]),
    "qtnh_permute_device": (i32, [vp, i32, P_i64, P_i32, vp, vp]),
    "qtnh_hash_counter": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]),
    "qtnh_rng_complex_normals": (None, [C.c_uint64, i64, vp]),
    "qtnh_counter_complex_normals": (None, [C.c_uint64, i64, i64, vp, i32]),
    "qtnh_counter_complex_normals_device": (i32, [vp, C.c_uint64, i64, i64, vp]),
    "qtnh_probe_fp64_peak": (i32, [vp, P_f64]),
    "qtnh_remap_plan_json": (i32, [i32, P_i64, i32, P_i64, P_i32, i32, P_i64, i32, i32, C.c_char_p, sz]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)  # AttributeError here = the .so does not export the ABI
    _f.restype = _res
    _f.argtypes = _args


def i64_array(vals):
    vals = list(vals)
    return (C.c_int64 * max(1, len(vals)))(*vals)


def i32_array(vals):
    vals = list(vals)
    return (C.c_int * max(1, len(vals)))(*vals)


def last_error() -> str:
    buf = C.create_string_buffer(4096)
    lib.qtnh_last_error(buf, 4096)
    return buf.value.decode(errors="replace")


def kernel_launches() -> int:
    return int(lib.qtnh_kernel_launch_count())
