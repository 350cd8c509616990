"""ctypes binding of the C-ABI (include/egt_b200.h) -> _lib/libegt_b200.so.

The library is built in-tree by paper_2605_11582_b200._build (nvcc,
sm_100a).  There is no fallback: if the shared object is missing the import
fails with the build command to run.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EGT_LIB_PATH") or os.path.join(_HERE, "_lib", "libegt_b200.so")

EGT_OK, EGT_EINVAL, EGT_EFORMAT, EGT_EINTERNAL, EGT_ECUDA = range(5)
KIND_F32, KIND_INT4 = 0, 1
FMT_NAMES = {0: "int4-2:4", 1: "int4-1:4", 2: "int4-dense", 3: "fp16-2:4", 4: "fp16-1:4"}
PATH_NAMES = {0: "tiled-mma.sp", 1: "general"}

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
szp = C.POINTER(C.c_size_t)


class PackedView(C.Structure):
    """egt_packed_view (PackedSparseMatrix, packed.hpp:37-67)."""

    _fields_ = [
        ("n", C.c_uint8), ("m", C.c_uint8), ("rows", C.c_uint32), ("cols", C.c_uint32),
        ("kind", C.c_uint8),
        ("index_words", u16p), ("n_index_words", C.c_size_t),
        ("value_bytes", u8p), ("n_value_bytes", C.c_size_t),
        ("group_sizes", u32p), ("n_group_sizes", C.c_size_t),
        ("group_offsets", u32p), ("n_group_offsets", C.c_size_t),
        ("scales", f32p), ("n_scales", C.c_size_t),
        ("zero_points", u8p), ("n_zero_points", C.c_size_t),
        ("values", f32p), ("n_values", C.c_size_t),
    ]


class QuantView(C.Structure):
    """egt_quant_view (QuantizedMatrix with every position kept)."""

    _fields_ = [
        ("rows", C.c_uint32), ("cols", C.c_uint32),
        ("group_sizes", u32p), ("group_offsets", u32p),
        ("scales", f32p), ("n_scales", C.c_size_t),
        ("zero_points", u8p),
        ("codes", u8p), ("n_codes", C.c_size_t),
    ]


class DevInfo(C.Structure):
    _fields_ = [
        ("rows", C.c_uint32), ("cols", C.c_uint32),
        ("n", C.c_uint8), ("m", C.c_uint8), ("kind", C.c_uint8), ("format", C.c_uint8),
        ("path", C.c_uint8),
        ("device_bytes", C.c_uint64), ("algorithmic_bytes", C.c_uint64), ("nnz", C.c_uint64),
    ]


class ModelConfig(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_ff", "max_positions")]


class TrieView(C.Structure):
    _fields_ = [("n_nodes", C.c_uint32), ("token", u32p), ("parent", u32p),
                ("payload", C.POINTER(C.c_int64))]


class SessionView(C.Structure):
    _fields_ = [("prompt", C.POINTER(C.c_int32)), ("prompt_len", C.c_uint32), ("n_beams", C.c_uint32),
                ("beam_node", u32p), ("beam_log_prob", f64p), ("beam_len", u32p),
                ("beam_tokens", C.POINTER(C.c_int32))]


class VerifyOut(C.Structure):
    _fields_ = [("n_selected", C.c_uint32), ("score", f64p), ("payload", C.POINTER(C.c_int64)),
                ("beam", u32p), ("len", u32p), ("tokens", C.POINTER(C.c_int32)),
                ("tokens_stride", C.c_uint32), ("flattened_nodes", C.c_uint32), ("rows", C.c_uint32)]


class DecodeOptions(C.Structure):
    _fields_ = [("beam_size", C.c_int), ("mode", C.c_int), ("forced_depth", C.c_int), ("t_step", C.c_double),
                ("alpha", C.c_double), ("beta", C.c_double), ("node_cap", C.c_uint64), ("kv_cache", C.c_int)]


INPUT_NONE, INPUT_RMSNORM, INPUT_SILU = 0, 1, 2
UPLOAD_ROUND_FP16 = 1  # egt_dev_packed_create_ex flag


class EgtqLayerInfo(C.Structure):
    _fields_ = [("name", C.c_char_p), ("pattern", C.c_uint8), ("has_quant", C.c_uint8), ("has_index", C.c_uint8),
                ("rows", C.c_uint32), ("cols", C.c_uint32)]

# every symbol include/egt_b200.h declares, with its signature
SIGNATURES = {
    "egt_abi_version": (C.c_int, []),
    "egt_last_error": (C.c_char_p, []),
    "egt_dev_packed_create": (C.c_int, [C.POINTER(PackedView), C.c_void_p, C.POINTER(C.c_void_p)]),
    "egt_dev_packed_create_ex": (C.c_int, [C.POINTER(PackedView), C.c_uint32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "egt_dev_dense_i4_create": (C.c_int, [C.POINTER(QuantView), C.c_void_p, C.POINTER(C.c_void_p)]),
    "egt_dev_packed_slice_rows": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    "egt_dev_packed_destroy": (C.c_int, [C.c_void_p]),
    "egt_dev_packed_query": (C.c_int, [C.c_void_p, C.POINTER(DevInfo)]),
    "egt_spmv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]),
    "egt_spmv_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                              C.c_void_p]),
    "egt_spmv_fused": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.c_void_p, C.c_uint32, C.c_uint32, C.c_float, C.c_uint32, C.c_void_p,
                                 C.c_void_p]),
    "egt_spmv_fused_multi": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, C.c_void_p, C.POINTER(C.c_void_p),
                                       C.c_uint32, C.c_float, C.c_uint32, C.c_void_p]),
    "egt_spmm_multi": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, C.c_void_p, C.c_uint32, C.c_uint32,
                                 C.POINTER(C.c_void_p), C.c_uint32, C.c_uint32, C.c_float, C.c_void_p]),
    "egt_spmv_host": (C.c_int, [C.c_void_p, f32p, C.c_size_t, f32p, C.c_void_p]),
    "egt_dequant": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "egt_set_pdl": (None, [C.c_int]),
    "egt_launch_count": (C.c_uint64, []),
    "egt_tune_force_plan": (None, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "egt_tune_read_trace": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_size_t, C.c_int]),
    "egt_host_fit_group": (None, [f64p, C.c_size_t, f32p, u8p]),
    "egt_host_group_count": (C.c_size_t, [C.c_uint32, C.c_uint32, u32p]),
    "egt_host_quantize": (C.c_int, [f32p, C.c_uint32, C.c_uint32, u32p, u8p, u32p, f32p, u8p, u8p, szp]),
    "egt_host_pack_int4": (C.c_int, [u8p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, u8p, C.c_size_t, C.c_int,
                                     u16p, szp, u8p, szp]),
    "egt_host_pack_f32": (C.c_int, [u8p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, f32p, u16p, szp, f32p, szp]),
    "egt_host_footprint": (C.c_int, [C.POINTER(PackedView), u64p, f64p]),
}

_MODEL_SIGNATURES = {
    "egt_model_create": (C.c_int, [C.POINTER(ModelConfig), f32p, C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p,
                                   C.POINTER(C.c_void_p)]),
    "egt_model_destroy": (C.c_int, [C.c_void_p]),
    "egt_model_query": (C.c_int, [C.c_void_p, C.POINTER(ModelConfig)]),
    "egt_forward": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), u8p, C.c_uint32,
                              C.c_void_p, C.c_void_p]),
    "egt_gather": (C.c_int, [C.c_void_p, C.c_uint64, u32p, u32p, C.c_uint32, f32p, C.c_void_p]),
    "egt_verify_parallel": (C.c_int, [C.c_void_p, C.POINTER(TrieView), C.POINTER(SessionView), C.c_int,
                                      C.POINTER(VerifyOut), C.c_void_p]),
    "egt_decode": (C.c_int, [C.c_void_p, C.POINTER(TrieView), C.POINTER(C.c_int32), C.c_uint32,
                             C.POINTER(DecodeOptions), C.POINTER(VerifyOut), C.POINTER(C.c_int32), C.c_void_p]),
    "egt_kv_pool_create": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "egt_kv_pool_destroy": (C.c_int, [C.c_void_p]),
    "egt_forward_kv": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_uint32,
                                 C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_uint32), C.c_void_p, C.c_void_p]),
}


class TreeView(C.Structure):
    _fields_ = [("n_beams", C.c_uint32), ("padded_len", C.c_uint32), ("committed_len", u32p),
                ("n_nodes", C.c_uint32), ("parent", C.POINTER(C.c_int32)), ("beam", u32p)]


_MODEL_SIGNATURES["egt_forward_tree"] = (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                                   C.POINTER(TreeView), C.c_void_p, C.c_void_p])

_PLANNING_SIGNATURES = {
    "egt_host_plan_sparsity": (C.c_int, [C.c_uint32, u32p, u32p, C.POINTER(f32p), C.POINTER(f32p), C.c_double, u8p]),
    "egt_cost_estimator_create": (C.c_int, [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_void_p)]),
    "egt_cost_estimator_observe_step": (C.c_int, [C.c_void_p, C.c_double]),
    "egt_cost_estimator_observe_verify": (C.c_int, [C.c_void_p, C.c_uint64, C.c_double]),
    "egt_cost_estimator_model": (C.c_int, [C.c_void_p, f64p]),
    "egt_cost_estimator_destroy": (C.c_int, [C.c_void_p]),
    "egt_measure_cost_model": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, u32p, C.c_uint32, C.c_int, C.c_void_p,
                                         C.c_void_p]),
    "egt_host_estimate_trigger": (C.c_int, [C.POINTER(TrieView), C.POINTER(SessionView), C.c_double, C.c_double,
                                            C.c_double, C.c_uint64, C.POINTER(C.c_int), f64p]),
    "egt_host_tree_mask": (C.c_int, [C.POINTER(TrieView), C.POINTER(SessionView), C.c_uint32, u32p, u32p,
                                     C.POINTER(C.c_int32), u32p, u32p, u32p, C.c_uint32, u32p, C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32), u8p, C.c_size_t, u32p, u32p]),
}

_MODEL_SIGNATURES.update({
    "egt_decoder_create": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "egt_decoder_start": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_uint32, C.c_void_p]),
    "egt_decoder_step": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "egt_decoder_read": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_uint32, u32p, C.c_void_p, C.c_void_p]),
    "egt_decoder_destroy": (C.c_int, [C.c_void_p]),
})

_MODEL_SIGNATURES.update({
    "egt_egtq_parse": (C.c_int, [u8p, C.c_size_t, C.c_char_p, C.POINTER(C.c_void_p)]),
    "egt_egtq_layer_count": (C.c_uint32, [C.c_void_p]),
    "egt_egtq_query": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(EgtqLayerInfo)]),
    "egt_egtq_upload": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "egt_egtq_upload_ex": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "egt_egtq_destroy": (C.c_int, [C.c_void_p]),
})



class IpcHandle(C.Structure):
    _fields_ = [("bytes", C.c_uint8 * 64)]


PEER_NOWAIT = 4
PEER_CTRL_BYTES = 512
MAX_PEERS = 8

_PEER_SIGNATURES = {
    "egt_peer_buffer_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p), C.POINTER(IpcHandle)]),
    "egt_peer_buffer_free": (C.c_int, [C.c_void_p]),
    "egt_peer_buffer_open": (C.c_int, [C.POINTER(IpcHandle), C.POINTER(C.c_void_p)]),
    "egt_peer_buffer_close": (C.c_int, [C.c_void_p]),
    "egt_peer_group_create": (C.c_int, [C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "egt_peer_group_destroy": (C.c_int, [C.c_void_p]),
    "egt_peer_group_y": (C.c_void_p, [C.c_void_p]),
    "egt_spmv_allgather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.c_void_p]),
    "egt_peer_wait": (C.c_int, [C.c_void_p, C.c_void_p]),
    "egt_peer_group_check": (C.c_int, [C.c_void_p]),
}

class GpuPackedOut(C.Structure):
    _fields_ = [("index_words", C.c_void_p), ("value_bytes", C.c_void_p), ("group_offsets", C.c_void_p),
                ("scales", C.c_void_p), ("zero_points", C.c_void_p)]


_COMPRESS_SIGNATURES = {
    "egt_gpu_importance": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                     C.c_void_p]),
    "egt_gpu_prune_nm": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "egt_gpu_quantize_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int, u32p,
                                        C.POINTER(GpuPackedOut), C.c_void_p, C.POINTER(C.c_void_p)]),
}

SIGNATURES.update(_MODEL_SIGNATURES)
SIGNATURES.update(_COMPRESS_SIGNATURES)
SIGNATURES["egt_gemv_f32"] = (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p])
SIGNATURES["egt_bench_spmv"] = (C.c_int, [u32p, u32p, C.c_uint32, C.c_int, C.c_uint64, C.c_char_p, C.c_size_t,
                                          C.POINTER(C.c_size_t)])
SIGNATURES.update(_PEER_SIGNATURES)
SIGNATURES.update(_PLANNING_SIGNATURES)

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2605_11582_b200._build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            try:
                fn = getattr(L, name)
            except AttributeError:
                if "EGT_LIB_PATH" in os.environ:  # tuning: an older build under test
                    continue
                raise
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class EgtError(Exception):
    """Maps egt_status onto the reference's exception classes."""

    KIND = {EGT_EINVAL: "invalid_argument", EGT_EFORMAT: "FormatError",
            EGT_EINTERNAL: "InvariantError", EGT_ECUDA: "CudaError"}

    def __init__(self, status: int, msg: str):
        self.status = status
        self.kind = self.KIND.get(status, "unknown")
        super().__init__(f"{self.kind}: {msg}")


class InvalidArgument(EgtError, ValueError):
    pass


class FormatError(EgtError):
    pass


def check(status: int) -> None:
    if status != EGT_OK:
        msg = lib().egt_last_error().decode(errors="replace")
        if status == EGT_EINVAL:
            raise InvalidArgument(status, msg)
        if status == EGT_EFORMAT:
            raise FormatError(status, msg)
        raise EgtError(status, msg)
