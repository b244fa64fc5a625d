"""ctypes binding of libmspq.so (include/mspq_capi.h).  No fallback: if the CUDA library is
missing the import of anything that needs it raises."""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmspq.so")

_lib = None

c_int, c_ll, c_ull, c_float, c_double, c_void_p, c_char_p = (
    ctypes.c_int, ctypes.c_longlong, ctypes.c_ulonglong, ctypes.c_float, ctypes.c_double,
    ctypes.c_void_p, ctypes.c_char_p)


class ModelDesc(ctypes.Structure):
    _fields_ = [("L", c_int), ("E", c_int), ("K", c_int), ("d", c_int), ("f", c_int),
                ("V", c_int), ("P", c_int), ("seed", c_ull), ("embed_scale", c_float),
                ("pos_scale", c_float), ("a_router", c_float), ("a_up", c_float),
                ("a_down", c_float), ("a_lm", c_float), ("eps", c_float),
                ("unique_experts", c_int), ("H", c_int), ("Hkv", c_int), ("Dh", c_int),
                ("a_qkv", c_float), ("a_o", c_float)]


class EngineOpts(ctypes.Structure):
    _fields_ = [("device", c_int), ("kmax", c_int), ("host_store_path", c_char_p),
                ("host_store_role", c_int), ("slot_extra", c_int), ("log_cap", c_int),
                ("trace_level", c_int), ("expert_codec", c_int), ("max_streams", c_int)]


# (name, restype, argtypes)
_SIGS = [
    ("mspq_status_string", c_char_p, [c_int]),
    ("mspq_last_error", c_char_p, []),
    ("mspq_free", None, [c_void_p]),
    ("mspq_version", c_int, []),
    ("mspq_fill_bf16", c_int, [c_ull, c_ull, c_float, c_int, c_void_p, c_ll, c_ll, c_void_p]),
    ("mspq_fill_expert", c_int, [c_ull, c_int, c_int, c_int, c_int, c_float, c_float, c_void_p, c_void_p]),
    ("mspq_quantize_int4", c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    ("mspq_embed", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p]),
    ("mspq_gate_topk", c_int, [c_void_p] * 4 + [c_int, c_ll] + [c_void_p] * 10 + [c_int] * 6 + [c_float, c_void_p]),
    ("mspq_build_schedule", c_int, [c_void_p, c_int, c_int, c_int] + [c_void_p] * 9),
    ("mspq_moe_bf16_tc_ws_bytes", c_ll, [c_int] * 6),
    ("mspq_moe_bf16_tc", c_int, [c_void_p] * 8 + [c_ll] + [c_int] * 7 + [c_void_p] * 3),
    ("mspq_moe_bf16_tc_part", c_int, [c_void_p] * 8 + [c_ll] + [c_int] * 7 + [c_void_p] * 3 + [c_int, c_void_p]),
    ("mspq_tile_bf16", c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p]),
    ("mspq_dense_ws_bytes", c_ll, [c_int, c_int]),
    ("mspq_dense_sched_fill", c_int, [c_void_p, c_int]),
    ("mspq_dense_bf16_tc", c_int, [c_void_p] * 3 + [c_int] * 4 + [c_void_p, c_void_p, c_ll, c_void_p]),
    ("mspq_attention_ws_bytes", c_ll, [c_int] * 4),
    ("mspq_attention_batched", c_int, [c_void_p, c_int, c_ll] + [c_int] * 5 + [c_void_p, c_ll] + [c_void_p] * 5),
    ("mspq_attention", c_int, [c_void_p, c_int, c_ll] + [c_int] * 5 + [c_void_p] * 7),
    ("mspq_gate_topk_img", c_int, [c_void_p] * 4 + [c_int, c_ll] + [c_void_p] * 10 + [c_int] * 6 + [c_float, c_void_p, c_void_p]),
    ("mspq_debug_gemv_variant", c_int, [c_int]),
    ("mspq_fragtile_int4", c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p]),
    ("mspq_moe_int4_gemv", c_int, [c_void_p] * 4 + [c_ll] + [c_int] * 6 + [c_void_p] * 3),
    ("mspq_moe_int4_tc", c_int, [c_void_p] * 8 + [c_ll] + [c_int] * 9 + [c_void_p] * 3),
    ("mspq_tile_int4", c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    ("mspq_debug_timeline", c_int, [c_void_p, c_int]),
    ("mspq_lm_head", c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p]),
    ("mspq_argmax", c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p]),
    ("mspq_argmax_advance", c_int, [c_void_p, c_int] + [c_void_p] * 6),
    ("mspq_accept_scan", c_int, [c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    ("mspq_accept_advance", c_int, [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    ("mspq_xc_max_blob_bytes", c_ll, [c_ll]),
    ("mspq_xc_scratch_bytes", c_ll, [c_ll]),
    ("mspq_xc_encode", c_int, [c_void_p, c_ll, c_void_p, c_void_p, c_ll, ctypes.POINTER(c_ll), c_void_p]),
    ("mspq_xc_decode", c_int, [c_void_p, c_int, c_int, c_void_p, c_int, c_void_p]),
    ("mspq_int4_blob_bytes", c_ll, [c_int, c_int]),
    ("mspq_bf16_blob_bytes", c_ll, [c_int, c_int]),
    ("mspq_cache_create", c_int, [c_int] * 6 + [c_void_p]),
    ("mspq_cache_destroy", c_int, [c_void_p]),
    ("mspq_cache_configure", c_int, [c_void_p, c_int, c_int, c_void_p, c_int, c_int, c_double, c_double, c_void_p]),
    ("mspq_cache_view_get", c_int, [c_void_p, c_void_p]),
    ("mspq_cache_set_staging", c_int, [c_void_p, c_int]),
    ("mspq_cache_begin_cycle", c_int, [c_void_p, c_int, c_void_p]),
    ("mspq_cache_plan_row", c_int, [c_void_p, c_int, c_void_p]),
    ("mspq_cache_verify_layer", c_int, [c_void_p, c_int, c_int] + [c_void_p] * 3),
    ("mspq_cache_replay_cycle", c_int, [c_void_p] * 4 + [c_int] * 3 + [c_void_p] * 7),
    ("mspq_cache_replay_all", c_int, [c_void_p] * 5 + [c_int, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_int]
     + [c_void_p] * 5),
    ("mspq_replay", c_int, [c_int, c_char_p, c_char_p, ctypes.POINTER(c_void_p)]),
    ("mspq_governor", c_int, [c_char_p, ctypes.POINTER(c_void_p)]),
    ("mspq_compare_policies", c_int, [c_int, c_char_p, c_char_p, c_char_p, c_char_p, ctypes.POINTER(c_void_p)]),
    ("mspq_sweep_k", c_int, [c_int, c_char_p, c_char_p, c_char_p, ctypes.POINTER(c_void_p)]),
    ("mspq_engine_create", c_int, [ctypes.POINTER(ModelDesc), ctypes.POINTER(EngineOpts), ctypes.POINTER(c_void_p)]),
    ("mspq_engine_destroy", c_int, [c_void_p]),
    ("mspq_engine_configure", c_int, [c_void_p, c_char_p]),
    ("mspq_generate", c_int, [c_void_p, c_void_p, c_int, c_int, ctypes.POINTER(c_void_p)]),
    ("mspq_generate_batch", c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, ctypes.POINTER(c_void_p)]),
    ("mspq_engine_info", c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    ("mspq_engine_read", c_int, [c_void_p, c_char_p, c_void_p, c_ll]),
    ("mspq_engine_home_create", c_int, [c_void_p, c_int, c_int, c_void_p]),
    ("mspq_engine_peer_attach_ipc", c_int, [c_void_p, c_int, c_void_p]),
    ("mspq_engine_peer_attach", c_int, [c_void_p, c_int, c_void_p]),
]

EXPORTS = [s[0] for s in _SIGS]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libmspq.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class CacheView(ctypes.Structure):
    _fields_ = [("elb_ids", c_void_p), ("elb_gates", c_void_p), ("scal", c_void_p), ("req", c_void_p),
                ("log", c_void_p), ("plan", c_void_p), ("cov", c_void_p), ("step", c_void_p),
                ("res", c_void_p), ("host_stat", ctypes.POINTER(ctypes.c_int32)),
                ("host_req", ctypes.POINTER(ctypes.c_int32)), ("host_sched", ctypes.POINTER(ctypes.c_int32)),
                ("req_cap", c_int), ("log_cap", c_int), ("plan_cap", c_int), ("nbuf", c_int)]


class MspqError(RuntimeError):
    """moespeq::Error analogue: .code = status (ErrorCode ordinal + 1, or 1000+)."""

    def __init__(self, code, msg):
        super().__init__(f"{lib().mspq_status_string(code).decode()}: {msg}")
        self.code = code
        self.name = lib().mspq_status_string(code).decode()


def check(status):
    if status != 0:
        raise MspqError(status, lib().mspq_last_error().decode())


def take_string(ptr) -> str:
    s = ctypes.cast(ptr, c_char_p).value.decode()
    lib().mspq_free(ptr)
    return s
