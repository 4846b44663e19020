"""ctypes loader for libsfg.so (the B200 engine's C ABI, include/sfg.h).

The product path has no CPU fallback: if the shared library is missing or no
B200 is present, the calls below raise.  ``build()`` compiles the library
in-tree (paper_2602_16760_b200/libsfg.so) with nvcc for sm_100a.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.path.join(PKG, "libsfg.so")
HEADER = os.path.join(ROOT, "include", "sfg.h")
CSRC = os.path.join(PKG, "csrc")

KINDS = ["ok", "config", "input", "protocol", "transport", "capacity", "session", "numeric",
         "training", "decomposition", "internal"]


class SplitError(RuntimeError):
    """Mirror of splitf::SplitError: ``str(e)`` is "<category>: <message>"."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = KINDS[code] if 0 <= code < len(KINDS) else "internal"


def build(jobs: int = 8) -> str:
    subprocess.run(["make", "-s", "-C", CSRC, f"-j{jobs}"], check=True)
    return LIB_PATH


class ModelConfig(C.Structure):
    """splitf::ModelConfig (tinyformer.hpp:15-33)."""
    _fields_ = [(n, C.c_int32) for n in ("vocab_size", "n_layers", "hidden_dim", "n_heads", "n_kv_heads",
                                          "head_dim", "ffn_dim", "max_seq_len")] + [
        ("rope_base", C.c_float), ("rms_eps", C.c_float), ("seed", C.c_uint64)]


class EngineOptions(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("device", "math", "weight_dtype", "layer_begin", "layer_end",
                                          "with_embedding", "with_head", "extended_shapes")]


class ServerConfig(C.Structure):
    _fields_ = [("layer_begin", C.c_int32), ("layer_end", C.c_int32), ("session_expiry_s", C.c_double),
                ("max_sessions", C.c_int32), ("response_dtype", C.c_int32)]


class ClientConfig(C.Structure):
    _fields_ = [("prefix_layers", C.c_int32), ("suffix_layers", C.c_int32), ("wire_dtype", C.c_int32),
                ("one_way_delay_ms", C.c_double)]


class DecodeConfig(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("mode", "window_w", "ngram_n", "max_candidates_g", "pool_capacity")]


class DecodeStats(C.Structure):
    _fields_ = [("steps", C.c_int32), ("tokens_committed", C.c_int32), ("wall_seconds", C.c_double),
                ("match_rate", C.c_double), ("clamped", C.c_uint64)]


class StepProfile(C.Structure):
    _fields_ = [("step_ms", C.c_double), ("server_ms", C.c_double), ("local_ms", C.c_double),
                ("launches", C.c_int32), ("batch", C.c_int32)]


FRAME_HANDLER = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_uint8), C.c_size_t,
                            C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.c_size_t))

_lib = None


def declared_symbols() -> list[str]:
    """Every function name declared in include/sfg.h."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sfg_[a-z0-9_]+)\s*\(", src)) - {"sfg_frame_handler"})


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(f"{LIB_PATH} not built — run paper_2602_16760_b200._lib.build() "
                                "(the B200 engine has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i32p, f32p = C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_float)
    sig = {
        "sfg_last_error": (C.c_char_p, []),
        "sfg_version": (C.c_char_p, []),
        "sfg_engine_create_seeded": (i32, [C.POINTER(ModelConfig), C.POINTER(EngineOptions), C.POINTER(vp)]),
        "sfg_engine_create_from_params": (i32, [C.POINTER(ModelConfig), C.POINTER(EngineOptions), f32p,
                                                C.POINTER(vp)]),
        "sfg_engine_destroy": (None, [vp]),
        "sfg_tp_unique_id": (i32, [C.POINTER(C.c_uint8)]),
        "sfg_engine_create_tp": (i32, [C.POINTER(ModelConfig), C.POINTER(EngineOptions), i32, i32,
                                       C.POINTER(C.c_uint8), C.POINTER(vp)]),
        "sfg_engine_weight_bytes": (C.c_int64, [vp]),
        "sfg_bank_create": (i32, [vp, i32, i32, C.POINTER(vp)]),
        "sfg_bank_destroy": (None, [vp]),
        "sfg_bank_resolve": (i32, [vp, i32p, i32]),
        "sfg_bank_crop": (i32, [vp, i32]),
        "sfg_bank_mark_committed": (None, [vp, i32]),
        "sfg_bank_reset": (None, [vp]),
        "sfg_bank_state": (None, [vp, i32p, i32p]),
        "sfg_bank_read_kv": (i32, [vp, i32, i32, i32, f32p, f32p]),
        "sfg_forward_layers": (i32, [vp, vp, i32, i32, i32, f32p, i32p, f32p, f32p]),
        "sfg_embed_at": (i32, [vp, i32, i32p, i32p, f32p]),
        "sfg_finalize": (i32, [vp, i32, f32p, f32p]),
        "sfg_finalize_argmax": (i32, [vp, i32, f32p, i32p]),
        "sfg_server_create": (i32, [vp, C.POINTER(ServerConfig), C.POINTER(vp)]),
        "sfg_server_destroy": (None, [vp]),
        "sfg_server_handle": (i32, [vp, C.POINTER(C.c_uint8), C.c_size_t, C.POINTER(C.POINTER(C.c_uint8)),
                                    C.POINTER(C.c_size_t)]),
        "sfg_server_handle_batch": (i32, [vp, i32, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                                          C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.c_size_t)]),
        "sfg_server_shared_passes": (C.c_uint64, [vp]),
        "sfg_server_expire_sessions": (C.c_size_t, [vp]),
        "sfg_server_session_count": (C.c_size_t, [vp]),
        "sfg_server_session_view": (i32, [vp, C.c_char_p, i32p, i32p, i32p]),
        "sfg_server_set_clock": (None, [vp, C.CFUNCTYPE(C.c_double, C.c_void_p), vp]),
        "sfg_router_create": (i32, [C.POINTER(vp), i32, C.c_double, C.POINTER(vp)]),
        "sfg_router_create_handlers": (i32, [C.POINTER(vp), C.POINTER(vp), i32, C.c_double, C.POINTER(vp)]),
        "sfg_router_destroy": (None, [vp]),
        "sfg_router_handle": (i32, [vp, C.POINTER(C.c_uint8), C.c_size_t, C.POINTER(C.POINTER(C.c_uint8)),
                                    C.POINTER(C.c_size_t)]),
        "sfg_router_session_device": (i32, [vp, C.c_char_p]),
        "sfg_router_load": (i32, [vp, i32p]),
        "sfg_router_set_clock": (None, [vp, C.CFUNCTYPE(C.c_double, C.c_void_p), vp]),
        "sfg_batcher_create": (i32, [vp, i32, C.POINTER(vp)]),
        "sfg_batcher_destroy": (None, [vp]),
        "sfg_batcher_handle": (i32, [vp, C.POINTER(C.c_uint8), C.c_size_t, C.POINTER(C.POINTER(C.c_uint8)),
                                     C.POINTER(C.c_size_t)]),
        "sfg_batcher_stats": (None, [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "sfg_client_create": (i32, [vp, C.POINTER(ClientConfig), vp, vp, C.c_char_p, C.POINTER(vp)]),
        "sfg_client_create_linked": (i32, [vp, C.POINTER(ClientConfig), vp, C.c_char_p, C.POINTER(vp)]),
        "sfg_client_destroy": (None, [vp]),
        "sfg_client_prefill": (i32, [vp, i32p, i32, i32p, f32p]),
        "sfg_client_decode_step": (i32, [vp, i32, i32p, i32p, f32p, i32p, i32, i32, f32p, i32p]),
        "sfg_decode": (i32, [vp, C.POINTER(DecodeConfig), vp, i32p, i32, i32, i32p, f32p, i32p, i32p,
                             C.POINTER(DecodeStats)]),
        "sfg_decoder_create": (i32, [vp, C.POINTER(DecodeConfig), vp, i32p, i32, i32, C.POINTER(vp)]),
        "sfg_decoder_step": (i32, [vp, i32p, i32p, i32p]),
        "sfg_decoder_done": (i32, [vp]),
        "sfg_decoder_destroy": (None, [vp]),
        "sfg_pool_create": (i32, [i32, C.c_size_t, C.POINTER(vp)]),
        "sfg_pool_destroy": (None, [vp]),
        "sfg_pool_update": (i32, [vp, i32p, i32p, i32]),
        "sfg_pool_lookup": (i32, [vp, i32, i32, i32p]),
        "sfg_pool_size": (C.c_size_t, [vp]),
        "sfg_f32_to_f16": (C.c_uint16, [C.c_float, C.POINTER(C.c_uint64)]),
        "sfg_f16_to_f32": (C.c_float, [C.c_uint16]),
        "sfg_selftest_wire_roundtrip": (i32, [f32p, f32p, i32, C.POINTER(C.c_uint64)]),
        "sfg_client_last_profile": (i32, [vp, C.POINTER(StepProfile)]),
        "sfg_set_graphs": (None, [i32]),
        "sfg_copy_bytes": (None, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "sfg_profiler_enable": (None, [i32]),
        "sfg_debug_mask_runs": (i32, [C.POINTER(C.c_uint16), i32, i32, i32p, i32p, i32p, i32, i32p, i32p]),
        "sfg_debug_set_mega": (None, [i32]),
        "sfg_debug_mega_trace": (None, [i32]),
        "sfg_debug_mega_trace_read": (i32, [vp, C.POINTER(C.c_uint64), C.c_size_t]),
        "sfg_debug_bank_buffer": (i32, [vp, i32, f32p, i32]),
        "sfg_profiler_reset": (None, []),
        "sfg_profiler_stats": (i32, [i32, C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int):
    if rc != 0:
        raise SplitError(rc, lib().sfg_last_error().decode())
