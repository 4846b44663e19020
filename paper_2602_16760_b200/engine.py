"""Python mirror of the reference splitf C++ interface for the lookahead hot
path, backed by libsfg.so (include/sfg.h).  Names, argument meaning and
error behaviour follow the reference so the parity tests read like the
reference's own tests:

  tinyformer.hpp  ModelConfig, CacheBank, forward_layers, embed_at, finalize,
                  argmax_row                          -> Engine / CacheBank
  server.hpp      ServerEngine::handle / expire_sessions / session_view
                                                      -> ServerEngine
  client.hpp      SplitClient::prefill / decode_step  -> SplitClient
  decoding.hpp    NGramPool, decode_sequential, decode_lookahead(_with_pool)

Every call goes to the B200 through the C ABI; there is no CPU fallback
(errors surface as ``SplitError`` with the reference's "<category>: <msg>").
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import SplitError, check

_i32p = C.POINTER(C.c_int32)
_f32p = C.POINTER(C.c_float)

EXACT, FAST = 0, 1
F16, F32 = 0, 1


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


@dataclass
class ModelConfig:
    """splitf::ModelConfig (tinyformer.hpp:15-33); defaults are the reference's."""
    vocab_size: int = 256
    n_layers: int = 8
    hidden_dim: int = 64
    n_heads: int = 4
    n_kv_heads: int = 2
    head_dim: int = 16
    ffn_dim: int = 256
    max_seq_len: int = 256
    rope_base: float = 10000.0
    rms_eps: float = 1e-5
    seed: int = 1234

    def to_c(self) -> _lib.ModelConfig:
        return _lib.ModelConfig(self.vocab_size, self.n_layers, self.hidden_dim, self.n_heads, self.n_kv_heads,
                                self.head_dim, self.ffn_dim, self.max_seq_len, self.rope_base, self.rms_eps,
                                self.seed)

    @classmethod
    def from_any(cls, c) -> "ModelConfig":
        return cls(**{k: getattr(c, k) for k in cls.__dataclass_fields__})


def tp_unique_id() -> bytes:
    """A fresh NCCL group id for a tensor-parallel engine group (rank 0 makes
    it and shares it with the other ranks)."""
    buf = (C.c_uint8 * 128)()
    check(_lib.lib().sfg_tp_unique_id(buf))
    return bytes(buf)


class Engine:
    """Weights of a layer range resident on one B200."""

    def __init__(self, cfg, math: int = EXACT, weights: str = "bf16", layers: tuple | None = None,
                 with_embedding: bool = True, with_head: bool = True, device: int = 0,
                 params: np.ndarray | None = None, tp: tuple | None = None, extended_shapes: bool = False):
        """tp = (size, rank, unique_id bytes): this engine is rank `rank` of a
        tensor-parallel group (see tp_unique_id; FAST math, seeded weights).
        extended_shapes: accept q_dim != hidden_dim (NeMo-12B), which the
        reference's validate() rejects (sfg.h sfg_engine_options)."""
        self.cfg = ModelConfig.from_any(cfg)
        L = _lib.lib()
        lb, le = layers if layers is not None else (0, self.cfg.n_layers)
        opt = _lib.EngineOptions(device, math, 0 if weights == "bf16" else 1, lb, le, int(with_embedding),
                                 int(with_head), int(extended_shapes))
        h = C.c_void_p()
        cc = self.cfg.to_c()
        if tp is not None and tp[0] > 1:
            if params is not None:
                raise ValueError("tensor-parallel engines take the seeded weights")
            uid = (C.c_uint8 * 128).from_buffer_copy(bytes(tp[2]))
            check(L.sfg_engine_create_tp(C.byref(cc), C.byref(opt), int(tp[0]), int(tp[1]), uid, C.byref(h)))
        elif params is None:
            check(L.sfg_engine_create_seeded(C.byref(cc), C.byref(opt), C.byref(h)))
        else:
            p = _f32(params)
            check(L.sfg_engine_create_from_params(C.byref(cc), C.byref(opt), _p(p, _f32p), C.byref(h)))
        self.h = h
        self.math = math

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().sfg_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def weight_bytes(self) -> int:
        return int(_lib.lib().sfg_engine_weight_bytes(self.h))

    def bank(self, layer_begin: int, layer_end: int) -> "CacheBank":
        return CacheBank(self, layer_begin, layer_end)

    # forward_layers (tinyformer.hpp:174-176)
    def forward_layers(self, layer_begin, layer_end, hidden, positions, bank, mask=None, out=None) -> np.ndarray:
        h = _f32(hidden)
        if out is None:
            out = np.empty_like(h)
        elif out.shape != h.shape or out.dtype != np.float32 or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float32 array shaped like hidden")
        m = None if mask is None else _f32(mask)
        check(_lib.lib().sfg_forward_layers(self.h, bank.h, layer_begin, layer_end, h.shape[0], _p(h, _f32p),
                                            _p(_i32(positions), _i32p), _p(m, _f32p), _p(out, _f32p)))
        return out

    def embed_at(self, ids, positions) -> np.ndarray:
        ids = _i32(ids)
        out = np.empty((len(ids), self.cfg.hidden_dim), dtype=np.float32)
        check(_lib.lib().sfg_embed_at(self.h, len(ids), _p(ids, _i32p), _p(_i32(positions), _i32p),
                                      _p(out, _f32p)))
        return out

    def finalize(self, hidden) -> np.ndarray:
        h = _f32(hidden)
        out = np.empty((h.shape[0], self.cfg.vocab_size), dtype=np.float32)
        check(_lib.lib().sfg_finalize(self.h, h.shape[0], _p(h, _f32p), _p(out, _f32p)))
        return out

    def finalize_argmax(self, hidden) -> np.ndarray:
        h = _f32(hidden)
        out = np.empty(h.shape[0], dtype=np.int32)
        check(_lib.lib().sfg_finalize_argmax(self.h, h.shape[0], _p(h, _f32p), _p(out, _i32p)))
        return out


class CacheBank:
    """CacheBank (tinyformer.hpp:131-156) with device-resident K/V."""

    def __init__(self, eng: Engine, lb: int, le: int):
        self.eng = eng
        h = C.c_void_p()
        check(_lib.lib().sfg_bank_create(eng.h, lb, le, C.byref(h)))
        self.h = h
        self.layer_begin, self.layer_end = lb, le

    def __del__(self):
        try:
            _lib.lib().sfg_bank_destroy(self.h)
        except Exception:
            pass

    def _state(self):
        a, b = C.c_int32(), C.c_int32()
        _lib.lib().sfg_bank_state(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    def len(self) -> int:
        return self._state()[0]

    def committed_len(self) -> int:
        return self._state()[1]

    def provisional(self) -> int:
        a, b = self._state()
        return a - b

    def resolve(self, keep):
        k = _i32(keep)
        check(_lib.lib().sfg_bank_resolve(self.h, _p(k, _i32p), len(k)))

    def crop(self, pos: int):
        check(_lib.lib().sfg_bank_crop(self.h, pos))

    def mark_committed(self, c: int):
        _lib.lib().sfg_bank_mark_committed(self.h, c)

    def reset(self):
        _lib.lib().sfg_bank_reset(self.h)

    def kv(self, layer, head, pos):
        hd = self.eng.cfg.head_dim
        k = np.empty(hd, dtype=np.float32)
        v = np.empty(hd, dtype=np.float32)
        check(_lib.lib().sfg_bank_read_kv(self.h, layer, head, pos, _p(k, _f32p), _p(v, _f32p)))
        return k, v


@dataclass
class ServerConfig:
    """splitf::ServerConfig (server.hpp:15-22)."""
    layer_begin: int = 2
    layer_end: int = 6
    session_expiry_s: float = 300.0
    max_sessions: int = 64
    response_dtype: int | None = None  # None mirrors the request


class ServerEngine:
    """ServerEngine (server.hpp:28-77) on the B200; ``handle`` takes and
    returns encoded frames (PROTOCOL.md)."""

    def __init__(self, eng: Engine, cfg: ServerConfig | None = None):
        cfg = cfg or ServerConfig()
        self.eng, self.cfg = eng, cfg
        c = _lib.ServerConfig(cfg.layer_begin, cfg.layer_end, cfg.session_expiry_s, cfg.max_sessions,
                              -1 if cfg.response_dtype is None else cfg.response_dtype)
        h = C.c_void_p()
        check(_lib.lib().sfg_server_create(eng.h, C.byref(c), C.byref(h)))
        self.h = h
        self._clock_cb = None

    def __del__(self):
        try:
            _lib.lib().sfg_server_destroy(self.h)
        except Exception:
            pass

    def handle(self, frame: bytes) -> bytes:
        buf = (C.c_uint8 * len(frame)).from_buffer_copy(frame)
        rp = C.POINTER(C.c_uint8)()
        rn = C.c_size_t()
        check(_lib.lib().sfg_server_handle(self.h, buf, len(frame), C.byref(rp), C.byref(rn)))
        return C.string_at(rp, rn.value)

    def handle_batch(self, frames) -> list:
        """handle() over several queued frames; step frames of distinct sessions
        share one weight pass (responses identical to handle() one by one)."""
        n = len(frames)
        bufs = [(C.c_uint8 * len(f)).from_buffer_copy(f) for f in frames]
        reqs = (C.c_void_p * n)(*[C.addressof(b) for b in bufs])
        lens = (C.c_size_t * n)(*[len(f) for f in frames])
        rps = (C.POINTER(C.c_uint8) * n)()
        rns = (C.c_size_t * n)()
        check(_lib.lib().sfg_server_handle_batch(self.h, n, reqs, lens, rps, rns))
        return [C.string_at(rps[i], rns[i]) for i in range(n)]

    @property
    def handler(self):
        """(C function pointer, ctx) usable as a FrameHandler by C clients."""
        fn = C.cast(_lib.lib().sfg_server_handle, C.c_void_p)
        return fn, self.h

    def shared_passes(self) -> int:
        return int(_lib.lib().sfg_server_shared_passes(self.h))

    def expire_sessions(self) -> int:
        return int(_lib.lib().sfg_server_expire_sessions(self.h))

    def session_count(self) -> int:
        return int(_lib.lib().sfg_server_session_count(self.h))

    def session_view(self, sid: str):
        a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
        if not _lib.lib().sfg_server_session_view(self.h, sid.encode(), C.byref(a), C.byref(b), C.byref(c)):
            return None
        return {"cache_len": a.value, "committed_len": b.value, "provisional": c.value}

    def set_clock(self, now_s):
        cb = C.CFUNCTYPE(C.c_double, C.c_void_p)(lambda _ctx: float(now_s()))
        self._clock_cb = cb
        _lib.lib().sfg_server_set_clock(self.h, cb, None)


def _handle_bytes(fn, h, frame: bytes) -> bytes:
    buf = (C.c_uint8 * len(frame)).from_buffer_copy(frame)
    rp = C.POINTER(C.c_uint8)()
    rn = C.c_size_t()
    check(fn(h, buf, len(frame), C.byref(rp), C.byref(rn)))
    return C.string_at(rp, rn.value)


class Router:
    """Frame router over one ServerEngine per device (or any frame handlers):
    sessions are placed on the least-loaded backend at their prompt frame and
    stay there (sfg.h sfg_router_*).  ``backends`` are ServerEngines or
    (C function pointer, ctx) handler pairs."""

    def __init__(self, backends, session_expiry_s: float = 300.0):
        L = _lib.lib()
        h = C.c_void_p()
        n = len(backends)
        if all(isinstance(b, ServerEngine) for b in backends):
            arr = (C.c_void_p * n)(*[b.h.value for b in backends])
            check(L.sfg_router_create(arr, n, session_expiry_s, C.byref(h)))
        else:
            fns = (C.c_void_p * n)(*[C.cast(b[0], C.c_void_p).value for b in backends])
            ctxs = (C.c_void_p * n)(*[b[1] for b in backends])
            check(L.sfg_router_create_handlers(fns, ctxs, n, session_expiry_s, C.byref(h)))
        self.h, self._backends, self._clock_cb = h, backends, None

    def __del__(self):
        try:
            _lib.lib().sfg_router_destroy(self.h)
        except Exception:
            pass

    def handle(self, frame: bytes) -> bytes:
        return _handle_bytes(_lib.lib().sfg_router_handle, self.h, frame)

    @property
    def handler(self):
        return C.cast(_lib.lib().sfg_router_handle, C.c_void_p), self.h

    def session_device(self, sid: str) -> int:
        return int(_lib.lib().sfg_router_session_device(self.h, sid.encode()))

    def load(self) -> list:
        out = (C.c_int32 * len(self._backends))()
        n = _lib.lib().sfg_router_load(self.h, out)
        return list(out[:n])

    def set_clock(self, now_s):
        cb = C.CFUNCTYPE(C.c_double, C.c_void_p)(lambda _ctx: float(now_s()))
        self._clock_cb = cb
        _lib.lib().sfg_router_set_clock(self.h, cb, None)


class Batcher:
    """Cross-session batching queue in front of a Router: a FrameHandler for
    concurrent connection threads (sfg.h sfg_batcher_*)."""

    def __init__(self, router: Router, max_frames: int = 0):
        h = C.c_void_p()
        check(_lib.lib().sfg_batcher_create(router.h, max_frames, C.byref(h)))
        self.h, self.router = h, router

    def __del__(self):
        try:
            _lib.lib().sfg_batcher_destroy(self.h)
        except Exception:
            pass

    def handle(self, frame: bytes) -> bytes:
        return _handle_bytes(_lib.lib().sfg_batcher_handle, self.h, frame)

    @property
    def handler(self):
        return C.cast(_lib.lib().sfg_batcher_handle, C.c_void_p), self.h

    def stats(self) -> dict:
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _lib.lib().sfg_batcher_stats(self.h, C.byref(a), C.byref(b), C.byref(c))
        return {"batches": a.value, "frames": b.value, "max_batch": c.value}


@dataclass
class SplitConfig:
    """splitf::SplitConfig (client.hpp:14-20) + the SimChannel one-way delay."""
    prefix_layers: int = 2
    suffix_layers: int = 2
    dtype: int = F16
    one_way_delay_ms: float = 0.0

    def to_c(self):
        return _lib.ClientConfig(self.prefix_layers, self.suffix_layers, self.dtype, self.one_way_delay_ms)


class SplitClient:
    """SplitClient (client.hpp:41-100) on the B200.

    ``server`` is either a ServerEngine in this process (device-linked: hidden
    rows never leave HBM) or a (C function pointer, ctx) frame handler."""

    def __init__(self, local: Engine, cfg: SplitConfig | None = None, server=None, session_id: str = "",
                 frames: bool = False):
        cfg = cfg or SplitConfig()
        self.local, self.cfg = local, cfg
        h = C.c_void_p()
        L = _lib.lib()
        if isinstance(server, ServerEngine) and not frames:
            check(L.sfg_client_create_linked(local.h, C.byref(cfg.to_c()), server.h, session_id.encode(),
                                             C.byref(h)))
        else:
            fn, ctx = server.handler if isinstance(server, ServerEngine) else server
            check(L.sfg_client_create(local.h, C.byref(cfg.to_c()), fn, ctx, session_id.encode(), C.byref(h)))
        self.h = h
        self._server = server  # keep alive

    def __del__(self):
        try:
            _lib.lib().sfg_client_destroy(self.h)
        except Exception:
            pass

    def prefill(self, prompt, want_logits=False):
        p = _i32(prompt)
        first = C.c_int32()
        lg = np.empty(self.local.cfg.vocab_size, dtype=np.float32) if want_logits else None
        check(_lib.lib().sfg_client_prefill(self.h, _p(p, _i32p), len(p), C.byref(first), _p(lg, _f32p)))
        return (first.value, lg) if want_logits else first.value

    def decode_step(self, tokens, positions, mask=None, keep=(), crop=None, want_logits=True):
        t = _i32(tokens)
        k = _i32(keep) if len(keep) else np.zeros(1, dtype=np.int32)
        m = None if mask is None else _f32(mask)
        lg = np.empty((len(t), self.local.cfg.vocab_size), dtype=np.float32) if want_logits else None
        am = np.empty(len(t), dtype=np.int32)
        check(_lib.lib().sfg_client_decode_step(self.h, len(t), _p(t, _i32p), _p(_i32(positions), _i32p),
                                                _p(m, _f32p), _p(k, _i32p), len(keep),
                                                -1 if crop is None else crop, _p(lg, _f32p), _p(am, _i32p)))
        return lg if want_logits else am

    def last_profile(self) -> dict:
        p = _lib.StepProfile()
        _lib.lib().sfg_client_last_profile(self.h, C.byref(p))
        return {"step_ms": p.step_ms, "server_ms": p.server_ms, "local_ms": p.local_ms,
                "launches": p.launches, "batch": p.batch}


class NGramPool:
    """NGramPool (decoding.hpp:35-60)."""

    def __init__(self, ngram_n: int, capacity: int):
        h = C.c_void_p()
        check(_lib.lib().sfg_pool_create(ngram_n, capacity, C.byref(h)))
        self.h, self.n = h, ngram_n

    def __del__(self):
        try:
            _lib.lib().sfg_pool_destroy(self.h)
        except Exception:
            pass

    def update(self, previous, current):
        a, b = _i32(previous), _i32(current)
        check(_lib.lib().sfg_pool_update(self.h, _p(a, _i32p), _p(b, _i32p), len(a)))

    def lookup(self, key, max_candidates):
        out = np.zeros(max(1, max_candidates) * (self.n - 1), dtype=np.int32)
        got = _lib.lib().sfg_pool_lookup(self.h, key, max_candidates, _p(out, _i32p))
        return [out[i * (self.n - 1):(i + 1) * (self.n - 1)].tolist() for i in range(got)]

    def size(self):
        return int(_lib.lib().sfg_pool_size(self.h))


@dataclass
class LookaheadConfig:
    """splitf::LookaheadConfig (decoding.hpp:25-30)."""
    ngram_n: int = 3
    window_w: int = 8
    max_candidates_g: int = 2
    pool_capacity: int = 4096


@dataclass
class DecodeResult:
    tokens: list
    committed_logits: np.ndarray | None
    step_batch: list
    step_accepted: list
    steps: int
    tokens_committed: int
    wall_seconds: float
    match_rate: float
    clamped: int
    extra: dict = field(default_factory=dict)


def _decode(client: SplitClient, mode, prompt, max_new, la: LookaheadConfig, pool, want_logits):
    p = _i32(prompt)
    toks = np.zeros(max(1, max_new), dtype=np.int32)
    V = client.local.cfg.vocab_size
    lg = np.zeros((max_new, V), dtype=np.float32) if want_logits else None
    sb = np.zeros(max(1, max_new), dtype=np.int32)
    sa = np.zeros(max(1, max_new), dtype=np.int32)
    st = _lib.DecodeStats()
    dc = _lib.DecodeConfig(mode, la.window_w, la.ngram_n, la.max_candidates_g, la.pool_capacity)
    check(_lib.lib().sfg_decode(client.h, C.byref(dc), pool.h if pool is not None else None, _p(p, _i32p), len(p),
                                max_new, _p(toks, _i32p), _p(lg, _f32p), _p(sb, _i32p), _p(sa, _i32p),
                                C.byref(st)))
    return DecodeResult(toks[:max_new].tolist(), lg, sb[:st.steps].tolist(), sa[:st.steps].tolist(), st.steps,
                        st.tokens_committed, st.wall_seconds, st.match_rate, st.clamped)


def decode_sequential(client, prompt, max_new, want_logits=False) -> DecodeResult:
    return _decode(client, 0, prompt, max_new, LookaheadConfig(), None, want_logits)


def decode_lookahead(client, prompt, max_new, cfg: LookaheadConfig | None = None, want_logits=False):
    return _decode(client, 2, prompt, max_new, cfg or LookaheadConfig(), None, want_logits)


def decode_lookahead_with_pool(client, prompt, max_new, cfg: LookaheadConfig, pool: NGramPool,
                               want_logits=False):
    return _decode(client, 2, prompt, max_new, cfg, pool, want_logits)


def f32_to_f16_bits(v: float, counter=None) -> int:
    c = C.c_uint64(0)
    b = _lib.lib().sfg_f32_to_f16(C.c_float(v), C.byref(c))
    if counter is not None:
        counter[0] += c.value
    return int(b)


def f16_bits_to_f32(b: int) -> float:
    return float(_lib.lib().sfg_f16_to_f32(C.c_uint16(b)))
