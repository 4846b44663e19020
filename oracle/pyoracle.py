"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle.

Two checkers live behind one interface:

* ``Port``  — oracle/liboracle.so, the plain-C restatement (splitf_oracle.c);
* ``Ref``   — oracle/_ref/libsplitf_ref.so, the UNMODIFIED reference sources
  (/root/reference/proj/src) compiled in place with ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) may import this module.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsplitf_ref.so")
REF_SRC = "/root/reference/proj/src"

_i32p = C.POINTER(C.c_int32)
_f32p = C.POINTER(C.c_float)
_u8p = C.POINTER(C.c_uint8)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = msg.split(":", 1)[0] if ":" in msg else "internal"


@dataclass
class ModelCfg:
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

    def q_dim(self):
        return self.n_heads * self.head_dim

    def kv_dim(self):
        return self.n_kv_heads * self.head_dim


class _CCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("vocab_size", "n_layers", "hidden_dim", "n_heads",
                                        "n_kv_heads", "head_dim", "ffn_dim", "max_seq_len")] + [
        ("rope_base", C.c_float), ("rms_eps", C.c_float), ("seed", C.c_uint64)]


def _ccfg(c: ModelCfg) -> _CCfg:
    return _CCfg(c.vocab_size, c.n_layers, c.hidden_dim, c.n_heads, c.n_kv_heads, c.head_dim,
                 c.ffn_dim, c.max_seq_len, c.rope_base, c.rms_eps, c.seed)


@dataclass
class DecodeCfg:
    mode: int = 2  # 0 sequential, 1 jacobi (ref only), 2 lookahead
    prefix_layers: int = 2
    suffix_layers: int = 2
    wire_f32: int = 1
    server_dtype: int = -1
    window_w: int = 5
    ngram_n: int = 3
    max_candidates_g: int = 5
    pool_capacity: int = 4096
    block_k: int = 4
    rtt_ms: float = 0.0


class _RefDecodeCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("mode", "prefix_layers", "suffix_layers", "wire_f32",
                                        "server_dtype", "window_w", "ngram_n", "max_candidates_g",
                                        "pool_capacity", "block_k")] + [("rtt_ms", C.c_double)]


class _OrcDecodeCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("mode", "prefix_layers", "suffix_layers", "wire_f32",
                                        "server_dtype", "window_w", "ngram_n", "max_candidates_g",
                                        "pool_capacity")]


class _RefStats(C.Structure):
    _fields_ = [("steps", C.c_int), ("tokens_committed", C.c_int), ("wall_seconds", C.c_double),
                ("acceptance_rate", C.c_double), ("match_rate", C.c_double),
                ("prefill_ms", C.c_double)]


class _OrcStats(C.Structure):
    _fields_ = [("steps", C.c_int), ("tokens_committed", C.c_int), ("clamped", C.c_uint64)]


@dataclass
class DecodeOut:
    tokens: list
    logits: np.ndarray | None
    step_batch: list
    step_accepted: list
    steps: int
    tokens_committed: int
    extra: dict = field(default_factory=dict)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def build_port():
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)


def build_ref():
    if not os.path.isdir(REF_SRC):
        return False
    subprocess.run(["make", "-s", "-C", HERE, "-j8", "ref"], check=True)
    return True


def ref_available() -> bool:
    return os.path.exists(REF_SO)


# ─────────────────────────────────────────────────────────────────────────
class _Base:
    lib: C.CDLL

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._errfn().decode())


class Port(_Base):
    """oracle/liboracle.so — the C restatement."""

    _lib = None

    def __init__(self):
        if Port._lib is None:
            if not os.path.exists(PORT_SO):
                build_port()
            lib = C.CDLL(PORT_SO)
            lib.orc_last_error.restype = C.c_char_p
            lib.orc_param_count.restype = C.c_int64
            lib.orc_model_params.restype = C.c_int64
            lib.orc_f32_to_f16.restype = C.c_uint16
            lib.orc_f32_to_f16.argtypes = [C.c_float, C.POINTER(C.c_uint64)]
            lib.orc_f16_to_f32.restype = C.c_float
            lib.orc_f16_to_f32.argtypes = [C.c_uint16]
            lib.orc_pool_size.restype = C.c_size_t
            lib.orc_pool_new.argtypes = [C.c_int, C.c_size_t, C.POINTER(C.c_void_p)]
            Port._lib = lib
        self.lib = Port._lib
        self._errfn = self.lib.orc_last_error

    # model -----------------------------------------------------------------
    def model(self, cfg: ModelCfg, bf16: bool = True, params: np.ndarray | None = None, layers: tuple | None = None):
        h = C.c_void_p()
        if layers is not None:  # decoder layers [lo, hi) of the init stream only
            self._check(self.lib.orc_model_new_layers(C.byref(_ccfg(cfg)), int(bf16), layers[0], layers[1],
                                                      C.byref(h)))
        elif params is None:
            self._check(self.lib.orc_model_new(C.byref(_ccfg(cfg)), int(bf16), C.byref(h)))
        else:
            p = np.ascontiguousarray(params, dtype=np.float32)
            self._check(self.lib.orc_model_from_params(C.byref(_ccfg(cfg)), _ptr(p, _f32p), C.byref(h)))
        return _Model(self, h, cfg, "orc")

    def set_relaxed_validate(self, on: bool):
        """Accept q_dim != hidden_dim (NeMo-12B); the reference's validate()
        rejects it while its arithmetic uses q_dim throughout."""
        self.lib.orc_set_relaxed_validate(int(on))

    def param_count(self, cfg: ModelCfg) -> int:
        return int(self.lib.orc_param_count(C.byref(_ccfg(cfg))))

    def f32_to_f16(self, v: float, counter=None) -> int:
        c = C.c_uint64(0)
        b = self.lib.orc_f32_to_f16(C.c_float(v), C.byref(c))
        if counter is not None:
            counter[0] += c.value
        return int(b)

    def f16_to_f32(self, b: int) -> float:
        return float(self.lib.orc_f16_to_f32(C.c_uint16(b)))

    def verify_greedy(self, logits: np.ndarray, row_begin, guesses, anchor):
        lg = np.ascontiguousarray(logits, dtype=np.float32)
        g = np.asarray(guesses, dtype=np.int32)
        out = np.zeros(len(g) + 1, dtype=np.int32)
        acc = self.lib.orc_verify_greedy(_ptr(lg, _f32p), lg.shape[1], row_begin, _ptr(g, _i32p),
                                         len(g), anchor, _ptr(out, _i32p))
        return acc, out[:acc + 1].tolist()

    def pool(self, n, cap):
        h = C.c_void_p()
        self._check(self.lib.orc_pool_new(n, cap, C.byref(h)))
        return _Pool(self, h, n, "orc")

    def decode(self, model, dc: DecodeCfg, prompt, max_new, pool=None, want_logits=False) -> DecodeOut:
        p = np.asarray(prompt, dtype=np.int32)
        toks = np.zeros(max_new, dtype=np.int32)
        lg = np.zeros((max_new, model.cfg.vocab_size), dtype=np.float32) if want_logits else None
        sb = np.zeros(max_new + 1, dtype=np.int32)
        sa = np.zeros(max_new + 1, dtype=np.int32)
        st = _OrcStats()
        c = _OrcDecodeCfg(dc.mode, dc.prefix_layers, dc.suffix_layers, dc.wire_f32, dc.server_dtype,
                          dc.window_w, dc.ngram_n, dc.max_candidates_g, dc.pool_capacity)
        self._check(self.lib.orc_decode(model.h, C.byref(c), pool.h if pool else None,
                                        _ptr(p, _i32p), len(p), max_new, _ptr(toks, _i32p),
                                        _ptr(lg, _f32p) if lg is not None else None,
                                        _ptr(sb, _i32p), _ptr(sa, _i32p), C.byref(st)))
        return DecodeOut(toks.tolist(), lg, sb[:st.steps].tolist(), sa[:st.steps].tolist(), st.steps,
                         st.tokens_committed, {"clamped": st.clamped})


class Ref(_Base):
    """oracle/_ref/libsplitf_ref.so — the reference sources, compiled in place."""

    _lib = None

    def __init__(self):
        if Ref._lib is None:
            if not os.path.exists(REF_SO) and not build_ref():
                raise FileNotFoundError("oracle/_ref/libsplitf_ref.so not built and /root/reference absent")
            lib = C.CDLL(REF_SO)
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_model_params.restype = C.c_int64
            lib.ref_f32_to_f16.restype = C.c_uint16
            lib.ref_f32_to_f16.argtypes = [C.c_float, C.POINTER(C.c_uint64)]
            lib.ref_f16_to_f32.restype = C.c_float
            lib.ref_f16_to_f32.argtypes = [C.c_uint16]
            lib.ref_pool_size.restype = C.c_size_t
            lib.ref_pool_new.argtypes = [C.c_int, C.c_size_t, C.POINTER(C.c_void_p)]
            lib.ref_server_expire.restype = C.c_size_t
            lib.ref_server_count.restype = C.c_size_t
            lib.ref_server_new.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                           C.POINTER(C.c_void_p)]
            lib.ref_server_handle.argtypes = [C.c_void_p, _u8p, C.c_size_t, C.POINTER(_u8p),
                                              C.POINTER(C.c_size_t)]
            lib.ref_time_forward.restype = C.c_double
            lib.ref_time_forward.argtypes = [C.c_void_p] + [C.c_int] * 5
            lib.ref_time_finalize.restype = C.c_double
            lib.ref_time_finalize.argtypes = [C.c_void_p, C.c_int, C.c_int]
            Ref._lib = lib
        self.lib = Ref._lib
        self._errfn = self.lib.ref_last_error

    def model(self, cfg: ModelCfg, bf16: bool = True, layers: tuple | None = None, with_head=True,
              unchecked: bool = False):
        """unchecked: skip ModelConfig::validate (q_dim != hidden, NeMo-12B);
        needs `layers` (ref_model_new_unchecked)."""
        h = C.c_void_p()
        lo, hi = layers if layers is not None else (-1, -1)
        if unchecked:
            self._check(self.lib.ref_model_new_unchecked(C.byref(_ccfg(cfg)), int(bf16), lo, hi, int(with_head),
                                                         C.byref(h)))
            return _Model(self, h, cfg, "ref")
        self._check(self.lib.ref_model_new(C.byref(_ccfg(cfg)), int(bf16), lo, hi, int(with_head),
                                           C.byref(h)))
        return _Model(self, h, cfg, "ref")

    def timing_model(self, cfg: ModelCfg, layers: tuple, with_head: bool):
        """Tensors of `layers` (+ head) filled with U[-a,a] values without
        walking the reference stream: for CPU-baseline timing only."""
        h = C.c_void_p()
        self._check(self.lib.ref_model_new_timing(C.byref(_ccfg(cfg)), layers[0], layers[1], int(with_head),
                                                  C.byref(h)))
        return _Model(self, h, cfg, "ref")

    def f32_to_f16(self, v: float, counter=None) -> int:
        c = C.c_uint64(0)
        b = self.lib.ref_f32_to_f16(C.c_float(v), C.byref(c))
        if counter is not None:
            counter[0] += c.value
        return int(b)

    def f16_to_f32(self, b: int) -> float:
        return float(self.lib.ref_f16_to_f32(C.c_uint16(b)))

    def verify_greedy(self, logits: np.ndarray, row_begin, guesses, anchor):
        lg = np.ascontiguousarray(logits, dtype=np.float32)
        g = np.asarray(guesses, dtype=np.int32)
        out = np.zeros(len(g) + 1, dtype=np.int32)
        acc = C.c_int(0)
        self._check(self.lib.ref_verify_greedy(lg.shape[0], lg.shape[1], _ptr(lg, _f32p), row_begin,
                                               _ptr(g, _i32p), len(g), anchor, C.byref(acc),
                                               _ptr(out, _i32p)))
        return acc.value, out[:acc.value + 1].tolist()

    def pool(self, n, cap):
        h = C.c_void_p()
        self._check(self.lib.ref_pool_new(n, cap, C.byref(h)))
        return _Pool(self, h, n, "ref")

    def corpus(self, kind: str, vocab: int, n_prompts: int, prompt_len: int, seed: int):
        out = np.zeros(n_prompts * prompt_len, dtype=np.int32)
        self._check(self.lib.ref_corpus(0 if kind == "repetitive" else 1, vocab, n_prompts,
                                        prompt_len, C.c_uint64(seed), _ptr(out, _i32p)))
        return out.reshape(n_prompts, prompt_len).tolist()

    def decode(self, model, dc: DecodeCfg, prompt, max_new, handler=None, handler_ctx=None,
               want_logits=False) -> DecodeOut:
        """run_decode through the reference client + decode loop; ``handler``
        is a C function pointer (ctypes) standing in for the server."""
        p = np.asarray(prompt, dtype=np.int32)
        toks = np.zeros(max_new, dtype=np.int32)
        lg = np.zeros((max_new, model.cfg.vocab_size), dtype=np.float32) if want_logits else None
        sb = np.zeros(max_new + 1, dtype=np.int32)
        sa = np.zeros(max_new + 1, dtype=np.int32)
        st = _RefStats()
        c = _RefDecodeCfg(dc.mode, dc.prefix_layers, dc.suffix_layers, dc.wire_f32, dc.server_dtype,
                          dc.window_w, dc.ngram_n, dc.max_candidates_g, dc.pool_capacity, dc.block_k,
                          dc.rtt_ms)
        self._check(self.lib.ref_decode(model.h, C.byref(c), _ptr(p, _i32p), len(p), max_new,
                                        handler, handler_ctx, _ptr(toks, _i32p),
                                        _ptr(lg, _f32p) if lg is not None else None,
                                        _ptr(sb, _i32p), _ptr(sa, _i32p), C.byref(st)))
        return DecodeOut(toks.tolist(), lg, sb[:st.steps].tolist(), sa[:st.steps].tolist(), st.steps,
                         st.tokens_committed,
                         {"wall_seconds": st.wall_seconds, "acceptance_rate": st.acceptance_rate,
                          "match_rate": st.match_rate, "prefill_ms": st.prefill_ms})

    def server(self, model, lb, le, expiry_s=300.0, max_sessions=64, response_dtype=-1):
        h = C.c_void_p()
        self._check(self.lib.ref_server_new(model.h, lb, le, expiry_s, max_sessions, response_dtype,
                                            C.byref(h)))
        return _RefServer(self, h)


class _Model:
    def __init__(self, owner, h, cfg, pfx):
        self.o, self.h, self.cfg, self.p = owner, h, cfg, pfx
        self.lib = owner.lib

    def __del__(self):
        try:
            getattr(self.lib, f"{self.p}_model_free")(self.h)
        except Exception:
            pass

    def params(self) -> np.ndarray:
        fn = getattr(self.lib, f"{self.p}_model_params")
        n = fn(self.h, None)
        out = np.empty(n, dtype=np.float32)
        fn(self.h, _ptr(out, _f32p))
        return out

    def bank(self, lb, le):
        h = C.c_void_p()
        self.o._check(getattr(self.lib, f"{self.p}_bank_new")(self.h, lb, le, C.byref(h)))
        return _Bank(self, h)

    def generate(self, prompt, max_new, want_logits=False):
        p = np.asarray(prompt, dtype=np.int32)
        toks = np.zeros(max_new, dtype=np.int32)
        lg = np.zeros((max_new, self.cfg.vocab_size), dtype=np.float32) if want_logits else None
        self.o._check(getattr(self.lib, f"{self.p}_generate")(
            self.h, _ptr(p, _i32p), len(p), max_new, _ptr(toks, _i32p),
            _ptr(lg, _f32p) if lg is not None else None))
        return (toks.tolist(), lg) if want_logits else toks.tolist()

    def embed_at(self, ids, pos):
        ids = np.asarray(ids, dtype=np.int32)
        pos = np.asarray(pos, dtype=np.int32)
        out = np.zeros((len(ids), self.cfg.hidden_dim), dtype=np.float32)
        self.o._check(getattr(self.lib, f"{self.p}_embed_at")(self.h, len(ids), _ptr(ids, _i32p),
                                                             _ptr(pos, _i32p), _ptr(out, _f32p)))
        return out

    def finalize(self, h):
        h = np.ascontiguousarray(h, dtype=np.float32)
        out = np.zeros((h.shape[0], self.cfg.vocab_size), dtype=np.float32)
        self.o._check(getattr(self.lib, f"{self.p}_finalize")(self.h, h.shape[0], _ptr(h, _f32p),
                                                             _ptr(out, _f32p)))
        return out


class _Bank:
    def __init__(self, model, h):
        self.m, self.h = model, h
        self.lib, self.p, self.o = model.lib, model.p, model.o

    def __del__(self):
        try:
            getattr(self.lib, f"{self.p}_bank_free")(self.h)
        except Exception:
            pass

    def forward(self, lb, le, h, pos, mask=None):
        h = np.ascontiguousarray(h, dtype=np.float32)
        pos = np.asarray(pos, dtype=np.int32)
        out = np.zeros_like(h)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.float32)
        self.o._check(getattr(self.lib, f"{self.p}_forward")(
            self.m.h, self.h, lb, le, h.shape[0], _ptr(h, _f32p), _ptr(pos, _i32p),
            _ptr(m, _f32p) if m is not None else None, _ptr(out, _f32p)))
        return out

    def resolve(self, keep):
        k = np.asarray(keep, dtype=np.int32)
        self.o._check(getattr(self.lib, f"{self.p}_bank_resolve")(self.h, _ptr(k, _i32p), len(k)))

    def crop(self, pos):
        self.o._check(getattr(self.lib, f"{self.p}_bank_crop")(self.h, pos))

    def mark_committed(self, c):
        getattr(self.lib, f"{self.p}_bank_mark_committed")(self.h, c)

    def state(self):
        a, b = C.c_int(), C.c_int()
        getattr(self.lib, f"{self.p}_bank_state")(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    def load_layer(self, layer, k, v, length):
        """(_ref only) install a layer's K/V slabs [n_kv x max_len x hd] and its length."""
        k = np.ascontiguousarray(k, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        self.o._check(self.lib.ref_bank_load_layer(self.h, layer, _ptr(k, _f32p), _ptr(v, _f32p), length))

    def kv(self, layer, head, pos):
        hd = self.m.cfg.head_dim
        k = np.zeros(hd, dtype=np.float32)
        v = np.zeros(hd, dtype=np.float32)
        self.o._check(getattr(self.lib, f"{self.p}_bank_kv")(self.h, layer, head, pos,
                                                            _ptr(k, _f32p), _ptr(v, _f32p)))
        return k, v


class _Pool:
    def __init__(self, owner, h, n, p):
        self.o, self.h, self.n, self.p, self.lib = owner, h, n, p, owner.lib

    def __del__(self):
        try:
            getattr(self.lib, f"{self.p}_pool_free")(self.h)
        except Exception:
            pass

    def update(self, prev, cur):
        a = np.asarray(prev, dtype=np.int32)
        b = np.asarray(cur, dtype=np.int32)
        self.o._check(getattr(self.lib, f"{self.p}_pool_update")(self.h, _ptr(a, _i32p), _ptr(b, _i32p), len(a)))

    def lookup(self, key, max_c):
        out = np.zeros(max(1, max_c) * (self.n - 1), dtype=np.int32)
        got = getattr(self.lib, f"{self.p}_pool_lookup")(self.h, key, max_c, _ptr(out, _i32p))
        return [out[i * (self.n - 1):(i + 1) * (self.n - 1)].tolist() for i in range(got)]

    def size(self):
        return int(getattr(self.lib, f"{self.p}_pool_size")(self.h))


class _RefServer:
    def __init__(self, owner, h):
        self.o, self.h, self.lib = owner, h, owner.lib
        self._clock = None

    def __del__(self):
        try:
            self.lib.ref_server_free(self.h)
        except Exception:
            pass

    def handle(self, req: bytes) -> bytes:
        buf = (C.c_uint8 * len(req)).from_buffer_copy(req)
        rp = _u8p()
        rn = C.c_size_t()
        self.o._check(self.lib.ref_server_handle(self.h, buf, len(req), C.byref(rp), C.byref(rn)))
        return C.string_at(rp, rn.value)

    def set_clock(self, now: float):
        if self._clock is None:
            self._clock = C.c_double(now)
            self.lib.ref_server_set_clock(self.h, C.byref(self._clock))
        self._clock.value = now

    def session_view(self, sid: str):
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        if not self.lib.ref_server_session_view(self.h, sid.encode(), C.byref(a), C.byref(b), C.byref(c)):
            return None
        return {"cache_len": a.value, "committed_len": b.value, "provisional": c.value}

    def expire_sessions(self):
        return int(self.lib.ref_server_expire(self.h))

    def session_count(self):
        return int(self.lib.ref_server_count(self.h))


# Model configs named by BASELINE.json (SURVEY §8 preamble) ----------------
def desk_cfg(seed=1234) -> ModelCfg:
    return ModelCfg(seed=seed)


def tiny_cfg(seed=1234) -> ModelCfg:
    """config 1: 4 layers, d=256, 4q/2kv x 64 (GQA), ffn 896, V=32768."""
    return ModelCfg(vocab_size=32768, n_layers=4, hidden_dim=256, n_heads=4, n_kv_heads=2,
                    head_dim=64, ffn_dim=896, max_seq_len=512, rope_base=1e6, rms_eps=1e-5, seed=seed)


def mistral7b_cfg(seed=1234, max_seq_len=4096) -> ModelCfg:
    return ModelCfg(vocab_size=32768, n_layers=32, hidden_dim=4096, n_heads=32, n_kv_heads=8,
                    head_dim=128, ffn_dim=14336, max_seq_len=max_seq_len, rope_base=1e6, rms_eps=1e-5,
                    seed=seed)


def nemo12b_cfg(seed=1234, max_seq_len=4096) -> ModelCfg:
    """Mistral NeMo 12B true shape: d=5120, 32 q heads x 128 = q_dim 4096 (!= d)."""
    return ModelCfg(vocab_size=131072, n_layers=40, hidden_dim=5120, n_heads=32, n_kv_heads=8,
                    head_dim=128, ffn_dim=14336, max_seq_len=max_seq_len, rope_base=1e6, rms_eps=1e-5,
                    seed=seed)


def nemo12b_parity_cfg(seed=1234, max_seq_len=4096) -> ModelCfg:
    """NeMo-12B width with head_dim 160 so the reference's validate() accepts it."""
    return ModelCfg(vocab_size=131072, n_layers=40, hidden_dim=5120, n_heads=32, n_kv_heads=8,
                    head_dim=160, ffn_dim=14336, max_seq_len=max_seq_len, rope_base=1e6, rms_eps=1e-5,
                    seed=seed)
