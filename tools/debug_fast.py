"""Dev check of the FAST (tcgen05) path on a B200: error vs the CPU oracle,
batch invariance, and per-kernel timing at the 7B shape (one layer)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import ctypes as C

import paper_2602_16760_b200 as sfg
import pyoracle as po
from paper_2602_16760_b200 import _lib


def scfg(c):
    return sfg.ModelConfig(**{k: getattr(c, k) for k in po.ModelCfg.__dataclass_fields__})


def rel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-30)))


port = po.Port()
for name, cfg in (("desk", po.desk_cfg()), ("tiny", po.tiny_cfg())):
    m = port.model(cfg, bf16=True)
    eng = sfg.Engine(scfg(cfg), math=sfg.FAST, params=m.params())
    rng = np.random.default_rng(1)
    L = cfg.n_layers
    for rows in (1, 5, 16, 21):
        bo, bg = m.bank(0, L), eng.bank(0, L)
        h = rng.standard_normal((rows, cfg.hidden_dim)).astype(np.float32)
        a = bo.forward(0, L, h, list(range(rows)))
        b = eng.forward_layers(0, L, h, list(range(rows)), bg)
        k1, _ = bo.kv(L - 1, 0, rows - 1)
        k2, _ = bg.kv(L - 1, 0, rows - 1)
        print(name, "rows", rows, "hidden rel err", rel(b, a), "kv rel", rel(k2[None], k1[None]), flush=True)
    h = rng.standard_normal((3, cfg.hidden_dim)).astype(np.float32)
    lo, lg = m.finalize(h), eng.finalize(h)
    print(name, "logits rel err", rel(lg, lo), "argmax eq", (lg.argmax(1) == lo.argmax(1)).all(),
          (eng.finalize_argmax(h) == lo.argmax(1)).all(), flush=True)
    # decode tokens vs oracle, lookahead vs sequential bitwise inside FAST
    srv = sfg.ServerEngine(eng, sfg.ServerConfig(2 if name == "desk" else 1, L - (2 if name == "desk" else 1)))
    sp = 2 if name == "desk" else 1
    la = sfg.LookaheadConfig(ngram_n=3, window_w=5, max_candidates_g=5)
    prompt = [3, 1, 4, 1, 5, 9, 2, 6]
    s = sfg.decode_sequential(sfg.SplitClient(eng, sfg.SplitConfig(sp, sp, sfg.F32), srv), prompt, 40, want_logits=True)
    la_ = sfg.decode_lookahead(sfg.SplitClient(eng, sfg.SplitConfig(sp, sp, sfg.F32), srv), prompt, 40, la, want_logits=True)
    ref = port.decode(m, po.DecodeCfg(mode=2, prefix_layers=sp, suffix_layers=sp, wire_f32=1, window_w=5, ngram_n=3,
                                      max_candidates_g=5), prompt, 40, want_logits=True)
    print(name, "fast seq==lookahead tokens", s.tokens == la_.tokens, "logits bitwise",
          np.array_equal(s.committed_logits, la_.committed_logits), "tokens==oracle", la_.tokens == ref.tokens,
          "logit rel", rel(la_.committed_logits, ref.logits), flush=True)

# 7B shape, one layer
cfg7 = po.mistral7b_cfg()
t = time.time()
eng = sfg.Engine(scfg(cfg7), math=sfg.FAST, layers=(2, 3), with_embedding=False, with_head=False)
print("7B 1-layer fast engine init", time.time() - t, "s", flush=True)
ref = po.Ref() if po.ref_available() else None
rng = np.random.default_rng(2)
h = (rng.standard_normal((16, 4096)) * 0.5).astype(np.float32)
bg = eng.bank(2, 3)
L = _lib.lib()
L.sfg_profiler_reset()
L.sfg_profiler_enable(1)
for it in range(5):
    bg.reset()
    out = eng.forward_layers(2, 3, h, list(range(16)), bg)
L.sfg_profiler_enable(0)
names = ["qkv", "attention", "o_proj", "gate_up", "down", "rmsnorm", "lm_head", "other"]
for ci, n in enumerate(names):
    cnt, ms, by, fl = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
    L.sfg_profiler_stats(ci, C.byref(cnt), C.byref(ms), C.byref(by), C.byref(fl))
    if cnt.value:
        print(f"{n:10s} launches {cnt.value} avg {ms.value / cnt.value * 1000:.1f} us  "
              f"{by.value / (ms.value / 1000) / 1e9:.0f} GB/s", flush=True)
if ref is not None:
    mr = ref.model(cfg7, bf16=True, layers=(2, 3), with_head=False)
    bo = mr.bank(2, 3)
    a = bo.forward(2, 3, h[:4], list(range(4)))
    print("7B layer rel err (4 rows)", rel(out[:4], a), flush=True)
