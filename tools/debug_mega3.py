"""Compare megakernel vs per-GEMM intermediate buffers (q, att, act, h)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import paper_2602_16760_b200 as sfg
import pyoracle as po
from paper_2602_16760_b200 import _lib

L = _lib.lib()


def scfg(c):
    return sfg.ModelConfig(**{k: getattr(c, k) for k in po.ModelCfg.__dataclass_fields__})


def buf(bank, which, n):
    out = np.zeros(n, dtype=np.float32)
    _lib.check(L.sfg_debug_bank_buffer(bank.h, which, out.ctypes.data_as(C.POINTER(C.c_float)), n))
    return out


port = po.Port()
cfg = po.tiny_cfg()
m = port.model(cfg, bf16=True)
eng = sfg.Engine(scfg(cfg), math=sfg.FAST, params=m.params())
rng = np.random.default_rng(1)
for rows in (1, 3):
    h = rng.standard_normal((rows, cfg.hidden_dim)).astype(np.float32)
    res = {}
    for mode in (1, 0):
        L.sfg_debug_set_mega(mode)
        b = eng.bank(0, 1)
        out = eng.forward_layers(0, 1, h, list(range(rows)), b)
        res[mode] = {"q": buf(b, 1, rows * cfg.q_dim()), "att": buf(b, 2, rows * cfg.q_dim()),
                     "act": buf(b, 3, rows * cfg.ffn_dim), "h": out}
    for k in ("q", "att", "act", "h"):
        a, bb = res[1][k], res[0][k]
        print("rows", rows, k, "max abs diff", float(np.max(np.abs(a - bb))), "max", float(np.max(np.abs(bb))),
              "first idx", int(np.argmax(np.abs(a - bb) > 1e-3 * max(1e-30, float(np.max(np.abs(bb)))))), flush=True)
# sum-of-squares partials after a 1-row forward, vs numpy on the returned rows
L.sfg_debug_set_mega(1)
h = rng.standard_normal((1, cfg.hidden_dim)).astype(np.float32)
b = eng.bank(0, 1)
out = eng.forward_layers(0, 1, h, [0], b)
tH = cfg.hidden_dim // 128
ssd = buf(b, 4, tH * 16).reshape(tH, 16)
sso = buf(b, 5, tH * 16).reshape(tH, 16)
print("ss_d tiles row0", ssd[:, 0], "expected (after down)", [float(np.sum(out[0, t*128:(t+1)*128].astype(np.float64)**2)) for t in range(tH)])
print("ss_o tiles row0", sso[:, 0])
