"""Dev check of the FAST megakernel path: tiny + 7B-shape decode through the
linked client with graphs off/on, error localisation (SFG_DEBUG=1)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import paper_2602_16760_b200 as sfg
import pyoracle as po
from paper_2602_16760_b200 import _lib


def scfg(c):
    return sfg.ModelConfig(**{k: getattr(c, k) for k in po.ModelCfg.__dataclass_fields__})


def rel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-30)))


port = po.Port()
cfg = po.tiny_cfg()
m = port.model(cfg, bf16=True)
eng = sfg.Engine(scfg(cfg), math=sfg.FAST, params=m.params())
rng = np.random.default_rng(1)
for rows in (1, 5, 16):
    bo, bg = m.bank(0, 4), eng.bank(0, 4)
    h = rng.standard_normal((rows, cfg.hidden_dim)).astype(np.float32)
    a = bo.forward(0, 4, h, list(range(rows)))
    b = eng.forward_layers(0, 4, h, list(range(rows)), bg)
    print("tiny mega rows", rows, "rel", rel(b, a), flush=True)
for graphs in (0, 1):
    _lib.lib().sfg_set_graphs(graphs)
    srv = sfg.ServerEngine(eng, sfg.ServerConfig(1, 3))
    la = sfg.LookaheadConfig(ngram_n=3, window_w=5, max_candidates_g=5)
    prompt = [3, 1, 4, 1, 5, 9, 2, 6]
    try:
        s = sfg.decode_sequential(sfg.SplitClient(eng, sfg.SplitConfig(1, 1, sfg.F32), srv), prompt, 30,
                                  want_logits=True)
        la_ = sfg.decode_lookahead(sfg.SplitClient(eng, sfg.SplitConfig(1, 1, sfg.F32), srv), prompt, 30, la,
                                   want_logits=True)
        ref = port.decode(m, po.DecodeCfg(mode=2, prefix_layers=1, suffix_layers=1, wire_f32=1, window_w=5,
                                          ngram_n=3, max_candidates_g=5), prompt, 30, want_logits=True)
        print("graphs", graphs, "seq==la tokens", s.tokens == la_.tokens, "bitwise",
              np.array_equal(s.committed_logits, la_.committed_logits), "tokens==oracle", la_.tokens == ref.tokens,
              "rel", rel(la_.committed_logits, ref.logits), flush=True)
    except Exception as e:
        print("graphs", graphs, "ERROR", e, flush=True)
