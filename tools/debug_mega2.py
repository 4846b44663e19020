"""Localise megakernel errors: one layer, tiny config, compare q/KV/h."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import paper_2602_16760_b200 as sfg
import pyoracle as po


def scfg(c):
    return sfg.ModelConfig(**{k: getattr(c, k) for k in po.ModelCfg.__dataclass_fields__})


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


port = po.Port()
for name, cfg in (("tiny", po.tiny_cfg()), ("7b", po.mistral7b_cfg())):
    if name == "tiny":
        m = port.model(cfg, bf16=True)
        eng = sfg.Engine(scfg(cfg), math=sfg.FAST, params=m.params())
        L0, L1 = 0, 1
    else:
        ref = po.Ref()
        m = ref.model(cfg, bf16=True, layers=(2, 3), with_head=False)
        eng = sfg.Engine(scfg(cfg), math=sfg.FAST, layers=(2, 3), with_embedding=False, with_head=False)
        L0, L1 = 2, 3
    rng = np.random.default_rng(1)
    for rows in (1, 2, 5):
        bo, bg = m.bank(L0, L1), eng.bank(L0, L1)
        h = rng.standard_normal((rows, cfg.hidden_dim)).astype(np.float32)
        a = bo.forward(L0, L1, h, list(range(rows)))
        b = eng.forward_layers(L0, L1, h, list(range(rows)), bg)
        kerr = max(rel(bg.kv(L0, hh, p)[0], bo.kv(L0, hh, p)[0]) for hh in range(cfg.n_kv_heads) for p in range(rows))
        verr = max(rel(bg.kv(L0, hh, p)[1], bo.kv(L0, hh, p)[1]) for hh in range(cfg.n_kv_heads) for p in range(rows))
        print(name, "rows", rows, "h rel", rel(b, a), "K rel", kerr, "V rel", verr, "nan", np.isnan(b).any(), flush=True)
