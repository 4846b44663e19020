"""Batch invariance of the FAST megakernel at the 7B shape (dev tool): row 0
of a 16-row batch must equal the same row run alone, bitwise."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import paper_2602_16760_b200 as sfg
import pyoracle as po

cfg = po.mistral7b_cfg(max_seq_len=512)
NL = int(os.environ.get("NL", "2"))
eng = sfg.Engine(sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__}), math=sfg.FAST,
                 layers=(2, 2 + NL), with_embedding=False, with_head=False)
rng = np.random.default_rng(0)
for prior in (20, 40, 120, 130):
    pre = (rng.standard_normal((prior, 4096)) * 0.5).astype(np.float32)
    h16 = (rng.standard_normal((16, 4096)) * 0.5).astype(np.float32)
    outs = {}
    for rows in (1, 16):
        bank = eng.bank(2, 2 + NL)
        eng.forward_layers(2, 2 + NL, pre, list(range(prior)), bank)
        bank.mark_committed(prior)
        # lookahead-like mask: every row sees the prefix and itself
        mask = np.full((rows, prior + rows), -np.inf, dtype=np.float32)
        mask[:, :prior] = 0.0
        for i in range(rows):
            mask[i, prior + i] = 0.0
        outs[rows] = eng.forward_layers(2, 2 + NL, h16[:rows], [prior + i for i in range(rows)], bank, mask)
    d = np.abs(outs[1][0] - outs[16][0]).max()
    print(f"prior {prior}: row0 bitwise {np.array_equal(outs[1][0], outs[16][0])} maxdiff {d:.3g}")
