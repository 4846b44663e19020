"""configs[3] at the TRUE Mistral NeMo 12B shape: d=5120, 32 q heads x 128
(q_dim 4096 != d), 8 kv heads, ffn 14336.  The reference's validate() rejects
q_dim != hidden (tinyformer.cpp:109-111) but its forward_layers uses q_dim()
throughout (:405-406, :444, :491); oracle/_ref builds that shape's weights
without validate (ref_model_new_unchecked) and runs its own forward_layers.
The engine accepts the shape with sfg_engine_options.extended_shapes = 1.

  * EXACT math: hidden states and K/V entries bitwise equal to the reference;
  * FAST math (the layer-stack megakernel at 16 rows, the prompt path at
    40 rows): per-row relative error <= 1e-5.
"""
import numpy as np
import pytest

import paper_2602_16760_b200 as sfg
import pyoracle as po

pytestmark = pytest.mark.gpu
TOL = 1e-5


def rel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-30)))


def scfg(c):
    return sfg.ModelConfig(**{k: getattr(c, k) for k in po.ModelCfg.__dataclass_fields__})


@pytest.fixture(scope="module")
def nemo_ref(ref):
    cfg = po.nemo12b_cfg(max_seq_len=256)
    return cfg, ref.model(cfg, bf16=True, layers=(2, 3), with_head=False, unchecked=True)


def test_engine_rejects_q_dim_ne_hidden_without_extension():
    cfg = po.nemo12b_cfg(max_seq_len=64)
    with pytest.raises(sfg.SplitError, match="n_heads \\* head_dim must equal hidden_dim"):
        sfg.Engine(scfg(cfg), math=sfg.FAST, layers=(2, 3), with_embedding=False, with_head=False)


def test_nemo12b_true_width_layer_exact_bitwise(nemo_ref):
    cfg, mr = nemo_ref
    eng = sfg.Engine(scfg(cfg), math=sfg.EXACT, layers=(2, 3), with_embedding=False, with_head=False,
                     extended_shapes=True)
    rng = np.random.default_rng(21)
    bg, br = eng.bank(2, 3), mr.bank(2, 3)
    pre = (rng.standard_normal((6, cfg.hidden_dim)) * 0.5).astype(np.float32)
    assert np.array_equal(eng.forward_layers(2, 3, pre, list(range(6)), bg), br.forward(2, 3, pre, list(range(6))))
    bg.mark_committed(6)
    br.mark_committed(6)
    h = (rng.standard_normal((4, cfg.hidden_dim)) * 0.5).astype(np.float32)
    assert np.array_equal(eng.forward_layers(2, 3, h, [6, 7, 8, 9], bg), br.forward(2, 3, h, [6, 7, 8, 9]))
    for pos in (0, 5, 9):
        kg, vg = bg.kv(2, cfg.n_kv_heads - 1, pos)
        kr, vr = br.kv(2, cfg.n_kv_heads - 1, pos)
        assert np.array_equal(kg, kr) and np.array_equal(vg, vr)


def test_nemo12b_true_width_layer_fast_within_tolerance(nemo_ref):
    cfg, mr = nemo_ref
    eng = sfg.Engine(scfg(cfg), math=sfg.FAST, layers=(2, 3), with_embedding=False, with_head=False,
                     extended_shapes=True)
    rng = np.random.default_rng(22)
    bg, br = eng.bank(2, 3), mr.bank(2, 3)
    # prompt path: 40 rows in one pass of three 16-row chunks
    pre = (rng.standard_normal((40, cfg.hidden_dim)) * 0.5).astype(np.float32)
    a0 = br.forward(2, 3, pre, list(range(40)))
    b0 = eng.forward_layers(2, 3, pre, list(range(40)), bg)
    assert rel(b0, a0) <= TOL
    bg.mark_committed(40)
    br.mark_committed(40)
    # a 16-row lookahead-shaped step through the layer-stack megakernel
    mask = np.zeros((16, 56), np.float32)
    for i in range(16):
        mask[i, 40 + i + 1:] = -np.inf
    mask[7:, 41:47] = -np.inf  # candidate rows: prefix + anchor + own branch
    pos = [40 + min(i, 6) for i in range(16)]
    x = (rng.standard_normal((16, cfg.hidden_dim)) * 0.5).astype(np.float32)
    a1 = br.forward(2, 3, x, pos, mask)
    b1 = eng.forward_layers(2, 3, x, pos, bg, mask=mask)
    assert rel(b1, a1) <= TOL
