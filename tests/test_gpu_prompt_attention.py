"""The tensor-core causal prompt attention (sfg_attn_tc.cu, head_dim 128) on
the FAST prompt path against the CPU oracle (tinyformer.cpp:442-489 attention
under the prefix mask law, server.cpp:203-224 prompt handling):

* every GQA group the kernel tiles (128 queries = 128 / G rows x G heads per
  CTA: G = 1, 2, 4, 8), so the query-block shapes and the (row, head) -> TMEM
  lane map are all exercised;
* ragged prompt lengths (the last query block is partial, the last 64-key
  block is partial);
* a second prompt appended to an already cached context (prior > 0: the
  causal limit of row r is prior + r + 1, key blocks span both parts).
    per-row ||h_gpu - h_ref||_2 / ||h_ref||_2 <= 1e-5 (the FAST tolerance)
Prompts longer than 16 rows take the per-GEMM prompt path, whose attention is
attn_prompt_tc_kernel at head_dim 128.
"""
import numpy as np
import pytest

import paper_2602_16760_b200 as sfg
import pyoracle as po

pytestmark = pytest.mark.gpu
TOL = 1e-5


def rel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-30)))


@pytest.mark.parametrize("n_heads,n_kv", [(2, 2), (4, 2), (4, 1), (8, 1)])
def test_prompt_attention_tc_gqa_groups_ragged_and_appended(port, n_heads, n_kv):
    cfg = po.ModelCfg(vocab_size=512, n_layers=4, hidden_dim=n_heads * 128, n_heads=n_heads, n_kv_heads=n_kv,
                      head_dim=128, ffn_dim=512, max_seq_len=1024, rope_base=1e6, rms_eps=1e-5, seed=91 + n_heads)
    m = port.model(cfg, bf16=True)
    eng = sfg.Engine(sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__}),
                     math=sfg.FAST, params=m.params())
    lb, le = 1, 2
    bo, bg = m.bank(lb, le), eng.bank(lb, le)
    rng = np.random.default_rng(n_heads * 10 + n_kv)
    # first prompt: 203 rows (partial last query block and key block)
    p1 = 203
    h = (rng.standard_normal((p1, cfg.hidden_dim)) * 0.5).astype(np.float32)
    a = bo.forward(lb, le, h, list(range(p1)))
    b = eng.forward_layers(lb, le, h, list(range(p1)), bg)
    assert rel(b, a) <= TOL, ("prompt 1", rel(b, a))
    bo.mark_committed(p1)
    bg.mark_committed(p1)
    # second prompt appended at prior 203: 77 rows see keys [0, 203 + r + 1)
    p2 = 77
    h2 = (rng.standard_normal((p2, cfg.hidden_dim)) * 0.5).astype(np.float32)
    pos2 = list(range(p1, p1 + p2))
    a2 = bo.forward(lb, le, h2, pos2)
    b2 = eng.forward_layers(lb, le, h2, pos2, bg)
    assert rel(b2, a2) <= TOL, ("prompt 2 (appended)", rel(b2, a2))
