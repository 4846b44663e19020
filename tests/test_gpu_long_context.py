"""Long-context parity of the FAST path (configs[4] builds a 2k-token KV
context): at >= 2048 cached keys the layer-stack megakernel's attention —
per-(row, kv head) items (SFG_ATTN=rows) or key-chunked items merged over
16+ chunks of 128 keys (SFG_ATTN=chunked) — and the prompt path (attention
sized by the cache length) must stay within the FAST tolerance of the CPU
oracle, including lookahead branch masks and a keep/compaction step at that
depth (tinyformer.cpp:442-489 attention, decoding.cpp:275-293 branch mask,
tinyformer.cpp:282-308 resolve).

    per-row ||h_gpu - h_ref||_2 / ||h_ref||_2 <= 1e-5

Shape: hidden 512 = 4 q heads x 128 over 1 kv head (GQA 4, head_dim 128),
ffn 512, max_seq_len 4096 — CPU-cheap for the oracle (2048-row prefill in
seconds) with the 7B head geometry.  The attention design is fixed per
process, so the chunked run re-executes this file in a child process.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2602_16760_b200 as sfg
import pyoracle as po

pytestmark = pytest.mark.gpu
TOL = 1e-5
PRIOR = 2048
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def long_cfg():
    return po.ModelCfg(vocab_size=512, n_layers=4, hidden_dim=512, n_heads=4, n_kv_heads=1, head_dim=128,
                       ffn_dim=512, max_seq_len=4096, rope_base=1e6, rms_eps=1e-5, seed=77)


def rel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-30)))


def lookahead_step(prior, n_cand=5, w=5):
    """decode_lookahead_with_pool's batch at context `prior`: anchor, W window
    rows (prefix law), then n_cand 2-token candidate branches that see the
    prefix + anchor + their own branch only (decoding.cpp:251-293)."""
    rows = 1 + w + 2 * n_cand
    kv = prior + rows
    mask = np.full((rows, kv), -np.inf, dtype=np.float32)
    pos = [prior] + [prior + 1 + i for i in range(w)]
    for i in range(1 + w):
        mask[i, :prior + i + 1] = 0.0
    for b in range(n_cand):
        r0 = 1 + w + 2 * b
        for j in range(2):
            mask[r0 + j, :prior + 1] = 0.0
            mask[r0 + j, prior + r0:prior + r0 + j + 1] = 0.0
            pos.append(prior + 1 + j)
    return mask, pos


def _run_long_context(port):
    cfg = long_cfg()
    m = port.model(cfg, bf16=True)
    eng = sfg.Engine(sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__}),
                     math=sfg.FAST, params=m.params())
    lb, le = 1, 3
    bo, bg = m.bank(lb, le), eng.bank(lb, le)
    rng = np.random.default_rng(5)
    # prompt pass: 2048 rows through the per-GEMM prompt path
    h = (rng.standard_normal((PRIOR, cfg.hidden_dim)) * 0.5).astype(np.float32)
    a = bo.forward(lb, le, h, list(range(PRIOR)))
    b = eng.forward_layers(lb, le, h, list(range(PRIOR)), bg)
    assert rel(b, a) <= TOL, ("prefill", rel(b, a))
    bo.mark_committed(PRIOR)
    bg.mark_committed(PRIOR)
    # lookahead step at prior 2048 (megakernel: 16 rows, branch mask)
    mask, pos = lookahead_step(PRIOR)
    x = (rng.standard_normal((len(pos), cfg.hidden_dim)) * 0.5).astype(np.float32)
    a1 = bo.forward(lb, le, x, pos, mask)
    b1 = eng.forward_layers(lb, le, x, pos, bg, mask=mask)
    assert rel(b1, a1) <= TOL, ("step 1", rel(b1, a1))
    # accept the anchor + candidate 0 (keep = [0, 6, 7]): in-place compaction at
    # depth 2048, then the next lookahead step over the compacted cache
    keep = [0, 6, 7]
    bo.resolve(keep)
    bg.resolve(keep)
    assert bo.state() == (PRIOR + 3, PRIOR + 3) and (bg.len(), bg.committed_len()) == (PRIOR + 3, PRIOR + 3)
    mask2, pos2 = lookahead_step(PRIOR + 3)
    x2 = (rng.standard_normal((len(pos2), cfg.hidden_dim)) * 0.5).astype(np.float32)
    a2 = bo.forward(lb, le, x2, pos2, mask2)
    b2 = eng.forward_layers(lb, le, x2, pos2, bg, mask=mask2)
    assert rel(b2, a2) <= TOL, ("step 2", rel(b2, a2))
    # a single sequential row at the same depth: its result is the lookahead
    # anchor's, bitwise (batch invariance over 2k keys)
    bg2 = eng.bank(lb, le)
    eng.forward_layers(lb, le, h, list(range(PRIOR)), bg2)
    bg2.mark_committed(PRIOR)
    one = eng.forward_layers(lb, le, x[:1], pos[:1], bg2)
    assert np.array_equal(one[0], b1[0])
    return rel(b, a), rel(b1, a1), rel(b2, a2)


def test_long_context_rows_attention(port):
    # at 2048 cached keys the automatic choice is the chunked design: the
    # per-row design is forced in a child process (the choice is read once)
    if os.environ.get("SFG_ATTN") == "rows":
        print("rel errors (prefill, step, step after resolve):", _run_long_context(port))
        return
    if os.environ.get("SFG_ATTN") == "chunked":
        pytest.skip("this process runs the chunked design")
    env = dict(os.environ, SFG_ATTN="rows")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu",
                        os.path.join(ROOT, "tests", "test_gpu_long_context.py") + "::test_long_context_rows_attention"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_long_context_auto_attention(port):
    """No SFG_ATTN: the session picks the key-chunked design at 2048 cached keys."""
    if os.environ.get("SFG_ATTN"):
        pytest.skip("a design is forced in this process")
    print("rel errors (prefill, step, step after resolve):", _run_long_context(port))


def test_long_context_chunked_attention(port):
    if os.environ.get("SFG_ATTN") == "chunked":
        print("rel errors (prefill, step, step after resolve):", _run_long_context(port))
        return
    env = dict(os.environ, SFG_ATTN="chunked")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu",
                        os.path.join(ROOT, "tests", "test_gpu_long_context.py") + "::test_long_context_chunked_attention"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def _run_7b_width(ref):
    """One Mistral-7B-width middle layer (d=4096, 32q/8kv x128, ffn 14336) at
    prior 512: the GPU bank's 512 cached entries (its own prompt pass) are
    installed in the reference's CacheBank, then a 16-row lookahead step with
    the branch mask runs on both (the reference's own forward_layers)."""
    cfg = po.mistral7b_cfg(max_seq_len=1024)
    prior = 512
    eng = sfg.Engine(sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__}),
                     math=sfg.FAST, layers=(2, 3), with_embedding=False, with_head=False)
    mr = ref.model(cfg, bf16=True, layers=(2, 3), with_head=False)
    rng = np.random.default_rng(12)
    bg, br = eng.bank(2, 3), mr.bank(2, 3)
    h = (rng.standard_normal((prior, cfg.hidden_dim)) * 0.5).astype(np.float32)
    eng.forward_layers(2, 3, h, list(range(prior)), bg)
    bg.mark_committed(prior)
    k = np.zeros((cfg.n_kv_heads, cfg.max_seq_len, cfg.head_dim), np.float32)
    v = np.zeros_like(k)
    for hh in range(cfg.n_kv_heads):
        for p_ in range(prior):
            k[hh, p_], v[hh, p_] = bg.kv(2, hh, p_)
    br.load_layer(2, k, v, prior)
    br.mark_committed(prior)
    mask, pos = lookahead_step(prior)
    x = (rng.standard_normal((len(pos), cfg.hidden_dim)) * 0.5).astype(np.float32)
    a = br.forward(2, 3, x, pos, mask)
    b = eng.forward_layers(2, 3, x, pos, bg, mask=mask)
    return rel(b, a)


def test_7b_width_layer_prior_512_rows_attention(ref):
    if os.environ.get("SFG_ATTN", "rows") != "rows":
        pytest.skip("this process runs the chunked design")
    e = _run_7b_width(ref)
    print("7B-width layer at prior 512, rel error:", e)
    assert e <= TOL


def test_7b_width_layer_prior_512_chunked_attention(ref):
    if os.environ.get("SFG_ATTN") == "chunked":
        e = _run_7b_width(ref)
        print("7B-width layer at prior 512 (chunked), rel error:", e)
        assert e <= TOL
        return
    env = dict(os.environ, SFG_ATTN="chunked")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu",
                        os.path.join(ROOT, "tests", "test_gpu_long_context.py") +
                        "::test_7b_width_layer_prior_512_chunked_attention"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("math", ["exact", "fast"])
def test_long_keep_list_compaction_equals_oracle(port, math):
    """CacheBank::resolve with a keep list longer than one 64-row compaction
    chunk (tinyformer.cpp:282-308): 150 kept entries of a 200-row provisional
    tail, each moved down by its own offset.  Every kept K/V entry equals the
    oracle's (bitwise in EXACT math, where the cached values themselves are
    bitwise), and the next step over the compacted cache stays in tolerance."""
    cfg = po.tiny_cfg()
    m = port.model(cfg, bf16=True)
    eng = sfg.Engine(sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__}),
                     math=sfg.EXACT if math == "exact" else sfg.FAST, params=m.params())
    lb, le = 1, 3
    bo, bg = m.bank(lb, le), eng.bank(lb, le)
    rng = np.random.default_rng(8)
    h = (rng.standard_normal((40, cfg.hidden_dim)) * 0.5).astype(np.float32)
    bo.forward(lb, le, h, list(range(40)))
    eng.forward_layers(lb, le, h, list(range(40)), bg)
    bo.mark_committed(40)
    bg.mark_committed(40)
    t = (rng.standard_normal((200, cfg.hidden_dim)) * 0.5).astype(np.float32)
    bo.forward(lb, le, t, list(range(40, 240)))
    eng.forward_layers(lb, le, t, list(range(40, 240)), bg)
    keep = sorted(rng.choice(200, size=150, replace=False).tolist())
    bo.resolve(keep)
    bg.resolve(keep)
    assert bo.state() == (190, 190) and (bg.len(), bg.committed_len()) == (190, 190)
    for layer in (lb, le - 1):
        for pos in list(range(38, 42)) + [100, 150, 188, 189]:
            kg, vg = bg.kv(layer, cfg.n_kv_heads - 1, pos)
            ko, vo = bo.kv(layer, cfg.n_kv_heads - 1, pos)
            if math == "exact":
                assert np.array_equal(kg, ko) and np.array_equal(vg, vo), (layer, pos)
            else:
                assert rel(kg[None], ko[None]) <= TOL and rel(vg[None], vo[None]) <= TOL, (layer, pos)
    x = (rng.standard_normal((3, cfg.hidden_dim)) * 0.5).astype(np.float32)
    a = bo.forward(lb, le, x, [190, 191, 192])
    b = eng.forward_layers(lb, le, x, [190, 191, 192], bg)
    assert (np.array_equal(a, b) if math == "exact" else rel(b, a) <= TOL)
