"""CPU tests: the oracle is pinned before it is trusted.

* the C restatement (oracle/liboracle.so) reproduces the reference's own
  known answers (frozen stream, binary16 constants, verify_greedy, NGramPool);
* it reproduces the golden fixtures generated from the UNMODIFIED reference
  (tests/golden/ref_*.json, made by tests/golden/make_golden.py);
* where oracle/_ref is available it is bit-identical to the reference on the
  split decode paths (tokens, committed logits, step logs);
* the device expf port (paper_2602_16760_b200/csrc/sfg_expf.h) matches the
  host libm on all 2^32 inputs.
"""
import hashlib
import math
import os
import subprocess

import numpy as np
import pytest

import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def _f(v):
    return float(v) if not isinstance(v, str) else float(v.replace("inf", "inf"))


# ── reference known answers ──────────────────────────────────────────────
def test_frozen_stream_port(port, golden):
    ka = golden["reference_known_answers"]["frozen_stream"]
    m = port.model(po.desk_cfg(), bf16=False)
    assert m.generate(ka["prompt"], 24) == ka["expected"]


def test_frozen_stream_ref(ref, golden):
    ka = golden["reference_known_answers"]["frozen_stream"]
    m = ref.model(po.desk_cfg(), bf16=False)
    assert m.generate(ka["prompt"], 24) == ka["expected"]


@pytest.mark.parametrize("which", ["port", "ref", "sfg"])
def test_f16_constants_and_clamp(which, request, golden):
    ka = golden["reference_known_answers"]
    if which == "sfg":
        import paper_2602_16760_b200 as sfg
        enc, dec = sfg.f32_to_f16_bits, sfg.f16_bits_to_f32
    else:
        lib = request.getfixturevalue(which)
        enc, dec = lib.f32_to_f16, lib.f16_to_f32
    for v, b in ka["f16_constants"]["encode"]:
        assert enc(_f(v)) == b
    for b, v in ka["f16_constants"]["decode"]:
        assert dec(b) == _f(v)
    cnt = [0]
    for v, b in ka["f16_clamp"]["encode"]:
        assert enc(v, cnt) == b
    assert cnt[0] == ka["f16_clamp"]["clamped_after_two"]
    cnt = [0]
    back = [dec(enc(v, cnt)) for v in ka["f16_clamp"]["values"]]
    assert cnt[0] == ka["f16_clamp"]["values_clamped"]
    assert back == ka["f16_clamp"]["values_back"]


def test_f16_roundtrip_within_one_ulp(port):
    # test_wire.cpp:78-88: |x| in [1e-5, 1e4), round trip within one half-ulp
    rng = np.random.default_rng(42)
    for _ in range(3000):
        mag = 10.0 ** (rng.integers(0, 9000) / 1000.0 - 5.0)
        x = float(np.float32(mag * (1 if rng.integers(0, 2) else -1)))
        rt = port.f16_to_f32(port.f32_to_f16(x))
        e = math.frexp(abs(x) if abs(x) >= 6.1e-5 else 6.1035156e-5)[1] - 1
        assert abs(rt - x) <= math.ldexp(1.0, e - 10)


def test_f16_codec_port_equals_ref_and_sfg(port, ref):
    import paper_2602_16760_b200 as sfg
    # every binary16 pattern decodes identically
    for b in range(0, 65536, 7):
        a, r, s = port.f16_to_f32(b), ref.f16_to_f32(b), sfg.f16_bits_to_f32(b)
        assert (math.isnan(a) and math.isnan(r) and math.isnan(s)) or (a == r == s and math.copysign(1, a) == math.copysign(1, r) == math.copysign(1, s))
    # encode: edge values + random bit patterns
    rng = np.random.default_rng(7)
    vals = list(np.frombuffer(rng.integers(0, 2**32, 20000, dtype=np.uint64).astype(np.uint32).tobytes(), dtype=np.float32))
    vals += [65504.0, 65519.0, 65520.0, 6.0e-8, 2.98e-8, 2.9802322e-8, 5.96e-8, -0.0, 1e-45, 3e38]
    for v in vals:
        c1, c2, c3 = [0], [0], [0]
        assert port.f32_to_f16(float(v), c1) == ref.f32_to_f16(float(v), c2) == sfg.f32_to_f16_bits(float(v), c3)
        assert c1 == c2 == c3


@pytest.mark.parametrize("which", ["port", "ref"])
def test_verify_greedy_known_answers(which, request, golden):
    lib = request.getfixturevalue(which)
    ka = golden["reference_known_answers"]["verify_greedy"]
    lg = np.asarray(ka["logits"], dtype=np.float32)
    for c in ka["cases"]:
        acc, com = lib.verify_greedy(lg, 0, c["guesses"], c["anchor"])
        assert acc == c["accepted"] and com == c["committed"]


def _pool_script(pool):
    # test_decoding.cpp:63-96
    pool.update([10, 11, 12, 13], [20, 21, 22, 23])
    assert pool.size() == 2
    assert pool.lookup(10, 2) == [[21, 22]]
    assert pool.lookup(99, 2) == []
    pool.update([10, 1, 2], [0, 30, 31])
    assert pool.lookup(10, 2) == [[30, 31], [21, 22]]
    assert pool.lookup(10, 1) == [[30, 31]]
    pool.update([50, 1, 2], [0, 60, 61])
    assert pool.size() == 4
    pool.update([51, 1, 2], [0, 70, 71])
    assert pool.size() == 4
    assert pool.lookup(10, 2) == [[30, 31]]
    pool.update([50, 1, 2], [0, 60, 61])
    assert pool.size() == 4


@pytest.mark.parametrize("which", ["port", "ref", "sfg"])
def test_ngram_pool_known_answers(which, request):
    if which == "sfg":
        import paper_2602_16760_b200 as sfg
        pool = sfg.NGramPool(3, 4)
    else:
        pool = request.getfixturevalue(which).pool(3, 4)
    _pool_script(pool)


def test_pool_randomised_port_ref_sfg(port, ref):
    import paper_2602_16760_b200 as sfg
    rng = np.random.default_rng(3)
    pools = [port.pool(3, 16), ref.pool(3, 16), sfg.NGramPool(3, 16)]
    for _ in range(300):
        w = int(rng.integers(3, 7))
        prev = rng.integers(0, 6, w).tolist()
        cur = rng.integers(0, 6, w).tolist()
        for p in pools:
            p.update(prev, cur)
        k = int(rng.integers(0, 6))
        g = int(rng.integers(0, 5))
        outs = [p.lookup(k, g) for p in pools]
        assert outs[0] == outs[1] == outs[2]
        assert pools[0].size() == pools[1].size() == pools[2].size()


# ── golden fixtures from the unmodified reference ─────────────────────────
def test_port_reproduces_ref_monolithic_golden(port, golden):
    for r in golden["ref_monolithic_desk"]["runs"]:
        m = port.model(po.desk_cfg(), bf16=r["bf16"])
        toks, lg = m.generate(r["prompt"], 24, want_logits=True)
        assert toks == r["tokens"]
        assert sha(lg) == r["logits_sha256"]


@pytest.mark.parametrize("name", ["ref_decode_desk", "ref_decode_tiny"])
def test_port_reproduces_ref_decode_golden(port, golden, name):
    g = golden[name]
    cfg = po.ModelCfg(**g["config"])
    m = port.model(cfg, bf16=True)
    runs = g["runs"] if name == "ref_decode_desk" else g["runs"][::3]
    for r in runs:
        dc = po.DecodeCfg(mode=r["mode"], prefix_layers=g["split"], suffix_layers=g["split"],
                          wire_f32=r["wire_f32"], window_w=5, ngram_n=3, max_candidates_g=5)
        out = port.decode(m, dc, r["prompt"], r["max_new"], want_logits=True)
        assert out.tokens == r["tokens"]
        assert out.step_batch == r["step_batch"]
        assert out.step_accepted == r["step_accepted"]
        assert sha(out.logits) == r["logits_sha256"]


# ── port == reference (live) ──────────────────────────────────────────────
def test_port_params_equal_ref(port, ref):
    for cfg in (po.desk_cfg(), po.desk_cfg(seed=777)):
        for bf16 in (False, True):
            assert np.array_equal(port.model(cfg, bf16=bf16).params(), ref.model(cfg, bf16=bf16).params())


def test_port_forward_resolve_crop_equal_ref(port, ref):
    cfg = po.desk_cfg()
    mp, mr = port.model(cfg, bf16=True), ref.model(cfg, bf16=True)
    rng = np.random.default_rng(11)
    bp, br = mp.bank(1, 5), mr.bank(1, 5)
    h = rng.standard_normal((5, cfg.hidden_dim)).astype(np.float32)
    a, b = bp.forward(1, 5, h, list(range(5))), br.forward(1, 5, h, list(range(5)))
    assert np.array_equal(a, b)
    bp.mark_committed(5), br.mark_committed(5)
    # branch-shaped mask: rows see prefix + own subset
    kv = 5 + 4
    mask = np.full((4, kv), -np.inf, dtype=np.float32)
    mask[:, :5] = 0
    mask[0, 5] = 0
    mask[1, 5:7] = 0
    mask[2, [5, 7]] = 0
    mask[3, [5, 7, 8]] = 0
    h2 = rng.standard_normal((4, cfg.hidden_dim)).astype(np.float32)
    a, b = bp.forward(1, 5, h2, [5, 6, 6, 7], mask), br.forward(1, 5, h2, [5, 6, 6, 7], mask)
    assert np.array_equal(a, b)
    for bank in (bp, br):
        bank.resolve([1, 3])
    assert bp.state() == br.state() == (7, 7)
    for layer in range(1, 5):
        for pos in range(7):
            ka, va = bp.kv(layer, 1, pos)
            kb, vb = br.kv(layer, 1, pos)
            assert np.array_equal(ka, kb) and np.array_equal(va, vb)
    for bank in (bp, br):
        bank.crop(6)
    assert bp.state() == br.state()
    with pytest.raises(po.OracleError) as e1:
        bp.resolve([0])
    with pytest.raises(po.OracleError) as e2:
        br.resolve([0])
    assert str(e1.value) == str(e2.value)


@pytest.mark.parametrize("mode", [0, 2])
@pytest.mark.parametrize("wire_f32", [1, 0])
def test_port_decode_equals_ref(port, ref, mode, wire_f32):
    cfg = po.desk_cfg(seed=4321)
    mp, mr = port.model(cfg, bf16=True), ref.model(cfg, bf16=True)
    rng = np.random.default_rng(5 + mode + 7 * wire_f32)
    for _ in range(3):
        prompt = rng.integers(0, cfg.vocab_size, int(rng.integers(3, 12))).tolist()
        dc = po.DecodeCfg(mode=mode, wire_f32=wire_f32, window_w=5, ngram_n=3, max_candidates_g=5)
        a = port.decode(mp, dc, prompt, 30, want_logits=True)
        b = ref.decode(mr, dc, prompt, 30, want_logits=True)
        assert a.tokens == b.tokens and a.step_batch == b.step_batch and a.step_accepted == b.step_accepted
        assert np.array_equal(a.logits, b.logits)


def test_lookahead_equals_sequential_oracle(port):
    # test_metrics.cpp:187-203: lookahead logits bit-identical to sequential
    cfg = po.desk_cfg()
    m = port.model(cfg, bf16=True)
    for prompt in ([3, 1, 4, 1, 5, 9, 2, 6], [9, 9, 9, 9, 9, 9]):
        s = port.decode(m, po.DecodeCfg(mode=0), prompt, 40, want_logits=True)
        la = port.decode(m, po.DecodeCfg(mode=2, window_w=5, ngram_n=3, max_candidates_g=5), prompt, 40,
                         want_logits=True)
        assert s.tokens == la.tokens
        assert np.array_equal(s.logits, la.logits)


# ── device expf port vs host libm, all 2^32 inputs ────────────────────────
def test_expf_port_exhaustive(tmp_path):
    src = os.path.join(ROOT, "tests", "tools", "expf_exhaustive.c")
    exe = str(tmp_path / "expf_exh")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe, src, "-lm", "-lpthread"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches 0" in r.stdout


def test_relaxed_port_equals_reference_forward_q_dim_ne_hidden(port, ref):
    """NeMo-12B geometry (q_dim != hidden_dim) at a small width: the relaxed C
    restatement is bit-identical to the reference's OWN forward_layers run on
    that shape (weights built without ModelConfig::validate, which is the only
    reference code that rejects it; forward_layers uses q_dim() throughout,
    tinyformer.cpp:405-406, :444, :491) - prompt pass, branch-masked step,
    resolve, and the K/V entries."""
    cfg = po.ModelCfg(vocab_size=256, n_layers=4, hidden_dim=160, n_heads=4, n_kv_heads=2, head_dim=32,
                      ffn_dim=192, max_seq_len=64, rope_base=1e6, seed=99)  # q_dim 128 != 160
    port.set_relaxed_validate(True)
    try:
        mp = port.model(cfg, bf16=True, layers=(1, 3))
        with pytest.raises(po.OracleError):
            port.set_relaxed_validate(False)
            port.model(cfg, bf16=True, layers=(1, 3))
        port.set_relaxed_validate(True)
        mr = ref.model(cfg, bf16=True, layers=(1, 3), with_head=False, unchecked=True)
        with pytest.raises(po.OracleError, match="n_heads \\* head_dim must equal hidden_dim"):
            ref.model(cfg, bf16=True, layers=(1, 3), with_head=False)
        rng = np.random.default_rng(3)
        bp, br = mp.bank(1, 3), mr.bank(1, 3)
        h = (rng.standard_normal((9, cfg.hidden_dim)) * 0.5).astype(np.float32)
        assert np.array_equal(bp.forward(1, 3, h, list(range(9))), br.forward(1, 3, h, list(range(9))))
        bp.mark_committed(9)
        br.mark_committed(9)
        mask = np.zeros((3, 12), np.float32)
        mask[1, 10] = -np.inf
        mask[2, 10:] = -np.inf
        x = (rng.standard_normal((3, cfg.hidden_dim)) * 0.5).astype(np.float32)
        assert np.array_equal(bp.forward(1, 3, x, [9, 10, 10], mask), br.forward(1, 3, x, [9, 10, 10], mask))
        bp.resolve([0, 2])
        br.resolve([0, 2])
        for l, hh, p in ((1, 0, 3), (2, 1, 9), (2, 1, 10)):
            kp, vp = bp.kv(l, hh, p)
            kr, vr = br.kv(l, hh, p)
            assert np.array_equal(kp, kr) and np.array_equal(vp, vr)
    finally:
        port.set_relaxed_validate(False)
