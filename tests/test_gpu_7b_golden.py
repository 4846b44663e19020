"""The measured path pinned to the CPU reference at the Mistral-7B shape.

tests/golden/ref_decode_7b_d{2,4,8}.json were produced by the UNMODIFIED
reference (oracle/_ref: SplitClient + decode loop + ServerEngine,
decoding.cpp:111-355, server.cpp:173-265) on the same seeded bf16 weights
(tests/golden/make_golden_7b.py).  The FAST engine — the tcgen05 layer-stack
megakernel that bench.py times, behind the same client/server — must
reproduce, per run:

  * the committed token sequence, bit for bit;
  * accepted-per-step and the batch size of every step;
  * the boundary rows at both crossings of the split (prefix-layer output as
    sent on the wire, middle-layer output as returned) within

        per-row ||h_gpu - h_ref||_2 / ||h_ref||_2 <= BOUNDARY_TOL

    (FAST math: bf16 weights x 3-way bf16-split fp32 activations with fp32
    accumulation in a different order from the reference's serial sums).

Modes: sequential (f32 wire), lookahead W5 N3 G5 (f16 wire, natural pool),
and the bench's forced-B16 workload (junk pool: G continuations for every
key, bench.py seed_pool) on both wires.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2602_16760_b200 as sfg
import pyoracle as po
import wirepy

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BOUNDARY_TOL = 1e-5
FIXTURES = sorted(f[:-5] for f in os.listdir(GOLD) if f.startswith("ref_decode_7b_d") and f.endswith(".json"))


def _load(stem):
    with open(os.path.join(GOLD, f"{stem}.json")) as f:
        doc = json.load(f)
    rows = np.load(os.path.join(GOLD, doc["boundary_rows_file"]))
    return doc, rows


def rel_rows(a, b):
    return np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-30)


@pytest.fixture(scope="module")
def eng7b():
    cfg = po.mistral7b_cfg()
    return sfg.Engine(sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__}),
                      math=sfg.FAST)


def junk_pool(vocab, seed, g, ng=3):
    """bench.py seed_pool: the same update sequence the golden's reference pool saw."""
    import bench
    pool = sfg.NGramPool(ng, 1 << 20)
    bench.seed_pool(sfg._lib, pool, vocab, g, np.random.default_rng(seed))
    return pool


class Recorder:
    """Frame handler between the GPU client and the GPU server that keeps the
    boundary rows (request = prefix output, response = middle-layer output)."""

    def __init__(self, srv, frames):
        self.srv, self.frames, self.req, self.resp = srv, frames, [], []
        self._buf = None
        self.fn = sfg._lib.FRAME_HANDLER(self._handle)

    def _handle(self, ctx, req, n, resp, resp_n):
        q = C.string_at(req, n)
        r = self.srv.handle(q)
        if len(self.req) < self.frames:
            hq, bq = wirepy.decode(q)
            hr, br = wirepy.decode(r)
            if hr["kind"] == "response":
                self.req.append(wirepy.rows_of(hq, bq))
                self.resp.append(wirepy.rows_of(hr, br))
        self._buf = (C.c_uint8 * len(r)).from_buffer_copy(r)
        resp[0] = C.cast(self._buf, C.POINTER(C.c_uint8))
        resp_n[0] = len(r)
        return 0


def _decode(eng, doc, run, client):
    la = sfg.LookaheadConfig(ngram_n=doc["lookahead"]["N"], window_w=doc["lookahead"]["W"],
                             max_candidates_g=doc["lookahead"]["G"], pool_capacity=4096)
    if run["mode"] == 0:
        return sfg.decode_sequential(client, run["prompt"], run["max_new"])
    if run["junk_pool"]:
        jp = doc["junk_pool"]
        pool = junk_pool(doc["config"]["vocab_size"], jp["seed"], jp["per_key"], doc["lookahead"]["N"])
        return sfg.decode_lookahead_with_pool(client, run["prompt"], run["max_new"], la, pool)
    return sfg.decode_lookahead(client, run["prompt"], run["max_new"], la)


@pytest.mark.parametrize("stem", FIXTURES)
def test_7b_tokens_and_acceptance_equal_reference(eng7b, stem):
    """Device-linked client (the bench's `value` path): tokens, accepted-per-step
    and batch sizes identical to the reference's decode."""
    doc, _ = _load(stem)
    depth = doc["split"]
    L = doc["config"]["n_layers"]
    srv = sfg.ServerEngine(eng7b, sfg.ServerConfig(depth, L - depth))
    bad = []
    for i, run in enumerate(doc["runs"]):
        wire = sfg.F32 if run["wire_f32"] else sfg.F16
        cl = sfg.SplitClient(eng7b, sfg.SplitConfig(depth, depth, wire), srv, session_id=f"g{i}")
        out = _decode(eng7b, doc, run, cl)
        if (out.tokens != run["tokens"] or out.step_accepted != run["step_accepted"]
                or out.step_batch != run["step_batch"]):
            bad.append((i, run["name"], out.tokens, run["tokens"], out.step_accepted, run["step_accepted"]))
    assert not bad, bad


@pytest.mark.parametrize("stem", FIXTURES)
def test_7b_boundary_rows_within_tolerance(eng7b, stem):
    """Frame-level client (the bench's `e2e` path): same tokens, and the rows at
    both crossings of the split within BOUNDARY_TOL of the reference's."""
    doc, rows = _load(stem)
    depth = doc["split"]
    L = doc["config"]["n_layers"]
    srv = sfg.ServerEngine(eng7b, sfg.ServerConfig(depth, L - depth))
    worst = {"req": 0.0, "resp": 0.0}
    checked = 0
    for i, run in enumerate(doc["runs"]):
        if not run["boundary_frames"]:
            continue
        rec = Recorder(srv, run["boundary_frames"])
        wire = sfg.F32 if run["wire_f32"] else sfg.F16
        cl = sfg.SplitClient(eng7b, sfg.SplitConfig(depth, depth, wire), (C.cast(rec.fn, C.c_void_p), None),
                             session_id=f"b{i}")
        out = _decode(eng7b, doc, run, cl)
        assert out.tokens == run["tokens"], (i, run["name"])
        for f, nrows in enumerate(run["boundary_rows"]):
            for side, got in (("req", rec.req[f]), ("resp", rec.resp[f])):
                want = rows[f"r{i}_f{f}_{side}"]
                assert got.shape == want.shape == (nrows, doc["config"]["hidden_dim"])
                worst[side] = max(worst[side], float(rel_rows(got, want).max()))
                checked += nrows
    print(f"7B {stem}: boundary rows checked {checked}, worst rel err {worst}")
    assert checked > 0
    assert worst["req"] <= BOUNDARY_TOL and worst["resp"] <= BOUNDARY_TOL, worst
