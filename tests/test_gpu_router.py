"""GPU tests of the multi-device front end: a Router over one FAST
ServerEngine per device (two engine replicas when the box has one GPU) and
the Batcher in front of it, driven by concurrent frame-level clients (one
thread each, like FrameServer's connection threads, transport.cpp:565-581).

Every session decoded through the batching queue reproduces, bit for bit
(tokens, committed logits, accepted-per-step), the same decode run alone
through one server: placement is sticky and every FAST kernel is batch
invariant, so sharing a weight pass never changes a row's result."""
import threading

import numpy as np
import pytest

import paper_2602_16760_b200 as sfg
import pyoracle as po

pytestmark = pytest.mark.gpu


def _devices():
    try:
        import torch
        return max(1, torch.cuda.device_count())
    except Exception:
        return 1


@pytest.fixture(scope="module")
def replicas(port):
    cfg = po.tiny_cfg()
    m = port.model(cfg, bf16=True)
    mc = sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__})
    ndev = min(2, _devices())
    engines = [sfg.Engine(mc, math=sfg.FAST, params=m.params(), device=i % ndev) for i in range(2)]
    return cfg, engines


def test_batched_sessions_across_replicas_equal_solo_decodes(replicas):
    cfg, engines = replicas
    split = 1
    servers = [sfg.ServerEngine(e, sfg.ServerConfig(split, cfg.n_layers - split)) for e in engines]
    router = sfg.Router(servers)
    bq = sfg.Batcher(router)
    la = sfg.LookaheadConfig(ngram_n=3, window_w=5, max_candidates_g=5)
    rng = np.random.default_rng(3)
    prompts = [rng.integers(0, cfg.vocab_size, 12).tolist() for _ in range(6)]
    prompts[1] = [7, 7, 7, 7, 7, 7, 7, 7]  # a repetitive prompt: pool hits, larger batches
    results, errors = [None] * len(prompts), []

    def client(i):
        try:
            cl = sfg.SplitClient(engines[0], sfg.SplitConfig(split, split, sfg.F32), bq.handler,
                                 session_id=f"sess-{i}")
            results[i] = sfg.decode_lookahead(cl, prompts[i], 24, la, want_logits=True)
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    ts = [threading.Thread(target=client, args=(i,)) for i in range(len(prompts))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errors, errors
    assert sorted(router.load()) == [3, 3]
    # solo reference: each prompt alone, one server, frame path, no queue
    solo_srv = sfg.ServerEngine(engines[0], sfg.ServerConfig(split, cfg.n_layers - split))
    for i, p in enumerate(prompts):
        solo = sfg.decode_lookahead(sfg.SplitClient(engines[0], sfg.SplitConfig(split, split, sfg.F32), solo_srv,
                                                    session_id=f"solo-{i}", frames=True), p, 24, la,
                                    want_logits=True)
        assert results[i].tokens == solo.tokens, i
        assert results[i].step_accepted == solo.step_accepted, i
        assert np.array_equal(results[i].committed_logits, solo.committed_logits), i
    st = bq.stats()
    print("batcher:", st, "shared weight passes:", [s.shared_passes() for s in servers])
    assert st["frames"] >= sum(r.steps + 1 for r in results)
