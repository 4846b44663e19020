"""configs[4] on ONE process over every visible GPU: 1..64 concurrent
Mistral-7B-shape lookahead sessions through the multi-device front end
(Router: sticky least-loaded placement over one FAST server per GPU;
Batcher: per-GPU queue feeding handle_batch), one client thread per session
(FrameServer's thread-per-connection model, transport.cpp:565-581).

    python tools/session_sweep.py [--sessions 1,4,16,64] [--ctx 24] [--tokens 24]

Each session's local side (2+2 layers, LM head) runs on the engine of the
GPU its index maps to; frames cross host memory.  Every session prefills its
prompt first; then all sessions decode together (a barrier), and the point
reports aggregate committed tok/s over that decode phase, the per-session step
time, the mean prefill time and batching statistics.
"""
import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_16760_b200 as sfg  # noqa: E402

H_7B = dict(vocab_size=32768, n_layers=32, hidden_dim=4096, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336,
            max_seq_len=4096, rope_base=1e6, rms_eps=1e-5, seed=1234)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sessions", default="1,4,16,64")
    ap.add_argument("--ctx", type=int, default=24)
    ap.add_argument("--tokens", type=int, default=24)
    ap.add_argument("--gpus", type=int, default=0, help="0: all visible")
    args = ap.parse_args()
    import torch
    ndev = args.gpus or torch.cuda.device_count()
    cfg = sfg.ModelConfig(**H_7B)
    engines = [None] * ndev
    t0 = time.time()

    def mk(d):
        engines[d] = sfg.Engine(cfg, math=sfg.FAST, device=d)

    ts = [threading.Thread(target=mk, args=(d,)) for d in range(ndev)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    print(json.dumps({"gpus": ndev, "engine_init_s": round(time.time() - t0, 1)}), flush=True)
    la = sfg.LookaheadConfig(ngram_n=3, window_w=5, max_candidates_g=5)
    split = 2
    for k in [int(x) for x in args.sessions.split(",")]:
        servers = [sfg.ServerEngine(e, sfg.ServerConfig(split, cfg.n_layers - split, max_sessions=64)) for e in engines]
        router = sfg.Router(servers)
        bq = sfg.Batcher(router)
        prompts = [np.random.default_rng(1000 + i).integers(0, cfg.vocab_size, args.ctx).tolist() for i in range(k)]
        res, errs = [None] * k, []
        # every session prefills first (its prompt frame), then all decode
        # together: aggregate tok/s is the DECODE phase with k sessions live
        gate = threading.Barrier(k)
        L = sfg.lib()
        la_c = sfg._lib.DecodeConfig(2, 5, 3, 5, 1 << 20)

        def client(i):
            d = None
            try:
                cl = sfg.SplitClient(engines[i % ndev], sfg.SplitConfig(split, split, sfg.F16), bq.handler,
                                     session_id=f"sweep-{k}-{i}")
                pool = sfg.NGramPool(3, 1 << 20)
                p = np.asarray(prompts[i], dtype=np.int32)
                d = C.c_void_p()
                tp = time.time()
                sfg._lib.check(L.sfg_decoder_create(cl.h, C.byref(la_c), pool.h, p.ctypes.data_as(C.POINTER(C.c_int32)),
                                                    len(p), args.tokens + 64, C.byref(d)))
                prefill = time.time() - tp
                committed = np.zeros(16, dtype=np.int32)
                n, b = C.c_int32(), C.c_int32()
                gate.wait()
                t0 = time.time()
                toks, steps = 0, 0
                while toks < args.tokens:
                    sfg._lib.check(L.sfg_decoder_step(d, committed.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(n),
                                                      C.byref(b)))
                    toks += n.value
                    steps += 1
                res[i] = (time.time() - t0, toks, steps, prefill)
            except Exception as e:
                errs.append(repr(e))
                try:
                    gate.abort()
                except Exception:
                    pass
            finally:
                if d is not None and d.value:
                    L.sfg_decoder_destroy(d)

        ts = [threading.Thread(target=client, args=(i,)) for i in range(k)]
        tw = time.time()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            print(json.dumps({"sessions": k, "gpus": ndev, "context": args.ctx, "error": errs[0]}), flush=True)
            continue
        dec = max(r[0] for r in res)
        toks = sum(r[1] for r in res)
        st = bq.stats()
        print(json.dumps({"sessions": k, "gpus": ndev, "context": args.ctx,
                          "aggregate_tok_s": toks / dec, "per_session_step_ms": dec / (sum(r[2] for r in res) / k) * 1e3,
                          "prefill_s_mean": round(float(np.mean([r[3] for r in res])), 3),
                          "placement": router.load(), "frames_per_server_batch": st["frames"] / max(1, st["batches"]),
                          "max_server_batch": st["max_batch"],
                          "shared_weight_passes": [s.shared_passes() for s in servers],
                          "attention": os.environ.get("SFG_ATTN", "auto"),
                          "wall_s": round(time.time() - tw, 1)}), flush=True)
        del bq, router, servers


if __name__ == "__main__":
    main()
