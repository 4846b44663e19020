"""Regenerates tests/golden/ref_decode_7b*.json (+ boundary rows .npz) from the
UNMODIFIED reference compiled in place (oracle/_ref/libsplitf_ref.so) at the
Mistral-7B shape the bench measures (BASELINE configs[1]/[2]).

    python tests/golden/make_golden_7b.py --depth 2 [--threads 8]
    python tests/golden/make_golden_7b.py --depth 4
    python tests/golden/make_golden_7b.py --depth 8

Weights: init_weights(seed 1234) rounded to bf16 RNE (SURVEY §8(c) parity
protocol step 1), materialised by ONE walk of the reference stream into a
client part (embedding, prefix + suffix layers, head) and a server part
(middle layers) so the 29 GB fp32 model is held once (ref_split_models).
Decodes run through the reference's own SplitClient + decode loop
(decoding.cpp:111-355) against one shared reference ServerEngine
(server.cpp:173-265), one host thread per decode.  Modes:

  seq-f32   decode_sequential, f32 wire             (records boundary rows)
  la-f16    decode_lookahead, W5 N3 G5, f16 wire     (natural pool)
  b16-f32   decode_lookahead_with_pool, junk pool (G continuations for
            every key, the bench's forced-B16 workload), f32 wire
                                                     (records boundary rows)
  b16-f16   the same on the f16 wire

The boundary rows are the fp32 rows each side of the server as the
reference saw them: request rows (prefix-layer output) and response rows
(middle-layer output) of the first exchanges.
"""
import argparse
import ctypes as C
import json
import os
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as po  # noqa: E402

_i32p = C.POINTER(C.c_int32)
_f32p = C.POINTER(C.c_float)
W, NG, G = 5, 3, 5
JUNK_SEED = 7  # bench.py seed_pool


def junk_pool(lib, vocab):
    """bench.py seed_pool: G junk continuations for every key, same update order."""
    conts = np.random.default_rng(JUNK_SEED).integers(0, vocab, size=(vocab, G, NG - 1)).astype(np.int32)
    h = C.c_void_p()
    if lib.ref_pool_new(NG, C.c_size_t(1 << 20), C.byref(h)):
        raise RuntimeError(lib.ref_last_error())
    prev = np.zeros(3, dtype=np.int32)
    cur = np.zeros(3, dtype=np.int32)
    pp, cp = prev.ctypes.data_as(_i32p), cur.ctypes.data_as(_i32p)
    for key in range(vocab):
        prev[0] = key
        for j in range(G):
            cur[1:] = conts[key, j]
            lib.ref_pool_update(h, pp, cp, 3)
    return h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depth", type=int, default=2, help="local layers each side (privacy depth)")
    ap.add_argument("--threads", type=int, default=8)
    ap.add_argument("--prompts", type=int, default=4)
    ap.add_argument("--quick", action="store_true", help="2 tokens per run (smoke of the generator)")
    args = ap.parse_args()

    ref = po.Ref()
    lib = ref.lib
    lib.ref_pool_new.argtypes = [C.c_int, C.c_size_t, C.POINTER(C.c_void_p)]
    cfg = po.mistral7b_cfg()
    d = args.depth
    lb, le = d, cfg.n_layers - d
    hd = cfg.hidden_dim

    nrep = args.prompts // 2
    prompts = ref.corpus("repetitive", cfg.vocab_size, nrep, 8, 100) + \
        ref.corpus("random", cfg.vocab_size, args.prompts - nrep, 8, 101)

    jobs = []  # (name, mode, wire_f32, pool, max_new, rec_frames, prompt)
    for pi, p in enumerate(prompts):
        if d == 2:
            jobs.append(("seq-f32", 0, 1, False, 17, 3, pi))
            jobs.append(("la-f16", 2, 0, False, 17, 0, pi))
            jobs.append(("b16-f32", 2, 1, True, 13, 2, pi))
            jobs.append(("b16-f16", 2, 0, True, 9, 0, pi))
        elif pi < 2:
            jobs.append(("seq-f32", 0, 1, False, 17, 2, pi))
            jobs.append(("la-f16", 2, 0, False, 17, 0, pi))
    if args.quick:
        jobs = [(n, m, w, p, 3, min(r, 2), pi) for (n, m, w, p, _mn, r, pi) in jobs]

    t0 = time.time()
    cw, sw = C.c_void_p(), C.c_void_p()
    ref._check(lib.ref_split_models(C.byref(po._ccfg(cfg)), 1, d, d, C.byref(cw), C.byref(sw)))
    srv = C.c_void_p()
    ref._check(lib.ref_server_new_move(sw, lb, le, 64, C.byref(srv)))
    print(f"[{time.time() - t0:.0f}s] weights ready (depth {d}, middle [{lb},{le}))", flush=True)
    base_pool = junk_pool(lib, cfg.vocab_size) if any(j[3] for j in jobs) else None
    print(f"[{time.time() - t0:.0f}s] junk pool ready", flush=True)

    lock = threading.Lock()
    results = [None] * len(jobs)
    rows_store = {}

    def run(idx):
        name, mode, wire_f32, use_pool, max_new, rec, pi = jobs[idx]
        pool = None
        if use_pool:
            pool = C.c_void_p()
            ref._check(lib.ref_pool_clone(base_pool, C.byref(pool)))
        dc = po._RefDecodeCfg(mode, d, d, wire_f32, -1, W, NG, G, 4096, 4, 0.0)
        p = np.asarray(prompts[pi], dtype=np.int32)
        maxr = 16
        req = np.zeros((max(rec, 1), maxr, hd), dtype=np.float32)
        resp = np.zeros_like(req)
        rrows = np.zeros(max(rec, 1), dtype=np.int32)
        toks = np.zeros(max_new, dtype=np.int32)
        sb = np.zeros(max_new + 1, dtype=np.int32)
        sa = np.zeros(max_new + 1, dtype=np.int32)
        st = po._RefStats()
        t1 = time.time()
        ref._check(lib.ref_decode_on(cw, srv, C.byref(dc), pool, f"golden-{idx}".encode(),
                                     p.ctypes.data_as(_i32p), len(p), max_new, rec, maxr,
                                     req.ctypes.data_as(_f32p), resp.ctypes.data_as(_f32p),
                                     rrows.ctypes.data_as(_i32p), toks.ctypes.data_as(_i32p),
                                     sb.ctypes.data_as(_i32p), sa.ctypes.data_as(_i32p), C.byref(st)))
        if pool is not None:
            lib.ref_pool_free(pool)
        out = {"name": name, "mode": mode, "wire_f32": wire_f32, "junk_pool": use_pool,
               "prompt": p.tolist(), "max_new": max_new, "tokens": toks.tolist(),
               "step_batch": sb[:st.steps].tolist(), "step_accepted": sa[:st.steps].tolist(),
               "boundary_frames": int(rec), "boundary_rows": rrows[:rec].tolist(),
               "cpu_seconds": round(time.time() - t1, 1)}
        with lock:
            results[idx] = out
            for f in range(rec):
                rows_store[f"r{idx}_f{f}_req"] = req[f, :rrows[f]].copy()
                rows_store[f"r{idx}_f{f}_resp"] = resp[f, :rrows[f]].copy()
            print(f"[{time.time() - t0:.0f}s] job {idx} {name} prompt {pi}: {out['cpu_seconds']}s "
                  f"tokens {out['tokens']} batch {out['step_batch']}", flush=True)

    with ThreadPoolExecutor(args.threads) as ex:
        # longest first
        order = sorted(range(len(jobs)), key=lambda i: -(jobs[i][4] * (16 if jobs[i][3] else 6 if jobs[i][1] else 1)))
        list(ex.map(run, order))

    cfgd = {k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__}
    suffix = "_quick" if args.quick else ""
    stem = f"ref_decode_7b_d{d}{suffix}"
    doc = {"name": f"mistral7b depth {d}", "source": "oracle/_ref (reference SplitClient + decode loop + "
           "ServerEngine, ref_shim.cpp ref_decode_on) — tests/golden/make_golden_7b.py",
           "config": cfgd, "weights": "init_weights(seed) rounded to bf16 RNE", "split": d,
           "lookahead": {"W": W, "N": NG, "G": G}, "junk_pool": {"seed": JUNK_SEED, "per_key": G,
                                                               "note": "bench.py seed_pool"},
           "boundary_rows_file": f"{stem}.npz", "host_threads": args.threads,
           "wall_seconds": round(time.time() - t0, 1), "runs": results}
    with open(os.path.join(HERE, f"{stem}.json"), "w") as f:
        json.dump(doc, f, indent=1)
    np.savez_compressed(os.path.join(HERE, f"{stem}.npz"), **rows_store)
    print(f"written {stem}.json / .npz in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
