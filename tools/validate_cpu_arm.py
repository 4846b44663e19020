"""Validates the extrapolated CPU baseline of bench.py: the
bench times ONE Mistral-7B middle layer over 16 rows (+ one LM-head row) on
the reference (oracle/_ref) and extrapolates to a whole forced-B16 lookahead
step.  Here the reference runs the real thing once — its own SplitClient +
decode_lookahead_with_pool (junk pool: every step B=16) + ServerEngine, an
8-token prompt and 2 lookahead steps, single-threaded like the reference —
and the measured per-step wall time is set against the extrapolation made
on the same host in the same run.

    python tools/validate_cpu_arm.py [--out profiles/r02_cpu_arm_validation.json]

Needs ~30 GB of host memory (the 7B weights in fp32, held once).
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import pyoracle as po  # noqa: E402
from make_golden_7b import junk_pool  # noqa: E402

_i32p = C.POINTER(C.c_int32)
_f32p = C.POINTER(C.c_float)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_cpu_arm_validation.json"))
    args = ap.parse_args()
    ref = po.Ref()
    lib = ref.lib
    lib.ref_pool_new.argtypes = [C.c_int, C.c_size_t, C.POINTER(C.c_void_p)]
    cfg = po.mistral7b_cfg()
    # 1) the bench's extrapolation (bench.py cpu_sample / cpu_head_time), same host, 1 thread
    tm = ref.timing_model(cfg, (2, 3), False)
    lib.ref_time_forward(tm.h, 2, 3, 1, 24, 1)  # first touch of the fresh weights (bench.py does the same)
    t_layer = lib.ref_time_forward(tm.h, 2, 3, 16, 24, 1)
    th = ref.timing_model(cfg, (0, 0), True)
    lib.ref_time_finalize(th.h, 1, 1)
    t_head = lib.ref_time_finalize(th.h, 1, 1)
    extrapolated = t_layer * cfg.n_layers + t_head * 16
    del tm, th
    # 2) the real step: reference client + decode loop + server, forced B=16
    t0 = time.time()
    cw, sw = C.c_void_p(), C.c_void_p()
    ref._check(lib.ref_split_models(C.byref(po._ccfg(cfg)), 1, 2, 2, C.byref(cw), C.byref(sw)))
    srv = C.c_void_p()
    ref._check(lib.ref_server_new_move(sw, 2, cfg.n_layers - 2, 64, C.byref(srv)))
    pool = junk_pool(lib, cfg.vocab_size)
    t_setup = time.time() - t0
    dc = po._RefDecodeCfg(2, 2, 2, 0, -1, 5, 3, 5, 4096, 4, 0.0)
    prompt = np.asarray(ref.corpus("random", cfg.vocab_size, 1, 8, 101)[0], dtype=np.int32)
    max_new = 3  # prefill's token + 2 lookahead steps
    toks = np.zeros(max_new, np.int32)
    sb = np.zeros(max_new + 1, np.int32)
    sa = np.zeros(max_new + 1, np.int32)
    st = po._RefStats()
    dummy = np.zeros(1, np.float32)
    rows = np.zeros(1, np.int32)
    t1 = time.time()
    ref._check(lib.ref_decode_on(cw, srv, C.byref(dc), pool, b"validate", prompt.ctypes.data_as(_i32p), len(prompt),
                                 max_new, 0, 1, dummy.ctypes.data_as(_f32p), dummy.ctypes.data_as(_f32p),
                                 rows.ctypes.data_as(_i32p), toks.ctypes.data_as(_i32p), sb.ctypes.data_as(_i32p),
                                 sa.ctypes.data_as(_i32p), C.byref(st)))
    t_decode = time.time() - t1
    measured = st.wall_seconds / max(1, st.steps)
    out = {"host_cpu": os.popen("lscpu | grep 'Model name'").read().strip(), "threads": 1,
           "extrapolated_step_s": extrapolated,
           "extrapolation": f"one 7B middle layer x 16 rows ({t_layer:.2f} s) x {cfg.n_layers} layers + "
                            f"LM head x 16 rows ({t_head:.3f} s/row)",
           "measured_step_s": measured, "steps": st.steps, "step_batch": sb[:st.steps].tolist(),
           "step_accepted": sa[:st.steps].tolist(), "prefill_ms": st.prefill_ms,
           "measured_over_extrapolated": measured / extrapolated,
           "decode_call_s": t_decode, "setup_s": t_setup, "tokens": toks.tolist(),
           "what": "reference SplitClient + decode_lookahead_with_pool (junk pool, forced B=16) + ServerEngine, "
                   "8-token prompt, 2 lookahead steps, 2+2 split, f16 wire, 1 host thread"}
    print(json.dumps(out, indent=1))
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
