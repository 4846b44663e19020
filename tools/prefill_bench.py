"""Time the prompt (prefill) forward of the 28 middle layers at the 7B shape.

handle_prompt (server.cpp:203-224) runs forward_layers over the whole prompt;
here: sfg_forward_layers over P rows with the causal mask, FAST math, host
buffers (sync call).  Prints one JSON line per prompt length.
    python tools/prefill_bench.py [P ...]
"""
import json
import os
import sys
import time

import ctypes as C

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_16760_b200 as sfg  # noqa: E402

H_7B = dict(vocab_size=32768, n_layers=32, hidden_dim=4096, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336,
            max_seq_len=4096, rope_base=1e6, rms_eps=1e-5, seed=1234)


def pin(arr):
    """Page-lock a numpy array (cudaHostRegister) so the engine's host<->device
    copies run at pinned-memory speed, as a serving front end's buffers would."""
    rt = C.CDLL("libcudart.so")
    rc = rt.cudaHostRegister(C.c_void_p(arr.ctypes.data), C.c_size_t(arr.nbytes), 0)
    if rc != 0:
        raise RuntimeError(f"cudaHostRegister failed: {rc}")
    return arr


def main():
    lens = [int(a) for a in sys.argv[1:]] or [256, 2048]
    eng = sfg.Engine(sfg.ModelConfig(**H_7B), math=sfg.FAST, layers=(2, 30), with_embedding=False, with_head=False)
    rng = np.random.default_rng(0)
    for P in lens:
        h = pin((rng.standard_normal((P, 4096)) * 0.5).astype(np.float32))
        out = pin(np.empty_like(h))
        pos = np.arange(P, dtype=np.int32)
        bank = eng.bank(2, 30)
        eng.forward_layers(2, 30, h, pos, bank, out=out)  # warm-up (workspace growth, graph-free path)
        ts = []
        for _ in range(3):
            bank.reset()
            t0 = time.perf_counter()
            eng.forward_layers(2, 30, h, pos, bank, out=out)
            ts.append(time.perf_counter() - t0)
        L = sfg.lib()
        L.sfg_profiler_reset()
        L.sfg_profiler_enable(1)
        bank.reset()
        eng.forward_layers(2, 30, h, pos, bank)
        L.sfg_profiler_enable(0)
        classes = {}
        for ci, name in enumerate(["qkv", "attention", "o_proj", "gate_up", "down"]):
            cnt, ms, by, fl = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            L.sfg_profiler_stats(ci, C.byref(cnt), C.byref(ms), C.byref(by), C.byref(fl))
            classes[name] = {"launches": cnt.value, "ms": round(ms.value, 3)}
        wbytes = 28 * 436.2e6
        print(json.dumps({"prompt_len": P, "middle_layers": 28, "ms": min(ts) * 1e3,
                          "host_buffers": "pinned (cudaHostRegister), copies inside the timed call",
                          "ms_per_token": min(ts) * 1e3 / P,
                          "weight_bytes_per_16_rows_gb": wbytes / 1e9,
                          "checksum": float(np.abs(out).astype(np.float64).sum()),
                          "classes": classes}), flush=True)


if __name__ == "__main__":
    main()
