"""Phase timeline of the FAST megakernel at the 7B shape (B200 dev tool).

Per barrier id: when the CTAs passed the phase's input barrier (X start),
finished building activation images (X done) and finished the phase
(arrive), relative to the earliest CTA entry; median / max over CTAs."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import paper_2602_16760_b200 as sfg
import pyoracle as po
from paper_2602_16760_b200 import _lib

L = _lib.lib()
NL = int(os.environ.get("NL", "6"))
cfg = po.mistral7b_cfg()
eng = sfg.Engine(sfg.ModelConfig(**{k: getattr(cfg, k) for k in po.ModelCfg.__dataclass_fields__}), math=sfg.FAST,
                 layers=(2, 2 + NL), with_embedding=False, with_head=False)
bank = eng.bank(2, 2 + NL)
rng = np.random.default_rng(0)
PRIOR = int(os.environ.get("PRIOR", "24"))
h = (rng.standard_normal((PRIOR, 4096)) * 0.5).astype(np.float32)
eng.forward_layers(2, 2 + NL, h, list(range(PRIOR)), bank)
bank.mark_committed(PRIOR)
L.sfg_debug_mega_trace(1)
h16 = (rng.standard_normal((16, 4096)) * 0.5).astype(np.float32)
times = []
for it in range(4):
    bank.crop(PRIOR)
    t0 = time.perf_counter()
    eng.forward_layers(2, 2 + NL, h16, list(range(PRIOR, PRIOR + 16)), bank)
    times.append(time.perf_counter() - t0)
print("wall per forward (ms):", [round(t * 1000, 3) for t in times])
G = 148
TW = 20
tr = np.zeros(G * 256 * TW, dtype=np.uint64)
L.sfg_debug_mega_trace_read(bank.h, tr.ctypes.data_as(C.POINTER(C.c_uint64)), tr.size)
tr = tr.reshape(G, 256, TW).astype(np.int64)
t0 = tr[:, 255, 0].min()
names = {1: "QKV", 2: "ATTN", 3: "O", 4: "GU", 5: "DOWN"}
print("kernel entry spread (us):", (tr[:, 255, 0].max() - t0) / 1000)
print(f"TOTAL layers {NL}: {(tr[:, 5 * NL, 2].max() - t0) / 1000:.1f} us")
print("stall columns: total wait (us, median/max over CTAs) of X-writer on empty, MMA on full, producer on empty")
print(f"{'id':>4} {'phase':>5} {'xstart med/max':>18} {'xdone med/max':>18} {'arrive med/max':>18}"
      f" {'xw-empty':>14} {'mma-full':>14} {'prod-empty':>14} {'last acc med/max':>18}")
for bid in range(0, 1 + 5 * NL):
    ph = "STAT" if bid == 0 else names[(bid - 1) % 5 + 1]
    def col(k):
        v = tr[:, bid, k]
        v = v[v > 0]
        if v.size == 0:
            return "-"
        return f"{(np.median(v) - t0) / 1000:8.1f}/{(v.max() - t0) / 1000:8.1f}"
    def dur(k):
        v = tr[:, bid, k]
        if not v.any():
            return "-"
        return f"{np.median(v) / 1000:6.1f}/{v.max() / 1000:6.1f}"
    print(f"{bid:4d} {ph:>5} {col(0):>18} {col(1):>18} {col(2):>18} {dur(3):>14} {dur(4):>14} {dur(5):>14}"
          f" {col(6):>18}")
# MMA issuer per phase of layer 2: first MMA, last commit (median/max), time
# waited for a free accumulator, and busy time = last - first - waits
print("MMA issuer (layer 2): phase  first med/max   last med/max   full-wait   acc-wait   span med")
for k, ph in enumerate(("QKV", "O", "GU", "DOWN")):
    in_id = {0: 5 * 2, 1: 5 * 2 + 2, 2: 5 * 2 + 3, 3: 5 * 2 + 4}[k]
    f, la = tr[:, in_id, 16], tr[:, in_id, 17]
    m = f > 0
    if not m.any():
        continue
    span = (la[m] - f[m]) / 1000
    print(f"   {ph:5s} {(np.median(f[m]) - t0) / 1000:7.1f}/{(f[m].max() - t0) / 1000:7.1f} "
          f"{(np.median(la[m]) - t0) / 1000:7.1f}/{(la[m].max() - t0) / 1000:7.1f} "
          f"{np.median(tr[m, in_id, 4]) / 1000:8.1f} {np.median(tr[m, in_id, 18]) / 1000:8.1f} {np.median(span):8.1f}")
# the latest CTAs of each phase of layer 1: last accumulator ready (slot 6 of
# the phase's input barrier) vs arrival at the phase's output barrier
phase_in = {1: 5, 3: 7, 4: 8, 5: 9}  # output barrier id -> input barrier id (layer 1)
for out_id, in_id in ((6, 5), (8, 7), (9, 8), (10, 9)):
    arr = tr[:, out_id, 2]
    order = np.argsort(arr)[::-1][:6]
    print(f"phase out {out_id} ({names[(out_id - 1) % 5 + 1]}): latest CTAs "
          "(cta: last acc, fenced, counter, loads, epi_final, epi done, arrive)")
    for c in order:
        def ts(k, row=in_id):
            v = tr[c, row, k]
            return f"{(v - t0) / 1000:7.1f}" if v > 0 else "      -"
        print(f"   {int(c):4d}:", " ".join(ts(k) for k in (6, 8, 9, 10, 11, 7)), ts(2, out_id),
              "| epi: h ready, stores done, sumsq done:", " ".join(ts(k) for k in (12, 13, 14)))
# per-phase critical path: input barrier complete (max arrive) -> output barrier
# complete, against the phase's weight bytes at the measured HBM peak
H, QD, KVD, F = 4096, 4096, 1024, 14336
wbytes = {"QKV": H * (QD + 2 * KVD) * 2, "ATTN": 0, "O": QD * H * 2, "GU": 2 * H * F * 2, "DOWN": F * H * 2}
print("phase      start    end   dur  ideal@6.55TB/s over")
tot = over_tot = 0.0
for l in range(1, NL - 1):
    for k, ph in enumerate(("QKV", "ATTN", "O", "GU", "DOWN")):
        out_id = 5 * l + 1 + k
        in_id = out_id - 1
        s0 = (tr[:, in_id, 2].max() - t0) / 1000
        s1 = (tr[:, out_id, 2].max() - t0) / 1000
        ideal = wbytes[ph] / 6.5488e12 * 1e6  # MEASURED_PEAKS.json hbm_gbs
        print(f"L{l} {ph:5s} {s0:7.1f} {s1:7.1f} {s1 - s0:5.1f} {ideal:8.1f} {s1 - s0 - ideal:6.1f}")
        tot += s1 - s0
        over_tot += s1 - s0 - ideal
print(f"per layer: {tot / (NL - 2):.1f} us, overhead {over_tot / (NL - 2):.1f} us")
# attention items (chunked design): start of the key walk (12) and its end (13)
for l in range(1, NL - 1):
    bid = 5 * l + 2
    st, en = tr[:, bid, 12], tr[:, bid, 13]
    m = (st > 0) & (en > 0)
    if m.any():
        d = (en[m] - st[m]) / 1000
        print(f"L{l} attention key walk per CTA: median {np.median(d):.1f} us max {d.max():.1f} us over {m.sum()} CTAs;"
              f" first start {(st[m].min() - t0) / 1000:.1f} last end {(en[m].max() - t0) / 1000:.1f}")
# per-row attention items (ids 200 + l): entry, flags ok, q staged, walk end
# per warp (8..15), combine end, published
for l in range(1, NL - 1):
    T = tr[:, 200 + l, :]
    m = T[:, 0] > 0
    if not m.any():
        continue
    T = T[m]
    qkv_done = (tr[:, 5 * l + 1, 2].max() - t0) / 1000
    rel = lambda v: (v - t0) / 1000  # noqa: E731
    walk_end = T[:, 8:16].max(axis=1)
    walk_first = np.where(T[:, 8:16] > 0, T[:, 8:16], np.iinfo(np.int64).max).min(axis=1)
    def md(x):
        return f"{np.median(x) / 1000:5.2f}/{x.max() / 1000:5.2f}"
    print(f"L{l} attention items ({m.sum()} CTAs), QKV complete at {qkv_done:.1f}: "
          f"entry med {np.median(rel(T[:, 0])):.1f} max {rel(T[:, 0]).max():.1f}; "
          f"flag wait {md(T[:, 1] - T[:, 0])}, q stage {md(T[:, 2] - T[:, 1])}, "
          f"walk first/last warp {md(walk_first - T[:, 2])} / {md(walk_end - T[:, 2])}, "
          f"combine {md(T[:, 3] - walk_end)}, publish {md(T[:, 4] - T[:, 3])}; "
          f"last published {rel(T[:, 4]).max():.1f}")
# per-warp key-walk end (relative to q staged), median over CTAs
for l in range(1, 3):
    T = tr[:, 200 + l, :]
    T = T[T[:, 0] > 0]
    if T.size:
        print(f"L{l} walk end per warp (us after q staged):",
              " ".join(f"{np.median(T[:, 8 + w] - T[:, 2]) / 1000:5.2f}" for w in range(8)))
# clock64 breakdown of the per-row attention key walk (debug builds that
# record ids 200/210/220 + l: scores, value loads, softmax + PV), cycles
for l in range(1, 3):
    parts = []
    for base, name in ((200, "K+scores"), (210, "V loads"), (220, "softmax+PV")):
        T = tr[:, base + l, :8]
        v = T[T > 0]
        if v.size:
            parts.append(f"{name} med {np.median(v):.0f} max {v.max():.0f}")
    if parts:
        print(f"L{l} walk cycles per warp:", "; ".join(parts))
# chunked attention items (ids 230 + l): 0 staged issue, 1 K landed, 2 scores done,
# 3 P^T written + V landed, 5 PV done, 6 partial published, 7 all chunks arrived, 8 merged + published
for l in range(1, NL - 1):
    T = tr[:, 230 + l, :]
    m = T[:, 0] > 0
    if not m.any():
        continue
    T = T[m]
    rel = lambda v: (v - t0) / 1000  # noqa: E731
    def md(x):
        return f"{np.median(x) / 1000:5.2f}/{x.max() / 1000:5.2f}"
    seg = [("K land", 0, 1), ("scores", 1, 2), ("P+V", 2, 3), ("PV", 3, 5)]
    if (T[:, 14] > 0).all() and (T[:, 15] > 0).all():  # tensor-core path: QKV wait | K load + split | Q + rest
        seg = [("QKV wait", 0, 14), ("K load+split", 14, 15), ("Q split+MMA in", 15, 1)] + seg[1:]
    parts = ", ".join(f"{n} {md(T[:, b] - T[:, a])}" for n, a, b in seg)
    has6 = T[:, 6] > 0
    if has6.any():
        parts += f", publish {md(T[has6, 6] - T[has6, 5])}, arrive-wait {md(T[has6, 7] - T[has6, 6])}, merge {md(T[has6, 8] - T[has6, 7])}"
        h9 = has6 & (T[:, 9] > 0)
        if h9.any():
            parts += (f" [merge: stage {md(T[h9, 9] - T[h9, 7])}, weights {md(T[h9, 10] - T[h9, 9])},"
                      f" o + stores {md(T[h9, 11] - T[h9, 10])}, proxy fence {md(T[h9, 12] - T[h9, 11])},"
                      f" gpu fence + flag {md(T[h9, 8] - T[h9, 12])}]")
    print(f"L{l} chunked attention ({m.sum()} CTAs): first start {rel(T[:, 0]).min():.1f} last publish "
          f"{rel(T[:, 8]).max():.1f}; {parts}")
