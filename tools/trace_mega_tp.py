"""Phase timeline of the FAST megakernel under tensor parallelism (dev tool, 2 GPUs).

    python tools/trace_mega_tp.py [NL]          # spawns the two ranks

Each rank builds its TP=2 shard of the Mistral-NeMo-12B true shape (layers
2 .. 2+NL), runs a 24-token prompt, then traces a 16-row forward (globaltimer
per CTA and phase, as tools/trace_mega.py) and prints per-phase durations
against that rank's weight bytes at the measured HBM peak, next to the same
numbers of a TP=1 engine on rank 0's GPU."""
import ctypes as C
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def phases(tr, NL, wb):
    G = tr.shape[0]
    t0 = tr[:, 255, 0].min()
    out = []
    for l in range(1, NL - 1):
        for k, ph in enumerate(("QKV", "ATTN", "O", "GU", "DOWN")):
            out_id = 5 * l + 1 + k
            s0 = (tr[:, out_id - 1, 2].max() - t0) / 1000
            s1 = (tr[:, out_id, 2].max() - t0) / 1000
            out.append((l, ph, s1 - s0, wb[ph] / 6.5488e12 * 1e6))
    return out


def run_rank(rank, size, uid, NL):
    import paper_2602_16760_b200 as sfg
    L = sfg.lib()
    H, nh, nkv, hd, F = 5120, 32, 8, 128, 14336
    mc = sfg.ModelConfig(vocab_size=131072, n_layers=40, hidden_dim=H, n_heads=nh, n_kv_heads=nkv, head_dim=hd,
                         ffn_dim=F, max_seq_len=4096, rope_base=1e6, rms_eps=1e-5, seed=1234)
    tp = (size, rank, uid) if size > 1 else None
    eng = sfg.Engine(mc, math=sfg.FAST, device=rank, layers=(2, 2 + NL), with_embedding=False, with_head=False,
                     extended_shapes=True, tp=tp)
    bank = eng.bank(2, 2 + NL)
    rng = np.random.default_rng(0)
    h = (rng.standard_normal((24, H)) * 0.5).astype(np.float32)
    eng.forward_layers(2, 2 + NL, h, list(range(24)), bank)
    bank.mark_committed(24)
    L.sfg_debug_mega_trace(1)
    h16 = (rng.standard_normal((16, H)) * 0.5).astype(np.float32)
    ts = []
    for _ in range(4):
        bank.crop(24)
        t = time.perf_counter()
        eng.forward_layers(2, 2 + NL, h16, list(range(24, 40)), bank)
        ts.append((time.perf_counter() - t) * 1e3)
    G = 148
    tr = np.zeros(G * 256 * 20, dtype=np.uint64)
    L.sfg_debug_mega_trace_read(bank.h, tr.ctypes.data_as(C.POINTER(C.c_uint64)), tr.size)
    tr = tr.reshape(G, 256, 20).astype(np.int64)
    qd = nh * hd // size
    kvd = nkv * hd // size
    Fl = F // size
    wb = {"QKV": H * (qd + 2 * kvd) * 2, "ATTN": 0, "O": qd * H * 2, "GU": 2 * H * Fl * 2, "DOWN": Fl * H * 2}
    rows = phases(tr, NL, wb)
    per = {}
    for l, ph, d, ideal in rows:
        per.setdefault(ph, []).append((d, ideal))
    msg = [f"tp{size} rank {rank}: wall per forward (ms) {[round(x, 3) for x in ts]}"]
    tot = 0.0
    for ph in ("QKV", "ATTN", "O", "GU", "DOWN"):
        d = np.mean([x[0] for x in per[ph]])
        tot += d
        msg.append(f"   {ph:5s} {d:6.1f} us (bytes at peak {per[ph][0][1]:5.1f})")
    msg.append(f"   per layer {tot:6.1f} us")
    t0 = tr[:, 255, 0].min()
    for base, nm in ((240, "O"), (248, "DOWN")):
        for l in (1, 2):
            T = tr[:, base + l, :5]
            mk = T[:, 0] > 0
            if not mk.any():
                continue
            T = T[mk]
            def md(x):
                return f"{np.median(x) / 1000:5.2f}/{x.max() / 1000:5.2f}"
            msg.append(f"   L{l} {nm} exchange ({mk.sum()} CTAs): entry {(T[:, 0].min() - t0) / 1000:.1f}..{(T[:, 0].max() - t0) / 1000:.1f} us;"
                       f" tagged stores {md(T[:, 1] - T[:, 0])}, peer words arrive {md(T[:, 3] - T[:, 1])},"
                       f" sum {md(T[:, 4] - T[:, 3])}")
    print("\n".join(msg), flush=True)


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--rank":
        rank, size, uid, NL = int(sys.argv[2]), int(sys.argv[3]), bytes.fromhex(sys.argv[4]), int(sys.argv[5])
        run_rank(rank, size, uid, NL)
        return
    NL = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    import paper_2602_16760_b200 as sfg
    uid = sfg.tp_unique_id()
    procs = [subprocess.Popen([sys.executable, __file__, "--rank", str(r), "2", uid.hex(), str(NL)]) for r in range(2)]
    for p in procs:
        p.wait()
    subprocess.run([sys.executable, __file__, "--rank", "0", "1", "00", str(NL)])


if __name__ == "__main__":
    main()
