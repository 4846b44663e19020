"""The server's frame-mask parser (mask_from_frame, server.cpp:148-171) on the
host: sfg_debug_mask_runs (word-wise scan, sfg_server.cpp runs_from_f16_mask)
against a direct NumPy restatement on random masks -- legal entries are +0,
-0 and -inf (server.cpp:165-169), visible = not -inf, runs are the maximal
visible intervals of each row.  CPU only: no device is touched."""
import ctypes as C

import numpy as np
import pytest

from paper_2602_16760_b200 import _lib

NEG_INF, POS0, NEG0 = 0xFC00, 0x0000, 0x8000


def reference_runs(m):
    q, kv = m.shape
    if not np.isin(m, [POS0, NEG0, NEG_INF]).all():
        return None
    row_off, runs = [0], []
    for i in range(q):
        vis = m[i] != NEG_INF
        j = 0
        while j < kv:
            if not vis[j]:
                j += 1
                continue
            e = j
            while e < kv and vis[e]:
                e += 1
            runs.append((j, e))
            j = e
        row_off.append(len(runs))
    empty = any(row_off[i + 1] == row_off[i] for i in range(q))
    return row_off, runs, empty


def parse(m):
    L = _lib.lib()
    q, kv = m.shape
    m = np.ascontiguousarray(m, dtype=np.uint16)
    cap = q * kv + 1
    row_off = np.zeros(q + 1, np.int32)
    st, en = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
    n, empty = C.c_int32(), C.c_int32()
    i32p = C.POINTER(C.c_int32)
    rc = L.sfg_debug_mask_runs(m.ctypes.data_as(C.POINTER(C.c_uint16)), q, kv, row_off.ctypes.data_as(i32p),
                               st.ctypes.data_as(i32p), en.ctypes.data_as(i32p), cap, C.byref(n), C.byref(empty))
    if rc != 0:
        return rc
    return row_off.tolist(), list(zip(st[:n.value].tolist(), en[:n.value].tolist())), bool(empty.value)


@pytest.mark.parametrize("seed", range(6))
def test_mask_parser_matches_restatement_on_random_masks(seed):
    rng = np.random.default_rng(seed)
    for _ in range(300):
        q, kv = int(rng.integers(1, 18)), int(rng.integers(1, 300))
        style = rng.integers(0, 4)
        if style == 0:    # lookahead shape: shared prefix, then branch columns
            m = np.full((q, kv), NEG_INF, np.uint16)
            prior = int(rng.integers(0, kv))
            m[:, :prior] = POS0
            for i in range(q):
                m[i, prior:][rng.random(kv - prior) < 0.3] = POS0
        elif style == 1:  # random entries incl. -0
            m = rng.choice(np.array([POS0, NEG0, NEG_INF], np.uint16), size=(q, kv), p=[0.45, 0.1, 0.45])
        elif style == 2:  # long uniform runs (the word-wise fast path)
            m = np.where(((np.arange(kv)[None, :] // int(rng.integers(1, 40))) % 2) == 0, POS0, NEG_INF)
            m = np.repeat(m.astype(np.uint16), q, axis=0)
        else:             # an illegal entry somewhere
            m = np.zeros((q, kv), np.uint16)
            m.flat[int(rng.integers(0, q * kv))] = 0x3C00
        want = reference_runs(m)
        got = parse(m)
        if want is None:
            assert isinstance(got, int) and got != 0  # protocol error, no runs
        else:
            assert got == want


def test_mask_parser_long_context_lookahead_mask():
    q, kv, prior = 16, 2064, 2048
    m = np.full((q, kv), NEG_INF, np.uint16)
    m[:, :prior] = POS0
    for i in range(q):
        m[i, prior:prior + i + 1] = POS0
    row_off, runs, empty = parse(m)
    assert not empty and row_off == list(range(q + 1))
    assert runs == [(0, prior + i + 1) for i in range(q)]
