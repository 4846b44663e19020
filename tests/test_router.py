"""CPU tests of the multi-device serving front end (sfg_router / sfg_batcher,
include/sfg.h): placement, stickiness and error behaviour of the router and
the per-backend batching queue, with Python frame handlers standing in for
the per-device servers (no GPU needed; the GPU path is
tests/test_gpu_router.py).

Reference behaviour mirrored: a step frame of a session the server does not
hold gets the error frame "session: unknown or expired session: <id>"
(server.cpp:226-232, error frames server.cpp:186-190); FrameServer calls the
handler from one thread per connection (transport.cpp:565-581)."""
import ctypes as C
import threading

import pytest

import paper_2602_16760_b200 as sfg
import wirepy
from paper_2602_16760_b200 import _lib


class FakeDevice:
    """A frame handler that behaves like a server for session bookkeeping:
    prompts create the session, steps of unknown sessions get the reference
    error frame, everything answered echoes the frame kind."""

    def __init__(self, idx):
        self.idx, self.sessions, self.seen = idx, set(), []
        self._buf = None
        self.fn = _lib.FRAME_HANDLER(self._handle)

    def _handle(self, ctx, req, n, resp, resp_n):
        h, _ = wirepy.decode(C.string_at(req, n))
        self.seen.append((h["kind"], h["session_id"]))
        sid = h["session_id"]
        if h["kind"] == "prompt":
            self.sessions.add(sid)
            r = wirepy.encode("response", sid, shape=(0,), srv_ms=float(self.idx))
        elif h["kind"] in ("step", "accept_and_step") and sid not in self.sessions:
            r = wirepy.encode("error", sid, shape=(0,), err="session: unknown or expired session: " + sid)
        else:
            r = wirepy.encode("response", sid, shape=(0,), srv_ms=float(self.idx))
        self._buf = (C.c_uint8 * len(r)).from_buffer_copy(r)
        resp[0] = C.cast(self._buf, C.POINTER(C.c_uint8))
        resp_n[0] = len(r)
        return 0

    @property
    def handler(self):
        return C.cast(self.fn, C.c_void_p), None


def prompt(sid):
    return wirepy.encode("prompt", sid, shape=(0,))


def step(sid):
    return wirepy.encode("step", sid, shape=(0,))


def test_router_places_least_loaded_and_is_sticky():
    devs = [FakeDevice(i) for i in range(3)]
    r = sfg.Router([d.handler for d in devs])
    for i in range(7):
        h, _ = wirepy.decode(r.handle(prompt(f"s{i}")))
        assert h["kind"] == "response"
    assert sorted(r.load()) == [2, 2, 3]
    placed = {f"s{i}": r.session_device(f"s{i}") for i in range(7)}
    assert placed["s0"] == 0 and placed["s1"] == 1 and placed["s2"] == 2  # ties -> lowest index
    for _ in range(3):  # steps and re-prompts go to the placing backend
        for sid, b in placed.items():
            h, _ = wirepy.decode(r.handle(step(sid)))
            assert h["kind"] == "response" and h["srv_ms"] == float(b)
    r.handle(prompt("s4"))
    assert r.session_device("s4") == placed["s4"]
    for d in devs:
        assert all(sid in d.sessions for _, sid in d.seen)


def test_router_unknown_session_gets_reference_error_frame():
    devs = [FakeDevice(i) for i in range(2)]
    r = sfg.Router([d.handler for d in devs])
    h, _ = wirepy.decode(r.handle(step("ghost")))
    assert h["kind"] == "error" and h["err"] == "session: unknown or expired session: ghost"
    assert h["session_id"] == "ghost"
    assert all(not d.seen for d in devs)  # no backend was bothered
    # malformed bytes: the protocol error frame, no backend involved
    h, _ = wirepy.decode(r.handle(b"\x05\x00"))
    assert h["kind"] == "error" and h["err"].startswith("protocol:")
    # ping: answered by a backend
    h, _ = wirepy.decode(r.handle(wirepy.encode("ping", "")))
    assert h["kind"] == "response"


def test_router_drops_sessions_the_backend_lost():
    devs = [FakeDevice(i) for i in range(2)]
    r = sfg.Router([d.handler for d in devs])
    r.handle(prompt("a"))
    b = r.session_device("a")
    devs[b].sessions.discard("a")  # the server expired it
    h, _ = wirepy.decode(r.handle(step("a")))
    assert h["kind"] == "error" and "unknown or expired session" in h["err"]
    assert r.session_device("a") == -1 and r.load() == [0, 0]
    h, _ = wirepy.decode(r.handle(step("a")))  # now refused at the router
    assert h["kind"] == "error" and len(devs[b].seen) == 2


def test_router_expiry_frees_placements():
    devs = [FakeDevice(i) for i in range(2)]
    r = sfg.Router([d.handler for d in devs], session_expiry_s=10.0)
    now = [100.0]
    r.set_clock(lambda: now[0])
    r.handle(prompt("old"))
    now[0] = 105.0
    r.handle(prompt("mid"))
    assert r.load() == [1, 1]
    now[0] = 112.0  # "old" idle 12 s > 10 s: dropped when the next session is placed
    r.handle(prompt("new"))
    assert r.session_device("old") == -1 and r.session_device("new") == 0 and r.load() == [1, 1]


def test_batcher_serves_concurrent_connections():
    devs = [FakeDevice(i) for i in range(2)]
    r = sfg.Router([d.handler for d in devs])
    bq = sfg.Batcher(r)
    n_threads, n_steps = 8, 25
    errors = []

    def client(i):
        sid = f"c{i}"
        try:
            h, _ = wirepy.decode(bq.handle(prompt(sid)))
            assert h["kind"] == "response" and h["session_id"] == sid
            for _ in range(n_steps):
                h, _ = wirepy.decode(bq.handle(step(sid)))
                assert h["kind"] == "response" and h["session_id"] == sid
                assert h["srv_ms"] == float(r.session_device(sid))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    ts = [threading.Thread(target=client, args=(i,)) for i in range(n_threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
    assert not errors, errors
    st = bq.stats()
    assert st["frames"] == n_threads * (n_steps + 1)
    assert sorted(r.load()) == [4, 4]
    # refused frames never reach a queue
    h, _ = wirepy.decode(bq.handle(step("nobody")))
    assert h["kind"] == "error"
    assert bq.stats()["frames"] == n_threads * (n_steps + 1)


def test_router_rejects_empty_backend_list():
    with pytest.raises(sfg.SplitError):
        sfg.Router([])
