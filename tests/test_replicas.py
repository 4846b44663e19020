"""Multi-GPU partitioning — host logic on CPU with gloo.

The N-GPU path is N independent replicas: sessions are assigned round-robin
to ranks, there is no data-path collective, and the measurement is reduced as
max-over-ranks (time) and sum-over-ranks (tokens).  These tests run that logic
with world_size 2 over gloo on 127.0.0.1, the same code bench.py runs over NCCL.
"""
import os
import socket
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_16760_b200 import replicas  # noqa: E402


def test_assign_sessions_round_robin():
    m = replicas.assign_sessions(64, 8)
    assert [len(x) for x in m] == [8] * 8
    assert sorted(s for r in m for s in r) == list(range(64))
    assert replicas.assign_sessions(5, 2) == [[0, 2, 4], [1, 3]]
    assert replicas.assign_sessions(0, 4) == [[], [], [], []]
    with pytest.raises(ValueError):
        replicas.assign_sessions(3, 0)


def test_single_process_group_is_identity():
    g = replicas.Group()
    assert replicas.max_over_ranks(g, 3.5) == 3.5
    assert replicas.sum_over_ranks(g, 2.0) == 2.0
    replicas.barrier(g)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WORKER = textwrap.dedent("""
    import os, sys, json
    sys.path.insert(0, {root!r})
    from paper_2602_16760_b200 import replicas
    g = replicas.setup("gloo")
    mine = replicas.assign_sessions(6, g.world)[g.rank]
    # each rank "times" its own sessions; the slowest rank defines the job time
    t = 1.0 + g.rank
    toks = float(10 * len(mine))
    replicas.barrier(g)
    out = {{"rank": g.rank, "world": g.world, "sessions": mine,
           "sids": [replicas.session_id(g.rank, i) for i in mine],
           "tmax": replicas.max_over_ranks(g, t), "toks": replicas.sum_over_ranks(g, toks)}}
    print(json.dumps(out), flush=True)
    replicas.teardown(g)
""")


def test_two_rank_gloo_reduction_and_sharding(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER.format(root=ROOT))
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, WORLD_SIZE="2", RANK=str(r), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    import json
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=240)
        assert p.returncode == 0, e
        outs.append(json.loads(o.strip().splitlines()[-1]))
    outs.sort(key=lambda d: d["rank"])
    assert [d["sessions"] for d in outs] == [[0, 2, 4], [1, 3, 5]]
    assert len({s for d in outs for s in d["sids"]}) == 6  # session ids never collide across ranks
    for d in outs:
        assert d["world"] == 2
        assert d["tmax"] == 2.0      # max over ranks
        assert d["toks"] == 60.0     # sum over ranks
