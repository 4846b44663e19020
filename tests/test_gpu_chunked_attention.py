"""The key-chunked attention design of the layer-stack megakernel (SFG_ATTN=
chunked: rows share K/V, for long contexts) must meet the same FAST-mode bar as
the default per-(row, kv head) design: the whole FAST suite (tolerances vs the
reference, determinism, batch invariance, lookahead == sequential bitwise at
the tiny/desk/7B shapes) is re-run in a fresh process with it selected (the
choice is read once per process)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_fast_suite_with_chunked_attention():
    env = dict(os.environ, SFG_ATTN="chunked")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", os.path.join(ROOT, "tests", "test_gpu_fast.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
