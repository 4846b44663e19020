"""bench.py must stay importable and parse its CLI on a CPU-only host (the
driver runs it unattended at round end)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_help_runs():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stderr
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--model", "--prompt-len"):
        assert flag in r.stdout


def test_bench_traffic_reads_committed_profile():
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    t = bench.ncu_traffic(argparse.Namespace(model="7b"))
    assert t["traffic"] is None or 0.9 < t["traffic"] / t["traffic_launch_algorithmic_bytes"] < 1.5
