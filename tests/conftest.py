import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.dirname(os.path.abspath(__file__))):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on a GPU box)")


@pytest.fixture(scope="session")
def port():
    import pyoracle
    return pyoracle.Port()


@pytest.fixture(scope="session")
def ref():
    import pyoracle
    if not pyoracle.ref_available() and not os.path.isdir(pyoracle.REF_SRC):
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return pyoracle.Ref()


@pytest.fixture(scope="session")
def golden():
    import json
    d = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    out = {}
    for f in sorted(os.listdir(d)):
        if f.endswith(".json"):
            with open(os.path.join(d, f)) as fh:
                out[f[:-5]] = json.load(fh)
    return out
