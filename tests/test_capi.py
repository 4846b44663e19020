"""CPU tests of the C ABI boundary (no device compute):

* libsfg.so loads and exports every function include/sfg.h declares;
* with no GPU visible the engine refuses to construct (no CPU fallback);
* host-side pieces of the boundary (binary16 codec, NGramPool) behave like
  the reference (see also test_oracle.py).
"""
import ctypes as C
import os
import subprocess

import pytest

import paper_2602_16760_b200 as sfg
from paper_2602_16760_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_built_for_sm100a():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build()"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    names = _lib.declared_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_python_mirror_binds_every_symbol():
    L = _lib.lib()
    for n in _lib.declared_symbols():
        assert getattr(L, n).restype is not None or getattr(L, n).argtypes is not None, n


def test_version_string():
    assert b"sm_100a" in _lib.lib().sfg_version()


def _have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU failure path")
def test_engine_fails_loudly_without_gpu():
    with pytest.raises(sfg.SplitError) as e:
        sfg.Engine(sfg.ModelConfig())
    assert e.value.kind == "internal"
    assert "no CPU fallback" in str(e.value)


def test_config_errors_use_reference_categories():
    # ModelConfig::validate fires before any device work (tinyformer.cpp:102-121)
    bad = sfg.ModelConfig(n_kv_heads=3)
    with pytest.raises(sfg.SplitError) as e:
        sfg.Engine(bad)
    assert str(e.value) == "config: n_kv_heads must divide n_heads"
    with pytest.raises(sfg.SplitError) as e:
        sfg.Engine(sfg.ModelConfig(head_dim=8))
    assert str(e.value) == "config: n_heads * head_dim must equal hidden_dim"


def test_pool_errors():
    with pytest.raises(sfg.SplitError) as e:
        sfg.NGramPool(1, 4)
    assert str(e.value) == "config: ngram_n must be >= 2"
