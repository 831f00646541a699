"""CPU: the C-ABI library builds for sm_100a, loads, exports every symbol include/blest_b200.h
declares, and fails loudly (no CPU fallback) when no B200 is present."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "blest_b200.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(blest_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2512_21967_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_library_is_sm100a_only():
    from paper_2512_21967_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout
    assert not re.search(r"sm_(8\d|9\d)\b", out.stdout)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2512_21967_b200 as B
    with pytest.raises(B.BlestCudaError):
        B.Graph.from_edges(4, np.array([[0, 1], [1, 2]]))
    with pytest.raises(B.BlestCudaError):
        B.device_info()


def test_permutation_host_logic():
    from paper_2512_21967_b200 import Permutation
    p = Permutation.from_forward([2, 0, 1])
    assert p.inverse(2) == 0 and p.forward(1) == 0
    q = Permutation.from_inverse([2, 0, 1])
    assert list(q.forward_map()) == [1, 2, 0]
    assert Permutation.composed(p, p.inverted()).is_identity()
    with pytest.raises(ValueError):
        Permutation.from_forward([0, 0, 1])


def test_engine_mode_names_round_trip():
    """R:tests/bfs_engine_test.cpp:362-366."""
    from paper_2512_21967_b200 import EngineMode, engine_mode_from_string
    for m in EngineMode:
        assert engine_mode_from_string(m.value) == m
    with pytest.raises(ValueError):
        engine_mode_from_string("turbo")
