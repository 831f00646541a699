"""The C++ drop-in façade (include/blest_b200.hpp): compiles here (CPU); on the B200 a
reference-style C++ program built against it runs and checks known answers
(tests/cpp/facade_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_facade_header_compiles():
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        "-I", os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "include"),
                        os.path.join(ROOT, "tests", "cpp", "facade_test.cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_c_header_is_plain_c():
    src = '#include "blest_b200.h"\nint main(void) { return blest_last_error() == 0; }\n'
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        "-x", "c", "-"], input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_facade_program_on_device():
    subprocess.check_call(["make", "-s", "-C", ROOT, "cpptest"])
    r = subprocess.run([os.path.join(ROOT, "tests", "cpp", "facade_test")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "facade_test: ok" in r.stdout
