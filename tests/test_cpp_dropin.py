"""The C++ boundary as a reference caller sees it: tests/cpp/test_dropin.cpp
includes include/levelrank/engine.hpp with an Eigen on the include path (the
Eigen overloads of compute_pagerank / compute_baseline / propagate_weights are
instantiated) and links liblevelrank_b200.so.  Building it needs no GPU;
running it (the reference's engine known answers) does."""
import os
import subprocess

import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp")


def _build():
    out = subprocess.run(["make", "-C", HERE, "-s"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    return os.path.join(HERE, "test_dropin")


def test_cpp_dropin_compiles(lr):
    assert os.path.exists(_build())


@pytest.mark.gpu
def test_cpp_dropin_known_answers(lr):
    exe = _build()
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ok: 0 failure(s)" in out.stdout
