"""Runs the C++ drop-in test binary (tests/cpp/test_dropin.cpp): the reference's
own test cases written against include/stagger_b200/stagger/*.hpp on the GPU,
checked against the C oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "test_dropin")


def test_cpp_dropin_builds():
    # the drop-in headers compile and link against libstagger_b200.so (no GPU needed)
    from paper_2312_12491_b200 import build

    build.build_cpp_tests()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_dropin_parity():
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(p.stdout, p.stderr[-3000:])
    assert p.returncode == 0, p.stderr[-3000:]
    assert " 0 failed" in p.stdout
