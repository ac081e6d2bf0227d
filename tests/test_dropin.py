"""The C++ drop-in headers (include/phgrms/*.hpp) compile against the reference's
test code shape (CPU) and pass the restated reference tests on a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def test_dropin_headers_compile():
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", f"-I{os.path.join(ROOT, 'include')}",
                    SRC], check=True)


@pytest.mark.gpu
def test_dropin_reference_tests_on_gpu():
    import __graft_entry__ as g
    g.build_dropin()
    r = subprocess.run([BIN, os.path.join(ROOT, "tests", "golden")], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "0 failures" in r.stdout
