"""Builds and runs tests/cpp/test_dropin.cpp: the reference's attention test cases driven through the C++ host
mirror (include/binattn_b200.hpp -> C ABI -> CUDA), checked against the CPU oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    import __graft_entry__ as g
    g.build()
    exe = str(tmp_path / "test_dropin")
    pkg, orc = os.path.join(ROOT, "paper_2603_09582_b200"), os.path.join(ROOT, "oracle")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"),
           "-o", exe, f"-L{pkg}", "-lbinattn_cuda", f"-L{orc}", "-lbinattn_oracle", f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{orc}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_mirror_compiles_and_links(tmp_path):
    """CPU-side: the header-only mirror compiles against the C ABI and links (no GPU needed to build)."""
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_dropin_against_oracle(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout + r.stderr
