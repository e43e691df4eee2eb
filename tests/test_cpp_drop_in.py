"""The reference-shaped C++ API (include/splatct_b200.hpp) compiled with g++
against libsplatct_b200.so and checked against the oracle (tests/cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(out):
    lib = os.path.join(ROOT, "paper_2405_20693_b200")
    orc = os.path.join(ROOT, "oracle")
    cmd = ["/usr/bin/g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_drop_in.cpp"), "-L", lib, "-lsplatct_b200", "-L", orc, "-lorc",
           f"-Wl,-rpath,{lib}:{orc}", "-o", out]
    subprocess.run(cmd, check=True)


def test_header_compiles(tmp_path):
    """CPU: the C++ mirror and the drop-in test compile and link against the C ABI."""
    from oracle import oracle as O
    O.build()
    _compile(str(tmp_path / "drop_in"))


@pytest.mark.gpu
def test_cpp_drop_in_parity(tmp_path):
    from oracle import oracle as O
    O.build()
    exe = str(tmp_path / "drop_in")
    _compile(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout
