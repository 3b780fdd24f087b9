"""The C++ drop-in facade (include/pfe/b200.hpp): compiles against the C ABI
on CPU; on the GPU its reference-style unit cases must pass."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_1612_06496_b200" / "lib"
BIN = ROOT / "tests" / "cpp" / "build" / "test_facade"


def build_facade_test() -> Path:
    BIN.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}", "-o", str(BIN),
           str(ROOT / "tests" / "cpp" / "test_facade.cpp"), f"-L{LIBDIR}", "-lpfe_b200", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return BIN


def test_facade_compiles_and_links():
    assert build_facade_test().exists()


@pytest.mark.gpu
def test_facade_reference_cases_pass_on_gpu():
    exe = build_facade_test()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "facade test passed" in r.stdout
