"""The C++ drop-in header (include/mcx/mcx.hpp) compiles against code written
for the reference API and, on a GPU, agrees with the oracle."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def build(tmp_path) -> Path:
    exe = tmp_path / "test_dropin"
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/test_dropin.cpp"),
           f"-L{ROOT / 'paper_1603_08390_b200/lib'}", "-lgenie_b200", f"-L{ROOT / 'oracle/_build'}", "-lgenie_oracle",
           f"-Wl,-rpath,{ROOT / 'paper_1603_08390_b200/lib'}", f"-Wl,-rpath,{ROOT / 'oracle/_build'}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_dropin_compiles_and_links(tmp_path):
    assert build(tmp_path).exists()


@pytest.mark.gpu
def test_dropin_runs_on_gpu(gpu, tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "dropin: ok" in r.stdout, r.stdout + r.stderr
