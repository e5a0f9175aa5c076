"""The C++ drop-in header (include/mcx/mcx.hpp) compiles against code written
for the reference API and, on a GPU, agrees with the oracle:

  tests/cpp/test_dropin.cpp         engine / partitions / LSH / documents
  tests/cpp/test_reference_api.cpp  the reference's test_index.cpp cases, the
                                    relational encoders, LshEncoder::token and
                                    acceptance criteria 1, 3, 10, 12 (engine half)
  tests/cpp/test_sequence.cpp       the reference's sequence-search tests
                                    (test_sa.cpp): SequenceSearcher with GPU
                                    retrieval + GPU edit-distance verification
  tests/cpp/test_dataset.cpp        the reference's dataset tests (CSV + schema,
                                    discretize, vector files, encoder sidecar);
                                    CPU, plus the fig1 pipeline on the GPU
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SOURCES = ["test_dropin", "test_reference_api", "test_dataset", "test_sequence"]


def build(tmp_path, name="test_dropin") -> Path:
    exe = tmp_path / name
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", f"-I{ROOT / 'include'}", str(ROOT / f"tests/cpp/{name}.cpp"),
           f"-L{ROOT / 'paper_1603_08390_b200/lib'}", "-lgenie_b200", f"-L{ROOT / 'oracle/_build'}", "-lgenie_oracle",
           f"-Wl,-rpath,{ROOT / 'paper_1603_08390_b200/lib'}", f"-Wl,-rpath,{ROOT / 'oracle/_build'}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return exe


@pytest.mark.parametrize("name", SOURCES)
def test_dropin_compiles_and_links(tmp_path, name):
    assert build(tmp_path, name).exists()


@pytest.mark.gpu
def test_dropin_runs_on_gpu(gpu, tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "dropin: ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_reference_api_on_gpu(gpu, tmp_path):
    exe = build(tmp_path, "test_reference_api")
    r = subprocess.run([str(exe), "120"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "reference api: ok" in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]


def test_dataset_adapters_cpu(tmp_path):
    exe = build(tmp_path, "test_dataset")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "dataset: ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_dataset_pipeline_on_gpu(gpu, tmp_path):
    exe = build(tmp_path, "test_dataset")
    r = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "dataset: ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_sequence_search_on_gpu(gpu, tmp_path):
    exe = build(tmp_path, "test_sequence")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "sequence: ok" in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]
