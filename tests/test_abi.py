"""The C-ABI libraries load and export every symbol their headers declare
(no compute calls: runs without a GPU)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_1603_08390_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent


def declared(header: Path):
    text = re.sub(r"/\*.*?\*/", "", header.read_text(), flags=re.S)
    names = re.findall(r"^[A-Za-z_][\w \*]*?\b(genie_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


@pytest.mark.parametrize("header,lib", [("include/genie/genie.h", N.ENGINE_LIB),
                                        ("include/genie/genie_synth.h", N.SYNTH_LIB)])
def test_library_exports_every_declared_symbol(header, lib):
    names = declared(ROOT / header)
    assert len(names) > 10
    dll = ctypes.CDLL(str(lib))
    missing = [n for n in names if not hasattr(dll, n)]
    assert not missing, f"{lib.name} lacks {missing}"


def test_ctypes_bindings_cover_the_header():
    names = declared(ROOT / "include/genie/genie.h")
    assert sorted(N.ENGINE_SYMBOLS) == names
    assert sorted(N.SYNTH_SYMBOLS) == declared(ROOT / "include/genie/genie_synth.h")


def test_engine_is_sm100a_only():
    # the fatbin carries sm_100a SASS and nothing else
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.ENGINE_LIB)], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_config_defaults_mirror_reference():
    c = N.engine().genie_config_default()
    assert c.selector == 0 and c.span_chunk > 0 and c.max_spans_per_task == 2  # engine.hpp:36-42
    l = N.engine().genie_lsh_config_default()  # lsh.hpp:132-145
    assert (l.family, l.m, l.rehash_domain, l.seed, l.w, l.bucket_count, l.bucket_min, l.rehash_pstable, l.sigma) == \
        (1, 237, 8192, 1, 4.0, 67, -33, 0, 1.0)


def test_null_index_is_a_contract_error():
    from paper_1603_08390_b200 import engine as E
    err = ctypes.create_string_buffer(256)
    rc = N.engine().genie_query_batch(None, None, 0, None, None, None, None, None, None, 0, None, None, None, None,
                                      None, None, err, 256)
    assert rc == N.GENIE_ERR_CONTRACT and b"null index" in err.value
    cfg = E.config(span_chunk=0)
    rc = N.engine().genie_query_batch(None, ctypes.byref(cfg), 0, None, None, None, None, None, None, 0, None, None,
                                      None, None, None, None, err, 256)
    assert rc == N.GENIE_ERR_CONTRACT and b"span_chunk and max_spans_per_task must be positive" in err.value
