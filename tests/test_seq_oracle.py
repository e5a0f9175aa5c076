"""The sequence-search oracle (oracle/pyoracle.py: edit_distance,
edit_distance_bounded, verify_candidates -- plain-Python restatements of
sa.hpp:109-162, 298-336) pinned against golden vectors the unmodified
reference computed (tests/golden/make_seq_golden.py), plus the reference's
own known answers (test_sa.cpp:119-183)."""
from pathlib import Path

import numpy as np
import pytest

from oracle.pyoracle import edit_distance, edit_distance_bounded, verify_candidates

GOLD = np.load(Path(__file__).parent / "golden" / "sequences.npz")


def strings(b, off):
    return [bytes(b[int(off[i]):int(off[i + 1])]) for i in range(off.shape[0] - 1)]


def test_known_answers():
    assert edit_distance(b"kitten", b"sitting") == 3
    assert edit_distance(b"same", b"same") == 0
    assert edit_distance(b"", b"abc") == 3 and edit_distance(b"abc", b"") == 3
    corpus = [b"abcdef", b"zzzzzz"]
    bid, bd, _, used, _ = verify_candidates(b"abcdxf", [(0, 4)], 3, corpus, 1)
    assert (bid, bd, used) == (0, 1, 1)
    out = verify_candidates(b"abcdefgh", [(0, 6), (1, 5)], 3, [b"abcdefgh", b"abcdefgx"], 2)
    assert out[0] == 0 and out[1] == 0 and out[3] == 1 and out[4] > 6
    with pytest.raises(ValueError):
        verify_candidates(b"abc", [], 3, corpus)


def test_edit_distance_matches_reference_vectors():
    A, B = strings(GOLD["a_bytes"], GOLD["a_off"]), strings(GOLD["b_bytes"], GOLD["b_off"])
    sel = [i for i in range(len(A)) if len(A[i]) * len(B[i]) <= 20_000][:400]
    assert len(sel) >= 200
    for i in sel:
        assert edit_distance(A[i], B[i]) == int(GOLD["exact"][i]), i
        assert edit_distance_bounded(A[i], B[i], int(GOLD["cap"][i])) == int(GOLD["bounded"][i]), i


def test_verify_candidates_matches_reference_vectors():
    qs = strings(GOLD["vq_bytes"], GOLD["vq_off"])
    flat = strings(GOLD["vc_bytes"], GOLD["vc_off"])
    per, nh = GOLD["vc_per"], GOLD["v_nhits"]
    ids, cnt, out = GOLD["v_ids"], GOLD["v_cnt"], GOLD["v_out"]
    c0 = h0 = 0
    for t in range(len(qs)):
        corpus = flat[c0:c0 + int(per[t])]
        hits = list(zip(ids[h0:h0 + int(nh[t])].tolist(), cnt[h0:h0 + int(nh[t])].tolist()))
        eb, req, bid, bd, cert, used, theta = (int(x) for x in out[t])
        assert verify_candidates(qs[t], hits, 3, corpus, req, bool(eb)) == (bid, bd, bool(cert), used, theta), t
        c0 += int(per[t])
        h0 += int(nh[t])
