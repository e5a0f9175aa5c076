"""GPU edit distances (genie_seqset_distances: bit-parallel Myers/Hyyro, one
thread per pair) against the reference's golden vectors (3000 pairs up to
~700 bytes: one- and multi-word queries, caps 0..1000) and the plain-Python
oracle on random corpora; the verification replay on GPU distances equals
the reference's verify_candidates (sa.hpp:298-336)."""
from pathlib import Path

import numpy as np
import pytest

from oracle.pyoracle import edit_distance, verify_candidates
from paper_1603_08390_b200.engine import ContractError, SeqSet

pytestmark = pytest.mark.gpu
GOLD = np.load(Path(__file__).parent / "golden" / "sequences.npz")


def strings(b, off):
    return [bytes(b[int(off[i]):int(off[i + 1])]) for i in range(off.shape[0] - 1)]


def test_pairs_equal_reference(gpu):
    A, B = strings(GOLD["a_bytes"], GOLD["a_off"]), strings(GOLD["b_bytes"], GOLD["b_off"])
    ss = SeqSet(B, device=gpu)
    for i in range(len(A)):  # one query per pair: its own candidate
        got = ss.distances(A[i], [i])
        assert int(got[0]) == int(GOLD["exact"][i]), (i, len(A[i]), len(B[i]))
        gb = ss.distances(A[i], [i], cap=int(GOLD["cap"][i]))
        assert int(gb[0]) == int(GOLD["bounded"][i]), i
    ss.close()


def test_scan_all_sequences(gpu):
    rng = np.random.default_rng(3)
    corpus = [bytes((97 + rng.integers(0, 4, int(rng.integers(0, 90)))).astype(np.uint8)) for _ in range(1500)]
    ss = SeqSet(corpus, device=gpu)
    for q in (corpus[7], corpus[100][:20] + b"zz", b"", b"a" * 300):
        want = [edit_distance(q, c) for c in corpus]
        assert ss.distances(q).tolist() == want
        assert ss.distances(q, cap=5).tolist() == [min(w, 6) for w in want]
    with pytest.raises(ContractError):
        ss.distances(b"abc", [1500])
    ss.close()


def test_verify_replay_on_gpu_distances(gpu):
    qs = strings(GOLD["vq_bytes"], GOLD["vq_off"])
    flat = strings(GOLD["vc_bytes"], GOLD["vc_off"])
    per, nh = GOLD["vc_per"], GOLD["v_nhits"]
    ids, cnt, out = GOLD["v_ids"], GOLD["v_cnt"], GOLD["v_out"]
    c0 = h0 = 0
    for t in range(len(qs)):
        corpus = flat[c0:c0 + int(per[t])]
        hits = list(zip(ids[h0:h0 + int(nh[t])].tolist(), cnt[h0:h0 + int(nh[t])].tolist()))
        ss = SeqSet(corpus, device=gpu)
        d = ss.distances(qs[t], [h[0] for h in hits])  # exact distances of every candidate, one launch
        exact = dict(zip((h[0] for h in hits), d.tolist()))
        got = verify_candidates(qs[t], hits, 3, corpus, int(out[t][1]), bool(out[t][0]),
                                dist=lambda i, cap: exact[i] if cap is None else min(exact[i], cap + 1))
        assert got == tuple([int(out[t][2]), int(out[t][3]), bool(out[t][4]), int(out[t][5]), int(out[t][6])]), t
        ss.close()
        c0 += int(per[t])
        h0 += int(nh[t])
