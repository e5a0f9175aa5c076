#!/usr/bin/env python
"""Golden vectors for sequence verification (sa.hpp), computed by the
UNMODIFIED reference (oracle/_ref -> mcx::edit_distance,
edit_distance_bounded, verify_candidates):

    make -C oracle && python tests/golden/make_seq_golden.py

  pairs   random byte strings (lengths 0..700, alphabets 2..26, mutated
          near-copies so distances span 0..hundreds), a cap per pair, the
          exact and the bounded distance
  verify  small corpora + queries + count-sorted candidate lists, with and
          without the early break: (best_id, best_distance, certified,
          candidates_used, threshold_at_stop)

Output: tests/golden/sequences.npz
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle.pyoracle import RefLib  # noqa: E402

OUT = HERE / "sequences.npz"


def rand_str(rng, n, alpha):
    return bytes((97 + rng.integers(0, alpha, n)).astype(np.uint8))


def mutate(rng, s: bytes, edits: int, alpha: int) -> bytes:
    b = bytearray(s)
    for _ in range(edits):
        if not b:
            break
        pos = int(rng.integers(0, len(b)))
        op = int(rng.integers(0, 3))
        ch = 97 + int(rng.integers(0, alpha))
        if op == 0:
            b[pos] = ch
        elif op == 1:
            del b[pos]
        else:
            b.insert(pos, ch)
    return bytes(b)


def shared_grams(s: bytes, q: bytes, n: int) -> int:
    from collections import Counter
    a = Counter(s[i:i + n] for i in range(len(s) - n + 1))
    b = Counter(q[i:i + n] for i in range(len(q) - n + 1))
    return sum(min(c, b[g]) for g, c in a.items() if g in b)


def main():
    ref = RefLib()
    rng = np.random.default_rng(20261017)
    A, B, caps, exact, bounded = [], [], [], [], []
    for t in range(3000):
        alpha = int(rng.choice([2, 4, 6, 26]))
        la = int(rng.choice([0, 1, 5, 40, 63, 64, 65, 100, 127, 128, 129, 200, 255, 256, 257, 300, 520, 700]))
        la = max(0, la + int(rng.integers(-2, 3)))
        a = rand_str(rng, la, alpha)
        b = mutate(rng, a, int(rng.integers(0, max(1, la // 3 + 2))), alpha) if rng.random() < 0.7 else \
            rand_str(rng, int(rng.integers(0, 300)), alpha)
        cap = int(rng.choice([0, 1, 3, 10, 50, 200, 1000]))
        A.append(a)
        B.append(b)
        caps.append(cap)
        exact.append(ref.edit_distance(a, b))
        bounded.append(ref.edit_distance(a, b, cap))
    # verify_candidates cases (test_sa.cpp:185-206 shape, wider)
    vq, vcorp, vids, vcnt, vout = [], [], [], [], []
    for t in range(200):
        alpha = int(rng.choice([3, 4, 6]))
        corpus = [rand_str(rng, 10 + int(rng.integers(0, 40)), alpha) for _ in range(30)]
        q = mutate(rng, corpus[int(rng.integers(0, len(corpus)))], int(rng.integers(0, 6)), alpha)
        hits = sorted(((i, shared_grams(c, q, 3)) for i, c in enumerate(corpus)), key=lambda h: (-h[1], h[0]))
        hits = [h for h in hits if h[1] > 0][: int(rng.choice([1, 4, 16, 30]))] or [(0, 0)]
        req = len(hits) + int(rng.integers(0, 3))
        for eb in (True, False):
            out = ref.verify_candidates(q, [h[0] for h in hits], [h[1] for h in hits], 3, corpus, req, eb)
            vq.append(q)
            vcorp.append(corpus)
            vids.append([h[0] for h in hits])
            vcnt.append([h[1] for h in hits])
            vout.append((int(eb), req) + tuple(int(x) for x in out))

    def pack(strs):
        off = np.zeros(len(strs) + 1, np.uint64)
        off[1:] = np.cumsum([len(s) for s in strs])
        return np.frombuffer(b"".join(strs) or b"\0", np.uint8)[: int(off[-1])].copy(), off

    a_b, a_o = pack(A)
    b_b, b_o = pack(B)
    q_b, q_o = pack(vq)
    flat = [s for c in vcorp for s in c]
    c_b, c_o = pack(flat)
    np.savez_compressed(OUT, a_bytes=a_b, a_off=a_o, b_bytes=b_b, b_off=b_o, cap=np.array(caps, np.uint32),
                        exact=np.array(exact, np.uint32), bounded=np.array(bounded, np.uint32),
                        vq_bytes=q_b, vq_off=q_o, vc_bytes=c_b, vc_off=c_o,
                        vc_per=np.array([len(c) for c in vcorp], np.uint32),
                        v_ids=np.array([x for v in vids for x in v], np.uint32),
                        v_cnt=np.array([x for v in vcnt for x in v], np.uint32),
                        v_nhits=np.array([len(v) for v in vids], np.uint32),
                        v_out=np.array(vout, np.int64))
    print(f"wrote {OUT}: {len(A)} pairs (max len {max(map(len, A + B))}), {len(vout)} verify cases")


if __name__ == "__main__":
    main()
