"""Shared helpers for the golden fixtures (tests only)."""
import hashlib

import numpy as np

from paper_1603_08390_b200 import synth


def digest_csr(csr) -> str:
    h = hashlib.sha256()
    for a in (np.array([csr.n], np.uint64), csr.keys, csr.key_off, csr.postings):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def digest_queries(qb) -> str:
    h = hashlib.sha256()
    for a in (qb.qid, qb.k, qb.item_off, qb.dim, qb.lo, qb.hi):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def config_dataset(name):
    if name == "adult":
        return synth.adult()
    if name == "tweets_200k":
        return synth.tweets(n=200_000, vocab=50_000, words=10, queries=64, k=100)
    if name == "tweets_1m":
        return synth.tweets(n=1_000_000, vocab=1_000_000, words=10, queries=32, k=100)
    raise KeyError(name)
