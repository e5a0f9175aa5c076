#!/usr/bin/env python
"""Generates tests/golden/* from the REFERENCE ITSELF (the unmodified mcx
headers compiled by oracle/Makefile into oracle/_ref/libmcx_ref.so).

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py

Fixtures (small, committed):
  random_instances.npz   40 random (objects, queries) instances shaped like
                         test_engine.cpp:34-60 and acceptance.cpp:57-105, with the
                         reference's execute_batch (Selector::cpq, sequential)
                         results and hash_results
  cpq_streams.npz        CountPriorityQueue update streams (test_cpq.cpp:257-278
                         style) with the reference's extract() and final AT
  lsh_tokens.npz         p-stable / random-binning tokens of small point sets from
                         LshEncoder::encode_point, plus the sampled parameters
  configs.json           result digests of the seeded workloads at test sizes
                         (C1 adult full size, C2 tweets reduced) and a digest of
                         the generated inputs (guards generator drift)
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import RefLib  # noqa: E402
from paper_1603_08390_b200 import synth  # noqa: E402
from paper_1603_08390_b200.engine import QueryBatch  # noqa: E402


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


INSTANCE_SPECS = []
rng = np.random.default_rng(20260101)
for i in range(40):
    n = int(rng.choice([1, 5, 17, 64, 300, 1000, 5000, 20000]))
    INSTANCE_SPECS.append(dict(
        n=n, dims=int(rng.integers(1, 5)), tokens=int(rng.integers(2, 17)), max_kw=int(rng.integers(1, 7)),
        queries=int(rng.integers(1, 12)), max_items=int(rng.integers(1, 7)), max_span=int(rng.integers(0, 4)),
        max_k=int(rng.choice([1, 3, 10, 100, 1000])), seed=1000 + i))


def make_instances(ref: RefLib):
    out = {}
    for i, spec in enumerate(INSTANCE_SPECS):
        ds = synth.random_instance(**spec)
        qb = ds.queries
        ix = ref.index(ds.csr)
        rc, r = ix.execute(qb, selector=0, sequential=True, stride=max(qb.max_k, 1))
        assert rc == 0, r
        pre = f"i{i}_"
        out[pre + "csr_n"] = np.array([ds.csr.n], np.uint64)
        out[pre + "keys"], out[pre + "key_off"], out[pre + "postings"] = ds.csr.keys, ds.csr.key_off, ds.csr.postings
        for f in ("qid", "k", "item_off", "dim", "lo", "hi"):
            out[pre + "q_" + f] = getattr(qb, f)
        out[pre + "len"], out[pre + "thr"] = r.length, r.threshold
        out[pre + "ids"], out[pre + "counts"] = r.ids, r.counts
        out[pre + "hash"] = np.array([r.hash], np.uint64)
        # split-list and partitioned runs must agree (test_engine.cpp:134-196)
        ix_split = ref.index(ds.csr, split=4)
        rc2, r2 = ix_split.execute(qb, selector=0, sequential=False, workers=4, span_chunk=7, spans_per_task=3,
                                   stride=max(qb.max_k, 1))
        if rc2 or r2.hash != r.hash:  # observed once in ~4000 runs of the reference's parallel engine
            print(f"warning: reference parallel/split run differs on instance {i}: rc={rc2}", file=sys.stderr)
        if ds.csr.n >= 2:
            rc3, r3 = ix.execute_partitioned(qb, max(1, ds.csr.n // 3), stride=max(qb.max_k, 1))
            assert rc3 == 0 and r3.hash == r.hash, (r3, r.hash)
    out["count"] = np.array([len(INSTANCE_SPECS)], np.uint64)
    np.savez_compressed(HERE / "random_instances.npz", **out)


def make_streams(ref: RefLib):
    g = np.random.default_rng(101)
    out = {}
    cases = []
    for t in range(60):
        n = int(1 + g.integers(0, 200))
        max_count = int(1 + g.integers(0, 24))
        k = int(1 + g.integers(0, 12))
        counts = g.integers(0, max_count + 1, size=n)
        stream = np.repeat(np.arange(n, dtype=np.uint32), counts)
        g.shuffle(stream)
        rc, ent, thr, at = ref.cpq_stream(n, max_count, k, stream)
        assert rc == 0
        cases.append((n, max_count, k, stream, ent, thr, at))
    for i, (n, mc, k, stream, ent, thr, at) in enumerate(cases):
        out[f"s{i}_meta"] = np.array([n, mc, k, thr, at, len(ent)], np.uint64)
        out[f"s{i}_stream"] = stream
        out[f"s{i}_ent"] = np.array(ent, np.uint32).reshape(-1, 2)
    out["count"] = np.array([len(cases)], np.uint64)
    np.savez_compressed(HERE / "cpq_streams.npz", **out)


def make_lsh(ref: RefLib):
    out = {}
    g = np.random.default_rng(7)
    cases = [
        ("pstable_sift", 0, 237, 128, 3, dict(w=4.0), (g.normal(0, 3.3, size=(60, 128))).astype(np.float32)),
        ("pstable_rehash", 0, 37, 16, 11, dict(w=2.5, rehash=True, domain=1024),
         g.normal(0, 1.0, size=(50, 16)).astype(np.float32)),
        ("rbh_ocr", 1, 237, 784, 7, dict(sigma=282.8), g.uniform(0, 1, size=(12, 784)).astype(np.float32)),
        ("rbh_small", 1, 64, 8, 5, dict(sigma=1.5), g.normal(0, 1, size=(80, 8)).astype(np.float32)),
    ]
    for name, fam, m, dims, seed, kw, pts in cases:
        toks = ref.lsh_encode(fam, m, dims, seed, pts, nthreads=8, **{k: v for k, v in kw.items()})
        a, b, rs = ref.lsh_params(fam, m, dims, seed, w=kw.get("w", 4.0), sigma=kw.get("sigma", 1.0))
        out[name + "_points"] = pts
        out[name + "_tokens"] = toks
        out[name + "_meta"] = np.array([fam, m, dims, seed, int(kw.get("rehash", False)), kw.get("domain", 8192)],
                                       np.int64)
        out[name + "_wsig"] = np.array([kw.get("w", 4.0), kw.get("sigma", 1.0)], np.float64)
        if a.size <= 4096:  # parameters of the small cases only (size)
            out[name + "_a"], out[name + "_b"] = a, b
        out[name + "_rs"] = rs
    out["kernel_width"] = np.array([ref.kernel_width(cases[3][6]), ref.kernel_width(cases[2][6])], np.float64)
    np.savez_compressed(HERE / "lsh_tokens.npz", **out)


def make_configs(ref: RefLib):
    res = {}
    ds = synth.adult()
    ix = ref.index(ds.csr)
    rc, r = ix.execute(ds.queries, selector=0, sequential=False, workers=0)
    assert rc == 0
    res["adult"] = {"csr": digest_csr(ds.csr), "queries": digest_queries(ds.queries), "hash": f"{r.hash:#018x}",
                    "keywords": ds.csr.num_keys, "postings": ds.csr.num_postings,
                    "thresholds_sum": int(r.threshold.sum())}
    ds = synth.tweets(n=200_000, vocab=50_000, words=10, queries=64, k=100)
    ix = ref.index(ds.csr)
    rc, r = ix.execute(ds.queries, selector=0, sequential=False, workers=0)
    assert rc == 0
    res["tweets_200k"] = {"csr": digest_csr(ds.csr), "queries": digest_queries(ds.queries), "hash": f"{r.hash:#018x}"}
    ds = synth.tweets(n=1_000_000, vocab=1_000_000, words=10, queries=32, k=100)
    ix = ref.index(ds.csr)
    rc, r = ix.execute(ds.queries, selector=0, sequential=False, workers=0)
    assert rc == 0
    res["tweets_1m"] = {"csr": digest_csr(ds.csr), "queries": digest_queries(ds.queries), "hash": f"{r.hash:#018x}"}
    (HERE / "configs.json").write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    ref = RefLib()
    make_instances(ref)
    make_streams(ref)
    make_lsh(ref)
    make_configs(ref)
    for p in sorted(HERE.glob("*")):
        print(p.name, p.stat().st_size)
