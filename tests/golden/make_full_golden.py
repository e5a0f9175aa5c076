#!/usr/bin/env python
"""Full-size parity pins for the five BASELINE.json configs,
computed on the CPU in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_full_golden.py [c1 c2 c3 c4 c5]

Every engine result comes from the UNMODIFIED reference (oracle/_ref ->
mcx::build_index + mcx::execute_batch, Selector::cpq, ExecMode::parallel over
all host threads) run on the same seeded inputs the GPU tests generate:

  c1  adult 48 842 x 14, 1024 queries                       reference engine
  c2  tweets 7M docs, V=1M, 1024 queries                    reference engine
  c3  sift 4M x 128 -> p-stable m=237 tokens, 1024 queries  reference encoder + engine
  c4  minhash 2M sets -> 128 minhash tokens, 4096 queries   oracle encoder (minHash has no
                                                            reference) + reference engine
  c5  ocr 1M x 784 -> RBH m=237 tokens, 2048 queries, k=1   reference encoder + engine

For C3/C5 the plain-C oracle's tokens are also computed and the number of
tokens that differ from the reference's is recorded (north_star: "fp32
boundary disagreements counted"; the fp64 path must show 0).

Output: tests/golden/full_configs.json -- per config the sha256 of the
generated inputs, of the index CSR and of the token matrices, the
hash_results digest (engine.hpp:141-153), the threshold sum, and timings.
The GPU tests (tests/test_gpu_full.py) regenerate the inputs with the same
seeds and compare against these digests only.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import Oracle, RefLib  # noqa: E402
from paper_1603_08390_b200 import synth  # noqa: E402
from paper_1603_08390_b200.engine import kernel_width_heuristic, point_queries  # noqa: E402

OUT = HERE / "full_configs.json"


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def csr_digest_from_ref(rix) -> tuple[str, int, int]:
    """sha of (n, keys, key_off, postings) of the reference index image; spans
    of an unsplit index tile the list array in keyword order
    (index_io.hpp:114-116), so key_off are the first spans' begins."""
    keys, first, cnt, sb, se, post = rix.export()
    key_off = np.concatenate([sb[first.astype(np.int64)], np.array([post.shape[0]], np.uint64)]).astype(np.uint64)
    return keys, key_off, post


def run_engine(rix, qb, label):
    t = time.perf_counter()
    rc, r = rix.execute(qb, selector=0, sequential=False, workers=0)
    dt = time.perf_counter() - t
    if rc:
        raise RuntimeError(f"{label}: reference error {rc}: {r}")
    print(f"  {label}: reference execute_batch {dt:.1f}s, hash {r.hash:#018x}", flush=True)
    return r, dt


def result_fields(r) -> dict:
    return {"hash": f"{r.hash:#018x}", "thresholds_sum": int(r.threshold.astype(np.int64).sum()),
            "lengths_sum": int(r.length.astype(np.int64).sum()),
            "top1_sum": int(r.counts[:, 0].astype(np.int64).sum()) if r.counts.shape[1] else 0}


def config_csr(ref, ds, name):
    t = time.perf_counter()
    rix = ref.index(ds.csr)
    build_s = time.perf_counter() - t
    keys, key_off, post = csr_digest_from_ref(rix)
    assert np.array_equal(keys, ds.csr.keys) and np.array_equal(key_off, ds.csr.key_off)
    assert np.array_equal(post, ds.csr.postings)
    r, q_s = run_engine(rix, ds.queries, name)
    return {"source": "reference", "n": int(ds.csr.n), "queries": len(ds.queries),
            "csr": sha(np.array([ds.csr.n], np.uint64), ds.csr.keys, ds.csr.key_off, ds.csr.postings),
            "query_items": sha(ds.queries.qid, ds.queries.k, ds.queries.item_off, ds.queries.dim, ds.queries.lo,
                               ds.queries.hi),
            "postings": int(ds.csr.num_postings), "keywords": int(ds.csr.num_keys),
            "ref_build_s": round(build_s, 1), "ref_query_s": round(q_s, 1), **result_fields(r)}


def tokens_config(ref, name, n, m, toks, qtoks, k, extra):
    """Reference index over LSH tokens (dim = function index) + engine."""
    t = time.perf_counter()
    obj_off = np.arange(n + 1, dtype=np.uint64) * np.uint64(m)
    dims = np.tile(np.arange(m, dtype=np.uint16), n)
    rix = ref.index_from_objects(n, obj_off, dims, toks.reshape(-1))
    del obj_off, dims
    build_s = time.perf_counter() - t
    print(f"  {name}: reference build_index {build_s:.1f}s", flush=True)
    keys, key_off, post = csr_digest_from_ref(rix)
    csr = sha(np.array([n], np.uint64), keys, key_off, post)
    nk, npost = int(keys.shape[0]), int(post.shape[0])
    del keys, key_off, post
    qb = point_queries(qtoks, k)
    r, q_s = run_engine(rix, qb, name)
    del rix
    return {"source": extra.pop("source"), "n": n, "queries": int(qtoks.shape[0]), "csr": csr,
            "tokens": sha(toks), "query_tokens": sha(qtoks), "postings": npost, "keywords": nk,
            "ref_build_s": round(build_s, 1), "ref_query_s": round(q_s, 1), **extra, **result_fields(r),
            "_result": r}


def c1(ref, o):
    return config_csr(ref, synth.adult(), "c1")


def c2(ref, o):
    return config_csr(ref, synth.tweets(), "c2")


def c3(ref, o):
    ds = synth.sift()
    t = time.perf_counter()
    toks = ref.lsh_encode(0, 237, 128, 3, ds.points, w=4.0)
    qt = ref.lsh_encode(0, 237, 128, 3, ds.query_points, w=4.0)
    enc_s = time.perf_counter() - t
    print(f"  c3: reference p-stable encode {enc_s:.1f}s", flush=True)
    otoks = o.lsh_encode(0, 237, 128, 3, points=ds.points, w=4.0)
    mism = int((otoks != toks).sum())
    del otoks
    pts_sha = sha(ds.points, ds.query_points)
    del ds
    out = tokens_config(ref, "c3", toks.shape[0], 237, toks, qt, 100,
                        {"source": "reference (encoder + engine)", "points": pts_sha, "ref_encode_s": round(enc_s, 1),
                         "oracle_token_mismatches": mism, "w": 4.0})
    out.pop("_result")
    return out


def c4(ref, o):
    ds = synth.sets()
    t = time.perf_counter()
    toks = o.lsh_encode(2, 128, 0, 5, set_off=ds.set_off, elems=ds.elems)
    qt = o.lsh_encode(2, 128, 0, 5, set_off=ds.query_set_off, elems=ds.query_elems)
    enc_s = time.perf_counter() - t
    sets_sha = sha(ds.set_off, ds.elems, ds.query_set_off, ds.query_elems)
    del ds
    out = tokens_config(ref, "c4", toks.shape[0], 128, toks, qt, 100,
                        {"source": "oracle minHash tokens (no reference minHash, SURVEY 8c) + reference engine",
                         "sets": sets_sha, "oracle_encode_s": round(enc_s, 1)})
    out.pop("_result")
    return out


def c5(ref, o):
    ds = synth.ocr()
    sigma = kernel_width_heuristic(ds.points[:10_000])
    t = time.perf_counter()
    toks = ref.lsh_encode(1, 237, 784, 7, ds.points, sigma=sigma, domain=8192)
    qt = ref.lsh_encode(1, 237, 784, 7, ds.query_points, sigma=sigma, domain=8192)
    enc_s = time.perf_counter() - t
    print(f"  c5: reference RBH encode {enc_s:.1f}s", flush=True)
    oq = o.lsh_encode(1, 237, 784, 7, points=ds.query_points, sigma=sigma)
    otoks = o.lsh_encode(1, 237, 784, 7, points=ds.points, sigma=sigma)
    mism = int((otoks != toks).sum()) + int((oq != qt).sum())
    del otoks, oq
    pts_sha = sha(ds.points, ds.query_points)
    labels, qlabels = ds.labels, ds.query_labels
    del ds
    out = tokens_config(ref, "c5", toks.shape[0], 237, toks, qt, 1,
                        {"source": "reference (encoder + engine)", "points": pts_sha, "ref_encode_s": round(enc_s, 1),
                         "oracle_token_mismatches": mism, "sigma_hex": float(sigma).hex()})
    r = out.pop("_result")
    out["top1_accuracy"] = round(float((labels[r.ids[:, 0]] == qlabels).mean()), 4)
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c4", "c3", "c5"]
    ref, o = RefLib(), Oracle()
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    res["_meta"] = {"host_threads": ref.hardware_threads(),
                    "engine": "mcx::execute_batch Selector::cpq ExecMode::parallel (unmodified reference headers)"}
    for name in which:
        print(name, flush=True)
        t = time.perf_counter()
        res[name] = globals()[name](ref, o)
        res[name]["wall_s"] = round(time.perf_counter() - t, 1)
        OUT.write_text(json.dumps(res, indent=1, sort_keys=True) + "\n")
        print(f"  {name}: {res[name]}", flush=True)
