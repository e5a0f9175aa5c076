#!/usr/bin/env python
"""Ultra-sparse set collections (live sets spread over tens of millions of ids): dense W = 8
tiles vs the hashed class at two tile sizes, same results (hash_results) required.  GPU box only:
`python tools/sparse_probe.py`."""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1603_08390_b200 import DeviceIndex, point_queries
from paper_1603_08390_b200.engine import CSR

def sparse_sets(n, live, m, domain, Q, seed=3):
    rng = np.random.default_rng(seed)
    ids = np.sort(rng.choice(n, size=live, replace=False)).astype(np.uint32)
    toks = rng.integers(0, domain, size=(live, m), dtype=np.uint32)
    flat = ((np.arange(m, dtype=np.uint64)[None, :] << np.uint64(32)) | toks.astype(np.uint64)).reshape(-1)
    oid = np.repeat(ids, m)
    order = np.argsort(flat, kind="stable")
    sk, sid = flat[order], oid[order]
    uniq, starts = np.unique(sk, return_index=True)
    off = np.concatenate([starts.astype(np.uint64), np.array([sk.shape[0]], np.uint64)])
    qt = toks[rng.integers(0, live, size=Q)].copy()
    flip = rng.random(qt.shape) < 0.5
    qt[flip] = rng.integers(0, domain, size=int(flip.sum()), dtype=np.uint32)
    return CSR(n, uniq, off, sid), qt

for (n, live, m, domain) in [(20_000_000, 1_000_000, 32, 4096), (50_000_000, 2_000_000, 64, 8192), (4_000_000, 1_000_000, 64, 4096)]:
    t = time.time(); csr, qt = sparse_sets(n, live, m, domain, 2048); gen = time.time() - t
    ix = DeviceIndex.from_csr(csr, device=0)
    qb = point_queries(qt, 100)
    res = {}
    for name, knobs in [("dense", {"GENIE_HASH_TILES": "0"}), ("hash4", {"GENIE_HASH_TILES": "4", "GENIE_HASH_LOAD_PCT": "100"}),
                        ("hash11", {"GENIE_HASH_TILES": "11", "GENIE_HASH_LOAD_PCT": "100"})]:
        os.environ.update(knobs)
        for _ in range(2): r = ix.query(qb)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); r = ix.query(qb, timings=True); ts.append(time.perf_counter() - t0)
        res[name] = r
        print(n, live, m, domain, name, "P/q", r.stats["postings"] // len(qb), "items", r.stats["work_items"], "fallback", r.stats["fallback_tiles"],
              "match_ms %.3f" % (r.timings["match_ns"] / 1e6), "total_ms %.3f" % (min(ts) * 1e3), "q/s %.0f" % (len(qb) / min(ts)), hex(r.hash()), flush=True)
    assert res["dense"].hash() == res["hash4"].hash() == res["hash11"].hash()
    ix.close()
