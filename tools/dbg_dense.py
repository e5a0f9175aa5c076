import os, sys
sys.path.insert(0, '.')
import numpy as np
from oracle.pyoracle import Oracle
from paper_1603_08390_b200 import DeviceIndex, config, synth
ds = synth.random_instance(n=40_000, dims=3, tokens=5, max_kw=8, queries=40, max_items=40, max_span=2, max_k=60, seed=5)
o = Oracle(); want = o.index(ds.csr).execute(ds.queries)
lens = np.diff(ds.csr.key_off)
print("n", ds.csr.n, "keys", ds.csr.num_keys, "list len min/max", lens.min(), lens.max())
for dens in ["0", "0.002", "0.05", "0.2"]:
    os.environ["GENIE_DENSE_MIN_DENSITY"] = dens
    ix = DeviceIndex.from_csr(ds.csr)
    for sel in (0, 1):
        for tb in (0, 4096, 16384):
            r = ix.query(ds.queries, config(selector=sel, tile_bytes=tb))
            bad = [q for q in range(40) if r.row(q) != want.row(q) or r.threshold[q] != want.threshold[q]]
            print(dens, sel, tb, "bad", bad[:10], [ (int(want.bound[q]), int(want.length[q]), int(r.length[q]), int(want.threshold[q]), int(r.threshold[q])) for q in bad[:4]])
