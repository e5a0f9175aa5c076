#!/usr/bin/env python
"""C3/C5 token diagnosis on the GPU box: host-sampled LSH parameters of the
GPU library vs the reference shim (oracle/_ref) and the oracle, bit for bit,
then GPU tokens vs the reference's tokens on the full config (mismatch count
and the first differing (point, function) pairs).  Test infrastructure."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import Oracle, RefLib  # noqa: E402
from paper_1603_08390_b200 import Encoder, lsh_config, synth  # noqa: E402
from paper_1603_08390_b200.engine import PSTABLE, RBH, lsh_sample  # noqa: E402


def main(which="c3", n=None):
    ref, o = RefLib(), Oracle()
    if which == "c3":
        ds = synth.sift(n=n or 4_000_000)
        fam, m, dims, seed, kw = PSTABLE, 237, 128, 3, dict(w=4.0)
        cfg = lsh_config(PSTABLE, m, dims, seed, w=4.0)
    else:
        import json
        g = json.loads((ROOT / "tests/golden/full_configs.json").read_text())["c5"]
        sigma = float.fromhex(g["sigma_hex"])
        ds = synth.ocr(n=n or 1_000_000)
        fam, m, dims, seed, kw = RBH, 237, 784, 7, dict(sigma=sigma)
        cfg = lsh_config(RBH, m, dims, seed, sigma=sigma, rehash_domain=8192)
    ga, gb, *_ = lsh_sample(cfg)
    ra, rb, _ = ref.lsh_params(fam, m, dims, seed, **kw)
    oa, ob, *_ = o.lsh_params(fam, m, dims, seed, **kw)
    for name, x, y in (("gpu-lib vs ref a", ga, ra), ("gpu-lib vs ref b", gb, rb), ("oracle vs ref a", oa, ra),
                       ("oracle vs ref b", ob, rb)):
        x = np.asarray(x, np.float64).reshape(-1)
        y = np.asarray(y, np.float64).reshape(-1)[: x.shape[0]]
        d = np.nonzero(x.view(np.uint64) != y.view(np.uint64))[0]
        print(f"{name}: {d.shape[0]} of {x.shape[0]} differ", d[:5], flush=True)
    enc = Encoder(cfg, 0)
    gt = enc.encode(ds.points)
    rt = ref.lsh_encode(fam, m, dims, seed, ds.points, **({"w": 4.0} if fam == PSTABLE else
                                                         {"sigma": kw["sigma"], "domain": 8192}))
    bad = np.argwhere(gt != rt)
    print(f"tokens: {bad.shape[0]} of {gt.size} differ", flush=True)
    for p, f in bad[:10]:
        print(f"  point {p} fn {f}: gpu {gt[p, f]} ref {rt[p, f]}", flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["c3"]), *(int(a) for a in sys.argv[2:3]))
