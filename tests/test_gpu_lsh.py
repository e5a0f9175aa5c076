"""LSH / minHash transforms on the GPU: bit-exact with the reference tokens
(golden fixtures from LshEncoder::encode_point) and with the oracle on larger
SIFT- and OCR-shaped samples; GPU index build from tokens equals the host CSR."""
from pathlib import Path

import numpy as np
import pytest

from paper_1603_08390_b200 import Encoder, lsh_config, synth
from paper_1603_08390_b200.engine import MINHASH, PSTABLE, RBH, DeviceIndex, csr_from_tokens

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("name", ["pstable_sift", "pstable_rehash", "rbh_ocr", "rbh_small"])
def test_tokens_equal_reference(gpu, name):
    g = np.load(GOLD / "lsh_tokens.npz")
    fam, m, dims, seed, rehash, domain = (int(x) for x in g[name + "_meta"])
    w, sigma = (float(x) for x in g[name + "_wsig"])
    enc = Encoder(lsh_config(fam, m, dims, seed, domain, w=w, sigma=sigma, rehash_pstable=bool(rehash)), gpu)
    assert np.array_equal(enc.encode(g[name + "_points"]), g[name + "_tokens"])


def test_pstable_sift_shaped_sample_equals_oracle(gpu, oracle):
    ds = synth.sift(n=20_000, dims=128, queries=16)
    enc = Encoder(lsh_config(PSTABLE, 237, 128, 3, w=4.0), gpu)
    got = enc.encode(ds.points)
    want = oracle.lsh_encode(0, 237, 128, 3, points=ds.points, w=4.0)
    assert np.array_equal(got, want), int((got != want).sum())


def test_rbh_ocr_shaped_sample_equals_oracle(gpu, oracle):
    ds = synth.ocr(n=1500, dims=784, queries=4)
    sigma = oracle.kernel_width(ds.points[:1000])
    enc = Encoder(lsh_config(RBH, 237, 784, 7, sigma=sigma), gpu)
    got = enc.encode(ds.points)
    want = oracle.lsh_encode(1, 237, 784, 7, points=ds.points, sigma=sigma)
    assert np.array_equal(got, want), int((got != want).sum())


def test_rbh_boundary_points_exact(gpu, oracle):
    # points sitting exactly on grid cell boundaries exercise the exact-division path
    from paper_1603_08390_b200.engine import lsh_sample
    cfg = lsh_config(RBH, 8, 4, 11, sigma=2.0)
    a, b, hs, rs = lsh_sample(cfg)
    pitch, shift = a.reshape(8, 4), b.reshape(8, 4)
    pts = []
    for f in range(8):
        for c in (-2, -1, 0, 1, 3):
            pts.append((shift[f] + c * pitch[f]).astype(np.float32))
    pts = np.array(pts, np.float32)
    got = Encoder(cfg, gpu).encode(pts)
    want = oracle.lsh_encode(1, 8, 4, 11, points=pts, sigma=2.0)
    assert np.array_equal(got, want)


def test_minhash_equals_oracle(gpu, oracle):
    ds = synth.sets(n=3000, queries=8)
    enc = Encoder(lsh_config(MINHASH, 128, 0, 5, rehash_domain=8192), gpu)
    got = enc.encode_sets(ds.set_off, ds.elems)
    want = oracle.lsh_encode(2, 128, 0, 5, set_off=ds.set_off, elems=ds.elems)
    assert np.array_equal(got, want)


def test_minhash_collision_rate_tracks_jaccard(gpu):
    # collision probability of a minHash function = Jaccard similarity
    rng = np.random.default_rng(3)
    base = rng.integers(0, 2**63, size=200, dtype=np.uint64)
    other = base.copy()
    other[:100] = rng.integers(0, 2**63, size=100, dtype=np.uint64)  # J = 100/300
    enc = Encoder(lsh_config(MINHASH, 4096, 0, 9, rehash_domain=1 << 30), gpu)
    t = enc.encode_sets(np.array([0, 200, 400], np.uint64), np.concatenate([base, other]))
    rate = float((t[0] == t[1]).mean())
    assert abs(rate - 1 / 3) < 4 * np.sqrt((1 / 3) * (2 / 3) / 4096)


def test_index_from_tokens_equals_host_csr(gpu):
    import torch
    rng = np.random.default_rng(5)
    toks = rng.integers(0, 67, size=(20_000, 37), dtype=np.uint32)
    d = torch.from_numpy(toks.astype(np.int32)).cuda(gpu)
    ix = DeviceIndex.from_tokens_device(d.data_ptr(), 20_000, 37, 67, device=gpu)
    want = csr_from_tokens(toks)
    got = ix.export()
    assert np.array_equal(got.keys, want.keys) and np.array_equal(got.key_off, want.key_off)
    assert np.array_equal(got.postings, want.postings)
    assert all(ix.dim_stats()[:37] == 1)
