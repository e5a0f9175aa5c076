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


@pytest.mark.parametrize("family", [PSTABLE, RBH])
def test_fp32_mode_disagreements_counted_and_bounded(gpu, oracle, family):
    """The opt-in fp32 transforms (genie_lsh_config.precision = GENIE_LSH_FP32)
    against the bit-exact fp64 path on SIFT-/OCR-shaped samples: tokens may
    differ only where the fp64 bucket value sits within fp32 rounding of a
    bucket boundary.  The count is printed (north_star: "fp32 boundary
    disagreements counted and bounded") and must stay below 1e-4 of the
    tokens (SURVEY 8c measured 1.9e-6 for p-stable, 0 for RBH)."""
    if family == PSTABLE:
        ds = synth.sift(n=200_000, dims=128, queries=16)
        kw = dict(w=4.0)
        cfg = lambda fp32: lsh_config(PSTABLE, 237, 128, 3, fp32=fp32, **kw)  # noqa: E731
    else:
        ds = synth.ocr(n=20_000, dims=784, queries=4)
        sigma = oracle.kernel_width(ds.points[:5000])
        cfg = lambda fp32: lsh_config(RBH, 237, 784, 7, sigma=sigma, fp32=fp32)  # noqa: E731
    exact = Encoder(cfg(False), gpu).encode(ds.points)
    fast = Encoder(cfg(True), gpu).encode(ds.points)
    bad = int((exact != fast).sum())
    print(f"fp32 {'p-stable' if family == PSTABLE else 'RBH'}: {bad} of {exact.size} tokens differ "
          f"({bad / exact.size:.2e})")
    assert bad <= 1e-4 * exact.size
    if family == PSTABLE:  # a disagreement is a neighbouring bucket, never further
        diff = np.abs(exact.astype(np.int64) - fast.astype(np.int64))
        assert int(diff.max(initial=0)) <= 1


@pytest.mark.parametrize("family", [PSTABLE, RBH, MINHASH])
def test_fused_query_path_equals_encode_then_query(gpu, oracle, family):
    """genie_lsh_query_batch (host points / sets in, tokens kept on the
    device) == the host encode followed by genie_query_batch."""
    from paper_1603_08390_b200.engine import point_queries

    if family == PSTABLE:
        ds = synth.sift(n=60_000, dims=128, queries=96)
        enc = Encoder(lsh_config(PSTABLE, 237, 128, 3, w=4.0), gpu)
        toks, qt, kw, k = enc.encode(ds.points), enc.encode(ds.query_points), dict(points=ds.query_points), 100
        dom = 67
    elif family == RBH:
        ds = synth.ocr(n=8_000, dims=784, queries=64)
        sigma = oracle.kernel_width(ds.points[:2000])
        enc = Encoder(lsh_config(RBH, 237, 784, 7, sigma=sigma), gpu)
        toks, qt, kw, k = enc.encode(ds.points), enc.encode(ds.query_points), dict(points=ds.query_points), 1
        dom = 8192
    else:
        ds = synth.sets(n=50_000, queries=128)
        enc = Encoder(lsh_config(MINHASH, 128, 0, 5, rehash_domain=8192), gpu)
        toks = enc.encode_sets(ds.set_off, ds.elems)
        qt = enc.encode_sets(ds.query_set_off, ds.query_elems)
        kw, k, dom = dict(set_off=ds.query_set_off, elems=ds.query_elems), 100, 8192
    ix = DeviceIndex.from_csr(csr_from_tokens(toks), device=gpu)
    want = ix.query(point_queries(qt, k, first_id=7))
    got = enc.query(ix, k, first_id=7, **kw)
    assert np.array_equal(got.qid, want.qid)
    assert np.array_equal(got.length, want.length) and np.array_equal(got.threshold, want.threshold)
    for q in range(len(got.length)):
        assert got.row(q) == want.row(q)
    assert dom > 0
