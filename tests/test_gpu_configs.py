"""The five BASELINE.json configs end to end on the GPU (transform -> index
-> scan/c-PQ -> merge) against the CPU oracle at test sizes, and the C2
headline config at full size on a query sample."""
import numpy as np
import pytest

from paper_1603_08390_b200 import DeviceIndex, Encoder, lsh_config, point_queries, synth
from paper_1603_08390_b200.engine import MINHASH, PSTABLE, RBH, csr_from_tokens

pytestmark = pytest.mark.gpu


def assert_same(got, want, label):
    assert np.array_equal(got.length, want.length), label
    assert np.array_equal(got.threshold, want.threshold), label
    for q in range(len(got.length)):
        assert got.row(q) == want.row(q), f"{label} q{q}"


def lsh_pipeline(gpu, oracle, family, m, dims, seed, points, qpoints, k, **kw):
    import torch
    enc = Encoder(lsh_config(family, m, dims, seed, **kw), gpu)
    dpts = torch.from_numpy(points).cuda(gpu)
    dtok = torch.zeros((points.shape[0], m), dtype=torch.int32, device=f"cuda:{gpu}")
    enc.encode_device(dpts, dtok)
    torch.cuda.synchronize()
    ix = DeviceIndex.from_tokens_device(dtok.data_ptr(), points.shape[0], m, kw.get("rehash_domain", 8192)
                                        if family == RBH else 67, device=gpu)
    qb = point_queries(enc.encode(qpoints), k)
    got = ix.query(qb)
    # the oracle path: oracle tokens -> host CSR -> oracle engine
    otoks = oracle.lsh_encode(family, m, dims, seed, points=points, w=kw.get("w", 4.0), sigma=kw.get("sigma", 1.0))
    assert np.array_equal(dtok.cpu().numpy().astype(np.uint32), otoks)
    oq = point_queries(oracle.lsh_encode(family, m, dims, seed, points=qpoints, w=kw.get("w", 4.0),
                                         sigma=kw.get("sigma", 1.0)), k)
    want = oracle.index(csr_from_tokens(otoks)).execute(oq)
    return got, want


def test_c3_sift_shaped(gpu, oracle):
    ds = synth.sift(n=200_000, dims=128, queries=64)
    got, want = lsh_pipeline(gpu, oracle, PSTABLE, 237, 128, 3, ds.points, ds.query_points, 100, w=4.0)
    assert_same(got, want, "C3")
    assert want.bound.max() == 237  # W = 8 counters


def test_c5_ocr_shaped_1nn(gpu, oracle):
    ds = synth.ocr(n=30_000, dims=784, queries=48)
    sigma = oracle.kernel_width(ds.points[:2000])
    got, want = lsh_pipeline(gpu, oracle, RBH, 237, 784, 7, ds.points, ds.query_points, 1, sigma=sigma,
                             rehash_domain=8192)
    assert_same(got, want, "C5")
    pred = ds.labels[got.ids[:, 0]]
    assert (pred == ds.query_labels).mean() > 0.8  # 1-NN prediction quality (side metric)


def test_c4_minhash(gpu, oracle):
    ds = synth.sets(n=100_000, queries=128)
    enc = Encoder(lsh_config(MINHASH, 128, 0, 5, rehash_domain=8192), gpu)
    toks = enc.encode_sets(ds.set_off, ds.elems)
    qt = enc.encode_sets(ds.query_set_off, ds.query_elems)
    assert np.array_equal(toks, oracle.lsh_encode(2, 128, 0, 5, set_off=ds.set_off, elems=ds.elems))
    csr = csr_from_tokens(toks)
    qb = point_queries(qt, 100)
    got = DeviceIndex.from_csr(csr, device=gpu).query(qb)
    want = oracle.index(csr).execute(qb)
    assert_same(got, want, "C4")
    # the query's source set is (almost always) its top-1 neighbour
    assert (got.counts[:, 0] > 64).mean() > 0.9


def test_c2_full_size_sample(gpu, oracle):
    ds = synth.tweets()  # 7M docs, vocab 1M, 1024 queries, k=100
    ix = DeviceIndex.from_csr(ds.csr, device=gpu)
    got = ix.query(ds.queries)
    sample = ds.queries.slice(0, 48)
    want = oracle.index(ds.csr).execute(sample)
    for q in range(48):
        assert got.row(q) == want.row(q) and got.threshold[q] == want.threshold[q], q
    # size-independent properties on the whole batch
    assert np.all(got.length == 100)
    assert np.all(np.diff(got.counts.astype(np.int64), axis=1) <= 0)
    assert np.all(got.threshold == got.counts[:, 99])
