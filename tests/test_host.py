"""Host-side logic (no GPU): synthetic workloads, host CSR build vs the
reference's build_index, the mcx mirror's construction rules, the sharding
and merge logic of the multi-GPU path, and LSH parameter sampling."""
import ctypes

import numpy as np
import pytest

from oracle.pyoracle import RefLib, ref_available
from paper_1603_08390_b200 import engine as E
from paper_1603_08390_b200 import mcx, synth
from paper_1603_08390_b200.dist import merge_host, shard_csr, shard_range

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def check_csr(csr):
    assert np.all(np.diff(csr.keys.astype(np.float64)) > 0)
    assert csr.key_off[0] == 0 and csr.key_off[-1] == csr.num_postings
    for j in range(min(csr.num_keys, 2000)):
        seg = csr.postings[csr.key_off[j]:csr.key_off[j + 1]]
        assert seg.size > 0 and np.all(np.diff(seg.astype(np.int64)) > 0) and seg.max() < csr.n


def test_adult_generator_shape():
    ds = synth.adult()
    check_csr(ds.csr)
    assert ds.csr.n == 48842 and ds.csr.num_postings == 48842 * 14
    assert ds.csr.num_keys == 5383  # SURVEY.md 8d probe
    assert len(ds.queries) == 1024 and np.all(ds.queries.k == 100)
    assert np.all(np.diff(ds.queries.item_off) == 14)


def test_tweets_generator_shape_and_determinism():
    a = synth.tweets(n=20_000, vocab=5_000, words=10, queries=16, k=100)
    b = synth.tweets(n=20_000, vocab=5_000, words=10, queries=16, k=100)
    check_csr(a.csr)
    assert a.csr.num_postings == 200_000
    assert np.array_equal(a.csr.postings, b.csr.postings) and np.array_equal(a.queries.lo, b.queries.lo)
    # Zipf(1): the most frequent word has the longest list
    lens = np.diff(a.csr.key_off)
    assert int(a.csr.keys[np.argmax(lens)]) == 0


def test_vector_and_set_generators():
    s = synth.sift(n=1000, dims=128, queries=8)
    assert s.points.shape == (1000, 128) and s.query_points.shape == (8, 128)
    o = synth.ocr(n=500, dims=784, queries=4)
    assert o.points.min() >= 0 and o.points.max() <= 1 and o.labels.max() < 10
    st = synth.sets(n=2000, queries=10)
    sizes = np.diff(st.set_off)
    assert sizes.min() >= 32 and sizes.max() <= 256 and len(st.query_set_off) == 11


@needs_ref
def test_host_csr_equals_reference_build_index():
    ref = RefLib()
    for seed in range(5):
        ds = synth.random_instance(n=400, dims=3, tokens=6, max_kw=6, queries=2, seed=seed)
        keys, first, cnt, sb, se, post = ref.index(ds.csr).export()
        assert np.array_equal(keys, ds.csr.keys) and np.array_equal(post, ds.csr.postings)
        assert np.array_equal(np.append(sb, post.size), ds.csr.key_off)
        # long-list splitting (index.hpp:229-238): spans tile each list
        keys2, first2, cnt2, sb2, se2, post2 = ref.index(ds.csr, split=4).export()
        assert np.array_equal(post2, post) and np.all(se2 - sb2 <= 4)


def test_mirror_construction_rules():
    with pytest.raises(E.ContractError):
        mcx.ObjectRecord(0, [(0, 1), (0, 1)])
    with pytest.raises(E.ContractError):
        mcx.QueryItem(0, 3, 2)
    with pytest.raises(E.ContractError):
        mcx.Query(1, [], 1)
    with pytest.raises(E.ContractError):
        mcx.Query(1, [mcx.QueryItem.point(0, 0)], 0)
    assert mcx.Keyword(3, 7).packed() == (3 << 32) | 7
    assert [mcx.width_for(x) for x in (1, 15, 16, 255, 256, 65535, 65536)] == [4, 4, 8, 8, 16, 16, 32]
    schema = mcx.RelationalSchema([10, 3])
    q = mcx.encode_relational_query(schema, [mcx.AttributeRange(0, -5, 4), mcx.AttributeRange(1, 2, 99)], 5)
    assert [(i.dim, i.lo, i.hi) for i in q.items] == [(0, 0, 4), (1, 2, 2)]
    with pytest.raises(E.DataError):
        mcx.encode_relational_query(schema, [mcx.AttributeRange(0, 20, 30)], 1)
    with pytest.raises(E.DataError):
        mcx.encode_relational_tuple(schema, [10, 0], 0)


def test_mirror_index_lookup_and_bound():
    objs = [mcx.ObjectRecord(0, [(0, 1), (1, 2), (2, 1)]), mcx.ObjectRecord(1, [(0, 2), (1, 1), (2, 2)]),
            mcx.ObjectRecord(2, [(0, 1), (1, 2), (2, 2)])]
    ix = mcx.build_index(objs)
    assert ix.num_objects() == 3 and ix.keyword_count() == 6
    assert sum(s.length() for s in ix.lookup(mcx.QueryItem(0, 1, 2))) == 3
    assert ix.lookup(mcx.QueryItem(9, 0, 100)) == []
    assert ix.max_token(0) == 2 and ix.max_multiplicity(1) == 1
    q = mcx.Query(0, [mcx.QueryItem(0, 1, 2), mcx.QueryItem(1, 1, 1), mcx.QueryItem(2, 2, 3)], 1)
    assert ix.max_count_bound(q) == 3
    with pytest.raises(E.DataError):
        mcx.build_index([mcx.ObjectRecord(0, [(0, 1)]), mcx.ObjectRecord(0, [(0, 2)])])
    # splitting at 4096 (test_index.cpp:87-99)
    big = mcx.build_index([mcx.ObjectRecord(i, [(0, 0)]) for i in range(10000)], 4096)
    assert [s.length() for s in big.lookup(mcx.QueryItem.point(0, 0))] == [4096, 4096, 1808]


def test_merge_topk_host_rules():
    a = mcx.TopKResult(0, [mcx.TopKEntry(1, 5)], 0)
    b = mcx.TopKResult(0, [mcx.TopKEntry(9, 7)], 0)
    m = mcx.merge_topk([a, b], 1, 0)
    assert m.entries == [mcx.TopKEntry(9, 7)] and m.threshold == 7
    with pytest.raises(E.ContractError):
        mcx.merge_topk([b, mcx.TopKResult(0, [mcx.TopKEntry(9, 3)], 0)], 2, 0)


def test_partition_dataset_offsets():
    objs = [mcx.ObjectRecord(i, [(0, i % 3)]) for i in range(10)]
    parts = mcx.partition_dataset(objs, 4)
    assert [(p.id_offset, p.size) for p in parts] == [(0, 4), (4, 4), (8, 2)]
    with pytest.raises(E.ContractError):
        mcx.partition_dataset(objs, 0)


def test_shard_ranges_tile_the_ids():
    for n in (0, 1, 7, 7_000_000):
        for world in (1, 2, 3, 8):
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n and all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))


def test_shard_csr_and_host_merge_equal_unsharded(oracle):
    ds = synth.tweets(n=30_000, vocab=2_000, words=10, queries=24, k=50)
    whole = oracle.index(ds.csr).execute(ds.queries)
    world = 3
    Q, K = len(ds.queries), 50
    ids = np.zeros((Q, world, K), np.uint32)
    cnt = np.zeros((Q, world, K), np.uint32)
    lens = np.zeros((Q, world), np.uint32)
    for r in range(world):
        lo, hi = shard_range(ds.csr.n, r, world)
        part = shard_csr(ds.csr, lo, hi)
        check_csr(part)
        res = oracle.index(part).execute(ds.queries, stride=K)
        ids[:, r], cnt[:, r], lens[:, r] = res.ids + lo, res.counts, res.length
    oi, oc, ol, ot = merge_host(ids, cnt, lens, ds.queries.k)
    assert np.array_equal(ol, whole.length) and np.array_equal(ot, whole.threshold)
    for q in range(Q):
        n = int(ol[q])
        assert np.array_equal(oi[q, :n], whole.ids[q, :n]) and np.array_equal(oc[q, :n], whole.counts[q, :n])


def test_lsh_parameter_sampling_equals_reference():
    g = np.load(__import__("pathlib").Path(__file__).parent / "golden" / "lsh_tokens.npz")
    for name in ("pstable_rehash", "rbh_small"):
        fam, m, dims, seed, rehash, domain = (int(x) for x in g[name + "_meta"])
        w, sigma = (float(x) for x in g[name + "_wsig"])
        a, b, hs, rs = E.lsh_sample(E.lsh_config(fam, m, dims, seed, domain, w=w, sigma=sigma))
        assert np.array_equal(a, g[name + "_a"]) and np.array_equal(b, g[name + "_b"]) and np.array_equal(rs, g[name + "_rs"])


def test_documents_deduplicate_and_intersect():
    # test_sa.cpp:208-226 (tokenize_document / DocumentCodec, sa.hpp:341-408)
    from paper_1603_08390_b200 import mcx

    assert len(mcx.tokenize_document("a b a")) == 2
    assert len(mcx.tokenize_document("The the THE")) == 1
    assert len(mcx.tokenize_document("the cat", {"the"})) == 1
    corpus = ["big data engine", "data data lake"]
    codec = mcx.DocumentCodec.build(corpus)
    assert codec.vocabulary_size() == 4
    d0, d1 = codec.encode(corpus[0], 0), codec.encode(corpus[1], 1)
    q = codec.encode_query("engine data", 2)
    assert q is not None
    assert mcx.match_count_reference(q, d0) == 2 and mcx.match_count_reference(q, d1) == 1
    assert mcx.match_count_reference(codec.encode_query(corpus[0], 1), d0) == 3
    assert codec.encode_query("unseen words only", 1) is None
    with pytest.raises(mcx.ContractError):
        codec.encode("unseen", 5)


def test_document_match_counts_equal_set_intersections():
    # test_sa.cpp:228-256
    import random

    from paper_1603_08390_b200 import mcx

    rng = random.Random(17)
    words = ["red", "green", "blue", "cyan", "teal", "gray", "pink", "gold", "jade", "rust"]
    for _ in range(100):
        def pick():
            s = set()
            n = 1 + rng.randrange(6)
            while len(s) < n:
                s.add(words[rng.randrange(len(words))])
            return " ".join(sorted(s)) + " ", s
        doc_text, doc_set = pick()
        q_text, q_set = pick()
        codec = mcx.DocumentCodec.build([doc_text])
        obj = codec.encode(doc_text, 0)
        query = codec.encode_query(q_text, 1)
        common = len(q_set & doc_set)
        if query is None:
            assert common == 0
        else:
            assert mcx.match_count_reference(query, obj) == common


# ----------------------------------------------------------------- MCIX files


@needs_ref
@pytest.mark.parametrize("seed,split", [(1, None), (2, 4096), (3, 16), (4, 1), (5, 7)])
def test_mcix_bytes_equal_reference_serializer(seed, split):
    # serialize_index (index_io.hpp:63-82) of build_index(objects, split): the
    # C ABI writer produces the reference's exact bytes, and reads them back
    ds = synth.random_instance(n=300 + 211 * seed, dims=3, tokens=4 + seed, max_kw=5, queries=2, seed=seed)
    want = RefLib().index(ds.csr, split=split or 0).serialize()
    got = E.mcix_serialize(ds.csr, split)
    assert got == want
    back = E.mcix_parse(want)
    assert back.n == ds.csr.n and np.array_equal(back.keys, ds.csr.keys)
    assert np.array_equal(back.key_off, ds.csr.key_off) and np.array_equal(back.postings, ds.csr.postings)
    idx = mcx.InvertedIndex(ds.csr, split)
    assert mcx.serialize_index(idx) == want
    assert np.array_equal(mcx.deserialize_index(want).csr.postings, ds.csr.postings)


@needs_ref
def test_mcix_rejects_what_the_reference_rejects():
    # deserialize_index's validation (index_io.hpp:84-146): same status, same message
    ref = RefLib()
    ds = synth.random_instance(n=200, dims=2, tokens=5, max_kw=4, queries=1, seed=11)
    img = bytearray(E.mcix_serialize(ds.csr, 8))
    K = ds.csr.num_keys

    def entry_offset(j):  # byte offset of keyword entry j
        pos = 16
        for i in range(j):
            spans = int.from_bytes(img[pos + 6:pos + 8], "little")
            pos += 8 + 16 * spans
        return pos

    list_at = entry_offset(K)
    cases = {
        "magic": bytes(b"MCIY" + img[4:]),
        "version": bytes(img[:4] + (2).to_bytes(4, "little") + img[8:]),
        "truncated": bytes(img[:list_at - 3]),
        "size": bytes(img[:-4]),
        "order": bytes(img[:entry_offset(1)] + (0).to_bytes(2, "little") + (0).to_bytes(4, "little") +
                       img[entry_offset(1) + 6:]),
        "tiling": bytes(img[:24] + (int.from_bytes(img[24:32], "little") + 1).to_bytes(8, "little") + img[32:]),
        "id range": bytes(img[:list_at] + (10**6).to_bytes(4, "little") + img[list_at + 4:]),
        "ascending": bytes(img[:list_at] + img[list_at + 4:list_at + 8] + img[list_at:list_at + 4] +
                           img[list_at + 8:]),
        "no spans": bytes(img[:22] + (0).to_bytes(2, "little") + img[24 + 16 * int.from_bytes(img[22:24], "little"):]),
    }
    for name, data in cases.items():
        rc, msg = ref.deserialize_status(data)
        assert rc == 2, (name, rc, msg)  # DataError
        with pytest.raises(E.DataError) as ex:
            E.mcix_parse(data)
        assert str(ex.value) == msg, (name, str(ex.value), msg)
