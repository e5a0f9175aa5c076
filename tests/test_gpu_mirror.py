"""The object-level mirror (paper_1603_08390_b200.mcx) exercised the way the
reference's own unit tests exercise mcx (test_engine.cpp, test_cpq.cpp,
acceptance criteria 1, 10, 12), with execution on the GPU."""
import random

import numpy as np
import pytest

from paper_1603_08390_b200 import mcx
from paper_1603_08390_b200.engine import ContractError

pytestmark = pytest.mark.gpu


def example_objects():
    return [mcx.ObjectRecord(0, [(0, 1), (1, 2), (2, 1)]), mcx.ObjectRecord(1, [(0, 2), (1, 1), (2, 2)]),
            mcx.ObjectRecord(2, [(0, 1), (1, 2), (2, 2)])]


def random_instance(rng, n, q_count):
    objects = []
    for i in range(n):
        kws = []
        for _ in range(rng.randint(0, 5)):
            kw = (rng.randint(0, 3), rng.randint(0, 7))
            if kw not in kws:
                kws.append(kw)
        objects.append(mcx.ObjectRecord(i, kws))
    queries = []
    for q in range(q_count):
        items = []
        for _ in range(rng.randint(1, 4)):
            lo = rng.randint(0, 7)
            items.append(mcx.QueryItem(rng.randint(0, 3), lo, lo + rng.randint(0, 7) % 3))
        queries.append(mcx.Query(q, items, 1 + rng.randrange(10)))
    return objects, queries


def oracle_result(query, objects):
    counts = [mcx.match_count_reference(query, o) for o in objects]
    ranked = sorted(((c, i) for i, c in enumerate(counts)), key=lambda t: (-t[0], t[1]))
    k_eff = min(query.k, len(counts))
    top = ranked[:k_eff]
    thr = top[-1][0] if query.k <= len(counts) and top else 0
    return [mcx.TopKEntry(i, c) for c, i in top if c > 0], thr


def test_running_example(gpu):
    index = mcx.build_index(example_objects())
    q1 = mcx.Query(0, [mcx.QueryItem(0, 1, 2), mcx.QueryItem(1, 1, 1), mcx.QueryItem(2, 2, 3)], 1)
    batch = mcx.execute_batch(index, [q1])
    assert len(batch.results) == 1
    assert batch.results[0].entries == [mcx.TopKEntry(1, 3)] and batch.results[0].threshold == 3
    assert mcx.execute_batch(index, []).results == []


def test_engine_equals_full_scan_oracle(gpu):
    rng = random.Random(29)
    for trial in range(20):
        objects, queries = random_instance(rng, 50 + rng.randrange(400), 8)
        index = mcx.build_index(objects)
        for sel in (mcx.Selector.cpq, mcx.Selector.bucket, mcx.Selector.sort):
            batch = mcx.execute_batch(index, queries, mcx.EngineConfig(selector=sel, mode=mcx.ExecMode.sequential))
            for q, query in enumerate(queries):
                ent, thr = oracle_result(query, objects)
                assert batch.results[q].entries == ent and batch.results[q].threshold == thr


def test_partitioned_equals_unpartitioned(gpu):
    rng = random.Random(41)
    for trial in range(6):
        n = 60 + rng.randrange(300)
        objects, queries = random_instance(rng, n, 5)
        whole = mcx.execute_batch(mcx.build_index(objects), queries)
        for cap in (n, n // 2 + 1, n // 6 + 1, 17):
            merged = mcx.execute_partitioned(mcx.partition_dataset(objects, cap), queries)
            for q in range(len(queries)):
                assert merged.results[q].entries == whole.results[q].entries
                assert merged.results[q].threshold == whole.results[q].threshold
            assert mcx.hash_results(merged.results) == mcx.hash_results(whole.results)


def test_timings_and_memory_accounting(gpu):
    rng = random.Random(43)
    objects, queries = random_instance(rng, 2000, 8)
    index = mcx.build_index(objects)
    batch = mcx.execute_batch(index, queries)
    t = batch.timings
    assert t.lookup_ns + t.match_ns + t.select_ns + t.merge_ns <= t.total_ns
    # acceptance criterion 12: counter_bytes = sum_q ceil(n * W_q / 8)
    want = sum((2000 * mcx.width_for(max(index.max_count_bound(q), 1)) + 7) // 8 for q in queries)
    assert batch.memory.counter_bytes == want > 0
    want_gate = sum((max(index.max_count_bound(q), 1) + 1) * 4 + 4 for q in queries)
    assert batch.memory.gate_bytes == want_gate


def test_knobs_must_be_positive(gpu):
    index = mcx.build_index(example_objects())
    q = mcx.Query(0, [mcx.QueryItem(0, 1, 2)], 1)
    with pytest.raises(ContractError):
        mcx.execute_batch(index, [q], mcx.EngineConfig(span_chunk=0))


def test_lsh_identical_point_matches_itself(gpu):
    # test_lsh.cpp:168-186
    cfg = mcx.LshEncoderConfig(family=mcx.LshFamily.random_binning, m=16, dims=4, sigma=1.5)
    enc = mcx.LshEncoder.create(cfg)
    p = np.array([0.1, -2.0, 3.0, 0.7], np.float32)
    obj = enc.encode_point(p, 0)
    q = enc.encode_query_point(p, 1)
    assert len(obj.keywords()) == 16 and len(q.items) == 16
    assert mcx.match_count_reference(q, obj) == 16


def test_documents_through_the_engine(gpu):
    # DocumentCodec (sa.hpp:361-408) -> build_index -> execute_batch: the top-k
    # of word-set intersections, equal to the full scan (the Tweets adapter)
    rng = random.Random(23)
    vocab = [f"w{i}" for i in range(60)] + ["The", "THE", "the"]
    docs = [" ".join(rng.choice(vocab) for _ in range(rng.randint(1, 12))) for _ in range(700)]
    codec = mcx.DocumentCodec.build(docs, stop_words={"the"})
    objects = [codec.encode(d, i) for i, d in enumerate(docs)]
    queries = []
    for q in range(40):
        text = " ".join(rng.choice(vocab + ["unseen"]) for _ in range(rng.randint(1, 8)))
        query = codec.encode_query(text, 1 + rng.randrange(30), q)
        if query is not None:
            queries.append(query)
    index = mcx.build_index(objects)
    batch = mcx.execute_batch(index, queries)
    for q, query in enumerate(queries):
        ent, thr = oracle_result(query, objects)
        assert batch.results[q].entries == ent and batch.results[q].threshold == thr
