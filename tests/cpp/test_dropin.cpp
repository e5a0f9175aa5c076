// Drop-in check of include/mcx/mcx.hpp: code written against the reference
// API (mcx::build_index / execute_batch / execute_partitioned / merge_topk /
// hash_results / LshEncoder) runs on the GPU and agrees with the CPU oracle
// (oracle/_build/libgenie_oracle.so, test infrastructure).
#include <mcx/mcx.hpp>

#include <cstdio>
#include <random>

extern "C" {
void* or_index_create(uint32_t, uint64_t, const uint64_t*, const uint64_t*, const uint32_t*);
void or_index_free(void*);
int or_execute(void*, uint32_t, const uint32_t*, const uint32_t*, const uint64_t*, const uint16_t*, const uint32_t*,
               const uint32_t*, uint32_t, uint32_t*, uint32_t*, uint32_t*, uint32_t*, uint64_t*, uint64_t*, uint32_t,
               uint32_t*);
uint64_t or_hash_results(uint32_t, const uint32_t*, const uint32_t*, const uint32_t*, uint32_t, const uint32_t*,
                         const uint32_t*);
}

static int failures = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        if (!(c)) {                                                       \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                   \
        }                                                                 \
    } while (0)

// oracle over the same objects (CSR built independently of the mirror)
static uint64_t oracle_hash(const std::vector<mcx::ObjectRecord>& objs, const std::vector<mcx::Query>& qs) {
    std::vector<std::pair<uint64_t, uint32_t>> pairs;
    for (const auto& o : objs)
        for (const auto& kw : o.keywords()) pairs.emplace_back(kw.packed(), o.id());
    std::sort(pairs.begin(), pairs.end());
    std::vector<uint64_t> keys, off{0};
    std::vector<uint32_t> post;
    for (size_t i = 0; i < pairs.size(); ++i) {
        if (i && pairs[i].first != pairs[i - 1].first) off.push_back(post.size());
        if (i == 0 || pairs[i].first != pairs[i - 1].first) keys.push_back(pairs[i].first);
        post.push_back(pairs[i].second);
    }
    if (!pairs.empty()) off.push_back(post.size());
    void* ix = or_index_create(uint32_t(objs.size()), keys.size(), keys.data(), off.data(), post.data());
    const uint32_t Q = uint32_t(qs.size());
    std::vector<uint32_t> qid(Q), k(Q), lo, hi;
    std::vector<uint64_t> ioff{0};
    std::vector<uint16_t> dim;
    uint32_t stride = 1;
    for (uint32_t q = 0; q < Q; ++q) {
        qid[q] = qs[q].id;
        k[q] = qs[q].k;
        stride = std::max(stride, k[q]);
        for (const auto& it : qs[q].items) {
            dim.push_back(it.dim);
            lo.push_back(it.lo);
            hi.push_back(it.hi);
        }
        ioff.push_back(dim.size());
    }
    std::vector<uint32_t> ids(size_t(Q) * stride), cnt(size_t(Q) * stride), len(Q), thr(Q);
    uint32_t bad = 0;
    or_execute(ix, Q, qid.data(), k.data(), ioff.data(), dim.data(), lo.data(), hi.data(), stride, ids.data(),
               cnt.data(), len.data(), thr.data(), nullptr, nullptr, 4, &bad);
    or_index_free(ix);
    return or_hash_results(Q, qid.data(), thr.data(), len.data(), stride, ids.data(), cnt.data());
}

int main() {
    using namespace mcx;
    // the running example (test_engine.cpp:80-89)
    std::vector<ObjectRecord> ex;
    ex.emplace_back(0, std::vector<Keyword>{{0, 1}, {1, 2}, {2, 1}});
    ex.emplace_back(1, std::vector<Keyword>{{0, 2}, {1, 1}, {2, 2}});
    ex.emplace_back(2, std::vector<Keyword>{{0, 1}, {1, 2}, {2, 2}});
    const auto index = build_index(ex);
    const Query q1(0, {QueryItem(0, 1, 2), QueryItem(1, 1, 1), QueryItem(2, 2, 3)}, 1);
    const auto b = execute_batch(index, std::vector<Query>{q1});
    CHECK(b.results.size() == 1 && b.results[0].entries.size() == 1);
    CHECK(b.results[0].entries[0] == (TopKEntry{1, 3}) && b.results[0].threshold == 3);
    CHECK(execute_batch(index, std::vector<Query>{}).results.empty());
    bool threw = false;
    try {
        execute_batch(index, std::vector<Query>{q1}, EngineConfig{.span_chunk = 0});
    } catch (const ContractError&) {
        threw = true;
    }
    CHECK(threw);

    // random instances: GPU == oracle, partitioned == whole (test_engine.cpp:97-196)
    std::mt19937 rng(29);
    for (int trial = 0; trial < 15; ++trial) {
        std::uniform_int_distribution<int> dimd(0, 3), tok(0, 7), klen(0, 5), items(1, 4);
        const size_t n = 50 + rng() % 400;
        std::vector<ObjectRecord> objs;
        for (size_t i = 0; i < n; ++i) {
            std::vector<Keyword> kws;
            for (int t = klen(rng); t > 0; --t) {
                const Keyword kw{DimId(dimd(rng)), Token(tok(rng))};
                if (std::find(kws.begin(), kws.end(), kw) == kws.end()) kws.push_back(kw);
            }
            objs.emplace_back(ObjectId(i), std::move(kws));
        }
        std::vector<Query> qs;
        for (uint32_t q = 0; q < 8; ++q) {
            std::vector<QueryItem> its;
            for (int i = items(rng); i > 0; --i) {
                const Token lo = Token(tok(rng));
                its.emplace_back(DimId(dimd(rng)), lo, lo + Token(tok(rng) % 3));
            }
            qs.emplace_back(q, its, 1 + uint32_t(rng() % 10));
        }
        const auto ix = build_index(objs);
        const auto whole = execute_batch(ix, qs);
        CHECK(hash_results(whole.results) == oracle_hash(objs, qs));
        const auto parts = partition_dataset(objs, uint32_t(n / 3 + 1));
        const auto merged = execute_partitioned(parts, qs);
        CHECK(hash_results(merged.results) == hash_results(whole.results));
        CHECK(whole.memory.counter_bytes > 0);
    }

    // LSH: an identical point matches itself on all m functions (test_lsh.cpp:168-186)
    LshEncoderConfig cfg;
    cfg.m = 16;
    cfg.dims = 4;
    cfg.sigma = 1.5;
    const auto enc = LshEncoder::create(cfg);
    const std::vector<float> p = {0.1f, -2.0f, 3.0f, 0.7f};
    CHECK(match_count_reference(enc.encode_query_point(p, 1), enc.encode_point(p, 0)) == 16);

    // documents (test_sa.cpp:208-226): DocumentCodec -> engine
    CHECK(tokenize_document("a b a").size() == 2);
    CHECK(tokenize_document("The the THE").size() == 1);
    CHECK(tokenize_document("the cat", {"the"}).size() == 1);
    const std::vector<std::string> corpus = {"big data engine", "data data lake"};
    const DocumentCodec codec = DocumentCodec::build(corpus);
    std::vector<ObjectRecord> docs = {codec.encode(corpus[0], 0), codec.encode(corpus[1], 1)};
    const auto dq = codec.encode_query("engine data", 2);
    CHECK(dq.has_value() && match_count_reference(*dq, docs[0]) == 2 && match_count_reference(*dq, docs[1]) == 1);
    CHECK(!codec.encode_query("unseen words only", 1).has_value());
    const auto dres = execute_batch(build_index(docs), std::vector<Query>{*dq});
    CHECK(dres.results[0].entries.size() == 2 && dres.results[0].entries[0] == (TopKEntry{0, 2}) &&
          dres.results[0].entries[1] == (TopKEntry{1, 1}) && dres.results[0].threshold == 1);

    // MCIX round trip (index_io.hpp): save -> load -> same answers
    {
        const auto img = serialize_index(build_index(docs, 1));
        const auto back = deserialize_index(img.data(), img.size());
        const auto r2 = execute_batch(back, std::vector<Query>{*dq});
        CHECK(hash_results(r2.results) == hash_results(dres.results));
        bool bad = false;
        try {
            std::vector<std::uint8_t> broken(img.begin(), img.end() - 1);
            (void)deserialize_index(broken.data(), broken.size());
        } catch (const DataError&) {
            bad = true;
        }
        CHECK(bad);
    }

    std::printf(failures ? "dropin: %d failures\n" : "dropin: ok\n", failures);
    return failures ? 1 : 0;
}
