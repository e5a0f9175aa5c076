// The reference's own checks, restated against the drop-in header
// include/mcx/mcx.hpp and run on the GPU (tests/test_cpp_dropin.py):
//
//   index   test_index.cpp:60-237 (running example, empty build, duplicate
//           ids, split at the threshold, split preserves postings, range
//           lookup, round trip, span increments == match_count_reference,
//           max_count_bound dominance, partition_dataset layout, MCIX
//           round trip byte-exact with split spans, corrupted images)
//   model   model.hpp:119-188 relational encoders (clamping, errors)
//   lsh     LshEncoder::token == encode_point's keyword (lsh.hpp:172-195)
//   accept  acceptance.cpp criterion 1 (exactness vs the CPU oracle),
//           3 (result independent of scheduling knobs, repeated runs),
//           10 (partition-capacity invariance through execute_partitioned),
//           12 engine half (counter_bytes accounting, acceptance.cpp:626-636)
//
// Usage: test_reference_api [corpus_size]  (acceptance corpus, default 120 of
// the reference's 1000 instances, same generator and seeds).
#include <mcx/mcx.hpp>

#include <cstdio>
#include <random>

extern "C" {
void* or_index_create(uint32_t, uint64_t, const uint64_t*, const uint64_t*, const uint32_t*);
void or_index_free(void*);
int or_execute(void*, uint32_t, const uint32_t*, const uint32_t*, const uint64_t*, const uint16_t*, const uint32_t*,
               const uint32_t*, uint32_t, uint32_t*, uint32_t*, uint32_t*, uint32_t*, uint64_t*, uint64_t*, uint32_t,
               uint32_t*);
}

using namespace mcx;

static int failures = 0, checks = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++checks;                                                             \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                       \
        }                                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, E)            \
    do {                                    \
        bool ok_ = false;                   \
        try {                               \
            (void)(expr);                   \
        } catch (const E&) {                \
            ok_ = true;                     \
        } catch (...) {                     \
        }                                   \
        CHECK(ok_ && #E);                   \
    } while (0)

namespace {

std::vector<ObjectRecord> example_objects() {
    std::vector<ObjectRecord> o;
    o.emplace_back(0, std::vector<Keyword>{{0, 1}, {1, 2}, {2, 1}});
    o.emplace_back(1, std::vector<Keyword>{{0, 2}, {1, 1}, {2, 2}});
    o.emplace_back(2, std::vector<Keyword>{{0, 1}, {1, 2}, {2, 2}});
    return o;
}

std::vector<ObjectId> ids_of(const InvertedIndex& index, Keyword kw) {
    std::vector<ObjectId> out;
    for (const auto& span : index.lookup(QueryItem::point(kw.dim, kw.token))) {
        const auto s = index.ids(span);
        out.insert(out.end(), s.begin(), s.end());
    }
    return out;
}

std::vector<ObjectRecord> random_objects(std::mt19937& rng, std::size_t n, int dims, int tokens) {
    std::uniform_int_distribution<int> dim(0, dims - 1), tok(0, tokens - 1), len(0, 6);
    std::vector<ObjectRecord> objs;
    for (std::size_t i = 0; i < n; ++i) {
        std::vector<Keyword> kws;
        for (int t = len(rng); t > 0; --t) {
            const Keyword kw{DimId(dim(rng)), Token(tok(rng))};
            if (std::find(kws.begin(), kws.end(), kw) == kws.end()) kws.push_back(kw);
        }
        objs.emplace_back(ObjectId(i), std::move(kws));
    }
    return objs;
}

void index_cases() {
    {  // postings of the running example
        const auto index = build_index(example_objects());
        CHECK(index.num_objects() == 3);
        CHECK(index.keyword_count() == 6);
        CHECK(ids_of(index, {0, 1}) == (std::vector<ObjectId>{0, 2}));
        CHECK(ids_of(index, {1, 2}) == (std::vector<ObjectId>{0, 2}));
        CHECK(ids_of(index, {2, 2}) == (std::vector<ObjectId>{1, 2}));
        CHECK(index.max_token(0) == Token{2});
        CHECK(!index.max_token(7).has_value());
        CHECK(index.max_multiplicity(1) == 1);
        CHECK(index.longest_list() == 2);
    }
    {  // empty dataset
        const auto index = build_index(std::vector<ObjectRecord>{});
        CHECK(index.num_objects() == 0 && index.keyword_count() == 0 && index.list_array().empty());
    }
    {  // duplicate ids
        std::vector<ObjectRecord> o;
        o.emplace_back(0, std::vector<Keyword>{{0, 1}});
        o.emplace_back(0, std::vector<Keyword>{{0, 2}});
        CHECK_THROWS_AS(build_index(o), DataError);
        CHECK_THROWS_AS(build_index(example_objects(), 0u), ContractError);
    }
    {  // long lists split at the threshold
        std::vector<ObjectRecord> o;
        for (std::size_t i = 0; i < 10000; ++i) o.emplace_back(ObjectId(i), std::vector<Keyword>{{0, 0}});
        const auto index = build_index(o, 4096);
        CHECK(index.keyword_count() == 1);
        const auto spans = index.lookup(QueryItem::point(0, 0));
        CHECK(spans.size() == 3);
        if (spans.size() == 3)
            CHECK(spans[0].length() == 4096 && spans[1].length() == 4096 && spans[2].length() == 1808);
        CHECK(index.spans_of(index.entries()[0]).size() == 3);
        CHECK(index.longest_list() == 10000);
    }
    {  // splitting preserves the postings multiset
        std::mt19937 rng(7);
        const auto objs = random_objects(rng, 500, 3, 4);
        const auto whole = build_index(objs);
        const auto split = build_index(objs, 32);
        for (const auto& e : whole.entries()) CHECK(ids_of(whole, e.keyword) == ids_of(split, e.keyword));
        for (const auto& s : split.spans()) CHECK(s.length() <= 32);
    }
    {  // lookup resolves range items
        const auto index = build_index(example_objects());
        std::size_t total = 0;
        for (const auto& s : index.lookup(QueryItem(0, 1, 2))) total += s.length();
        CHECK(total == 3);
        CHECK(index.lookup(QueryItem(9, 0, 100)).empty());
        std::size_t full = 0;
        for (const auto& s : index.lookup(QueryItem(2, 0, 0xffffffffu))) full += s.length();
        CHECK(full == 3);
        std::vector<PostingsSpan> acc;
        index.lookup_into(QueryItem(0, 1, 1), acc);
        index.lookup_into(QueryItem(0, 2, 2), acc);
        CHECK(acc.size() == 2);
    }
    {  // round trip: every keyword of every object found once
        std::mt19937 rng(11);
        const auto objs = random_objects(rng, 300, 4, 6);
        const auto index = build_index(objs, 16);
        for (const auto& o : objs)
            for (const auto& kw : o.keywords()) {
                const auto ids = ids_of(index, kw);
                CHECK(std::count(ids.begin(), ids.end(), o.id()) == 1);
            }
    }
    {  // per-query span increments == match_count_reference; bound dominance
        std::mt19937 rng(13);
        const auto objs = random_objects(rng, 200, 3, 5);
        const auto index = build_index(objs, 8);
        std::uniform_int_distribution<int> dim(0, 2), tok(0, 4), items(1, 4);
        for (int trial = 0; trial < 50; ++trial) {
            std::vector<QueryItem> qi;
            for (int i = items(rng); i > 0; --i) {
                const Token lo = Token(tok(rng));
                qi.push_back(QueryItem(DimId(dim(rng)), lo, lo + Token(tok(rng))));
            }
            const Query q(0, qi, 1);
            std::vector<std::uint32_t> counts(objs.size(), 0);
            for (const auto& it : q.items)
                for (const auto& span : index.lookup(it))
                    for (ObjectId id : index.ids(span)) ++counts[id];
            const std::uint64_t bound = index.max_count_bound(q);
            for (const auto& o : objs) {
                CHECK(counts[o.id()] == match_count_reference(q, o));
                CHECK(match_count_reference(q, o) <= bound);
            }
        }
    }
    {  // partitioning covers the dataset in order
        std::mt19937 rng(19);
        const auto o36 = random_objects(rng, 36, 3, 4);
        const auto p6 = partition_dataset(o36, 6);
        CHECK(p6.size() == 6);
        for (const auto& p : p6) CHECK(p.size == 6);
        const auto one = partition_dataset(o36, 100);
        CHECK(one.size() == 1 && one[0].size == 36 && one[0].id_offset == 0);
        const auto o10 = random_objects(rng, 10, 3, 4);
        const auto parts = partition_dataset(o10, 4);
        CHECK(parts.size() == 3);
        if (parts.size() == 3) {
            CHECK(parts[0].size == 4 && parts[1].size == 4 && parts[2].size == 2);
            CHECK(parts[0].id_offset == 0 && parts[1].id_offset == 4 && parts[2].id_offset == 8);
        }
        for (const auto& p : parts)
            for (const auto& e : p.index.entries())
                for (ObjectId local : ids_of(p.index, e.keyword)) {
                    const auto& kws = o10[local + p.id_offset].keywords();
                    CHECK(std::find(kws.begin(), kws.end(), e.keyword) != kws.end());
                }
        CHECK_THROWS_AS(partition_dataset(o10, 0), ContractError);
    }
    {  // MCIX round trip, byte-exact, split spans kept
        std::mt19937 rng(23);
        const auto objs = random_objects(rng, 400, 4, 6);
        const auto index = build_index(objs, 64);
        const auto bytes = serialize_index(index);
        const auto reloaded = deserialize_index(bytes.data(), bytes.size());
        CHECK(serialize_index(reloaded) == bytes);
        CHECK(reloaded.num_objects() == index.num_objects());
        CHECK(reloaded.keyword_count() == index.keyword_count());
        CHECK(reloaded.spans() == index.spans());
        CHECK(!reloaded.split_threshold().has_value());
        for (const auto& e : index.entries())
            CHECK(reloaded.max_multiplicity(e.keyword.dim) == index.max_multiplicity(e.keyword.dim));
        // the reloaded (split) index answers like the original
        const Query q(5, {QueryItem(0, 0, 3), QueryItem(2, 1, 1)}, 10);
        const auto a = execute_batch(index, std::vector<Query>{q});
        const auto b = execute_batch(reloaded, std::vector<Query>{q});
        CHECK(a.results[0].entries == b.results[0].entries && a.results[0].threshold == b.results[0].threshold);
        CHECK(fnv1a64(bytes.data(), bytes.size()) == fnv1a64(bytes.data(), bytes.size()));
    }
    {  // corrupted images
        const auto bytes = serialize_index(build_index(example_objects()));
        auto bad_magic = bytes;
        bad_magic[0] = 'X';
        CHECK_THROWS_AS(deserialize_index(bad_magic.data(), bad_magic.size()), DataError);
        CHECK_THROWS_AS(deserialize_index(bytes.data(), bytes.size() - 2), DataError);
        auto unsorted = bytes;
        unsorted[unsorted.size() - 4] = 0;
        CHECK_THROWS_AS(deserialize_index(unsorted.data(), unsorted.size()), DataError);
        auto bad_id = bytes;
        bad_id[bad_id.size() - 4] = 0x7f;
        CHECK_THROWS_AS(deserialize_index(bad_id.data(), bad_id.size()), DataError);
    }
}

void model_cases() {
    const RelationalSchema schema({1024, 9, 2});
    const std::vector<Token> row{700, 3, 1};
    const auto rec = encode_relational_tuple(schema, row, 4);
    CHECK(rec.id() == 4 && rec.keywords().size() == 3);
    CHECK(rec.keywords()[1] == (Keyword{1, 3}));
    CHECK_THROWS_AS(encode_relational_tuple(schema, std::vector<Token>{1, 2}, 0), ContractError);
    CHECK_THROWS_AS(encode_relational_tuple(schema, std::vector<Token>{1, 9, 0}, 0), DataError);
    CHECK_THROWS_AS(RelationalSchema({}), ContractError);
    CHECK_THROWS_AS(RelationalSchema({3, 0}), ContractError);
    const std::vector<AttributeRange> ranges{{0, -50, 40}, {1, 8, 20}, {2, 1, 1}};
    const auto q = encode_relational_query(schema, ranges, 7, 9);
    CHECK(q.id == 9 && q.k == 7 && q.items.size() == 3);
    CHECK(q.items[0].lo == 0 && q.items[0].hi == 40 && q.items[1].lo == 8 && q.items[1].hi == 8);
    CHECK_THROWS_AS(encode_relational_query(schema, std::vector<AttributeRange>{{3, 0, 1}}, 1), ContractError);
    CHECK_THROWS_AS(encode_relational_query(schema, std::vector<AttributeRange>{{1, 9, 12}}, 1), DataError);
    // a relational table through the engine equals the reference count
    std::mt19937 rng(5);
    std::vector<ObjectRecord> objs;
    for (ObjectId i = 0; i < 3000; ++i)
        objs.push_back(encode_relational_tuple(
            schema, std::vector<Token>{Token(rng() % 1024), Token(rng() % 9), Token(rng() % 2)}, i));
    const auto index = build_index(objs);
    const auto res = execute_batch(index, std::vector<Query>{q}).results[0];
    std::vector<TopKEntry> want;
    for (const auto& o : objs)
        if (const auto c = match_count_reference(q, o)) want.push_back({o.id(), c});
    std::sort(want.begin(), want.end(), TopKEntry::better);
    if (want.size() > q.k) want.resize(q.k);
    CHECK(res.entries == want);
}

void lsh_cases() {
    LshEncoderConfig c;
    c.family = LshFamily::p_stable;
    c.m = 17;
    c.dims = 8;
    c.seed = 3;
    const auto enc = LshEncoder::create(c);
    std::vector<float> p(8);
    for (int i = 0; i < 8; ++i) p[i] = 0.37f * float(i) - 1.1f;
    const auto rec = enc.encode_point(p, 0);
    for (std::uint32_t i = 0; i < c.m; ++i) CHECK(enc.token(i, p) == rec.keywords()[i].token);
    CHECK_THROWS_AS(enc.token(c.m, p), ContractError);
    CHECK_THROWS_AS(enc.token(0, std::vector<float>(3)), ContractError);
}

// acceptance.cpp:62-140 corpus generator
struct Instance {
    std::vector<ObjectRecord> objects;
    Query query;
};

Instance make_instance(std::size_t i) {
    constexpr std::uint64_t kMasterSeed = 0x6d63782d616363ull;
    std::mt19937_64 rng(mix64(kMasterSeed ^ (0x9e37 + i)));
    std::size_t n;
    const std::uint64_t bucket = rng() % 100;
    if (bucket < 85) n = 5 + rng() % 800;
    else if (bucket < 97) n = 800 + rng() % 7200;
    else if (bucket < 99) n = 8000 + rng() % 42000;
    else n = 100000;
    const int dims = 2 + int(rng() % 3);
    const int tokens = 4 + int(rng() % 13);
    Instance inst;
    inst.objects.reserve(n);
    for (std::size_t id = 0; id < n; ++id) {
        std::vector<Keyword> kws;
        const int count = 1 + int(rng() % 6);
        for (int t = 0; t < count; ++t) {
            const Keyword kw{DimId(rng() % dims), Token(rng() % tokens)};
            if (std::find(kws.begin(), kws.end(), kw) == kws.end()) kws.push_back(kw);
        }
        inst.objects.emplace_back(ObjectId(id), std::move(kws));
    }
    std::vector<QueryItem> items;
    const int item_count = 1 + int(rng() % 6);
    for (int t = 0; t < item_count; ++t) {
        const Token lo = Token(rng() % tokens);
        items.push_back(QueryItem(DimId(rng() % dims), lo, lo + Token(rng() % 4)));
    }
    const std::uint32_t ks[3] = {1, 10, 100};
    inst.query = Query(std::uint32_t(i), items, ks[i % 3]);
    return inst;
}

bool same_result(const TopKResult& a, const TopKResult& b) {
    return a.entries == b.entries && a.threshold == b.threshold;
}

// the CPU oracle's answer (oracle/genie_oracle.c, pinned to the reference)
TopKResult oracle_result(const InvertedIndex& index, const Query& q) {
    std::vector<std::uint64_t> keys = index.packed_keys(), off(index.keyword_count() + 1, 0);
    std::vector<ObjectId> post;
    for (std::size_t j = 0; j < index.keyword_count(); ++j) {
        for (const auto& s : index.spans_of(index.entries()[j])) {
            const auto v = index.ids(s);
            post.insert(post.end(), v.begin(), v.end());
        }
        off[j + 1] = post.size();
    }
    void* ox = or_index_create(index.num_objects(), keys.size(), keys.data(), off.data(), post.data());
    std::vector<std::uint16_t> dim;
    std::vector<std::uint32_t> lo, hi;
    for (const auto& it : q.items) {
        dim.push_back(it.dim);
        lo.push_back(it.lo);
        hi.push_back(it.hi);
    }
    const std::uint64_t ioff[2] = {0, q.items.size()};
    const std::uint32_t stride = q.k;
    std::vector<std::uint32_t> ids(stride), cnt(stride);
    std::uint32_t len = 0, thr = 0, bad = 0;
    or_execute(ox, 1, &q.id, &q.k, ioff, dim.data(), lo.data(), hi.data(), stride, ids.data(), cnt.data(), &len, &thr,
               nullptr, nullptr, 1, &bad);
    or_index_free(ox);
    TopKResult r;
    r.query_id = q.id;
    r.threshold = thr;
    for (std::uint32_t e = 0; e < len; ++e) r.entries.push_back({ids[e], cnt[e]});
    return r;
}

void acceptance(std::size_t corpus) {
    std::size_t exact_bad = 0, knob_bad = 0, part_bad = 0;
    for (std::size_t i = 0; i < corpus; ++i) {
        const Instance inst = make_instance(i);
        const auto index = build_index(inst.objects);
        const std::vector<Query> queries = {inst.query};
        EngineConfig seq;
        seq.mode = ExecMode::sequential;
        const BatchResult expected = execute_batch(index, queries, seq);
        // criterion 1: exactness against the pinned CPU oracle
        if (!same_result(expected.results[0], oracle_result(index, inst.query))) ++exact_bad;
        // criterion 3: scheduling knobs (workers, small chunks) and repeats
        for (std::uint32_t workers : {2u, 4u, 8u}) {
            EngineConfig par;
            par.workers = workers;
            par.span_chunk = 64;
            for (int rep = 0; rep < 3; ++rep)
                if (!same_result(execute_batch(index, queries, par).results[0], expected.results[0])) ++knob_bad;
        }
        // criterion 10: partition-capacity invariance
        const auto n = std::uint32_t(inst.objects.size());
        for (std::uint32_t cap : {n, std::max(1u, n / 2), std::max(1u, n / 6), 1000u}) {
            // capacity 1000 on the corpus' 8K-100K-object tail means 9-100 device
            // indexes per instance: kept for n <= 24 000 (up to 24 parts)
            if (cap == 1000u && n > 24000u) continue;
            const auto parts = partition_dataset(inst.objects, cap);
            const BatchResult merged = execute_partitioned(parts, queries, seq);
            if (!same_result(merged.results[0], expected.results[0])) ++part_bad;
            CHECK(merged.timings.total_ns >= merged.timings.merge_ns);
        }
    }
    CHECK(exact_bad == 0);
    CHECK(knob_bad == 0);
    CHECK(part_bad == 0);
    std::printf("acceptance: %zu instances, exactness %zu, knobs %zu, partitions %zu mismatches\n", corpus, exact_bad,
                knob_bad, part_bad);
    // criterion 12, engine half: 4-bit accounting = ceil(n / 2) bytes
    std::vector<ObjectRecord> objs;
    for (ObjectId i = 0; i < 101; ++i) objs.emplace_back(i, std::vector<Keyword>{{0, i % 7}});
    const auto index = build_index(objs);
    const Query q(0, {QueryItem(0, 0, 6)}, 5);
    const auto batch = execute_batch(index, std::vector<Query>{q});
    CHECK(batch.memory.counter_bytes == (101 + 1) / 2);
}

}  // namespace

int main(int argc, char** argv) {
    const std::size_t corpus = argc > 1 ? std::size_t(std::atol(argv[1])) : 120;
    try {
        index_cases();
        model_cases();
        lsh_cases();
        acceptance(corpus);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "unexpected exception: %s\n", e.what());
        return 2;
    }
    std::printf("reference api: %d checks, %d failures\n", checks, failures);
    if (failures) return 1;
    std::printf("reference api: ok\n");
    return 0;
}
