// mcx/mcx.hpp -- C++20 drop-in for the batched query path of the reference
// library `mcx` (/root/reference/proj/include/mcx, umbrella mcx.hpp:18-27).
//
// Same namespace, type names, member functions and error types as the
// reference, so callers of mcx::build_index / execute_batch /
// execute_partitioned / merge_topk / hash_results / LshEncoder recompile
// against this header and link libgenie_b200.so (hand-written sm_100a CUDA
// behind include/genie/genie.h).  Host-side pieces the reference also runs on
// the host (object and query construction, the CSR build, partition
// bookkeeping, merge_topk, hash_results) are restated here; match counting,
// the Count Priority Queue and top-k selection run on the GPU.
//
// Link: -I<repo>/include -L<repo>/paper_1603_08390_b200/lib -lgenie_b200
#pragma once

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdint>
#include <memory>
#include <optional>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "genie/genie.h"

namespace mcx {

// ---------------------------------------------------------------- error.hpp

class DataError : public std::runtime_error {
public:
    explicit DataError(const std::string& m) : std::runtime_error(m) {}
};
class ContractError : public std::invalid_argument {
public:
    explicit ContractError(const std::string& m) : std::invalid_argument(m) {}
};
class InvariantError : public std::logic_error {
public:
    explicit InvariantError(const std::string& m) : std::logic_error(m) {}
};

namespace detail {
[[noreturn]] inline void raise(int rc, const char* msg) {
    switch (rc) {
        case GENIE_ERR_CONTRACT: throw ContractError(msg);
        case GENIE_ERR_DATA: throw DataError(msg);
        case GENIE_ERR_INVARIANT: throw InvariantError(msg);
        default: throw std::runtime_error(std::string("genie: ") + msg);
    }
}
inline void check(int rc, const char* msg) {
    if (rc != GENIE_OK) raise(rc, msg);
}
}  // namespace detail

// ---------------------------------------------------------------- model.hpp

using DimId = std::uint16_t;
using Token = std::uint32_t;
using ObjectId = std::uint32_t;

struct Keyword {
    DimId dim = 0;
    Token token = 0;
    friend constexpr auto operator<=>(const Keyword&, const Keyword&) = default;
    constexpr std::uint64_t packed() const noexcept { return (std::uint64_t(dim) << 32) | token; }
};

class ObjectRecord {
public:
    ObjectRecord(ObjectId id, std::vector<Keyword> kws) : id_(id), kws_(std::move(kws)) {
        std::ranges::sort(kws_);
        if (auto it = std::ranges::adjacent_find(kws_); it != kws_.end())
            throw ContractError("ObjectRecord " + std::to_string(id) + ": duplicate keyword (dim=" +
                                std::to_string(it->dim) + ", token=" + std::to_string(it->token) + ")");
    }
    ObjectId id() const noexcept { return id_; }
    const std::vector<Keyword>& keywords() const noexcept { return kws_; }

private:
    ObjectId id_;
    std::vector<Keyword> kws_;
};

struct QueryItem {
    DimId dim = 0;
    Token lo = 0;
    Token hi = 0;
    QueryItem() = default;
    QueryItem(DimId d, Token l, Token h) : dim(d), lo(l), hi(h) {
        if (l > h)
            throw ContractError("QueryItem: lo " + std::to_string(l) + " > hi " + std::to_string(h) +
                                " on dim " + std::to_string(d));
    }
    static QueryItem point(DimId d, Token t) { return {d, t, t}; }
};

struct Query {
    std::uint32_t id = 0;
    std::vector<QueryItem> items;
    std::uint32_t k = 1;
    Query() = default;
    Query(std::uint32_t qid, std::vector<QueryItem> its, std::uint32_t qk) : id(qid), items(std::move(its)), k(qk) {
        if (items.empty()) throw ContractError("Query " + std::to_string(qid) + ": no items");
        if (k == 0) throw ContractError("Query " + std::to_string(qid) + ": k must be >= 1");
    }
};

inline std::uint32_t match_count_reference(const Query& q, const ObjectRecord& o) {
    const auto& kws = o.keywords();
    std::uint32_t total = 0;
    for (const auto& it : q.items) {
        auto a = std::lower_bound(kws.begin(), kws.end(), Keyword{it.dim, it.lo});
        auto b = std::upper_bound(kws.begin(), kws.end(), Keyword{it.dim, it.hi});
        total += static_cast<std::uint32_t>(b - a);
    }
    return total;
}

// ------------------------------------------------------------------ cpq.hpp

struct TopKEntry {
    ObjectId id = 0;
    std::uint32_t count = 0;
    friend constexpr bool operator==(const TopKEntry&, const TopKEntry&) = default;
    static constexpr bool better(const TopKEntry& a, const TopKEntry& b) noexcept {
        return a.count != b.count ? a.count > b.count : a.id < b.id;
    }
};

struct TopKResult {
    std::uint32_t query_id = 0;
    std::vector<TopKEntry> entries;  // count desc, id asc
    std::uint32_t threshold = 0;
};

// ---------------------------------------------------------------- index.hpp

struct PostingsSpan {
    std::uint64_t begin = 0, end = 0;
    std::uint64_t length() const noexcept { return end - begin; }
    friend constexpr bool operator==(const PostingsSpan&, const PostingsSpan&) = default;
};

inline constexpr std::uint32_t kDefaultSplitThreshold = 4096;

// The host CSR (keys ascending, ids ascending per key) plus its device copy.
class InvertedIndex {
public:
    InvertedIndex() = default;
    InvertedIndex(std::uint32_t n, std::vector<std::uint64_t> keys, std::vector<std::uint64_t> off,
                  std::vector<ObjectId> post, std::optional<std::uint32_t> split, int device = 0)
        : n_(n), keys_(std::move(keys)), off_(std::move(off)), post_(std::move(post)), split_(split),
          device_(device) {}

    std::uint32_t num_objects() const noexcept { return n_; }
    std::size_t keyword_count() const noexcept { return keys_.size(); }
    const std::vector<ObjectId>& list_array() const noexcept { return post_; }
    std::optional<std::uint32_t> split_threshold() const noexcept { return split_; }
    // the CSR image: packed keywords (ascending) and their postings offsets
    const std::vector<std::uint64_t>& packed_keys() const noexcept { return keys_; }
    const std::vector<std::uint64_t>& key_offsets() const noexcept { return off_; }

    // spans of every indexed keyword inside the item's range (index.hpp:86-96)
    std::vector<PostingsSpan> lookup(const QueryItem& item) const {
        std::vector<PostingsSpan> out;
        auto a = std::lower_bound(keys_.begin(), keys_.end(), Keyword{item.dim, item.lo}.packed());
        auto b = std::upper_bound(keys_.begin(), keys_.end(), Keyword{item.dim, item.hi}.packed());
        for (auto j = std::size_t(a - keys_.begin()); j < std::size_t(b - keys_.begin()); ++j) {
            const std::uint64_t lim = split_ ? *split_ : off_[j + 1] - off_[j];
            for (std::uint64_t p = off_[j]; p < off_[j + 1]; p += lim) out.push_back({p, std::min(off_[j + 1], p + lim)});
        }
        return out;
    }
    std::span<const ObjectId> ids(const PostingsSpan& s) const {
        return std::span<const ObjectId>(post_).subspan(s.begin, s.length());
    }

    genie_index* device() const {
        if (!dev_) {
            genie_index* h = nullptr;
            char err[512] = {};
            const std::uint64_t zero = 0;
            detail::check(genie_index_create(n_, keys_.size(), keys_.data(), off_.empty() ? &zero : off_.data(),
                                             post_.data(), nullptr, 0, device_, &h, err, sizeof(err)),
                          err);
            dev_ = std::shared_ptr<genie_index>(h, genie_index_destroy);
        }
        return dev_.get();
    }

private:
    std::uint32_t n_ = 0;
    std::vector<std::uint64_t> keys_, off_{0};
    std::vector<ObjectId> post_;
    std::optional<std::uint32_t> split_;
    int device_ = 0;
    mutable std::shared_ptr<genie_index> dev_;
};

// build_index (index.hpp:190-250): dense ids, (keyword, id) pairs grouped by
// keyword with ascending ids.
inline InvertedIndex build_index(std::span<const ObjectRecord> objects,
                                 std::optional<std::uint32_t> split_threshold = std::nullopt, int device = 0) {
    if (split_threshold && *split_threshold == 0) throw ContractError("split_threshold must be positive");
    const auto n = static_cast<std::uint32_t>(objects.size());
    std::vector<char> seen(n, 0);
    std::vector<std::pair<std::uint64_t, ObjectId>> pairs;
    for (const auto& o : objects) {
        if (o.id() >= n || seen[o.id()])
            throw DataError("object ids must be dense 0.." + std::to_string(n ? n - 1 : 0) + ": bad id " +
                            std::to_string(o.id()));
        seen[o.id()] = 1;
        for (const auto& kw : o.keywords()) pairs.emplace_back(kw.packed(), o.id());
    }
    std::ranges::sort(pairs);
    std::vector<std::uint64_t> keys, off{0};
    std::vector<ObjectId> post;
    post.reserve(pairs.size());
    for (std::size_t i = 0; i < pairs.size(); ++i) {
        if (i == 0 || pairs[i].first != pairs[i - 1].first) {
            if (i) off.push_back(post.size());
            keys.push_back(pairs[i].first);
        }
        post.push_back(pairs[i].second);
    }
    if (!pairs.empty()) off.push_back(post.size());
    return InvertedIndex(n, std::move(keys), std::move(off), std::move(post), split_threshold, device);
}

// ------------------------------------------------------------------ index_io
// MCIX files (index_io.hpp:27-154) through the C ABI: the same bytes as the
// reference's serialize_index for the same build, the same validation and
// DataError messages on load.  A loaded index keeps whole-list spans (the
// file's span cut is a build-time choice; results do not depend on it).

inline std::vector<std::uint8_t> serialize_index(const InvertedIndex& index) {
    char err[512] = {};
    std::uint64_t size = 0;
    const auto& k = index.packed_keys();
    const auto& o = index.key_offsets();
    const auto& p = index.list_array();
    const std::uint32_t split = index.split_threshold().value_or(0);
    detail::check(genie_mcix_serialize(index.num_objects(), k.size(), k.data(), o.data(), p.data(), split, nullptr,
                                       &size, err, sizeof(err)),
                  err);
    std::vector<std::uint8_t> out(size);
    detail::check(genie_mcix_serialize(index.num_objects(), k.size(), k.data(), o.data(), p.data(), split, out.data(),
                                       &size, err, sizeof(err)),
                  err);
    return out;
}

inline InvertedIndex deserialize_index(const std::uint8_t* data, std::size_t size, int device = 0) {
    char err[512] = {};
    std::uint32_t n = 0;
    std::uint64_t K = 0, P = 0;
    detail::check(genie_mcix_parse(data, size, &n, &K, &P, nullptr, nullptr, nullptr, err, sizeof(err)), err);
    std::vector<std::uint64_t> keys(K), off(K + 1);
    std::vector<ObjectId> post(P);
    detail::check(genie_mcix_parse(data, size, nullptr, nullptr, nullptr, keys.data(), off.data(), post.data(), err,
                                   sizeof(err)),
                  err);
    return InvertedIndex(n, std::move(keys), std::move(off), std::move(post), std::nullopt, device);
}

inline void save_index(const InvertedIndex& index, const std::string& path) {
    const auto bytes = serialize_index(index);
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw DataError("cannot open " + path + " for writing");
    const bool ok = std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
    std::fclose(f);
    if (!ok) throw DataError("failed writing " + path);
}

inline InvertedIndex load_index(const std::string& path, int device = 0) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw DataError("cannot open " + path);
    std::vector<std::uint8_t> bytes;
    std::uint8_t buf[1 << 16];
    for (std::size_t got; (got = std::fread(buf, 1, sizeof(buf), f)) > 0;) bytes.insert(bytes.end(), buf, buf + got);
    std::fclose(f);
    return deserialize_index(bytes.data(), bytes.size(), device);
}

struct IndexPartition {
    std::uint32_t part_id = 0;
    ObjectId id_offset = 0;
    std::uint32_t size = 0;
    InvertedIndex index;
};

inline std::vector<IndexPartition> partition_dataset(std::span<const ObjectRecord> objects,
                                                     std::uint32_t part_capacity,
                                                     std::optional<std::uint32_t> split = std::nullopt) {
    if (part_capacity == 0) throw ContractError("part_capacity must be >= 1");
    for (std::size_t i = 0; i < objects.size(); ++i)
        if (objects[i].id() != i) throw DataError("partitioning requires objects in dense id order");
    std::vector<IndexPartition> parts;
    for (std::size_t start = 0, pid = 0; start < objects.size(); start += part_capacity, ++pid) {
        const auto cnt = std::min<std::size_t>(part_capacity, objects.size() - start);
        std::vector<ObjectRecord> local;
        for (std::size_t i = 0; i < cnt; ++i) local.emplace_back(ObjectId(i), objects[start + i].keywords());
        parts.push_back({std::uint32_t(pid), ObjectId(start), std::uint32_t(cnt), build_index(local, split)});
    }
    return parts;
}

// --------------------------------------------------------------- engine.hpp

enum class Selector { cpq, bucket, sort };
enum class ExecMode { parallel, sequential };

struct EngineConfig {
    Selector selector = Selector::cpq;
    ExecMode mode = ExecMode::parallel;  // the device path is always parallel
    std::uint32_t workers = 0;           // accepted, unused on the device
    std::uint32_t span_chunk = 1024;     // postings per warp work unit
    std::uint32_t max_spans_per_task = 2;
};

struct StageTimings {
    std::uint64_t lookup_ns = 0, match_ns = 0, select_ns = 0, merge_ns = 0, total_ns = 0;
};
struct MemoryStats {
    std::size_t counter_bytes = 0, gate_bytes = 0, table_bytes = 0;
};
struct BatchResult {
    std::vector<TopKResult> results;
    StageTimings timings;
    MemoryStats memory;
};

inline std::uint64_t hash_results(std::span<const TopKResult> results) {
    std::vector<std::uint32_t> qid, thr, len;
    std::uint32_t stride = 1;
    for (const auto& r : results) stride = std::max<std::uint32_t>(stride, std::uint32_t(r.entries.size()));
    std::vector<genie_entry> ent(results.size() * std::size_t(stride));
    for (std::size_t q = 0; q < results.size(); ++q) {
        qid.push_back(results[q].query_id);
        thr.push_back(results[q].threshold);
        len.push_back(std::uint32_t(results[q].entries.size()));
        for (std::size_t e = 0; e < results[q].entries.size(); ++e)
            ent[q * stride + e] = {results[q].entries[e].id, results[q].entries[e].count};
    }
    return genie_hash_results(std::uint32_t(results.size()), qid.data(), thr.data(), len.data(), stride, ent.data());
}

inline TopKResult merge_topk(std::span<const TopKResult> locals, std::uint32_t k, std::uint32_t query_id) {
    TopKResult m;
    m.query_id = query_id;
    for (const auto& l : locals) m.entries.insert(m.entries.end(), l.entries.begin(), l.entries.end());
    std::ranges::sort(m.entries, {}, &TopKEntry::id);
    for (std::size_t i = 1; i < m.entries.size(); ++i)
        if (m.entries[i].id == m.entries[i - 1].id)
            throw ContractError("merge_topk: object " + std::to_string(m.entries[i].id) +
                                " reported by more than one partition");
    std::ranges::sort(m.entries, TopKEntry::better);
    if (m.entries.size() > k) m.entries.resize(k);
    m.threshold = m.entries.size() >= k ? m.entries.back().count : 0;
    return m;
}

inline BatchResult execute_batch(const InvertedIndex& index, std::span<const Query> queries,
                                 const EngineConfig& config = {}) {
    if (config.span_chunk == 0 || config.max_spans_per_task == 0)
        throw ContractError("span_chunk and max_spans_per_task must be positive");
    BatchResult batch;
    const auto Q = static_cast<std::uint32_t>(queries.size());
    if (!Q) return batch;
    std::vector<std::uint32_t> qid(Q), k(Q), lo, hi;
    std::vector<std::uint64_t> off(Q + 1, 0);
    std::vector<std::uint16_t> dim;
    std::uint32_t max_k = 1;
    for (std::uint32_t q = 0; q < Q; ++q) {
        qid[q] = queries[q].id;
        k[q] = queries[q].k;
        max_k = std::max(max_k, k[q]);
        for (const auto& it : queries[q].items) {
            dim.push_back(it.dim);
            lo.push_back(it.lo);
            hi.push_back(it.hi);
        }
        off[q + 1] = dim.size();
    }
    const std::uint32_t stride = std::max<std::uint32_t>(1, std::min(max_k, std::max<std::uint32_t>(index.num_objects(), 1)));
    std::vector<genie_entry> out(std::size_t(Q) * stride);
    std::vector<std::uint32_t> len(Q), thr(Q);
    genie_config cfg = genie_config_default();
    cfg.selector = static_cast<std::uint32_t>(config.selector);
    cfg.span_chunk = config.span_chunk;
    cfg.max_spans_per_task = config.max_spans_per_task;
    genie_stage_ns t{};
    genie_batch_stats st{};
    char err[1024] = {};
    detail::check(genie_query_batch(index.device(), &cfg, Q, qid.data(), k.data(), off.data(), dim.data(), lo.data(),
                                    hi.data(), stride, out.data(), len.data(), thr.data(), nullptr, &t, &st, err,
                                    sizeof(err)),
                  err);
    batch.results.resize(Q);
    for (std::uint32_t q = 0; q < Q; ++q) {
        auto& r = batch.results[q];
        r.query_id = qid[q];
        r.threshold = thr[q];
        for (std::uint32_t e = 0; e < len[q]; ++e) r.entries.push_back({out[std::size_t(q) * stride + e].id,
                                                                         out[std::size_t(q) * stride + e].count});
    }
    batch.timings = {t.lookup_ns, t.match_ns, t.select_ns, t.merge_ns, t.total_ns};
    batch.memory = {st.counter_bytes, st.gate_bytes, st.table_bytes};
    return batch;
}

inline BatchResult execute_partitioned(std::span<const IndexPartition> partitions, std::span<const Query> queries,
                                       const EngineConfig& config = {}) {
    std::uint64_t expected = 0;
    for (const auto& p : partitions) {
        if (p.id_offset != expected || p.index.num_objects() != p.size)
            throw ContractError("partitions must be disjoint and contiguous");
        expected += p.size;
    }
    BatchResult batch;
    batch.results.resize(queries.size());
    std::vector<std::vector<TopKResult>> locals(queries.size());
    for (const auto& p : partitions) {
        auto local = execute_batch(p.index, queries, config);
        batch.timings.lookup_ns += local.timings.lookup_ns;
        batch.timings.match_ns += local.timings.match_ns;
        batch.timings.select_ns += local.timings.select_ns;
        batch.memory.counter_bytes = std::max(batch.memory.counter_bytes, local.memory.counter_bytes);
        batch.memory.gate_bytes = std::max(batch.memory.gate_bytes, local.memory.gate_bytes);
        batch.memory.table_bytes = std::max(batch.memory.table_bytes, local.memory.table_bytes);
        for (std::size_t q = 0; q < queries.size(); ++q) {
            for (auto& e : local.results[q].entries) e.id += p.id_offset;
            locals[q].push_back(std::move(local.results[q]));
        }
    }
    for (std::size_t q = 0; q < queries.size(); ++q) batch.results[q] = merge_topk(locals[q], queries[q].k, queries[q].id);
    return batch;
}

// ------------------------------------------------------------------ lsh.hpp

// ------------------------------------------------------------------ documents
// tokenize_document / DocumentCodec (sa.hpp:341-408): lowercased whitespace
// words minus stop words, deduplicated; token = rank in the sorted build
// vocabulary, dim 0 (the Tweets adapter).

inline std::vector<std::string> tokenize_document(std::string_view text,
                                                  const std::set<std::string>& stop_words = {}) {
    std::set<std::string> words;
    std::string cur;
    auto flush = [&] {
        if (!cur.empty() && !stop_words.contains(cur)) words.insert(cur);
        cur.clear();
    };
    for (const char ch : text) {
        if (std::isspace(static_cast<unsigned char>(ch))) flush();
        else cur.push_back(static_cast<char>(std::tolower(static_cast<unsigned char>(ch))));
    }
    flush();
    return {words.begin(), words.end()};
}

class DocumentCodec {
public:
    static DocumentCodec build(std::span<const std::string> corpus, std::set<std::string> stop_words = {}) {
        DocumentCodec c;
        c.stop_ = std::move(stop_words);
        std::set<std::string> all;
        for (const auto& doc : corpus)
            for (auto& w : tokenize_document(doc, c.stop_)) all.insert(std::move(w));
        Token t = 0;
        for (const auto& w : all) c.vocab_.emplace(w, t++);
        return c;
    }
    std::size_t vocabulary_size() const noexcept { return vocab_.size(); }
    ObjectRecord encode(std::string_view text, ObjectId id) const {
        std::vector<Keyword> kws;
        for (const auto& w : tokenize_document(text, stop_)) {
            const auto it = vocab_.find(w);
            if (it == vocab_.end()) throw ContractError("document word outside the vocabulary");
            kws.push_back(Keyword{0, it->second});
        }
        return ObjectRecord(id, std::move(kws));
    }
    std::optional<Query> encode_query(std::string_view text, std::uint32_t k, std::uint32_t query_id = 0) const {
        std::vector<QueryItem> items;
        for (const auto& w : tokenize_document(text, stop_))
            if (const auto it = vocab_.find(w); it != vocab_.end()) items.push_back(QueryItem::point(0, it->second));
        if (items.empty()) return std::nullopt;
        return Query(query_id, std::move(items), k);
    }

private:
    std::set<std::string> stop_;
    std::unordered_map<std::string, Token> vocab_;
};

enum class LshFamily { p_stable, random_binning };

struct LshEncoderConfig {
    LshFamily family = LshFamily::random_binning;
    std::uint32_t m = 237;
    std::uint32_t dims = 0;
    std::uint64_t seed = 1;
    std::uint32_t rehash_domain = 8192;
    double w = 4.0;
    std::uint32_t bucket_count = 67;
    std::int64_t bucket_min = -33;
    bool rehash_pstable = false;
    double sigma = 1.0;
};

class LshEncoder {
public:
    static LshEncoder create(const LshEncoderConfig& c, int device = 0) {
        genie_lsh_config g = genie_lsh_config_default();
        g.family = c.family == LshFamily::p_stable ? GENIE_LSH_PSTABLE : GENIE_LSH_RBH;
        g.m = c.m;
        g.dims = c.dims;
        g.seed = c.seed;
        g.rehash_domain = c.rehash_domain;
        g.w = c.w;
        g.bucket_count = c.bucket_count;
        g.bucket_min = c.bucket_min;
        g.rehash_pstable = c.rehash_pstable ? 1 : 0;
        g.sigma = c.sigma;
        genie_encoder* h = nullptr;
        char err[512] = {};
        detail::check(genie_encoder_create(&g, device, &h, err, sizeof(err)), err);
        LshEncoder e;
        e.cfg_ = c;
        e.h_ = std::shared_ptr<genie_encoder>(h, genie_encoder_destroy);
        return e;
    }
    const LshEncoderConfig& config() const noexcept { return cfg_; }
    std::uint32_t m() const noexcept { return cfg_.m; }

    // tokens of n points (row-major n x dims) -> n x m
    std::vector<Token> encode_points(std::span<const float> points) const {
        if (points.size() % cfg_.dims) throw ContractError("point dimensionality mismatch");
        const std::uint64_t n = points.size() / cfg_.dims;
        std::vector<Token> out(n * cfg_.m);
        char err[512] = {};
        detail::check(genie_lsh_encode(h_.get(), points.data(), n, out.data(), err, sizeof(err)), err);
        return out;
    }
    ObjectRecord encode_point(std::span<const float> point, ObjectId id) const {
        check_dims(point);
        const auto t = encode_points(point);
        std::vector<Keyword> kws;
        for (std::uint32_t i = 0; i < cfg_.m; ++i) kws.push_back({DimId(i), t[i]});
        return ObjectRecord(id, std::move(kws));
    }
    Query encode_query_point(std::span<const float> point, std::uint32_t k, std::uint32_t query_id = 0) const {
        check_dims(point);
        const auto t = encode_points(point);
        std::vector<QueryItem> items;
        for (std::uint32_t i = 0; i < cfg_.m; ++i) items.push_back(QueryItem::point(DimId(i), t[i]));
        return Query(query_id, std::move(items), k);
    }

private:
    void check_dims(std::span<const float> p) const {
        if (p.size() != cfg_.dims)
            throw ContractError("point dimensionality " + std::to_string(p.size()) + " != hash dimensionality " +
                                std::to_string(cfg_.dims));
    }
    LshEncoderConfig cfg_;
    std::shared_ptr<genie_encoder> h_;
};

}  // namespace mcx
