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
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <memory>
#include <mutex>
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

// ------------------------------------------------------------------ rng.hpp

// splitmix64 finalizer (rng.hpp:25-30): the hash every seed and table home uses
inline constexpr std::uint64_t mix64(std::uint64_t x) noexcept {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

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

// Relational tables (model.hpp:119-188): one keyword per attribute (dim =
// attribute index); query ranges are clamped into the attribute's domain.
class RelationalSchema {
public:
    explicit RelationalSchema(std::vector<Token> domain_sizes) : dom_(std::move(domain_sizes)) {
        if (dom_.empty()) throw ContractError("RelationalSchema: empty schema");
        for (std::size_t a = 0; a < dom_.size(); ++a)
            if (!dom_[a]) throw ContractError("RelationalSchema: attribute " + std::to_string(a) + " has empty domain");
    }
    std::size_t attribute_count() const noexcept { return dom_.size(); }
    Token domain_size(std::size_t attr) const { return dom_.at(attr); }

private:
    std::vector<Token> dom_;
};

inline ObjectRecord encode_relational_tuple(const RelationalSchema& schema, std::span<const Token> values,
                                            ObjectId id) {
    if (values.size() != schema.attribute_count())
        throw ContractError("tuple arity " + std::to_string(values.size()) + " != schema arity " +
                            std::to_string(schema.attribute_count()));
    std::vector<Keyword> kws(values.size());
    for (std::size_t a = 0; a < values.size(); ++a) {
        if (values[a] >= schema.domain_size(a))
            throw DataError("attribute " + std::to_string(a) + ": token " + std::to_string(values[a]) +
                            " outside domain [0, " + std::to_string(schema.domain_size(a)) + ")");
        kws[a] = Keyword{DimId(a), values[a]};
    }
    return ObjectRecord(id, std::move(kws));
}

struct AttributeRange {
    std::size_t attr = 0;
    std::int64_t lo = 0;  // before clamping; may lie outside the domain
    std::int64_t hi = 0;
};

inline Query encode_relational_query(const RelationalSchema& schema, std::span<const AttributeRange> ranges,
                                     std::uint32_t k, std::uint32_t query_id = 0) {
    std::vector<QueryItem> items;
    items.reserve(ranges.size());
    for (const auto& r : ranges) {
        if (r.attr >= schema.attribute_count())
            throw ContractError("range on unknown attribute " + std::to_string(r.attr));
        const std::int64_t dom = schema.domain_size(r.attr);
        const std::int64_t lo = std::max<std::int64_t>(r.lo, 0), hi = std::min<std::int64_t>(r.hi, dom - 1);
        if (lo > hi)
            throw DataError("attribute " + std::to_string(r.attr) + ": range [" + std::to_string(r.lo) + ", " +
                            std::to_string(r.hi) + "] is empty after clamping to [0, " + std::to_string(dom) + ")");
        items.emplace_back(DimId(r.attr), Token(lo), Token(hi));
    }
    return Query(query_id, std::move(items), k);
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

// InvertedIndex (index.hpp:41-182): the reference's host view -- keyword
// entries sorted by keyword, each owning span_count consecutive spans of one
// list array -- kept verbatim so callers that walk entries()/spans() work
// unchanged.  Queries run on the device copy, a CSR image of the same lists
// uploaded on first use (device()); the spans of a keyword are contiguous, so
// the CSR row of entry j is [spans[first_span].begin, last span's end).
class InvertedIndex {
public:
    struct KeywordEntry {
        Keyword keyword;
        std::uint32_t first_span = 0;
        std::uint16_t span_count = 0;
    };
    struct DimStats {
        DimId dim = 0;
        Token max_token = 0;
        std::uint32_t max_multiplicity = 0;  // most tokens one object carries in the dim
    };

    InvertedIndex() = default;
    InvertedIndex(std::uint32_t num_objects, std::vector<KeywordEntry> entries, std::vector<PostingsSpan> spans,
                  std::vector<ObjectId> list_array, std::optional<std::uint32_t> split_threshold, int device = 0)
        : n_(num_objects), entries_(std::move(entries)), spans_(std::move(spans)), list_(std::move(list_array)),
          split_(split_threshold), device_(device), lazy_(std::make_shared<Lazy>()) {}

    std::uint32_t num_objects() const noexcept { return n_; }
    std::size_t keyword_count() const noexcept { return entries_.size(); }
    const std::vector<KeywordEntry>& entries() const noexcept { return entries_; }
    const std::vector<PostingsSpan>& spans() const noexcept { return spans_; }
    const std::vector<ObjectId>& list_array() const noexcept { return list_; }
    std::optional<std::uint32_t> split_threshold() const noexcept { return split_; }
    int device_id() const noexcept { return device_; }

    std::span<const ObjectId> ids(const PostingsSpan& s) const {
        return std::span<const ObjectId>(list_).subspan(s.begin, s.length());
    }
    std::span<const PostingsSpan> spans_of(const KeywordEntry& e) const {
        return std::span<const PostingsSpan>(spans_).subspan(e.first_span, e.span_count);
    }

    // index.hpp:86-96: the spans of every indexed keyword of the item's range
    void lookup_into(const QueryItem& item, std::vector<PostingsSpan>& out) const {
        const auto [a, b] = keyword_range(item);
        for (auto j = a; j < b; ++j) {
            const auto ss = spans_of(entries_[j]);
            out.insert(out.end(), ss.begin(), ss.end());
        }
    }
    std::vector<PostingsSpan> lookup(const QueryItem& item) const {
        std::vector<PostingsSpan> out;
        lookup_into(item, out);
        return out;
    }

    std::optional<Token> max_token(DimId dim) const {
        const DimStats* s = find_dim(dim);
        if (!s) return std::nullopt;
        return s->max_token;
    }
    std::uint32_t max_multiplicity(DimId dim) const {
        const DimStats* s = find_dim(dim);
        return s ? s->max_multiplicity : 0;
    }
    // index.hpp:118-133: sum over items of min(#keywords in range, max multiplicity)
    std::uint64_t max_count_bound(const Query& q) const {
        std::uint64_t bound = 0;
        for (const auto& it : q.items) {
            const auto [a, b] = keyword_range(it);
            bound += std::min<std::uint64_t>(b - a, max_multiplicity(it.dim));
        }
        return bound;
    }
    std::uint64_t longest_list() const {
        std::uint64_t best = 0;
        for (const auto& e : entries_) {
            std::uint64_t len = 0;
            for (const auto& s : spans_of(e)) len += s.length();
            best = std::max(best, len);
        }
        return best;
    }

    // CSR image of the lists (packed keywords ascending, row offsets, ids)
    std::vector<std::uint64_t> packed_keys() const {
        std::vector<std::uint64_t> k(entries_.size());
        for (std::size_t j = 0; j < entries_.size(); ++j) k[j] = entries_[j].keyword.packed();
        return k;
    }

    // adopt an existing device copy of exactly these lists (build_index's
    // device build), so the first query does not upload them again
    void adopt_device(std::shared_ptr<genie_index> h) const {
        std::call_once(lazy_->dev_once, [&] { lazy_->dev = std::move(h); });
    }

    // the device index (uploaded once; shared by copies of this object)
    genie_index* device() const {
        std::call_once(lazy_->dev_once, [&] {
            std::vector<std::uint64_t> off(entries_.size() + 1, 0);
            std::vector<ObjectId> gathered;
            const ObjectId* post = list_.data();
            if (tiles_in_order()) {
                for (std::size_t j = 0; j < entries_.size(); ++j)
                    off[j] = entries_[j].span_count ? spans_[entries_[j].first_span].begin : (j ? off[j - 1] : 0);
                off[entries_.size()] = list_.size();
            } else {  // arbitrary span placement: gather each keyword's spans into one row
                for (std::size_t j = 0; j < entries_.size(); ++j) {
                    for (const auto& s : spans_of(entries_[j])) {
                        const auto v = ids(s);
                        gathered.insert(gathered.end(), v.begin(), v.end());
                    }
                    off[j + 1] = gathered.size();
                }
                post = gathered.data();
            }
            const auto keys = packed_keys();
            genie_index* h = nullptr;
            char err[512] = {};
            detail::check(genie_index_create(n_, keys.size(), keys.data(), off.data(), post, nullptr, 0, device_, &h,
                                             err, sizeof(err)),
                          err);
            lazy_->dev = std::shared_ptr<genie_index>(h, genie_index_destroy);
        });
        return lazy_->dev.get();
    }

private:
    struct Lazy {
        std::once_flag dev_once, stats_once;
        std::shared_ptr<genie_index> dev;
        std::vector<DimStats> stats;  // sorted by dim
    };

    std::pair<std::size_t, std::size_t> keyword_range(const QueryItem& item) const {
        auto key_less = [](const KeywordEntry& e, const Keyword& k) { return e.keyword < k; };
        auto less_key = [](const Keyword& k, const KeywordEntry& e) { return k < e.keyword; };
        const auto a = std::lower_bound(entries_.begin(), entries_.end(), Keyword{item.dim, item.lo}, key_less);
        const auto b = std::upper_bound(a, entries_.end(), Keyword{item.dim, item.hi}, less_key);
        return {std::size_t(a - entries_.begin()), std::size_t(b - entries_.begin())};
    }

    bool tiles_in_order() const {
        std::uint64_t at = 0;
        for (const auto& e : entries_)
            for (const auto& s : spans_of(e)) {
                if (s.begin != at) return false;
                at = s.end;
            }
        return at == list_.size();
    }

    // DimStats (index.hpp:153-174), computed on first use: per dim the largest
    // token and the most keywords of that dim any one object carries
    const DimStats* find_dim(DimId dim) const {
        if (!lazy_) return nullptr;
        std::call_once(lazy_->stats_once, [&] {
            std::vector<std::uint32_t> per_obj(n_, 0);
            std::vector<ObjectId> touched;
            for (std::size_t j = 0; j < entries_.size();) {
                DimStats st;
                st.dim = entries_[j].keyword.dim;
                for (; j < entries_.size() && entries_[j].keyword.dim == st.dim; ++j) {
                    st.max_token = std::max(st.max_token, entries_[j].keyword.token);
                    for (const auto& s : spans_of(entries_[j]))
                        for (const ObjectId id : ids(s)) {
                            if (per_obj[id]++ == 0) touched.push_back(id);
                            st.max_multiplicity = std::max(st.max_multiplicity, per_obj[id]);
                        }
                }
                for (const ObjectId id : touched) per_obj[id] = 0;
                touched.clear();
                lazy_->stats.push_back(st);
            }
        });
        const auto& v = lazy_->stats;
        const auto it = std::lower_bound(v.begin(), v.end(), dim, [](const DimStats& s, DimId d) { return s.dim < d; });
        return it != v.end() && it->dim == dim ? &*it : nullptr;
    }

    std::uint32_t n_ = 0;
    std::vector<KeywordEntry> entries_;
    std::vector<PostingsSpan> spans_;
    std::vector<ObjectId> list_;
    std::optional<std::uint32_t> split_;
    int device_ = 0;
    std::shared_ptr<Lazy> lazy_ = std::make_shared<Lazy>();
};

namespace detail {
// entries/spans of a CSR image cut at the split threshold (index.hpp:229-243)
inline InvertedIndex from_csr(std::uint32_t n, const std::vector<std::uint64_t>& keys,
                              const std::vector<std::uint64_t>& off, std::vector<ObjectId> post,
                              std::optional<std::uint32_t> split, int device) {
    std::vector<InvertedIndex::KeywordEntry> entries(keys.size());
    std::vector<PostingsSpan> spans;
    for (std::size_t j = 0; j < keys.size(); ++j) {
        auto& e = entries[j];
        e.keyword = Keyword{DimId(keys[j] >> 32), Token(keys[j] & 0xffffffffu)};
        e.first_span = std::uint32_t(spans.size());
        const std::uint64_t len = off[j + 1] - off[j];
        const std::uint64_t lim = split ? *split : len;
        for (std::uint64_t p = off[j]; p < off[j + 1]; p += lim) spans.push_back({p, std::min(off[j + 1], p + lim)});
        const std::size_t made = spans.size() - e.first_span;
        if (made > 0xffff) throw DataError("keyword has too many sub-lists (" + std::to_string(made) + ")");
        e.span_count = std::uint16_t(made);
    }
    return InvertedIndex(n, std::move(entries), std::move(spans), std::move(post), split, device);
}
}  // namespace detail

// build_index (index.hpp:190-250).  Ids are checked on the host with the
// reference's message; the (keyword, id) sort and run-length CSR run on the
// device (genie_index_build: CUB radix sort), and the CSR comes back to fill
// the host view.  Same entries, spans and list array as the reference build.
inline InvertedIndex build_index(std::span<const ObjectRecord> objects,
                                 std::optional<std::uint32_t> split_threshold = std::nullopt, int device = 0) {
    if (split_threshold && *split_threshold == 0) throw ContractError("split_threshold must be positive");
    const auto n = static_cast<std::uint32_t>(objects.size());
    std::vector<const ObjectRecord*> by_id(n, nullptr);
    for (const auto& o : objects) {
        if (o.id() >= n || by_id[o.id()])
            throw DataError("object ids must be dense 0.." + std::to_string(n ? n - 1 : 0) + ": bad id " +
                            std::to_string(o.id()));
        by_id[o.id()] = &o;
    }
    std::vector<std::uint64_t> obj_off(std::size_t(n) + 1, 0);
    for (std::uint32_t i = 0; i < n; ++i) obj_off[i + 1] = obj_off[i] + by_id[i]->keywords().size();
    std::vector<std::uint16_t> dims(obj_off[n]);
    std::vector<std::uint32_t> toks(obj_off[n]);
    for (std::uint32_t i = 0; i < n; ++i) {
        std::size_t at = obj_off[i];
        for (const auto& kw : by_id[i]->keywords()) {
            dims[at] = kw.dim;
            toks[at++] = kw.token;
        }
    }
    char err[512] = {};
    genie_index* h = nullptr;
    detail::check(genie_index_build(n, obj_off.data(), dims.data(), toks.data(), device, &h, err, sizeof(err)), err);
    std::shared_ptr<genie_index> dev_ix(h, genie_index_destroy);
    std::uint32_t nn = 0, off_unused = 0;
    std::uint64_t K = 0, P = 0;
    int dev = 0;
    genie_index_info(h, &nn, &K, &P, &off_unused, &dev);
    std::vector<std::uint64_t> keys(K), off(K + 1, 0);
    std::vector<ObjectId> post(P);
    detail::check(genie_index_export(h, keys.data(), off.data(), post.data(), err, sizeof(err)), err);
    InvertedIndex index = detail::from_csr(n, keys, off, std::move(post), split_threshold, device);
    index.adopt_device(std::move(dev_ix));  // the built device CSR serves the queries
    return index;
}

// ------------------------------------------------------------------ index_io
// MCIX files (index_io.hpp:27-154) through the C ABI: the same bytes as the
// reference's serialize_index, the same validation and DataError messages on
// load; a loaded index keeps the file's spans (so it re-serializes
// byte-identically) and, like the reference, no split threshold.

inline std::vector<std::uint8_t> serialize_index(const InvertedIndex& index) {
    char err[512] = {};
    const auto keys = index.packed_keys();
    std::vector<std::uint16_t> cnt(keys.size());
    std::vector<std::uint64_t> bounds;
    bounds.reserve(index.spans().size() * 2);
    for (std::size_t j = 0; j < keys.size(); ++j) {
        const auto& e = index.entries()[j];
        cnt[j] = e.span_count;
        for (const auto& s : index.spans_of(e)) bounds.insert(bounds.end(), {s.begin, s.end});
    }
    const auto& p = index.list_array();
    std::uint64_t size = 0;
    detail::check(genie_mcix_serialize_spans(index.num_objects(), keys.size(), keys.data(), cnt.data(), bounds.data(),
                                             p.size(), p.data(), nullptr, &size, err, sizeof(err)),
                  err);
    std::vector<std::uint8_t> out(size);
    detail::check(genie_mcix_serialize_spans(index.num_objects(), keys.size(), keys.data(), cnt.data(), bounds.data(),
                                             p.size(), p.data(), out.data(), &size, err, sizeof(err)),
                  err);
    return out;
}

inline InvertedIndex deserialize_index(const std::uint8_t* data, std::size_t size, int device = 0) {
    char err[512] = {};
    std::uint32_t n = 0;
    std::uint64_t K = 0, P = 0, S = 0;
    detail::check(genie_mcix_parse(data, size, &n, &K, &P, nullptr, nullptr, nullptr, err, sizeof(err)), err);
    std::vector<std::uint64_t> keys(K), off(K + 1);
    std::vector<ObjectId> post(P);
    detail::check(genie_mcix_parse(data, size, nullptr, nullptr, nullptr, keys.data(), off.data(), post.data(), err,
                                   sizeof(err)),
                  err);
    detail::check(genie_mcix_parse_spans(data, size, &S, nullptr, nullptr, err, sizeof(err)), err);
    std::vector<std::uint16_t> cnt(K);
    std::vector<std::uint64_t> bounds(2 * S);
    detail::check(genie_mcix_parse_spans(data, size, &S, cnt.data(), bounds.data(), err, sizeof(err)), err);
    std::vector<InvertedIndex::KeywordEntry> entries(K);
    std::vector<PostingsSpan> spans(S);
    for (std::uint64_t s = 0; s < S; ++s) spans[s] = {bounds[2 * s], bounds[2 * s + 1]};
    for (std::uint64_t j = 0, first = 0; j < K; first += cnt[j], ++j)
        entries[j] = {Keyword{DimId(keys[j] >> 32), Token(keys[j] & 0xffffffffu)}, std::uint32_t(first), cnt[j]};
    return InvertedIndex(n, std::move(entries), std::move(spans), std::move(post), std::nullopt, device);
}

inline void save_index(const InvertedIndex& index, const std::string& path) {
    const auto bytes = serialize_index(index);
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw DataError("cannot open " + path + " for writing");
    const bool ok = std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
    std::fclose(f);
    if (!ok) throw DataError("write failed: " + path);
}

inline std::vector<std::uint8_t> read_file_bytes(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw DataError("cannot open " + path);
    std::vector<std::uint8_t> bytes;
    std::uint8_t buf[1 << 16];
    for (std::size_t got; (got = std::fread(buf, 1, sizeof(buf), f)) > 0;) bytes.insert(bytes.end(), buf, buf + got);
    const bool bad = std::ferror(f) != 0;
    std::fclose(f);
    if (bad) throw DataError("read failed: " + path);
    return bytes;
}

inline InvertedIndex load_index(const std::string& path, int device = 0) {
    const auto bytes = read_file_bytes(path);
    return deserialize_index(bytes.data(), bytes.size(), device);
}

// FNV-1a over a byte image (index_io.hpp:182-189): ties encoder sidecars to
// index files
inline std::uint64_t fnv1a64(const std::uint8_t* data, std::size_t size) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (std::size_t i = 0; i < size; ++i) h = (h ^ data[i]) * 0x100000001b3ull;
    return h;
}

struct IndexPartition {
    std::uint32_t part_id = 0;
    ObjectId id_offset = 0;
    std::uint32_t size = 0;
    InvertedIndex index;
};

// partition_dataset (index.hpp:263-291): consecutive parts of part_capacity
// objects over local ids.  `devices` (optional) places part p on
// devices[p % devices.size()], so execute_partitioned spreads over GPUs.
inline std::vector<IndexPartition> partition_dataset(std::span<const ObjectRecord> objects,
                                                     std::uint32_t part_capacity,
                                                     std::optional<std::uint32_t> split = std::nullopt,
                                                     std::span<const int> devices = {}) {
    if (part_capacity == 0) throw ContractError("part_capacity must be >= 1");
    for (std::size_t i = 0; i < objects.size(); ++i)
        if (objects[i].id() != i) throw DataError("partitioning requires objects in dense id order");
    std::vector<IndexPartition> parts;
    for (std::size_t start = 0, pid = 0; start < objects.size(); start += part_capacity, ++pid) {
        const auto cnt = std::min<std::size_t>(part_capacity, objects.size() - start);
        std::vector<ObjectRecord> local;
        local.reserve(cnt);
        for (std::size_t i = 0; i < cnt; ++i) local.emplace_back(ObjectId(i), objects[start + i].keywords());
        const int dev = devices.empty() ? 0 : devices[pid % devices.size()];
        parts.push_back({std::uint32_t(pid), ObjectId(start), std::uint32_t(cnt), build_index(local, split, dev)});
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
    std::uint32_t span_chunk = 4096;     // ids per chunk (engine.hpp:40); the device warp unit is a quarter
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

namespace detail {
// A batch flattened into the C ABI's arrays (queries in request order).
struct FlatBatch {
    std::vector<std::uint32_t> qid, k, lo, hi;
    std::vector<std::uint64_t> off{0};
    std::vector<std::uint16_t> dim;
    std::uint32_t max_k = 1;
    explicit FlatBatch(std::span<const Query> queries) {
        for (const auto& q : queries) {
            qid.push_back(q.id);
            k.push_back(q.k);
            max_k = std::max(max_k, q.k);
            for (const auto& it : q.items) {
                dim.push_back(it.dim);
                lo.push_back(it.lo);
                hi.push_back(it.hi);
            }
            off.push_back(dim.size());
        }
    }
};

inline genie_config to_genie(const EngineConfig& config) {
    if (config.span_chunk == 0 || config.max_spans_per_task == 0)
        throw ContractError("span_chunk and max_spans_per_task must be positive");
    genie_config cfg = genie_config_default();
    cfg.selector = static_cast<std::uint32_t>(config.selector);
    cfg.span_chunk = config.span_chunk;
    cfg.max_spans_per_task = config.max_spans_per_task;
    return cfg;
}

// rows of the C ABI -> TopKResults, plus timings and memory accounting
inline BatchResult to_batch(const FlatBatch& f, std::uint32_t stride, const std::vector<genie_entry>& out,
                            const std::vector<std::uint32_t>& len, const std::vector<std::uint32_t>& thr,
                            const genie_stage_ns& t, const genie_batch_stats& st) {
    BatchResult batch;
    batch.results.resize(f.qid.size());
    for (std::size_t q = 0; q < f.qid.size(); ++q) {
        auto& r = batch.results[q];
        r.query_id = f.qid[q];
        r.threshold = thr[q];
        r.entries.reserve(len[q]);
        for (std::uint32_t e = 0; e < len[q]; ++e) r.entries.push_back({out[q * stride + e].id, out[q * stride + e].count});
    }
    batch.timings = {t.lookup_ns, t.match_ns, t.select_ns, t.merge_ns, t.total_ns};
    batch.memory = {st.counter_bytes, st.gate_bytes, st.table_bytes};
    return batch;
}
}  // namespace detail

// execute_batch (engine.hpp:184-304): lookup, counting, the Count Priority
// Queue and top-k selection on the index's GPU; results in request order.
inline BatchResult execute_batch(const InvertedIndex& index, std::span<const Query> queries,
                                 const EngineConfig& config = {}) {
    const genie_config cfg = detail::to_genie(config);
    if (queries.empty()) return {};
    const detail::FlatBatch f(queries);
    const auto Q = static_cast<std::uint32_t>(queries.size());
    const std::uint32_t stride = std::max<std::uint32_t>(1, std::min(f.max_k, std::max<std::uint32_t>(index.num_objects(), 1)));
    std::vector<genie_entry> out(std::size_t(Q) * stride);
    std::vector<std::uint32_t> len(Q), thr(Q);
    genie_stage_ns t{};
    genie_batch_stats st{};
    char err[1024] = {};
    detail::check(genie_query_batch(index.device(), &cfg, Q, f.qid.data(), f.k.data(), f.off.data(), f.dim.data(),
                                    f.lo.data(), f.hi.data(), stride, out.data(), len.data(), thr.data(), nullptr, &t,
                                    &st, err, sizeof(err)),
                  err);
    return detail::to_batch(f, stride, out, len, thr, t, st);
}

// execute_partitioned (engine.hpp:308-347).  The reference runs the parts one
// after another; here all parts run at once -- each on its own device / stream
// (partition_dataset's `devices`), one host thread -- and their top-k rows are
// merged on the first part's device (genie_group_*: NCCL all-gather across
// distinct GPUs, peer copies otherwise).  Same results, timings and
// per-part-maximum memory accounting as the reference.
inline BatchResult execute_partitioned(std::span<const IndexPartition> partitions, std::span<const Query> queries,
                                       const EngineConfig& config = {}) {
    std::uint64_t expected = 0;
    for (const auto& p : partitions) {
        if (p.id_offset != expected || p.index.num_objects() != p.size)
            throw ContractError("partitions must be disjoint and contiguous");
        expected += p.size;
    }
    const genie_config cfg = detail::to_genie(config);
    if (queries.empty()) return {};
    if (partitions.empty()) {  // nothing indexed: every merged list is empty (engine.hpp:158-177)
        BatchResult batch;
        for (const auto& q : queries) batch.results.push_back(TopKResult{q.id, {}, 0});
        return batch;
    }
    std::vector<genie_index*> handles;
    std::vector<std::uint32_t> offsets;
    for (const auto& p : partitions) {
        handles.push_back(p.index.device());
        offsets.push_back(p.id_offset);
    }
    char err[1024] = {};
    genie_group* g = nullptr;
    detail::check(genie_group_from_indexes(handles.data(), offsets.data(), std::uint32_t(handles.size()),
                                           GENIE_EXCHANGE_AUTO, &g, err, sizeof(err)),
                  err);
    std::unique_ptr<genie_group, void (*)(genie_group*)> guard(g, genie_group_destroy);
    const detail::FlatBatch f(queries);
    const auto Q = static_cast<std::uint32_t>(queries.size());
    const std::uint32_t stride = std::max<std::uint32_t>(1, std::min<std::uint64_t>(f.max_k, std::max<std::uint64_t>(expected, 1)));
    std::vector<genie_entry> out(std::size_t(Q) * stride);
    std::vector<std::uint32_t> len(Q), thr(Q);
    genie_stage_ns t{};
    genie_batch_stats st{};
    detail::check(genie_group_query_batch(g, &cfg, Q, f.qid.data(), f.k.data(), f.off.data(), f.dim.data(),
                                          f.lo.data(), f.hi.data(), stride, out.data(), len.data(), thr.data(), &t,
                                          &st, err, sizeof(err)),
                  err);
    return detail::to_batch(f, stride, out, len, thr, t, st);
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

    // f_function(point) (lsh.hpp:172-175)
    Token token(std::uint32_t function, std::span<const float> point) const {
        if (function >= cfg_.m) throw ContractError("hash function index out of range");
        check_dims(point);
        return encode_points(point)[function];
    }

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
