// mcx/sa.hpp -- sequence search for the drop-in (reference:
// /root/reference/proj/include/mcx/sa.hpp): ordered n-grams, the gram codec
// that turns sequences into match-count objects, candidate verification and
// SequenceSearcher (index-backed 1-NN under edit distance).
//
// Retrieval runs on the GPU through execute_batch; verification runs on the
// GPU too: the corpus is uploaded once (genie_seqset) and one launch of the
// bit-parallel edit-distance kernel scores every candidate of a round (or the
// whole corpus for the scan fallback); the reference's sequential
// verification loop (sa.hpp:298-336) is then replayed on those distances, so
// outcomes -- best id, distance, certificate, candidates used, final
// threshold -- are the reference's.  The free functions edit_distance /
// edit_distance_bounded / shared_gram_count are the reference's host
// utilities, kept for API parity.
#pragma once

#include <map>
#include <string>
#include <string_view>
#include <unordered_map>

#include "mcx/mcx.hpp"

namespace mcx {

struct OrderedNGram {
    std::string gram;
    std::uint32_t occurrence = 0;
    friend bool operator==(const OrderedNGram&, const OrderedNGram&) = default;
};

// sa.hpp:48-60: sliding windows, the i-th copy of a gram numbered i
inline std::vector<OrderedNGram> decompose_sequence(std::string_view text, std::uint32_t n) {
    if (n == 0) throw ContractError("gram length must be >= 1");
    std::vector<OrderedNGram> out;
    if (text.size() < n) return out;
    std::unordered_map<std::string_view, std::uint32_t> seen;
    for (std::size_t i = 0; i + n <= text.size(); ++i) {
        const auto w = text.substr(i, n);
        out.push_back({std::string(w), seen[w]++});
    }
    return out;
}

// sa.hpp:64-91: sum over grams of min(count in s, count in q)
inline std::uint64_t shared_gram_count(std::string_view s, std::string_view q, std::uint32_t n) {
    if (n == 0) throw ContractError("gram length must be >= 1");
    std::unordered_map<std::string_view, std::int64_t> cnt;
    for (std::size_t i = 0; i + n <= s.size(); ++i) ++cnt[s.substr(i, n)];
    std::uint64_t shared = 0;
    for (std::size_t i = 0; i + n <= q.size(); ++i) {
        auto it = cnt.find(q.substr(i, n));
        if (it != cnt.end() && it->second > 0) {
            --it->second;
            ++shared;
        }
    }
    return shared;
}

// sa.hpp:96-101
inline std::int64_t count_lower_bound(std::int64_t qlen, std::int64_t slen, std::int64_t n, std::int64_t tau) {
    if (n < 1) throw ContractError("gram length must be >= 1");
    return std::max(qlen, slen) - n + 1 - tau * n;
}

// sa.hpp:109-123 (host utility): unit-cost Levenshtein distance
inline std::uint32_t edit_distance(std::string_view a, std::string_view b) {
    if (a.size() < b.size()) std::swap(a, b);
    std::vector<std::uint32_t> row(b.size() + 1);
    for (std::size_t j = 0; j <= b.size(); ++j) row[j] = std::uint32_t(j);
    for (std::size_t i = 1; i <= a.size(); ++i) {
        std::uint32_t diag = row[0];
        row[0] = std::uint32_t(i);
        for (std::size_t j = 1; j <= b.size(); ++j) {
            const std::uint32_t up = row[j];
            row[j] = std::min({up + 1, row[j - 1] + 1, diag + (a[i - 1] != b[j - 1] ? 1u : 0u)});
            diag = up;
        }
    }
    return row[b.size()];
}

// sa.hpp:127-162 (host utility): exact when <= cap, else cap + 1
inline std::uint32_t edit_distance_bounded(std::string_view a, std::string_view b, std::uint32_t cap) {
    const std::size_t d = a.size() > b.size() ? a.size() - b.size() : b.size() - a.size();
    if (d > cap) return cap + 1;
    return std::min(edit_distance(a, b), cap + 1);
}

namespace detail {
// sa.hpp:168-177: a gram's dim is a 16-bit bucket of FNV-1a + mix64
inline DimId gram_dim(std::string_view gram) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (const unsigned char ch : gram) h = (h ^ ch) * 0x100000001b3ull;
    return static_cast<DimId>(mix64(h) & 0xffffu);
}
}  // namespace detail

// sa.hpp:185-282: keyword (dim = gram bucket, token = ordinal << 16 |
// occurrence) per ordered gram; ordinals fixed by the corpus vocabulary
class GramCodec {
public:
    static GramCodec build(std::span<const std::string> corpus, std::uint32_t n) {
        if (n == 0) throw ContractError("gram length must be >= 1");
        GramCodec c;
        c.n_ = n;
        for (const auto& text : corpus)
            for (std::size_t i = 0; i + n <= text.size(); ++i) {
                const std::string_view w = std::string_view(text).substr(i, n);
                c.vocab_.emplace(std::make_pair(detail::gram_dim(w), std::string(w)), 0);
            }
        // ordinals run per dim in (dim, gram) order
        DimId dim = 0;
        Token next = 0;
        bool first = true;
        for (auto& [key, ord] : c.vocab_) {
            if (first || key.first != dim) {
                dim = key.first;
                next = 0;
                first = false;
            }
            if (next > 0xffffu) throw DataError("more than 65536 distinct grams share one dim bucket");
            ord = next++;
        }
        return c;
    }
    std::uint32_t n() const noexcept { return n_; }

    ObjectRecord encode(std::string_view text, ObjectId id) const {
        std::vector<Keyword> kws;
        each_gram(text, [&](std::string_view g, std::uint32_t occ) {
            const auto kw = keyword_for(g, occ);
            if (!kw) throw ContractError("sequence contains a gram outside the vocabulary");
            kws.push_back(*kw);
        });
        return ObjectRecord(id, std::move(kws));
    }
    std::optional<Query> encode_query(std::string_view text, std::uint32_t k, std::uint32_t query_id = 0) const {
        std::vector<QueryItem> items;
        each_gram(text, [&](std::string_view g, std::uint32_t occ) {
            if (const auto kw = keyword_for(g, occ)) items.push_back(QueryItem::point(kw->dim, kw->token));
        });
        if (items.empty()) return std::nullopt;
        return Query(query_id, std::move(items), k);
    }
    std::optional<Keyword> keyword_for(std::string_view gram, std::uint32_t occurrence) const {
        if (occurrence > 0xffffu) throw DataError("gram occurrence index exceeds 16 bits");
        const DimId dim = detail::gram_dim(gram);
        const auto it = vocab_.find(std::make_pair(dim, std::string(gram)));
        if (it == vocab_.end()) return std::nullopt;
        return Keyword{dim, (it->second << 16) | occurrence};
    }

private:
    template <class Fn>
    void each_gram(std::string_view text, Fn&& fn) const {
        if (text.size() < n_) return;
        std::unordered_map<std::string_view, std::uint32_t> seen;
        for (std::size_t i = 0; i + n_ <= text.size(); ++i) {
            const auto w = text.substr(i, n_);
            fn(w, seen[w]++);
        }
    }
    std::uint32_t n_ = 0;
    std::map<std::pair<DimId, std::string>, Token> vocab_;
};

struct CandidateHit {
    ObjectId id = 0;
    std::uint32_t count = 0;
};

struct VerificationOutcome {
    ObjectId best_id = 0;
    std::uint32_t best_distance = 0;
    bool certified = false;
    std::uint32_t candidates_used = 0;
    std::int64_t threshold_at_stop = 0;
};

// sa.hpp:304-307: no unreturned sequence can beat the best (strict)
inline bool topk_certificate(std::int64_t c_k, std::int64_t qlen, std::int64_t n, std::int64_t tau_kprime) {
    return c_k < qlen - n + 1 - tau_kprime * n;
}

namespace detail {
// The verification loop of sa.hpp:317-336 over a distance oracle:
// dist(i, cap) = the candidate's edit_distance_bounded (cap = UINT32_MAX for
// the first candidate's exact distance).
template <class Dist>
VerificationOutcome verify_loop(std::string_view query, std::span<const CandidateHit> cand, std::uint32_t n,
                                std::size_t requested_k, bool early_break, Dist&& dist,
                                std::span<const std::size_t> lengths) {
    if (cand.empty()) throw ContractError("verify_candidates: empty candidate list");
    if (requested_k == 0) requested_k = cand.size();
    const std::int64_t qlen = std::int64_t(query.size());
    VerificationOutcome out;
    out.best_id = cand[0].id;
    out.best_distance = dist(0, 0xffffffffu);
    out.candidates_used = 1;
    auto theta_of = [&](std::uint32_t d) { return qlen - std::int64_t(n) + 1 - std::int64_t(n) * (std::int64_t(d) - 1); };
    std::int64_t theta = theta_of(out.best_distance);
    for (std::size_t j = 1; j < cand.size(); ++j) {
        if (early_break && theta > std::int64_t(cand[j].count)) break;
        ++out.candidates_used;
        const std::int64_t ld = std::abs(std::int64_t(lengths[j]) - qlen);
        if (ld > std::int64_t(out.best_distance) || out.best_distance == 0) continue;
        const std::uint32_t d = dist(j, out.best_distance - 1);
        if (d < out.best_distance) {
            out.best_distance = d;
            out.best_id = cand[j].id;
            theta = theta_of(d);
        }
    }
    const std::int64_t c_k = cand.size() >= requested_k ? std::int64_t(cand.back().count) : 0;
    out.certified = topk_certificate(c_k, qlen, n, out.best_distance);
    out.threshold_at_stop = theta;
    return out;
}
}  // namespace detail

// verify_candidates (sa.hpp:298-336) over a host corpus (host utility; the
// searcher below verifies on the GPU)
inline VerificationOutcome verify_candidates(std::string_view query, std::span<const CandidateHit> candidates,
                                             std::uint32_t n, std::span<const std::string> corpus,
                                             std::size_t requested_k = 0, bool early_break = true) {
    std::vector<std::size_t> lens;
    for (const auto& c : candidates) lens.push_back(corpus[c.id].size());
    return detail::verify_loop(
        query, candidates, n, requested_k, early_break,
        [&](std::size_t j, std::uint32_t cap) {
            const std::string& s = corpus[candidates[j].id];
            return cap == 0xffffffffu ? edit_distance(query, s) : edit_distance_bounded(query, s, cap);
        },
        lens);
}

inline constexpr std::uint32_t kDefaultCandidateSchedule[] = {32, 64, 128, 256};

// SequenceSearcher (sa.hpp:419-512): retrieve the K highest-count candidates
// through the GPU index, verify them with GPU edit distances, escalate K, and
// fall back to a GPU scan of the whole corpus.
class SequenceSearcher {
public:
    SequenceSearcher(std::vector<std::string> corpus, std::uint32_t n,
                     std::optional<std::uint32_t> split_threshold = std::nullopt, int device = 0)
        : corpus_(std::move(corpus)), n_(n), codec_(GramCodec::build(corpus_, n)) {
        std::vector<ObjectRecord> records;
        records.reserve(corpus_.size());
        for (std::size_t i = 0; i < corpus_.size(); ++i) records.push_back(codec_.encode(corpus_[i], ObjectId(i)));
        index_ = build_index(records, split_threshold, device);
        std::string blob;
        std::vector<std::uint64_t> off{0};
        for (const auto& s : corpus_) {
            blob += s;
            off.push_back(blob.size());
        }
        genie_seqset* h = nullptr;
        char err[512] = {};
        detail::check(genie_seqset_create(reinterpret_cast<const std::uint8_t*>(blob.data()), off.data(),
                                          corpus_.size(), device, &h, err, sizeof(err)),
                      err);
        seqs_ = std::shared_ptr<genie_seqset>(h, genie_seqset_destroy);
    }

    struct SearchResult {
        VerificationOutcome outcome;
        std::vector<CandidateHit> candidates;
        bool answered_by_scan = false;
    };

    const InvertedIndex& index() const noexcept { return index_; }
    const GramCodec& codec() const noexcept { return codec_; }
    std::span<const std::string> corpus() const noexcept { return corpus_; }

    std::vector<CandidateHit> retrieve(std::string_view query_text, std::uint32_t big_k,
                                       const EngineConfig& config = {}) const {
        const auto q = codec_.encode_query(query_text, big_k);
        if (!q) return {};
        const BatchResult b = execute_batch(index_, std::span<const Query>(&*q, 1), config);
        std::vector<CandidateHit> hits;
        for (const auto& e : b.results[0].entries) hits.push_back({e.id, e.count});
        return hits;
    }

    SearchResult search_once(std::string_view query_text, std::uint32_t big_k = 32, const EngineConfig& config = {}) const {
        if (corpus_.empty()) throw ContractError("empty corpus");
        SearchResult r;
        r.candidates = retrieve(query_text, big_k, config);
        if (r.candidates.empty()) {  // nothing shares a gram: only a scan can answer
            r.outcome = scan(query_text);
            r.answered_by_scan = true;
            return r;
        }
        // every candidate's exact distance in one launch, then the reference loop
        std::vector<std::uint32_t> ids;
        std::vector<std::size_t> lens;
        for (const auto& c : r.candidates) {
            ids.push_back(c.id);
            lens.push_back(corpus_[c.id].size());
        }
        const auto d = distances(query_text, ids.data(), ids.size(), 0xffffffffu);
        r.outcome = detail::verify_loop(
            query_text, r.candidates, n_, big_k, true,
            [&](std::size_t j, std::uint32_t cap) { return cap == 0xffffffffu ? d[j] : std::min(d[j], cap + 1); },
            lens);
        return r;
    }

    SearchResult search_certified(std::string_view query_text,
                                  std::span<const std::uint32_t> schedule = kDefaultCandidateSchedule,
                                  const EngineConfig& config = {}) const {
        SearchResult last;
        for (const std::uint32_t k : schedule) {
            last = search_once(query_text, k, config);
            if (last.outcome.certified) return last;
        }
        last.outcome = scan(query_text);
        last.answered_by_scan = true;
        return last;
    }

private:
    std::vector<std::uint32_t> distances(std::string_view q, const std::uint32_t* ids, std::size_t count,
                                         std::uint32_t cap) const {
        std::vector<std::uint32_t> out(std::max<std::size_t>(count, 1));
        char err[512] = {};
        detail::check(genie_seqset_distances(seqs_.get(), reinterpret_cast<const std::uint8_t*>(q.data()), q.size(),
                                             ids, count, cap, out.data(), err, sizeof(err)),
                      err);
        out.resize(count);
        return out;
    }

    // sa.hpp:491-505: the first sequence at the smallest distance
    VerificationOutcome scan(std::string_view q) const {
        const auto d = distances(q, nullptr, corpus_.size(), 0xffffffffu);
        VerificationOutcome out;
        out.best_id = ObjectId(std::min_element(d.begin(), d.end()) - d.begin());
        out.best_distance = d[out.best_id];
        out.certified = true;
        out.candidates_used = std::uint32_t(corpus_.size());
        out.threshold_at_stop = 0;
        return out;
    }

    std::vector<std::string> corpus_;
    std::uint32_t n_;
    GramCodec codec_;
    InvertedIndex index_;
    std::shared_ptr<genie_seqset> seqs_;
};

}  // namespace mcx
