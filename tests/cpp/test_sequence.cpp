// The reference's sequence-search tests (test_sa.cpp:64-206, 258-286)
// restated against include/mcx/sa.hpp; SequenceSearcher retrieves on the GPU
// index and verifies with GPU edit distances, and must agree with the
// exhaustive CPU DP on every query (plus the reference's known answers).
#include <mcx/sa.hpp>

#include <cstdio>
#include <random>

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

static std::uint32_t dp(std::string_view a, std::string_view b) {
    std::vector<std::vector<std::uint32_t>> t(a.size() + 1, std::vector<std::uint32_t>(b.size() + 1));
    for (std::size_t i = 0; i <= a.size(); ++i) t[i][0] = std::uint32_t(i);
    for (std::size_t j = 0; j <= b.size(); ++j) t[0][j] = std::uint32_t(j);
    for (std::size_t i = 1; i <= a.size(); ++i)
        for (std::size_t j = 1; j <= b.size(); ++j)
            t[i][j] = std::min({t[i - 1][j] + 1, t[i][j - 1] + 1, t[i - 1][j - 1] + (a[i - 1] != b[j - 1] ? 1u : 0u)});
    return t[a.size()][b.size()];
}

static std::string rnd(std::mt19937& rng, std::size_t len, int alpha) {
    std::uniform_int_distribution<int> ch(0, alpha - 1);
    std::string s(len, 'a');
    for (auto& c : s) c = char('a' + ch(rng));
    return s;
}

static std::string mutate(std::string s, std::mt19937& rng, std::size_t edits, int alpha) {
    std::uniform_int_distribution<int> op(0, 2), ch(0, alpha - 1);
    for (std::size_t e = 0; e < edits && !s.empty(); ++e) {
        const std::size_t pos = rng() % s.size();
        switch (op(rng)) {
            case 0: s[pos] = char('a' + ch(rng)); break;
            case 1: s.erase(pos, 1); break;
            default: s.insert(pos, 1, char('a' + ch(rng))); break;
        }
    }
    return s;
}

int main() {
    try {
        // ordered grams on the worked sequence
        CHECK(decompose_sequence("aabaab", 3) ==
              (std::vector<OrderedNGram>{{"aab", 0}, {"aba", 0}, {"baa", 0}, {"aab", 1}}));
        CHECK(decompose_sequence("ab", 3).empty());
        CHECK(decompose_sequence("aaaa", 2) == (std::vector<OrderedNGram>{{"aa", 0}, {"aa", 1}, {"aa", 2}}));
        // shared grams, bounds, certificate
        CHECK(shared_gram_count("aabaab", "aabaab", 3) == 4);
        CHECK(shared_gram_count("aabaab", "abab", 3) == 1);
        CHECK(shared_gram_count("aaaa", "bbbb", 2) == 0);
        CHECK(count_lower_bound(40, 40, 3, 2) == 32);
        CHECK(count_lower_bound(10, 10, 3, 5) <= 0);
        CHECK(topk_certificate(5, 40, 3, 2) && !topk_certificate(32, 40, 3, 2) && !topk_certificate(33, 40, 3, 2));
        // edit distance classics and random pairs (host utilities)
        CHECK(edit_distance("kitten", "sitting") == 3 && edit_distance("", "abc") == 3);
        std::mt19937 rng(7);
        for (int t = 0; t < 300; ++t) {
            const auto a = rnd(rng, rng() % 40, 3), b = rnd(rng, rng() % 40, 3);
            const std::uint32_t e = dp(a, b), cap = rng() % 12;
            CHECK(edit_distance(a, b) == e);
            CHECK(edit_distance_bounded(a, b, cap) == (e <= cap ? e : cap + 1));
        }
        // the gram encoding realizes the min-count rule through match counts
        std::mt19937 r5(5);
        for (int t = 0; t < 200; ++t) {
            const auto s = rnd(r5, 3 + r5() % 25, 2), q = rnd(r5, 3 + r5() % 25, 2);
            const std::vector<std::string> corpus = {s, q};
            const auto codec = GramCodec::build(corpus, 3);
            const auto obj = codec.encode(s, 0);
            const auto query = codec.encode_query(q, 1);
            const auto want = shared_gram_count(s, q, 3);
            CHECK(query ? match_count_reference(*query, obj) == want : want == 0);
        }
        // verification known answers (host loop)
        {
            const std::vector<std::string> corpus = {"abcdef", "zzzzzz"};
            const std::vector<CandidateHit> hits = {{0, 4}};
            const auto o = verify_candidates("abcdxf", hits, 3, corpus, 1);
            CHECK(o.best_id == 0 && o.best_distance == 1 && o.candidates_used == 1);
            const std::vector<std::string> c2 = {"abcdefgh", "abcdefgx"};
            const std::vector<CandidateHit> h2 = {{0, 6}, {1, 5}};
            const auto o2 = verify_candidates("abcdefgh", h2, 3, c2, 2);
            CHECK(o2.best_id == 0 && o2.best_distance == 0 && o2.candidates_used == 1 && o2.threshold_at_stop > 6);
        }
        // certified searches match the exhaustive scan (GPU retrieval + GPU verification)
        std::mt19937 r19(19);
        std::vector<std::string> corpus;
        for (int i = 0; i < 400; ++i) corpus.push_back(rnd(r19, 20, 6));
        const SequenceSearcher searcher(corpus, 3);
        EngineConfig cfg;
        cfg.mode = ExecMode::sequential;
        int certified = 0, scans = 0;
        for (int t = 0; t < 60; ++t) {
            const auto q = mutate(corpus[r19() % corpus.size()], r19, 1 + r19() % 3, 6);
            const auto res = searcher.search_once(q, 16, cfg);
            std::uint32_t best = dp(q, corpus[0]);
            std::size_t best_id = 0;
            for (std::size_t i = 1; i < corpus.size(); ++i)
                if (const auto d = dp(q, corpus[i]); d < best) best = d, best_id = i;
            // the GPU-verified round equals the reference loop on host distances
            if (!res.answered_by_scan) {
                const auto host = verify_candidates(q, res.candidates, 3, corpus, 16);
                CHECK(host.best_id == res.outcome.best_id && host.best_distance == res.outcome.best_distance &&
                      host.certified == res.outcome.certified &&
                      host.candidates_used == res.outcome.candidates_used &&
                      host.threshold_at_stop == res.outcome.threshold_at_stop);
            }
            if (res.outcome.certified) {
                ++certified;
                CHECK(res.outcome.best_distance == best);
            }
            const std::vector<std::uint32_t> sched{16, 64};
            const auto sure = searcher.search_certified(q, sched, cfg);
            CHECK(sure.outcome.certified && sure.outcome.best_distance == best);
            if (sure.answered_by_scan) {
                ++scans;
                CHECK(sure.outcome.best_id == best_id && sure.outcome.candidates_used == corpus.size());
            }
        }
        CHECK(certified > 0);
        // a query sharing no gram goes to the scan
        const auto none = searcher.search_once("!!!!!!!!", 16, cfg);
        CHECK(none.answered_by_scan && none.outcome.certified);
        std::printf("sequence: certified %d / 60, scans %d\n", certified, scans);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "unexpected exception: %s\n", e.what());
        return 2;
    }
    std::printf("sequence: %d checks, %d failures\n", checks, failures);
    if (failures) return 1;
    std::printf("sequence: ok\n");
    return 0;
}
