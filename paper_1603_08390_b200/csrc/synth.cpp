// Seeded synthetic workloads (SURVEY.md 8d shapes) + host CSR construction.
// Input preparation only; see include/genie/genie_synth.h.
#include "genie/genie_synth.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// SplitMix64 with the reference's uniform / normal conventions (rng.hpp).
struct Rng {
    uint64_t s;
    double spare = 0.0;
    bool has = false;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        s += 0x9e3779b97f4a7c15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double normal() {
        if (has) {
            has = false;
            return spare;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare = r * std::sin(th);
        has = true;
        return r * std::cos(th);
    }
};

// Per-object stream: generation parallelises over objects.
Rng stream_for(uint64_t seed, uint64_t i) { return Rng(mix64(seed) ^ mix64(0x5eed0000ull + i)); }

unsigned nthreads() { return std::max(1u, std::min(32u, std::thread::hardware_concurrency())); }

template <typename Fn>
void parallel_for(uint64_t n, Fn&& fn) {
    const unsigned T = nthreads();
    if (n < 4096 || T == 1) {
        fn(0, n, 0u);
        return;
    }
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t) {
        const uint64_t a = n * t / T, b = n * (t + 1) / T;
        pool.emplace_back([&, a, b, t] { fn(a, b, t); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

struct genie_dataset {
    // CSR
    uint32_t n = 0;
    std::vector<uint64_t> keys, key_off{0};
    std::vector<uint32_t> postings;
    // queries
    std::vector<uint32_t> qid, k;
    std::vector<uint64_t> item_off{0};
    std::vector<uint16_t> dim;
    std::vector<uint32_t> lo, hi;
    // points
    uint32_t pn = 0, dims = 0, pq = 0;
    std::vector<float> points, qpoints;
    std::vector<uint32_t> labels, qlabels;
    // sets
    uint32_t sn = 0, sq = 0;
    std::vector<uint64_t> set_off{0}, elems, qset_off{0}, qelems;
};

namespace {

// Stable counting sort of (packed keyword, id) by keyword over a dense
// keyword index: build_index (index.hpp:190-250) without splitting.  Objects
// are scanned in id order, so every list comes out ascending.
void build_csr(genie_dataset& ds, uint32_t n, const std::vector<uint64_t>& obj_off,
               const std::vector<uint64_t>& kw) {
    ds.n = n;
    const uint64_t total = kw.size();
    // dense index: per dim, tokens [0, max_token]
    std::vector<uint64_t> dim_max(65536, 0);
    std::vector<uint8_t> dim_used(65536, 0);
    for (uint64_t x : kw) {
        const uint32_t d = static_cast<uint32_t>(x >> 32);
        dim_used[d] = 1;
        dim_max[d] = std::max<uint64_t>(dim_max[d], x & 0xffffffffu);
    }
    std::vector<uint64_t> base(65537, 0);
    for (uint32_t d = 0; d < 65536; ++d) base[d + 1] = base[d] + (dim_used[d] ? dim_max[d] + 1 : 0);
    const uint64_t space = base[65536];
    if (space > std::max<uint64_t>(total * 8, 1ull << 22))
        throw std::runtime_error("keyword space too sparse for the dense CSR builder");
    auto slot = [&](uint64_t x) { return base[x >> 32] + (x & 0xffffffffu); };
    const unsigned T = nthreads();
    std::vector<std::vector<uint32_t>> cnt(T, std::vector<uint32_t>(space, 0));
    parallel_for(n, [&](uint64_t a, uint64_t b, unsigned t) {
        auto& c = cnt[t];
        for (uint64_t i = a; i < b; ++i)
            for (uint64_t j = obj_off[i]; j < obj_off[i + 1]; ++j) ++c[slot(kw[j])];
    });
    // thread-major offsets inside each keyword keep ids ascending
    std::vector<uint64_t> key_start(space + 1, 0);
    for (uint64_t s = 0; s < space; ++s) {
        uint64_t tot = 0;
        for (unsigned t = 0; t < T; ++t) tot += cnt[t][s];
        key_start[s + 1] = key_start[s] + tot;
    }
    std::vector<std::vector<uint64_t>> cursor(T);
    for (unsigned t = 0; t < T; ++t) cursor[t].resize(space);
    for (uint64_t s = 0; s < space; ++s) {
        uint64_t o = key_start[s];
        for (unsigned t = 0; t < T; ++t) {
            cursor[t][s] = o;
            o += cnt[t][s];
        }
    }
    cnt.clear();
    ds.postings.assign(total, 0);
    // the same partition of objects per thread as the count pass
    const bool serial = n < 4096 || T == 1;
    parallel_for(n, [&](uint64_t a, uint64_t b, unsigned t) {
        auto& cur = cursor[serial ? 0 : t];
        for (uint64_t i = a; i < b; ++i)
            for (uint64_t j = obj_off[i]; j < obj_off[i + 1]; ++j)
                ds.postings[cur[slot(kw[j])]++] = static_cast<uint32_t>(i);
    });
    ds.keys.clear();
    ds.key_off.assign(1, 0);
    for (uint32_t d = 0; d < 65536; ++d) {
        if (!dim_used[d]) continue;
        for (uint64_t t = 0; t <= dim_max[d]; ++t) {
            const uint64_t s = base[d] + t;
            if (key_start[s + 1] > key_start[s]) {
                ds.keys.push_back((uint64_t(d) << 32) | t);
                ds.key_off.push_back(key_start[s + 1]);
            }
        }
    }
}

void add_query(genie_dataset& ds, uint32_t id, uint32_t k) {
    ds.qid.push_back(id);
    ds.k.push_back(k);
    ds.item_off.push_back(ds.dim.size());
}

}  // namespace

extern "C" {

int genie_synth_adult(uint32_t n, uint32_t Q, uint32_t k, uint64_t seed, genie_dataset** out) {
    auto* ds = new genie_dataset;
    static const uint32_t cat_domain[8] = {9, 16, 7, 15, 6, 5, 2, 42};
    Rng rng(seed);
    std::vector<uint32_t> rows(size_t(n) * 14);
    for (uint32_t i = 0; i < n; ++i) {
        for (uint32_t a = 0; a < 6; ++a) {
            uint32_t v;
            if ((a == 3 || a == 4) && rng.uniform() < 0.9) {
                v = 0;  // capital gain / loss are mostly zero
            } else {
                const double x = std::min(1023.0, std::max(0.0, 512.0 + 150.0 * rng.normal()));
                v = static_cast<uint32_t>(x);
            }
            rows[size_t(i) * 14 + a] = v;
        }
        for (uint32_t a = 0; a < 8; ++a) {
            uint32_t c = 0;
            while (c + 1 < cat_domain[a] && rng.uniform() < 0.45) ++c;
            rows[size_t(i) * 14 + 6 + a] = c;
        }
    }
    std::vector<uint64_t> obj_off(n + 1), kw(size_t(n) * 14);
    for (uint32_t i = 0; i < n; ++i) {
        obj_off[i] = uint64_t(i) * 14;
        for (uint32_t a = 0; a < 14; ++a) kw[size_t(i) * 14 + a] = (uint64_t(a) << 32) | rows[size_t(i) * 14 + a];
    }
    obj_off[n] = uint64_t(n) * 14;
    build_csr(*ds, n, obj_off, kw);
    for (uint32_t q = 0; q < Q && n; ++q) {
        const uint32_t r = static_cast<uint32_t>(rng.next() % n);
        for (uint32_t a = 0; a < 14; ++a) {
            const uint32_t v = rows[size_t(r) * 14 + a];
            ds->dim.push_back(static_cast<uint16_t>(a));
            if (a < 6) {  // +-50 window clamped to the 1024-bin domain
                ds->lo.push_back(v >= 50 ? v - 50 : 0);
                ds->hi.push_back(std::min<uint32_t>(v + 50, 1023));
            } else {
                ds->lo.push_back(v);
                ds->hi.push_back(v);
            }
        }
        add_query(*ds, q, k);
    }
    *out = ds;
    return 0;
}

int genie_synth_tweets(uint32_t n, uint32_t vocab, uint32_t words, uint32_t Q, uint32_t k,
                       uint64_t seed, genie_dataset** out) {
    if (vocab == 0 || words == 0 || words > vocab) return 1;
    auto* ds = new genie_dataset;
    // Zipf(1) inverse CDF over ranks 0..vocab-1, with a guide table
    std::vector<double> cdf(vocab);
    double h = 0.0;
    for (uint32_t r = 0; r < vocab; ++r) {
        h += 1.0 / (r + 1.0);
        cdf[r] = h;
    }
    for (auto& c : cdf) c /= h;
    cdf[vocab - 1] = 1.0;
    const uint32_t G = 1u << 20;
    std::vector<uint32_t> guide(G + 1);
    {
        uint32_t r = 0;
        for (uint32_t j = 0; j <= G; ++j) {
            const double u = double(j) / G;
            while (r + 1 < vocab && cdf[r] < u) ++r;
            guide[j] = r;
        }
    }
    auto draw = [&](Rng& g) {
        const double u = g.uniform();
        uint32_t r = guide[static_cast<uint32_t>(u * G)];
        while (r + 1 < vocab && cdf[r] < u) ++r;
        return r;
    };
    auto make_doc = [&](uint64_t i, uint32_t* dst) {
        Rng g = stream_for(seed, i);
        for (uint32_t w = 0; w < words;) {
            const uint32_t r = draw(g);
            bool dup = false;
            for (uint32_t x = 0; x < w; ++x) dup |= dst[x] == r;
            if (!dup) dst[w++] = r;  // duplicate words are redrawn
        }
    };
    std::vector<uint32_t> docs(size_t(n) * words);
    parallel_for(n, [&](uint64_t a, uint64_t b, unsigned) {
        for (uint64_t i = a; i < b; ++i) make_doc(i, &docs[i * words]);
    });
    std::vector<uint64_t> obj_off(n + 1), kw(size_t(n) * words);
    for (uint64_t i = 0; i <= n; ++i) obj_off[i] = i * words;
    parallel_for(size_t(n) * words, [&](uint64_t a, uint64_t b, unsigned) {
        for (uint64_t i = a; i < b; ++i) kw[i] = docs[i];  // dim 0
    });
    docs.clear();
    docs.shrink_to_fit();
    build_csr(*ds, n, obj_off, kw);
    std::vector<uint32_t> qd(words);
    for (uint32_t q = 0; q < Q; ++q) {
        make_doc(uint64_t(n) + q, qd.data());
        for (uint32_t w = 0; w < words; ++w) {
            ds->dim.push_back(0);
            ds->lo.push_back(qd[w]);
            ds->hi.push_back(qd[w]);
        }
        add_query(*ds, q, k);
    }
    *out = ds;
    return 0;
}

int genie_synth_sift(uint32_t n, uint32_t dims, uint32_t Q, uint64_t seed, genie_dataset** out) {
    auto* ds = new genie_dataset;
    const uint32_t C = 64;
    Rng rng(seed);
    std::vector<double> centre(size_t(C) * dims);
    for (auto& c : centre) c = 3.12 * rng.normal();
    ds->pn = n;
    ds->dims = dims;
    ds->pq = Q;
    ds->points.resize(size_t(n) * dims);
    ds->qpoints.resize(size_t(Q) * dims);
    auto gen = [&](uint64_t i, float* dst) {
        Rng g = stream_for(seed, i);
        const uint64_t c = g.next() % C;
        for (uint32_t j = 0; j < dims; ++j)
            dst[j] = static_cast<float>(centre[c * dims + j] + 2.34 * g.normal());
    };
    parallel_for(n, [&](uint64_t a, uint64_t b, unsigned) {
        for (uint64_t i = a; i < b; ++i) gen(i, &ds->points[i * dims]);
    });
    for (uint32_t q = 0; q < Q; ++q) gen(uint64_t(n) + q, &ds->qpoints[size_t(q) * dims]);
    *out = ds;
    return 0;
}

int genie_synth_ocr(uint32_t n, uint32_t dims, uint32_t Q, uint64_t seed, genie_dataset** out) {
    auto* ds = new genie_dataset;
    const uint32_t C = 10;
    Rng rng(seed);
    std::vector<double> centre(size_t(C) * dims);
    for (auto& c : centre) c = rng.uniform();
    ds->pn = n;
    ds->dims = dims;
    ds->pq = Q;
    ds->points.resize(size_t(n) * dims);
    ds->qpoints.resize(size_t(Q) * dims);
    ds->labels.resize(n);
    ds->qlabels.resize(Q);
    auto gen = [&](uint64_t i, float* dst, uint32_t* label) {
        Rng g = stream_for(seed, i);
        const uint32_t c = static_cast<uint32_t>(g.next() % C);
        *label = c;
        for (uint32_t j = 0; j < dims; ++j) {
            const double x = centre[size_t(c) * dims + j] + 0.25 * g.normal();
            dst[j] = static_cast<float>(std::min(1.0, std::max(0.0, x)));
        }
    };
    parallel_for(n, [&](uint64_t a, uint64_t b, unsigned) {
        for (uint64_t i = a; i < b; ++i) gen(i, &ds->points[i * dims], &ds->labels[i]);
    });
    for (uint32_t q = 0; q < Q; ++q) gen(uint64_t(n) + q, &ds->qpoints[size_t(q) * dims], &ds->qlabels[q]);
    *out = ds;
    return 0;
}

int genie_synth_sets(uint32_t n, uint32_t Q, uint64_t seed, genie_dataset** out) {
    auto* ds = new genie_dataset;
    ds->sn = n;
    ds->sq = Q;
    // decisions first (cheap, sequential): size, duplicate source, mutation rate
    std::vector<uint32_t> size(n), src(n);
    std::vector<double> frac(n, 0.0);
    for (uint32_t i = 0; i < n; ++i) {
        Rng g = stream_for(seed, i);
        size[i] = 32 + static_cast<uint32_t>(g.next() % 225);
        src[i] = i;
        if (i > 0 && g.uniform() < 0.2) {
            uint32_t j = static_cast<uint32_t>(g.next() % i);
            src[i] = src[j];  // root of the duplicate chain (always a base set)
            frac[i] = 0.1 + 0.2 * g.uniform();
            size[i] = size[src[i]];
        }
    }
    ds->set_off.resize(size_t(n) + 1);
    ds->set_off[0] = 0;
    for (uint32_t i = 0; i < n; ++i) ds->set_off[i + 1] = ds->set_off[i] + size[i];
    ds->elems.resize(ds->set_off[n]);
    // base sets
    parallel_for(n, [&](uint64_t a, uint64_t b, unsigned) {
        for (uint64_t i = a; i < b; ++i) {
            if (src[i] != i) continue;
            Rng g = stream_for(seed ^ 0xe1e5ull, i);
            for (uint64_t j = ds->set_off[i]; j < ds->set_off[i + 1]; ++j) ds->elems[j] = g.next();
        }
    });
    // near-duplicates: copy the root, replace a fraction with fresh draws
    parallel_for(n, [&](uint64_t a, uint64_t b, unsigned) {
        for (uint64_t i = a; i < b; ++i) {
            if (src[i] == i) continue;
            Rng g = stream_for(seed ^ 0xd0bull, i);
            const uint64_t s0 = ds->set_off[src[i]], d0 = ds->set_off[i];
            for (uint32_t j = 0; j < size[i]; ++j)
                ds->elems[d0 + j] = g.uniform() < frac[i] ? g.next() : ds->elems[s0 + j];
        }
    });
    // queries: copies of indexed sets with 10% replaced
    Rng rq(mix64(seed) ^ 0x9ull);
    ds->qset_off.assign(1, 0);
    for (uint32_t q = 0; q < Q && n; ++q) {
        const uint32_t s = static_cast<uint32_t>(rq.next() % n);
        for (uint64_t j = ds->set_off[s]; j < ds->set_off[s + 1]; ++j)
            ds->qelems.push_back(rq.uniform() < 0.1 ? rq.next() : ds->elems[j]);
        ds->qset_off.push_back(ds->qelems.size());
    }
    *out = ds;
    return 0;
}

int genie_synth_random(uint32_t n, uint32_t dims, uint32_t tokens, uint32_t max_kw, uint32_t Q,
                       uint32_t max_items, uint32_t max_span, uint32_t max_k, uint64_t seed,
                       genie_dataset** out) {
    if (!dims || !tokens || !max_items || !max_k) return 1;
    auto* ds = new genie_dataset;
    Rng g(seed);
    std::vector<uint64_t> obj_off(1, 0), kw;
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t cnt = max_kw ? static_cast<uint32_t>(g.next() % (max_kw + 1)) : 0;
        const size_t start = kw.size();
        for (uint32_t t = 0; t < cnt; ++t) {
            const uint64_t x = (uint64_t(g.next() % dims) << 32) | (g.next() % tokens);
            if (std::find(kw.begin() + start, kw.end(), x) == kw.end()) kw.push_back(x);
        }
        obj_off.push_back(kw.size());
    }
    build_csr(*ds, n, obj_off, kw);
    for (uint32_t q = 0; q < Q; ++q) {
        const uint32_t items = 1 + static_cast<uint32_t>(g.next() % max_items);
        for (uint32_t i = 0; i < items; ++i) {
            const uint32_t lo = static_cast<uint32_t>(g.next() % tokens);
            const uint32_t span = max_span ? static_cast<uint32_t>(g.next() % (max_span + 1)) : 0;
            ds->dim.push_back(static_cast<uint16_t>(g.next() % dims));
            ds->lo.push_back(lo);
            ds->hi.push_back(lo + span);
        }
        add_query(*ds, q, 1 + static_cast<uint32_t>(g.next() % max_k));
    }
    *out = ds;
    return 0;
}

void genie_dataset_free(genie_dataset* ds) { delete ds; }

void genie_dataset_csr(const genie_dataset* ds, uint32_t* n, uint64_t* K, const uint64_t** keys,
                       const uint64_t** key_off, const uint32_t** postings) {
    *n = ds->n;
    *K = ds->keys.size();
    *keys = ds->keys.data();
    *key_off = ds->key_off.data();
    *postings = ds->postings.data();
}

void genie_dataset_queries(const genie_dataset* ds, uint32_t* Q, const uint32_t** qid,
                           const uint32_t** k, const uint64_t** item_off, const uint16_t** dim,
                           const uint32_t** lo, const uint32_t** hi) {
    *Q = static_cast<uint32_t>(ds->qid.size());
    *qid = ds->qid.data();
    *k = ds->k.data();
    *item_off = ds->item_off.data();
    *dim = ds->dim.data();
    *lo = ds->lo.data();
    *hi = ds->hi.data();
}

void genie_dataset_points(const genie_dataset* ds, uint32_t* n, uint32_t* dims, const float** pts,
                          uint32_t* Q, const float** qpts, const uint32_t** labels,
                          const uint32_t** qlabels) {
    *n = ds->pn;
    *dims = ds->dims;
    *pts = ds->points.data();
    *Q = ds->pq;
    *qpts = ds->qpoints.data();
    *labels = ds->labels.data();
    *qlabels = ds->qlabels.data();
}

void genie_dataset_sets(const genie_dataset* ds, uint32_t* n, const uint64_t** set_off,
                        const uint64_t** elems, uint32_t* Q, const uint64_t** qoff,
                        const uint64_t** qelems) {
    *n = ds->sn;
    *set_off = ds->set_off.data();
    *elems = ds->elems.data();
    *Q = ds->sq;
    *qoff = ds->qset_off.data();
    *qelems = ds->qelems.data();
}

int genie_synth_csr_from_objects(uint32_t n, const uint64_t* obj_off, const uint16_t* dims,
                                 const uint32_t* tokens, genie_dataset** out, char* err,
                                 size_t errlen) {
    try {
        auto* ds = new genie_dataset;
        std::vector<uint64_t> off(obj_off, obj_off + n + 1), kw(obj_off[n] - obj_off[0]);
        for (auto& o : off) o -= obj_off[0];
        for (uint64_t j = 0; j < kw.size(); ++j)
            kw[j] = (uint64_t(dims[obj_off[0] + j]) << 32) | tokens[obj_off[0] + j];
        for (uint32_t i = 0; i < n; ++i) {
            std::vector<uint64_t> s(kw.begin() + off[i], kw.begin() + off[i + 1]);
            std::sort(s.begin(), s.end());
            if (std::adjacent_find(s.begin(), s.end()) != s.end()) {
                delete ds;
                const std::string m = "ObjectRecord " + std::to_string(i) + ": duplicate keyword";
                if (err && errlen) {
                    std::strncpy(err, m.c_str(), errlen - 1);
                    err[errlen - 1] = 0;
                }
                return 1;
            }
        }
        build_csr(*ds, n, off, kw);
        *out = ds;
        return 0;
    } catch (const std::exception& e) {
        if (err && errlen) {
            std::strncpy(err, e.what(), errlen - 1);
            err[errlen - 1] = 0;
        }
        return 2;
    }
}

}  // extern "C"
