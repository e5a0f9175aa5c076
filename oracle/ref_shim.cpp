// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// A C-ABI shim around the UNMODIFIED reference headers (mcx, header-only
// C++20, /root/reference/proj/include).  Built by oracle/Makefile into
// oracle/_ref/libmcx_ref.so; no reference source is copied into this repo,
// the headers are consumed through -I at compile time only.
//
// Consumers: tests/ (golden-vector generation and parity pinning),
// __graft_entry__.smoke() (checker), bench.py (`cpu_baseline` leg and
// `--impl reference`).  Every entry point calls the reference's own public
// API (mcx::build_index, mcx::execute_batch, mcx::execute_partitioned,
// mcx::merge_topk, mcx::hash_results, mcx::LshEncoder, ...).
#include <mcx/mcx.hpp>

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

namespace {

int fail(char* err, size_t errlen, int code, const char* what) {
    if (err && errlen) {
        std::strncpy(err, what, errlen - 1);
        err[errlen - 1] = 0;
    }
    return code;
}

// 1 contract, 2 data, 3 invariant, 9 other -- the same taxonomy as genie.h
template <typename Fn>
int guarded(char* err, size_t errlen, Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const mcx::ContractError& e) {
        return fail(err, errlen, 1, e.what());
    } catch (const mcx::DataError& e) {
        return fail(err, errlen, 2, e.what());
    } catch (const mcx::InvariantError& e) {
        return fail(err, errlen, 3, e.what());
    } catch (const std::exception& e) {
        return fail(err, errlen, 9, e.what());
    }
}

struct RefIndex {
    std::uint32_t n = 0;
    std::vector<mcx::ObjectRecord> objects;  // kept for partitioned runs
    mcx::InvertedIndex index;
};

std::vector<mcx::ObjectRecord> objects_from_csr(std::uint32_t n, std::uint64_t K,
                                                const std::uint64_t* keys,
                                                const std::uint64_t* key_off,
                                                const std::uint32_t* postings) {
    std::vector<std::vector<mcx::Keyword>> kws(n);
    for (std::uint64_t j = 0; j < K; ++j) {
        const mcx::Keyword kw{static_cast<mcx::DimId>(keys[j] >> 32),
                              static_cast<mcx::Token>(keys[j] & 0xffffffffu)};
        for (std::uint64_t p = key_off[j]; p < key_off[j + 1]; ++p) {
            if (postings[p] >= n) throw mcx::DataError("posting id out of range");
            kws[postings[p]].push_back(kw);
        }
    }
    std::vector<mcx::ObjectRecord> objects;
    objects.reserve(n);
    for (std::uint32_t i = 0; i < n; ++i) objects.emplace_back(i, std::move(kws[i]));
    return objects;
}

std::vector<mcx::Query> make_queries(std::uint32_t Q, const std::uint32_t* qid,
                                     const std::uint32_t* k, const std::uint64_t* item_off,
                                     const std::uint16_t* dim, const std::uint32_t* lo,
                                     const std::uint32_t* hi) {
    std::vector<mcx::Query> queries;
    queries.reserve(Q);
    for (std::uint32_t q = 0; q < Q; ++q) {
        std::vector<mcx::QueryItem> items;
        for (std::uint64_t i = item_off[q]; i < item_off[q + 1]; ++i) {
            items.emplace_back(dim[i], lo[i], hi[i]);
        }
        queries.emplace_back(qid[q], std::move(items), k[q]);
    }
    return queries;
}

void write_batch(const mcx::BatchResult& batch, std::uint32_t out_stride, std::uint32_t* out_ids,
                 std::uint32_t* out_counts, std::uint32_t* out_len, std::uint32_t* out_thr,
                 std::uint64_t* out_hash, std::uint64_t* timings5, std::uint64_t* mem3) {
    for (std::size_t q = 0; q < batch.results.size(); ++q) {
        const auto& r = batch.results[q];
        const std::size_t m = std::min<std::size_t>(r.entries.size(), out_stride);
        if (out_len) out_len[q] = static_cast<std::uint32_t>(r.entries.size());
        if (out_thr) out_thr[q] = r.threshold;
        for (std::size_t e = 0; e < m; ++e) {
            if (out_ids) out_ids[q * out_stride + e] = r.entries[e].id;
            if (out_counts) out_counts[q * out_stride + e] = r.entries[e].count;
        }
    }
    if (out_hash) *out_hash = mcx::hash_results(batch.results);
    if (timings5) {
        timings5[0] = batch.timings.lookup_ns;
        timings5[1] = batch.timings.match_ns;
        timings5[2] = batch.timings.select_ns;
        timings5[3] = batch.timings.merge_ns;
        timings5[4] = batch.timings.total_ns;
    }
    if (mem3) {
        mem3[0] = batch.memory.counter_bytes;
        mem3[1] = batch.memory.gate_bytes;
        mem3[2] = batch.memory.table_bytes;
    }
}

mcx::EngineConfig make_config(int selector, int mode, std::uint32_t workers,
                              std::uint32_t span_chunk, std::uint32_t spans_per_task) {
    mcx::EngineConfig c;
    c.selector = selector == 1 ? mcx::Selector::bucket
                 : selector == 2 ? mcx::Selector::sort
                                 : mcx::Selector::cpq;
    c.mode = mode == 1 ? mcx::ExecMode::sequential : mcx::ExecMode::parallel;
    c.workers = workers;
    c.span_chunk = span_chunk;
    c.max_spans_per_task = spans_per_task;
    return c;
}

}  // namespace

extern "C" {

unsigned mcxref_hardware_threads() { return std::thread::hardware_concurrency(); }

// CSR input: K keys (packed dim<<32|token, ascending), key_off[K+1], postings
// ascending per key.  split = 0 builds without long-list splitting.
int mcxref_index_from_csr(std::uint32_t n, std::uint64_t K, const std::uint64_t* keys,
                          const std::uint64_t* key_off, const std::uint32_t* postings,
                          std::uint32_t split, void** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto* ix = new RefIndex;
        ix->n = n;
        ix->objects = objects_from_csr(n, K, keys, key_off, postings);
        ix->index = split ? mcx::build_index(ix->objects, split) : mcx::build_index(ix->objects);
        *out = ix;
    });
}

// Object input: object i owns keywords [obj_off[i], obj_off[i+1]).
int mcxref_index_from_objects(std::uint32_t n, const std::uint64_t* obj_off,
                              const std::uint16_t* dims, const std::uint32_t* tokens,
                              std::uint32_t split, void** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto* ix = new RefIndex;
        ix->n = n;
        ix->objects.reserve(n);
        for (std::uint32_t i = 0; i < n; ++i) {
            std::vector<mcx::Keyword> kws;
            for (std::uint64_t j = obj_off[i]; j < obj_off[i + 1]; ++j) {
                kws.push_back(mcx::Keyword{dims[j], tokens[j]});
            }
            ix->objects.emplace_back(i, std::move(kws));
        }
        ix->index = split ? mcx::build_index(ix->objects, split) : mcx::build_index(ix->objects);
        *out = ix;
    });
}

void mcxref_index_free(void* p) { delete static_cast<RefIndex*>(p); }

// Exports the reference index image: sizes first (pass nulls), then arrays.
void mcxref_index_shape(void* p, std::uint64_t* K, std::uint64_t* P, std::uint64_t* S) {
    auto* ix = static_cast<RefIndex*>(p);
    *K = ix->index.entries().size();
    *P = ix->index.list_array().size();
    *S = ix->index.spans().size();
}

void mcxref_index_export(void* p, std::uint64_t* keys, std::uint32_t* first_span,
                         std::uint16_t* span_count, std::uint64_t* span_begin,
                         std::uint64_t* span_end, std::uint32_t* postings) {
    auto* ix = static_cast<RefIndex*>(p);
    const auto& e = ix->index.entries();
    for (std::size_t j = 0; j < e.size(); ++j) {
        keys[j] = e[j].keyword.packed();
        first_span[j] = e[j].first_span;
        span_count[j] = e[j].span_count;
    }
    const auto& s = ix->index.spans();
    for (std::size_t j = 0; j < s.size(); ++j) {
        span_begin[j] = s[j].begin;
        span_end[j] = s[j].end;
    }
    const auto& l = ix->index.list_array();
    std::memcpy(postings, l.data(), l.size() * sizeof(std::uint32_t));
}

// serialize_index (index_io.hpp:63-82): size query with out == nullptr.
int mcxref_index_serialize(void* p, std::uint8_t* out, std::uint64_t* size, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const auto img = mcx::serialize_index(static_cast<RefIndex*>(p)->index);
        if (out) {
            if (*size < img.size()) throw mcx::ContractError("serialize buffer too small");
            std::memcpy(out, img.data(), img.size());
        }
        *size = img.size();
    });
}

// deserialize_index (index_io.hpp:84-146) of an image: the status and message
// the reference produces for it (0 when it loads).
int mcxref_deserialize(const std::uint8_t* data, std::uint64_t size, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { (void)mcx::deserialize_index(data, size); });
}

std::uint32_t mcxref_max_multiplicity(void* p, std::uint16_t dim) {
    return static_cast<RefIndex*>(p)->index.max_multiplicity(dim);
}

int mcxref_max_count_bound(void* p, std::uint32_t n_items, const std::uint16_t* dim,
                           const std::uint32_t* lo, const std::uint32_t* hi,
                           std::uint64_t* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<mcx::QueryItem> items;
        for (std::uint32_t i = 0; i < n_items; ++i) items.emplace_back(dim[i], lo[i], hi[i]);
        const mcx::Query q(0, std::move(items), 1);
        *out = static_cast<RefIndex*>(p)->index.max_count_bound(q);
    });
}

// selector: 0 cpq, 1 bucket, 2 sort.  mode: 0 parallel, 1 sequential.
int mcxref_execute(void* p, std::uint32_t Q, const std::uint32_t* qid, const std::uint32_t* k,
                   const std::uint64_t* item_off, const std::uint16_t* dim,
                   const std::uint32_t* lo, const std::uint32_t* hi, int selector, int mode,
                   std::uint32_t workers, std::uint32_t span_chunk, std::uint32_t spans_per_task,
                   std::uint32_t out_stride, std::uint32_t* out_ids, std::uint32_t* out_counts,
                   std::uint32_t* out_len, std::uint32_t* out_thr, std::uint64_t* out_hash,
                   std::uint64_t* timings5, std::uint64_t* mem3, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto* ix = static_cast<RefIndex*>(p);
        const auto queries = make_queries(Q, qid, k, item_off, dim, lo, hi);
        const auto batch = mcx::execute_batch(
            ix->index, queries, make_config(selector, mode, workers, span_chunk, spans_per_task));
        write_batch(batch, out_stride, out_ids, out_counts, out_len, out_thr, out_hash, timings5,
                    mem3);
    });
}

int mcxref_execute_partitioned(void* p, std::uint32_t capacity, std::uint32_t Q,
                               const std::uint32_t* qid, const std::uint32_t* k,
                               const std::uint64_t* item_off, const std::uint16_t* dim,
                               const std::uint32_t* lo, const std::uint32_t* hi, int mode,
                               std::uint32_t out_stride, std::uint32_t* out_ids,
                               std::uint32_t* out_counts, std::uint32_t* out_len,
                               std::uint32_t* out_thr, std::uint64_t* out_hash, char* err,
                               size_t errlen) {
    return guarded(err, errlen, [&] {
        auto* ix = static_cast<RefIndex*>(p);
        const auto parts = mcx::partition_dataset(ix->objects, capacity);
        const auto queries = make_queries(Q, qid, k, item_off, dim, lo, hi);
        const auto batch =
            mcx::execute_partitioned(parts, queries, make_config(0, mode, 0, 4096, 2));
        write_batch(batch, out_stride, out_ids, out_counts, out_len, out_thr, out_hash, nullptr,
                    nullptr);
    });
}

// Lists: list l holds entries [off[l], off[l+1]) of (ids, counts).
int mcxref_merge_topk(std::uint32_t n_lists, const std::uint64_t* off, const std::uint32_t* ids,
                      const std::uint32_t* counts, std::uint32_t k, std::uint32_t query_id,
                      std::uint32_t out_cap, std::uint32_t* out_ids, std::uint32_t* out_counts,
                      std::uint32_t* out_len, std::uint32_t* out_thr, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<mcx::TopKResult> locals(n_lists);
        for (std::uint32_t l = 0; l < n_lists; ++l) {
            for (std::uint64_t e = off[l]; e < off[l + 1]; ++e) {
                locals[l].entries.push_back(mcx::TopKEntry{ids[e], counts[e]});
            }
        }
        const auto r = mcx::merge_topk(locals, k, query_id);
        *out_len = static_cast<std::uint32_t>(r.entries.size());
        *out_thr = r.threshold;
        for (std::size_t e = 0; e < r.entries.size() && e < out_cap; ++e) {
            out_ids[e] = r.entries[e].id;
            out_counts[e] = r.entries[e].count;
        }
    });
}

// c-PQ driven by an explicit update stream (reference CountPriorityQueue).
int mcxref_cpq_stream(std::uint32_t n, std::uint32_t max_count, std::uint32_t k,
                      std::uint64_t n_updates, const std::uint32_t* stream,
                      std::uint32_t out_cap, std::uint32_t* out_ids, std::uint32_t* out_counts,
                      std::uint32_t* out_len, std::uint32_t* out_thr, std::uint32_t* out_at,
                      char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        mcx::CountPriorityQueue pq(n, max_count, k);
        for (std::uint64_t i = 0; i < n_updates; ++i) pq.update(stream[i]);
        const auto r = pq.extract();
        *out_len = static_cast<std::uint32_t>(r.entries.size());
        *out_thr = r.threshold;
        *out_at = pq.audit_threshold();
        for (std::size_t e = 0; e < r.entries.size() && e < out_cap; ++e) {
            out_ids[e] = r.entries[e].id;
            out_counts[e] = r.entries[e].count;
        }
    });
}

std::uint64_t mcxref_mix64(std::uint64_t x) { return mcx::mix64(x); }

// family: 0 p-stable, 1 random binning.  tokens: n_points x m, row-major.
int mcxref_lsh_encode(int family, std::uint32_t m, std::uint32_t dims, std::uint64_t seed,
                      std::uint32_t rehash_domain, double w, std::uint32_t bucket_count,
                      std::int64_t bucket_min, int rehash_pstable, double sigma,
                      const float* points, std::uint64_t n_points, std::uint32_t n_threads,
                      std::uint32_t* tokens, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        mcx::LshEncoderConfig c;
        c.family = family == 0 ? mcx::LshFamily::p_stable : mcx::LshFamily::random_binning;
        c.m = m;
        c.dims = dims;
        c.seed = seed;
        c.rehash_domain = rehash_domain;
        c.w = w;
        c.bucket_count = bucket_count;
        c.bucket_min = bucket_min;
        c.rehash_pstable = rehash_pstable != 0;
        c.sigma = sigma;
        const auto enc = mcx::LshEncoder::create(c);
        const std::uint32_t T = std::max<std::uint32_t>(1, n_threads);
        std::vector<std::thread> pool;
        std::vector<std::exception_ptr> errs(T);
        for (std::uint32_t t = 0; t < T; ++t) {
            pool.emplace_back([&, t] {
                try {
                    for (std::uint64_t i = t; i < n_points; i += T) {
                        const std::span<const float> pt(points + i * dims, dims);
                        const auto obj = enc.encode_point(pt, static_cast<mcx::ObjectId>(i));
                        // one keyword per function, dim == function index
                        for (const auto& kw : obj.keywords()) tokens[i * m + kw.dim] = kw.token;
                    }
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        }
        for (auto& th : pool) th.join();
        for (auto& e : errs) {
            if (e) std::rethrow_exception(e);
        }
    });
}

// Parameter export via the reference's public samplers, seeded exactly as
// LshEncoder::create seeds them (lsh.hpp:156-164).  p-stable: a[m*dims], b[m],
// RBH: pitch[m*dims] -> a, shift[m*dims] -> b.  rehash_seed[m].
int mcxref_lsh_params(int family, std::uint32_t m, std::uint32_t dims, std::uint64_t seed,
                      double w, double sigma, double* a, double* b, std::uint64_t* rehash_seed,
                      char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        for (std::uint32_t i = 0; i < m; ++i) {
            mcx::SplitMix64 fn_rng(mcx::mix64(seed) ^ mcx::mix64(0x9e3779b9u + i));
            if (family == 0) {
                const auto h = mcx::sample_pstable(dims, w, fn_rng);
                for (std::uint32_t j = 0; j < dims; ++j) a[std::size_t(i) * dims + j] = h.a[j];
                b[i] = h.b;
            } else {
                const auto h = mcx::sample_rbh(sigma, dims, fn_rng);
                for (std::uint32_t j = 0; j < dims; ++j) {
                    a[std::size_t(i) * dims + j] = h.pitch[j];
                    b[std::size_t(i) * dims + j] = h.shift[j];
                }
            }
            rehash_seed[i] = fn_rng.next();
        }
    });
}

double mcxref_kernel_width(const float* points, std::uint64_t n, std::uint32_t dims,
                           std::uint64_t max_pairs) {
    std::vector<std::vector<float>> pts(n);
    for (std::uint64_t i = 0; i < n; ++i) pts[i].assign(points + i * dims, points + (i + 1) * dims);
    return mcx::kernel_width_heuristic(pts, max_pairs);
}

std::uint64_t mcxref_hash_results(std::uint32_t Q, const std::uint32_t* qid,
                                  const std::uint32_t* thr, const std::uint32_t* len,
                                  std::uint32_t stride, const std::uint32_t* ids,
                                  const std::uint32_t* counts) {
    std::vector<mcx::TopKResult> rs(Q);
    for (std::uint32_t q = 0; q < Q; ++q) {
        rs[q].query_id = qid[q];
        rs[q].threshold = thr[q];
        for (std::uint32_t e = 0; e < len[q]; ++e) {
            rs[q].entries.push_back(
                mcx::TopKEntry{ids[std::size_t(q) * stride + e], counts[std::size_t(q) * stride + e]});
        }
    }
    return mcx::hash_results(rs);
}

// sa.hpp:127-162: the reference's edit distances (golden vectors)
std::uint32_t mcxref_edit_distance_bounded(const char* a, std::uint64_t la, const char* b, std::uint64_t lb,
                                           std::uint32_t cap, int bounded) {
    const std::string_view x(a, la), y(b, lb);
    return bounded ? mcx::edit_distance_bounded(x, y, cap) : mcx::edit_distance(x, y);
}

// sa.hpp:298-336: verify_candidates over a corpus (strings at off[i]..off[i+1])
int mcxref_verify_candidates(const char* query, std::uint64_t qlen, std::uint32_t n_cand, const std::uint32_t* ids,
                             const std::uint32_t* counts, std::uint32_t n, const char* corpus_bytes,
                             const std::uint64_t* off, std::uint64_t n_corpus, std::uint64_t requested_k,
                             int early_break, std::uint32_t* best_id, std::uint32_t* best_distance, int* certified,
                             std::uint32_t* used, std::int64_t* theta, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<std::string> corpus(n_corpus);
        for (std::uint64_t i = 0; i < n_corpus; ++i) corpus[i].assign(corpus_bytes + off[i], off[i + 1] - off[i]);
        std::vector<mcx::CandidateHit> hits(n_cand);
        for (std::uint32_t i = 0; i < n_cand; ++i) hits[i] = {ids[i], counts[i]};
        const auto o = mcx::verify_candidates(std::string_view(query, qlen), hits, n, corpus, requested_k,
                                              early_break != 0);
        *best_id = o.best_id;
        *best_distance = o.best_distance;
        *certified = o.certified;
        *used = o.candidates_used;
        *theta = o.threshold_at_stop;
    });
}

}  // extern "C"
