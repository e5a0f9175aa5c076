// Host-side C-ABI entry points of the query path (include/genie/genie.h):
// validation with the reference's messages, staging, launch, readback.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <initializer_list>
#include <vector>

#include "internal.cuh"

namespace genie {

}  // namespace genie

namespace genie {
// Every pointer is page-locked host memory (a captured graph may copy only
// from / to pinned memory).
static bool all_pinned(std::initializer_list<const void*> ptrs) {
    for (const void* ptr : ptrs) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (a.type != cudaMemoryTypeHost) return false;
    }
    return true;
}
}  // namespace genie

using namespace genie;

extern "C" {

int genie_query_batch(genie_index* ix, const genie_config* cfg_in, uint32_t Q, const uint32_t* qid,
                      const uint32_t* k, const uint64_t* item_off, const uint16_t* item_dim,
                      const uint32_t* item_lo, const uint32_t* item_hi, uint32_t out_stride,
                      genie_entry* out, uint32_t* out_len, uint32_t* out_threshold,
                      uint64_t* out_bound, genie_stage_ns* timings, genie_batch_stats* stats,
                      char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        const auto t0 = std::chrono::steady_clock::now();
        const genie_config cfg = cfg_in ? *cfg_in : genie_config_default();
        validate_config(cfg);
        if (!ix) throw Error(GENIE_ERR_CONTRACT, "null index");
        if (Q && (!qid || !k || !item_off || !out || !out_len || !out_threshold))
            throw Error(GENIE_ERR_CONTRACT, "genie_query_batch: null argument");
        validate_offsets(Q, item_off);
        uint32_t max_k = 0;
        for (uint32_t q = 0; q < Q; ++q) max_k = std::max(max_k, k[q]);
        // a row never holds more than min(k, n) entries
        if (Q && out_stride < std::min<uint64_t>(max_k, std::max<uint32_t>(ix ? ix->n : 0, 1)))
            throw Error(GENIE_ERR_CONTRACT, "out_stride must be >= min(largest k, num_objects)");
        ensure_device(ix->device);
        Workspace& w = ix->ws;
        cudaStream_t s = ix->stream;
        const uint64_t items = Q ? item_off[Q] - item_off[0] : 0;
        if (items >= (1ull << 32)) throw Error(GENIE_ERR_CONTRACT, "too many query items");
        std::vector<uint64_t> off_rebased;
        const uint64_t* offs = item_off;
        if (Q && item_off[0] != 0) {
            off_rebased.assign(item_off, item_off + Q + 1);
            for (auto& o : off_rebased) o -= item_off[0];
            offs = off_rebased.data();
        }
        const uint64_t i0 = Q ? item_off[0] : 0;
        int rc = GENIE_RETRY;
        std::string msg;
        genie_batch_stats local_stats{};
        const uint32_t stride = std::max<uint32_t>(out_stride, 1);
        std::vector<uint64_t> bounds(Q);
        bool have_results = false;
        if ((cfg.flags & GENIE_FLAG_GRAPH) && Q && out_stride && i0 == 0 && all_pinned({qid, k, item_off, item_dim + i0, item_lo + i0,
                                                                            item_hi + i0, out, out_len, out_threshold})) {
            // One CUDA graph per batch shape and buffer set: the six uploads,
            // the 11-launch pipeline and the read-backs replay with one launch.
            w.d_out.reserve(uint64_t(Q) * stride);
            w.d_out_len.reserve(Q + 1);
            w.d_out_thr.reserve(Q + 1);
            w.d_qid.reserve(Q);
            w.d_k.reserve(Q);
            w.d_item_off.reserve(Q + 1);
            w.d_dim.reserve(items);
            w.d_lo.reserve(items);
            w.d_hi.reserve(items);
            if (ix->h_bounds_cap < Q) {
                if (ix->h_bounds) cudaFreeHost(ix->h_bounds);
                ix->h_bounds = nullptr;
                GENIE_CUDA(cudaMallocHost(&ix->h_bounds, Q * sizeof(uint64_t)));
                ix->h_bounds_cap = Q;
            }
            genie_config inner = cfg;
            inner.flags &= ~GENIE_FLAG_GRAPH;
            const uint64_t sig = prepare_batch(ix, inner, Q, static_cast<uint32_t>(items), max_k, stride, s);
            uint64_t cfgw = 0;
            std::memcpy(&cfgw, &inner, std::min(sizeof(cfgw), sizeof(inner)));
            const uint64_t key[16] = {reinterpret_cast<uint64_t>(qid), reinterpret_cast<uint64_t>(k),
                                      reinterpret_cast<uint64_t>(item_off), reinterpret_cast<uint64_t>(item_dim),
                                      reinterpret_cast<uint64_t>(item_lo), reinterpret_cast<uint64_t>(item_hi),
                                      reinterpret_cast<uint64_t>(out), reinterpret_cast<uint64_t>(out_len),
                                      reinterpret_cast<uint64_t>(out_threshold), Q, items, out_stride,
                                      max_k | (uint64_t(timings != nullptr) << 32), sig,
                                      mix64(cfgw ^ (uint64_t(inner.tile_bytes) << 32 | inner.ctas_per_sm)),
                                      reinterpret_cast<uint64_t>(ix->h_bounds)};
            if (!ix->host_graph || std::memcmp(key, ix->host_graph_key, sizeof(key)) != 0) {
                cudaGraph_t g = nullptr;
                // relaxed: launch_batch may set launch attributes on its first use
                GENIE_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
                try {
                    GENIE_CUDA(cudaMemcpyAsync(w.d_qid.p, qid, Q * 4, cudaMemcpyHostToDevice, s));
                    GENIE_CUDA(cudaMemcpyAsync(w.d_k.p, k, Q * 4, cudaMemcpyHostToDevice, s));
                    GENIE_CUDA(cudaMemcpyAsync(w.d_item_off.p, item_off, (Q + 1) * 8, cudaMemcpyHostToDevice, s));
                    GENIE_CUDA(cudaMemcpyAsync(w.d_dim.p, item_dim, items * 2, cudaMemcpyHostToDevice, s));
                    GENIE_CUDA(cudaMemcpyAsync(w.d_lo.p, item_lo, items * 4, cudaMemcpyHostToDevice, s));
                    GENIE_CUDA(cudaMemcpyAsync(w.d_hi.p, item_hi, items * 4, cudaMemcpyHostToDevice, s));
                    launch_batch(ix, inner, Q, w.d_qid.p, w.d_k.p, w.d_item_off.p, w.d_dim.p, w.d_lo.p, w.d_hi.p,
                                 static_cast<uint32_t>(items), max_k, stride, w.d_out.p, w.d_out_len.p, w.d_out_thr.p, s,
                                 timings != nullptr);
                    GENIE_CUDA(cudaMemcpyAsync(out, w.d_out.p, uint64_t(Q) * out_stride * sizeof(genie_entry),
                                               cudaMemcpyDeviceToHost, s));
                    GENIE_CUDA(cudaMemcpyAsync(out_len, w.d_out_len.p, Q * 4, cudaMemcpyDeviceToHost, s));
                    GENIE_CUDA(cudaMemcpyAsync(out_threshold, w.d_out_thr.p, Q * 4, cudaMemcpyDeviceToHost, s));
                    GENIE_CUDA(cudaMemcpyAsync(ix->h_bounds, w.q_bound.p, Q * 8, cudaMemcpyDeviceToHost, s));
                } catch (...) {
                    cudaStreamEndCapture(s, &g);
                    if (g) cudaGraphDestroy(g);
                    throw;
                }
                GENIE_CUDA(cudaStreamEndCapture(s, &g));
                bool updated = false;
                if (ix->host_graph) {
                    cudaGraphExecUpdateResultInfo info{};
                    updated = cudaGraphExecUpdate(ix->host_graph, g, &info) == cudaSuccess;
                    if (!updated) {
                        cudaGetLastError();
                        cudaGraphExecDestroy(ix->host_graph);
                        ix->host_graph = nullptr;
                    }
                }
                if (!updated) GENIE_CUDA(cudaGraphInstantiate(&ix->host_graph, g, 0));
                cudaGraphDestroy(g);
                std::memcpy(ix->host_graph_key, key, sizeof(key));
                ++ix->host_graph_captures;
            }
            GENIE_CUDA(cudaGraphLaunch(ix->host_graph, s));
            rc = finish_batch(ix, &local_stats, msg, qid);  // synchronises: results are in place
            if (rc == GENIE_OK) {
                have_results = true;
                std::copy(ix->h_bounds, ix->h_bounds + Q, bounds.begin());
            } else if (rc != GENIE_RETRY) {
                if (rc == GENIE_ERR_CONTRACT) validate_queries(Q, qid, k, item_off, item_dim, item_lo, item_hi);
                throw Error(rc, msg);
            }  // RETRY (the workspace grew): the direct path below re-issues the batch
        }
        for (int attempt = 0; attempt < 4 && rc == GENIE_RETRY; ++attempt) {
            h2d(w.d_qid, qid, Q, s);
            h2d(w.d_k, k, Q, s);
            h2d(w.d_item_off, offs, Q + 1, s);
            h2d(w.d_dim, item_dim + i0, items, s);
            h2d(w.d_lo, item_lo + i0, items, s);
            h2d(w.d_hi, item_hi + i0, items, s);
            w.d_out.reserve(uint64_t(Q) * std::max<uint32_t>(out_stride, 1));
            w.d_out_len.reserve(Q + 1);
            w.d_out_thr.reserve(Q + 1);
            launch_batch(ix, cfg, Q, w.d_qid.p, w.d_k.p, w.d_item_off.p, w.d_dim.p, w.d_lo.p,
                         w.d_hi.p, static_cast<uint32_t>(items), max_k, std::max<uint32_t>(out_stride, 1),
                         w.d_out.p, w.d_out_len.p, w.d_out_thr.p, s, timings != nullptr);
            rc = finish_batch(ix, &local_stats, msg, qid);
        }
        if (rc == GENIE_ERR_CONTRACT)  // the device flagged an input: the reference's exact message
            validate_queries(Q, qid, k, item_off, item_dim, item_lo, item_hi);
        if (rc != GENIE_OK) throw Error(rc, msg);
        if (Q && !have_results) {
            if (out_stride) {
                GENIE_CUDA(cudaMemcpyAsync(out, w.d_out.p, uint64_t(Q) * out_stride * sizeof(genie_entry),
                                           cudaMemcpyDeviceToHost, s));
            }
            GENIE_CUDA(cudaMemcpyAsync(out_len, w.d_out_len.p, Q * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
            GENIE_CUDA(cudaMemcpyAsync(out_threshold, w.d_out_thr.p, Q * sizeof(uint32_t),
                                       cudaMemcpyDeviceToHost, s));
        }
        if (Q && !have_results && (out_bound || stats))
            GENIE_CUDA(cudaMemcpyAsync(bounds.data(), w.q_bound.p, Q * sizeof(uint64_t),
                                       cudaMemcpyDeviceToHost, s));
        GENIE_CUDA(cudaStreamSynchronize(s));
        if (out_bound) std::copy(bounds.begin(), bounds.end(), out_bound);
        if (stats) {
            *stats = local_stats;
            memory_stats(ix->n, Q, k, bounds.data(), stats);
        }
        if (timings) {
            float ms_lookup = 0, ms_match = 0, ms_merge = 0;
            cudaEventElapsedTime(&ms_lookup, ix->ev[0], ix->ev[1]);
            cudaEventElapsedTime(&ms_match, ix->ev[1], ix->ev[2]);
            cudaEventElapsedTime(&ms_merge, ix->ev[2], ix->ev[3]);
            timings->lookup_ns = static_cast<uint64_t>(ms_lookup * 1e6);
            timings->match_ns = static_cast<uint64_t>(ms_match * 1e6);
            timings->select_ns = 0;  // fused into the match kernel (per-tile c-PQ extract)
            timings->merge_ns = static_cast<uint64_t>(ms_merge * 1e6);
            const auto t1 = std::chrono::steady_clock::now();
            timings->total_ns = static_cast<uint64_t>(
                std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
            const uint64_t sum = timings->lookup_ns + timings->match_ns + timings->merge_ns;
            if (sum > timings->total_ns) timings->total_ns = sum;
        }
        return GENIE_OK;
    });
}

int genie_query_batch_device(genie_index* ix, const genie_config* cfg_in, uint32_t Q,
                             const uint32_t* d_qid, const uint32_t* d_k, const uint64_t* d_item_off,
                             const uint16_t* d_item_dim, const uint32_t* d_item_lo,
                             const uint32_t* d_item_hi, uint32_t max_k, uint32_t total_items,
                             uint32_t out_stride, genie_entry* d_out, uint32_t* d_out_len,
                             uint32_t* d_out_threshold, void* stream, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        const genie_config cfg = cfg_in ? *cfg_in : genie_config_default();
        validate_config(cfg);
        if (!ix) throw Error(GENIE_ERR_CONTRACT, "null index");
        if (Q >= (1u << 21)) throw Error(GENIE_ERR_CONTRACT, "batch exceeds 2^21 queries");
        if (Q && out_stride < std::min<uint64_t>(max_k, std::max<uint32_t>(ix->n, 1)))
            throw Error(GENIE_ERR_CONTRACT, "out_stride must be >= min(max_k, num_objects)");
        ensure_device(ix->device);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ix->stream;
        launch_batch(ix, cfg, Q, d_qid, d_k, d_item_off, d_item_dim, d_item_lo, d_item_hi, total_items,
                     max_k, std::max<uint32_t>(out_stride, 1), d_out, d_out_len, d_out_threshold, s,
                     (cfg.flags & GENIE_FLAG_STAGE_EVENTS) != 0);
        if (s != ix->stream) {
            // make genie_query_status's synchronisation cover the caller's stream
            cudaEvent_t e = ix->ev[5];
            GENIE_CUDA(cudaEventRecord(e, s));
            GENIE_CUDA(cudaStreamWaitEvent(ix->stream, e, 0));
        }
        return GENIE_OK;
    });
}

int genie_query_status(genie_index* ix, genie_batch_stats* stats, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        ensure_device(ix->device);
        std::string msg;
        const int rc = finish_batch(ix, stats, msg, nullptr);
        if (rc != GENIE_OK) throw Error(rc, msg);
        return GENIE_OK;
    });
}

uint32_t genie_last_launch_count(const genie_index* ix) { return ix ? ix->last_launches : 0; }

uint64_t genie_graph_captures(const genie_index* ix) { return ix ? graph_captures(ix) + ix->host_graph_captures : 0; }

int genie_debug_status(genie_index* ix, uint64_t* words, uint32_t n_words, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        if (!ix || !ix->ws.h_status) throw Error(GENIE_ERR_CONTRACT, "no batch has run on this index");
        ensure_device(ix->device);
        GENIE_CUDA(cudaStreamSynchronize(ix->stream));
        for (uint32_t i = 0; i < n_words && i < ST_WORDS; ++i) words[i] = ix->ws.h_status[i];
        return GENIE_OK;
    });
}

int genie_last_stage_ns(genie_index* ix, genie_stage_ns* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        if (!ix || !out) throw Error(GENIE_ERR_CONTRACT, "null argument");
        if (!ix->last_timed) throw Error(GENIE_ERR_CONTRACT, "last batch was not launched with stage events");
        ensure_device(ix->device);
        GENIE_CUDA(cudaEventSynchronize(ix->ev[3]));
        float a = 0, b = 0, c = 0;
        GENIE_CUDA(cudaEventElapsedTime(&a, ix->ev[0], ix->ev[1]));
        GENIE_CUDA(cudaEventElapsedTime(&b, ix->ev[1], ix->ev[2]));
        GENIE_CUDA(cudaEventElapsedTime(&c, ix->ev[2], ix->ev[3]));
        out->lookup_ns = static_cast<uint64_t>(double(a) * 1e6);
        out->match_ns = static_cast<uint64_t>(double(b) * 1e6);
        out->select_ns = 0;
        out->merge_ns = static_cast<uint64_t>(double(c) * 1e6);
        out->total_ns = out->lookup_ns + out->match_ns + out->merge_ns;
        return GENIE_OK;
    });
}

int genie_merge_topk_device(genie_index* ix, uint32_t Q, uint32_t L, const genie_entry* d_in,
                            const uint32_t* d_in_len, uint32_t in_stride, const uint32_t* d_k,
                            uint32_t out_stride, genie_entry* d_out, uint32_t* d_out_len,
                            uint32_t* d_out_threshold, void* stream, char* err, size_t errlen) {
    return genie_merge_topk_device_layout(ix, Q, L, d_in, d_in_len, in_stride, 0, d_k, out_stride, d_out, d_out_len,
                                          d_out_threshold, stream, err, errlen);
}

int genie_merge_topk_device_layout(genie_index* ix, uint32_t Q, uint32_t L, const genie_entry* d_in,
                                   const uint32_t* d_in_len, uint32_t in_stride, uint32_t list_major,
                                   const uint32_t* d_k, uint32_t out_stride, genie_entry* d_out, uint32_t* d_out_len,
                                   uint32_t* d_out_threshold, void* stream, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        if (!ix) throw Error(GENIE_ERR_CONTRACT, "null index");
        ensure_device(ix->device);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ix->stream;
        // max_k is unknown on the host here; rows are bounded by L * in_stride
        const uint32_t max_rows = std::min<uint32_t>(out_stride, L * in_stride);
        launch_list_merge(ix, Q, L, d_in, d_in_len, in_stride, d_k, out_stride, d_out, d_out_len,
                          d_out_threshold, max_rows, s, list_major != 0);
        if (s != ix->stream) {
            GENIE_CUDA(cudaEventRecord(ix->ev[5], s));
            GENIE_CUDA(cudaStreamWaitEvent(ix->stream, ix->ev[5], 0));
        }
        return GENIE_OK;
    });
}

int genie_merge_topk(int device, uint32_t Q, uint32_t L, const genie_entry* in, const uint32_t* in_len,
                     uint32_t in_stride, const uint32_t* k, uint32_t out_stride, genie_entry* out,
                     uint32_t* out_len, uint32_t* out_threshold, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        ensure_device(device);
        uint32_t max_k = 0;
        for (uint32_t q = 0; q < Q; ++q) {
            if (k[q] == 0) throw Error(GENIE_ERR_CONTRACT, "merge_topk: k must be >= 1");
            max_k = std::max(max_k, k[q]);
        }
        if (Q && out_stride < std::min<uint64_t>(max_k, uint64_t(L) * in_stride))
            throw Error(GENIE_ERR_CONTRACT, "out_stride too small");
        for (uint64_t i = 0; i < uint64_t(Q) * L; ++i)
            if (in_len[i] > in_stride) throw Error(GENIE_ERR_CONTRACT, "list longer than in_stride");
        // a transient handle carries the stream and workspace
        genie_index tmp;
        tmp.device = device;
        tmp.sms = sm_count(device);
        GENIE_CUDA(cudaStreamCreateWithFlags(&tmp.stream, cudaStreamNonBlocking));
        struct Guard {
            genie_index& t;
            ~Guard() {
                if (t.ws.h_status) cudaFreeHost(t.ws.h_status);
                t.ws.h_status = nullptr;
                cudaStreamDestroy(t.stream);
                t.stream = nullptr;
            }
        } guard{tmp};
        DevBuf<genie_entry> d_in, d_out;
        DevBuf<uint32_t> d_len, d_k, d_olen, d_othr;
        h2d(d_in, in, uint64_t(Q) * L * in_stride, tmp.stream);
        h2d(d_len, in_len, uint64_t(Q) * L, tmp.stream);
        h2d(d_k, k, Q, tmp.stream);
        const uint32_t stride = std::max<uint32_t>(out_stride, 1);
        d_out.reserve(uint64_t(Q) * stride);
        d_olen.reserve(Q + 1);
        d_othr.reserve(Q + 1);
        // host lists (mcx::merge_topk) may come in any order: no list floors
        launch_list_merge(&tmp, Q, L, d_in.p, d_len.p, in_stride, d_k.p, stride, d_out.p, d_olen.p,
                          d_othr.p, max_k, tmp.stream, false, false);
        std::string msg;
        const int rc = finish_batch(&tmp, nullptr, msg, nullptr);
        if (rc != GENIE_OK) throw Error(rc, msg);
        if (Q) {
            GENIE_CUDA(cudaMemcpy(out, d_out.p, uint64_t(Q) * stride * sizeof(genie_entry),
                                  cudaMemcpyDeviceToHost));
            GENIE_CUDA(cudaMemcpy(out_len, d_olen.p, Q * sizeof(uint32_t), cudaMemcpyDeviceToHost));
            GENIE_CUDA(cudaMemcpy(out_threshold, d_othr.p, Q * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        }
        return GENIE_OK;
    });
}

// engine.hpp:141-153
uint64_t genie_hash_results(uint32_t Q, const uint32_t* qid, const uint32_t* thr, const uint32_t* len,
                            uint32_t stride, const genie_entry* entries) {
    uint64_t h = 0xcbf29ce484222325ull;
    auto mix_in = [&h](uint64_t v) { h = mix64(h ^ v); };
    for (uint32_t q = 0; q < Q; ++q) {
        mix_in(qid[q]);
        mix_in(thr[q]);
        mix_in(len[q]);
        for (uint32_t e = 0; e < len[q]; ++e) {
            const genie_entry& x = entries[uint64_t(q) * stride + e];
            mix_in((uint64_t(x.id) << 32) | x.count);
        }
    }
    return h;
}

}  // extern "C"
