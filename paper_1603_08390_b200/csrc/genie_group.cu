// A device group: object-id-range shards of one index on several GPUs, all
// driven by ONE host thread.  The concurrent counterpart of
// execute_partitioned (engine.hpp:308-347), which runs its parts one after
// another: here every shard's batch is in flight on its own device / stream
// at once, then the per-shard top-k rows (global ids) are exchanged and merged
// on the group's root device with merge_topk's rule (engine.hpp:158-177).
//
// Exchange: an NCCL all-gather over NVLink (ncclCommInitAll over the group's
// devices, one communicator per shard) when every shard sits on a distinct
// device and libnccl.so.2 can be loaded; otherwise (shards sharing a device,
// e.g. the single-GPU test box) peer / device-to-device copies of the rows
// into the root's gather buffer.  Both produce the list-major layout
// [shard][query][stride] that k_merge reads in place.
//
// NCCL is loaded at run time (dlopen) so the library has no link-time NCCL
// dependency; nccl.h supplies the types only.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <memory>
#include <vector>

#include "internal.cuh"

namespace genie {
namespace {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi* nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            return fn != nullptr;
        };
        a.ok = sym(a.comm_init_all, "ncclCommInitAll") && sym(a.comm_destroy, "ncclCommDestroy") &&
               sym(a.all_gather, "ncclAllGather") && sym(a.group_start, "ncclGroupStart") &&
               sym(a.group_end, "ncclGroupEnd") && sym(a.error_string, "ncclGetErrorString");
        return a;
    }();
    return api.ok ? &api : nullptr;
}

#define GENIE_NCCL(api, call)                                                                     \
    do {                                                                                          \
        ncclResult_t r_ = (call);                                                                 \
        if (r_ != ncclSuccess) throw ::genie::Error(GENIE_ERR_NCCL, std::string(#call) + ": " +   \
                                                                        (api)->error_string(r_)); \
    } while (0)

struct Shard {
    genie_index* ix = nullptr;
    bool owned = false;
    uint32_t extra = 0;                 // added to the shard's reported ids (on top of its own id_offset)
    DevBuf<genie_entry> gather;         // NCCL exchange: every shard's rows, on this shard's device
    DevBuf<uint32_t> gather_len;
    cudaEvent_t done = nullptr;         // rows ready on the shard's stream
    std::vector<uint64_t> bounds;       // max_count_bound per query (memory accounting)
    genie_batch_stats stats{};
    ncclComm_t comm = nullptr;
};

}  // namespace
}  // namespace genie

struct genie_group {
    std::vector<std::unique_ptr<genie::Shard>> shards;
    int exchange = GENIE_EXCHANGE_PEER;
    genie_index* root = nullptr;  // merge context on shards[0]'s device (stream, workspace, events)
    genie::DevBuf<genie_entry> peer_in, fin;
    genie::DevBuf<uint32_t> peer_len, d_k, fin_len, fin_thr;
    uint32_t total_objects = 0;
    genie_stage_ns last{};
};

namespace genie {
namespace {

genie_index* make_context(int device) {
    ensure_device(device);
    auto* ix = new genie_index;
    ix->device = device;
    ix->sms = sm_count(device);
    GENIE_CUDA(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
    for (auto& e : ix->ev) GENIE_CUDA(cudaEventCreate(&e));
    return ix;
}

void destroy_group(genie_group* g) {
    if (!g) return;
    const NcclApi* api = nccl_api();
    for (auto& s : g->shards) {
        if (!s) continue;
        cudaSetDevice(s->ix ? s->ix->device : 0);
        if (s->comm && api) api->comm_destroy(s->comm);
        if (s->done) cudaEventDestroy(s->done);
        s->gather.release();
        s->gather_len.release();
        if (s->owned) genie_index_destroy(s->ix);
    }
    if (g->root) {
        cudaSetDevice(g->root->device);
        g->peer_in.release();
        g->peer_len.release();
        g->fin.release();
        g->fin_len.release();
        g->fin_thr.release();
        g->d_k.release();
        genie_index_destroy(g->root);
    }
    delete g;
}

// Shards on distinct devices -> one NCCL communicator per shard; otherwise
// the peer-copy exchange.
void setup_exchange(genie_group* g, int mode) {
    std::vector<int> devs;
    for (auto& s : g->shards) devs.push_back(s->ix->device);
    std::vector<int> sorted = devs;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    const NcclApi* api = nccl_api();
    if (mode == GENIE_EXCHANGE_NCCL && (!distinct || !api))
        throw Error(GENIE_ERR_CONTRACT, !api ? "NCCL exchange requested but libnccl.so.2 cannot be loaded"
                                              : "NCCL exchange needs every shard on a distinct device");
    const bool use_nccl = mode == GENIE_EXCHANGE_NCCL || (mode == GENIE_EXCHANGE_AUTO && distinct && api);
    g->exchange = use_nccl ? GENIE_EXCHANGE_NCCL : GENIE_EXCHANGE_PEER;
    for (auto& s : g->shards) {
        ensure_device(s->ix->device);
        GENIE_CUDA(cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming));
    }
    if (use_nccl) {
        std::vector<ncclComm_t> comms(devs.size());
        GENIE_NCCL(api, api->comm_init_all(comms.data(), static_cast<int>(devs.size()), devs.data()));
        for (size_t i = 0; i < devs.size(); ++i) g->shards[i]->comm = comms[i];
    } else {
        // direct peer access where the hardware offers it (NVLink); copies
        // fall back to staged transfers otherwise
        const int r = g->root->device;
        for (int d : devs) {
            if (d == r) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, r, d);
            if (can) {
                ensure_device(r);
                const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) GENIE_CUDA(e);
                cudaGetLastError();
            }
        }
    }
}

}  // namespace
}  // namespace genie

using namespace genie;

extern "C" {

int genie_group_create(uint32_t num_objects, uint64_t num_keys, const uint64_t* keys, const uint64_t* key_off,
                       const uint32_t* postings, uint32_t num_shards, const int* devices, int exchange,
                       genie_group** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        if (!out || !devices || num_shards == 0) throw Error(GENIE_ERR_CONTRACT, "genie_group_create: bad argument");
        *out = nullptr;
        auto* g = new genie_group;
        try {
            g->total_objects = num_objects;
            for (uint32_t p = 0; p < num_shards; ++p) {
                // shard p owns ids [p n / G, (p + 1) n / G)
                const uint32_t b = static_cast<uint32_t>(uint64_t(num_objects) * p / num_shards);
                const uint32_t e = static_cast<uint32_t>(uint64_t(num_objects) * (p + 1) / num_shards);
                auto s = std::make_unique<Shard>();
                const int rc = genie_index_create_shard(num_objects, num_keys, keys, key_off, postings, b, e,
                                                        devices[p], &s->ix, err, errlen);
                if (rc != GENIE_OK) throw Error(rc, err ? std::string(err) : "shard creation failed");
                s->owned = true;
                g->shards.push_back(std::move(s));
            }
            g->root = make_context(devices[0]);
            setup_exchange(g, exchange);
        } catch (...) {
            destroy_group(g);
            throw;
        }
        *out = g;
        return GENIE_OK;
    });
}

int genie_group_from_indexes(genie_index* const* indexes, const uint32_t* id_offsets, uint32_t num_shards,
                             int exchange, genie_group** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        if (!out || !indexes || num_shards == 0) throw Error(GENIE_ERR_CONTRACT, "genie_group_from_indexes: bad argument");
        *out = nullptr;
        auto* g = new genie_group;
        try {
            uint64_t total = 0;
            for (uint32_t p = 0; p < num_shards; ++p) {
                if (!indexes[p]) throw Error(GENIE_ERR_CONTRACT, "genie_group_from_indexes: null index");
                auto s = std::make_unique<Shard>();
                s->ix = indexes[p];
                s->extra = id_offsets ? id_offsets[p] : 0;
                total += indexes[p]->n;
                g->shards.push_back(std::move(s));
            }
            if (total > 0xffffffffull) throw Error(GENIE_ERR_CONTRACT, "genie_group_from_indexes: too many objects");
            g->total_objects = static_cast<uint32_t>(total);
            g->root = make_context(indexes[0]->device);
            setup_exchange(g, exchange);
        } catch (...) {
            destroy_group(g);
            throw;
        }
        *out = g;
        return GENIE_OK;
    });
}

void genie_group_destroy(genie_group* g) { destroy_group(g); }

int genie_group_info(const genie_group* g, uint32_t* num_shards, int* exchange, uint32_t* num_objects) {
    if (!g) return GENIE_ERR_CONTRACT;
    if (num_shards) *num_shards = static_cast<uint32_t>(g->shards.size());
    if (exchange) *exchange = g->exchange;
    if (num_objects) *num_objects = g->total_objects;
    return GENIE_OK;
}

int genie_group_query_batch(genie_group* g, const genie_config* cfg_in, uint32_t Q, const uint32_t* qid,
                            const uint32_t* k, const uint64_t* item_off, const uint16_t* item_dim,
                            const uint32_t* item_lo, const uint32_t* item_hi, uint32_t out_stride, genie_entry* out,
                            uint32_t* out_len, uint32_t* out_threshold, genie_stage_ns* timings,
                            genie_batch_stats* stats, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        const auto t0 = std::chrono::steady_clock::now();
        const genie_config cfg = cfg_in ? *cfg_in : genie_config_default();
        validate_config(cfg);
        if (!g) throw Error(GENIE_ERR_CONTRACT, "null group");
        if (Q && (!qid || !k || !item_off || !out || !out_len || !out_threshold))
            throw Error(GENIE_ERR_CONTRACT, "genie_group_query_batch: null argument");
        validate_queries(Q, qid, k, item_off, item_dim, item_lo, item_hi);
        uint32_t max_k = 0;
        for (uint32_t q = 0; q < Q; ++q) max_k = std::max(max_k, k[q]);
        const uint32_t N = g->total_objects;
        if (Q && out_stride < std::min<uint64_t>(max_k, std::max<uint32_t>(N, 1)))
            throw Error(GENIE_ERR_CONTRACT, "out_stride must be >= min(largest k, num_objects)");
        const uint32_t P = static_cast<uint32_t>(g->shards.size());
        // one row stride for every shard: a shard row holds <= min(k, n_p) entries
        const uint32_t S = std::max<uint32_t>(1, static_cast<uint32_t>(std::min<uint64_t>(max_k, std::max<uint32_t>(N, 1))));
        const uint64_t items = Q ? item_off[Q] - item_off[0] : 0;
        if (items >= (1ull << 32)) throw Error(GENIE_ERR_CONTRACT, "too many query items");
        std::vector<uint64_t> offs(item_off, item_off + Q + 1);
        for (auto& o : offs) o -= item_off[0];
        const uint64_t i0 = item_off[0];
        const bool timed = timings != nullptr;

        // 1. every shard's batch in flight on its own device / stream
        auto launch = [&](Shard& s) {
            genie_index* ix = s.ix;
            ensure_device(ix->device);
            Workspace& w = ix->ws;
            cudaStream_t st = ix->stream;
            h2d(w.d_qid, qid, Q, st);
            h2d(w.d_k, k, Q, st);
            h2d(w.d_item_off, offs.data(), Q + 1, st);
            h2d(w.d_dim, item_dim + i0, items, st);
            h2d(w.d_lo, item_lo + i0, items, st);
            h2d(w.d_hi, item_hi + i0, items, st);
            w.d_out.reserve(uint64_t(Q) * S);
            w.d_out_len.reserve(Q + 1);
            w.d_out_thr.reserve(Q + 1);
            launch_batch(ix, cfg, Q, w.d_qid.p, w.d_k.p, w.d_item_off.p, w.d_dim.p, w.d_lo.p, w.d_hi.p,
                         static_cast<uint32_t>(items), max_k, S, w.d_out.p, w.d_out_len.p, w.d_out_thr.p, st, timed,
                         s.extra);
        };
        for (auto& s : g->shards) launch(*s);
        // 2. statuses (a workspace overflow re-issues that shard alone)
        for (auto& sp : g->shards) {
            Shard& s = *sp;
            ensure_device(s.ix->device);
            std::string msg;
            int rc = finish_batch(s.ix, &s.stats, msg, qid);
            for (int attempt = 0; rc == GENIE_RETRY && attempt < 3; ++attempt) {
                launch(s);
                rc = finish_batch(s.ix, &s.stats, msg, qid);
            }
            if (rc != GENIE_OK) throw Error(rc, msg);
            s.bounds.resize(Q);
            if (Q)
                GENIE_CUDA(cudaMemcpyAsync(s.bounds.data(), s.ix->ws.q_bound.p, Q * sizeof(uint64_t),
                                           cudaMemcpyDeviceToHost, s.ix->stream));
            GENIE_CUDA(cudaEventRecord(s.done, s.ix->stream));
        }
        // 3. exchange into list-major [shard][query][S] on the root device
        genie_index* root = g->root;
        const genie_entry* rows = nullptr;
        const uint32_t* lens = nullptr;
        const uint64_t row_elems = uint64_t(Q) * S;
        if (Q && g->exchange == GENIE_EXCHANGE_NCCL) {
            const NcclApi* api = nccl_api();
            for (auto& s : g->shards) {
                ensure_device(s->ix->device);
                s->gather.reserve(row_elems * P);
                s->gather_len.reserve(uint64_t(Q) * P);
            }
            GENIE_NCCL(api, api->group_start());
            for (auto& s : g->shards) {
                ensure_device(s->ix->device);
                GENIE_NCCL(api, api->all_gather(s->ix->ws.d_out.p, s->gather.p, row_elems * 2, ncclUint32, s->comm,
                                                s->ix->stream));
                GENIE_NCCL(api, api->all_gather(s->ix->ws.d_out_len.p, s->gather_len.p, Q, ncclUint32, s->comm,
                                                s->ix->stream));
            }
            GENIE_NCCL(api, api->group_end());
            Shard& s0 = *g->shards[0];
            ensure_device(root->device);
            GENIE_CUDA(cudaEventRecord(s0.done, s0.ix->stream));
            GENIE_CUDA(cudaStreamWaitEvent(root->stream, s0.done, 0));
            rows = s0.gather.p;
            lens = s0.gather_len.p;
        } else if (Q) {
            ensure_device(root->device);
            g->peer_in.reserve(row_elems * P);
            g->peer_len.reserve(uint64_t(Q) * P);
            for (uint32_t p = 0; p < P; ++p) {
                Shard& s = *g->shards[p];
                GENIE_CUDA(cudaStreamWaitEvent(root->stream, s.done, 0));
                GENIE_CUDA(cudaMemcpyPeerAsync(g->peer_in.p + p * row_elems, root->device, s.ix->ws.d_out.p,
                                               s.ix->device, row_elems * sizeof(genie_entry), root->stream));
                GENIE_CUDA(cudaMemcpyPeerAsync(g->peer_len.p + uint64_t(p) * Q, root->device, s.ix->ws.d_out_len.p,
                                               s.ix->device, Q * sizeof(uint32_t), root->stream));
            }
            rows = g->peer_in.p;
            lens = g->peer_len.p;
        }
        // 4. merge_topk on the root device, results to the host
        ensure_device(root->device);
        if (Q) {
            if (timed) GENIE_CUDA(cudaEventRecord(root->ev[2], root->stream));
            h2d(g->d_k, k, Q, root->stream);
            g->fin.reserve(row_elems);
            g->fin_len.reserve(Q + 1);
            g->fin_thr.reserve(Q + 1);
            launch_list_merge(root, Q, P, rows, lens, S, g->d_k.p, S, g->fin.p, g->fin_len.p, g->fin_thr.p, max_k,
                              root->stream, true);
            if (timed) GENIE_CUDA(cudaEventRecord(root->ev[3], root->stream));
            std::string msg;
            const int rc = finish_batch(root, nullptr, msg, qid);
            if (rc != GENIE_OK) throw Error(rc, msg);
            GENIE_CUDA(cudaMemcpy2DAsync(out, size_t(out_stride) * sizeof(genie_entry), g->fin.p,
                                         size_t(S) * sizeof(genie_entry), size_t(S) * sizeof(genie_entry), Q,
                                         cudaMemcpyDeviceToHost, root->stream));
            GENIE_CUDA(cudaMemcpyAsync(out_len, g->fin_len.p, Q * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                       root->stream));
            GENIE_CUDA(cudaMemcpyAsync(out_threshold, g->fin_thr.p, Q * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                       root->stream));
            GENIE_CUDA(cudaStreamSynchronize(root->stream));
        }
        for (auto& s : g->shards) {
            ensure_device(s->ix->device);
            GENIE_CUDA(cudaStreamSynchronize(s->ix->stream));
        }
        // 5. execute_partitioned's accounting: per-part maximum of the memory
        // stats (engine.hpp:330-333), work summed; stage times: the slowest shard
        if (stats) {
            *stats = genie_batch_stats{};
            for (auto& s : g->shards) {
                genie_batch_stats m{};
                memory_stats(s->ix->n, Q, k, s->bounds.data(), &m);
                stats->counter_bytes = std::max(stats->counter_bytes, m.counter_bytes);
                stats->gate_bytes = std::max(stats->gate_bytes, m.gate_bytes);
                stats->table_bytes = std::max(stats->table_bytes, m.table_bytes);
                stats->postings += s->stats.postings;
                stats->work_items += s->stats.work_items;
                stats->fallback_tiles += s->stats.fallback_tiles;
            }
        }
        if (timings) {
            *timings = genie_stage_ns{};
            for (auto& s : g->shards) {
                ensure_device(s->ix->device);
                float a = 0, b = 0;
                cudaEventElapsedTime(&a, s->ix->ev[0], s->ix->ev[1]);
                cudaEventElapsedTime(&b, s->ix->ev[1], s->ix->ev[3]);
                timings->lookup_ns = std::max<uint64_t>(timings->lookup_ns, static_cast<uint64_t>(double(a) * 1e6));
                timings->match_ns = std::max<uint64_t>(timings->match_ns, static_cast<uint64_t>(double(b) * 1e6));
            }
            if (Q) {
                ensure_device(root->device);
                float c = 0;
                cudaEventElapsedTime(&c, root->ev[2], root->ev[3]);
                timings->merge_ns = static_cast<uint64_t>(double(c) * 1e6);
            }
            timings->total_ns = static_cast<uint64_t>(
                std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
            const uint64_t sum = timings->lookup_ns + timings->match_ns + timings->merge_ns;
            if (sum > timings->total_ns) timings->total_ns = sum;
        }
        return GENIE_OK;
    });
}

}  // extern "C"
