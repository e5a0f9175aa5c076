// Device inverted index: CSR upload, validation, id-range shards, per-dim
// statistics, export.  Replaces the product of mcx::build_index
// (index.hpp:190-250) and the InvertedIndex accessors (index.hpp:41-182).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>

#include <algorithm>
#include <cstdlib>
#include <thread>
#include <vector>

#include "block.cuh"
#include "internal.cuh"

namespace genie {

void build_dense_containers(genie_index* ix, const uint64_t* h_off);

// ---- max_multiplicity per dim (index.hpp:110-113, 153-174) on the device:
// pass 1 counts the dim's keywords per object, pass 2 takes the max while
// clearing the scratch (atomicExch), touching only the dim's postings.
__global__ void k_dim_count(const uint32_t* post, uint64_t b, uint64_t e, uint32_t* cnt) {
    for (uint64_t i = b + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < e;
         i += uint64_t(gridDim.x) * blockDim.x)
        atomicAdd(&cnt[post[i]], 1u);
}

__global__ void k_dim_max(const uint32_t* post, uint64_t b, uint64_t e, uint32_t* cnt,
                          uint32_t* out) {
    uint32_t best = 0;
    for (uint64_t i = b + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < e;
         i += uint64_t(gridDim.x) * blockDim.x)
        best = max(best, atomicExch(&cnt[post[i]], 0u));
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, d));
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

__global__ void k_max_into(const uint32_t* src, uint32_t* dst, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[i] = max(dst[i], src[i]);
}

// max_multiplicity per dim (index.hpp:110-113, 153-174): per dim with more
// than one keyword, count each object's postings of that dim and take the
// max (two passes over only the dim's postings); a one-keyword dim has
// multiplicity 1 (ObjectRecord rejects duplicate keywords) -- gram-coded
// corpora have tens of thousands of such dims.
static void compute_dim_stats(genie_index* ix, const uint64_t* h_keys, const uint64_t* h_off) {
    GENIE_CUDA(cudaMemsetAsync(ix->dim_mult.p, 0, 65536 * sizeof(uint32_t), ix->stream));
    if (!ix->K || !ix->n) return;
    DevBuf<uint32_t> scratch;
    scratch.reserve(ix->n);
    GENIE_CUDA(cudaMemsetAsync(scratch.p, 0, size_t(ix->n) * sizeof(uint32_t), ix->stream));
    std::vector<uint32_t> single(65536, 0);  // dims with one keyword: every object carries it at most once
    bool any_single = false;
    uint64_t j = 0;
    while (j < ix->K) {
        const uint32_t d = static_cast<uint32_t>(h_keys[j] >> 32);
        uint64_t e = j;
        while (e < ix->K && static_cast<uint32_t>(h_keys[e] >> 32) == d) ++e;
        const uint64_t pb = h_off[j], pe = h_off[e];
        if (e - j == 1) {
            if (pe > pb) single[d] = 1, any_single = true;
        } else if (pe > pb) {
            const uint64_t blocks = std::min<uint64_t>((pe - pb + 255) / 256, uint64_t(ix->sms) * 16);
            k_dim_count<<<static_cast<unsigned>(blocks), 256, 0, ix->stream>>>(ix->postings.p, pb, pe,
                                                                              scratch.p);
            k_dim_max<<<static_cast<unsigned>(blocks), 256, 0, ix->stream>>>(ix->postings.p, pb, pe,
                                                                            scratch.p, ix->dim_mult.p + d);
        }
        j = e;
    }
    if (any_single) {  // the multi-keyword dims' maxima were atomicMax'ed into zeros: merge by max
        DevBuf<uint32_t> ones;
        ones.reserve(65536);
        GENIE_CUDA(cudaMemcpyAsync(ones.p, single.data(), 65536 * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                   ix->stream));
        k_max_into<<<256, 256, 0, ix->stream>>>(ones.p, ix->dim_mult.p, 65536);
        GENIE_CUDA(cudaStreamSynchronize(ix->stream));
    }
    GENIE_CUDA(cudaStreamSynchronize(ix->stream));
    GENIE_CUDA(cudaGetLastError());
}

// ---- dense containers: bit i of a dense key's bitmap is set iff object i
// carries the key.  Built from the CSR (ascending ids per list).
__global__ void k_build_bitmap(const uint32_t* post, uint64_t b, uint64_t e, uint32_t* bm) {
    for (uint64_t i = b + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < e;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t id = post[i];
        atomicOr(&bm[id >> 5], 1u << (id & 31));
    }
}

// Lists covering at least 1/64 of the objects carry a bitmap (at most twice
// their posting bytes).  Whether a query uses it depends on its counter width
// (k_cut): W = 4 from density 1/32, W >= 8 from 1/64 -- measured break-even of
// the bitmap adds (bit-sliced past 2W lists) against one shared atomic per
// posting.  GENIE_DENSE_MIN_DENSITY=<d> overrides both with one fixed
// threshold (0 disables the containers).
static double dense_density(genie_index* ix) {
    const char* v = std::getenv("GENIE_DENSE_MIN_DENSITY");
    if (!v || !*v) {
        ix->dense_inv[0] = 32;
        ix->dense_inv[1] = 64;
        ix->dense_inv[2] = 64;
        return 1.0 / 64;
    }
    ix->dense_inv[0] = ix->dense_inv[1] = ix->dense_inv[2] = 0;
    return std::atof(v);
}

// Per-dim key ranges (k_resolve): dim d's keywords are keys[first, first +
// count); when its tokens are exactly tok0 .. tok0 + count - 1 (LSH tokens,
// categorical domains) the count carries a flag and a point item resolves by
// arithmetic instead of a binary search over all K keys.
__global__ void k_dim_ranges(const uint64_t* keys, uint64_t K, DimRange* out) {
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < K; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t d = static_cast<uint32_t>(keys[j] >> 32);
        if (j > 0 && static_cast<uint32_t>(keys[j - 1] >> 32) == d) continue;  // first key of its dim only
        uint64_t lo = j, hi = K;  // end of the dim: first key with a larger dim
        while (lo < hi) {
            const uint64_t m = (lo + hi) >> 1;
            if (static_cast<uint32_t>(keys[m] >> 32) <= d) lo = m + 1;
            else hi = m;
        }
        const uint64_t cnt = lo - j;
        const uint32_t t0 = static_cast<uint32_t>(keys[j]), t1 = static_cast<uint32_t>(keys[lo - 1]);
        DimRange r{};
        r.first = j;
        r.count = static_cast<uint32_t>(cnt) | ((uint64_t(t1) - t0 + 1 == cnt) ? kDimDenseFlag : 0u);
        r.tok0 = t0;
        r.pad = t1;  // the dim's last token (the host sizes the token maps from it)
        out[d] = r;
    }
}

// Which gapped dims get a token map (span <= 8 x keys, total <= 2^28 entries)
// and where: one CTA, 64 dims per thread, a block scan of the map sizes.
__global__ void __launch_bounds__(1024) k_tokmap_plan(DimRange* ranges, unsigned long long* total_out) {
    __shared__ unsigned long long sums[32];
    constexpr uint32_t kPer = 65536 / 1024;
    unsigned long long mine = 0;
    for (uint32_t i = 0; i < kPer; ++i) {
        const DimRange& r = ranges[threadIdx.x * kPer + i];
        const uint32_t cnt = r.count & ~kDimDenseFlag;
        if (!cnt || (r.count & kDimDenseFlag)) continue;
        const uint64_t span = uint64_t(r.pad) - r.tok0 + 1;
        if (span <= 8ull * cnt) mine += span + 1;
    }
    unsigned long long total = 0;
    unsigned long long at = block_exclusive_scan<unsigned long long>(mine, sums, total);
    const bool fits = total <= (1ull << 28);  // all or nothing: the maps are an accelerator
    for (uint32_t i = 0; i < kPer; ++i) {
        DimRange& r = ranges[threadIdx.x * kPer + i];
        const uint32_t cnt = r.count & ~kDimDenseFlag;
        r.map_span = 0;
        if (!fits || !cnt || (r.count & kDimDenseFlag)) continue;
        const uint64_t span = uint64_t(r.pad) - r.tok0 + 1;
        if (span <= 8ull * cnt) {
            r.map_off = at;
            r.map_span = static_cast<uint32_t>(span);
            at += span + 1;
        }
    }
    if (threadIdx.x == 0) *total_out = fits ? total : 0;
}

// Fills the token maps: key j (rank i in its dim, token t) owns map entries
// (t - tok0, t_next - tok0], i.e. every token up to its successor's has
// i + 1 keys below it.
__global__ void k_tokmap(const uint64_t* keys, uint64_t K, const DimRange* ranges, uint32_t* map) {
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < K; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t d = static_cast<uint32_t>(keys[j] >> 32);
        const DimRange r = ranges[d];
        if (!r.map_span) continue;
        const uint32_t cnt = r.count & ~kDimDenseFlag;
        const uint64_t i = j - r.first;
        const uint32_t x0 = static_cast<uint32_t>(keys[j]) - r.tok0;
        const uint32_t x1 = i + 1 < cnt ? static_cast<uint32_t>(keys[j + 1]) - r.tok0 : r.map_span;
        for (uint32_t x = x0 + 1; x <= x1; ++x) map[r.map_off + x] = static_cast<uint32_t>(i + 1);
    }
}

// Index finalization shared by every construction path: the per-dim key
// ranges, then the dense containers.
void build_dense_containers(genie_index* ix, const uint64_t* h_off) {
    ix->dim_range.reserve(65536);
    GENIE_CUDA(cudaMemsetAsync(ix->dim_range.p, 0, 65536 * sizeof(DimRange), ix->stream));
    if (ix->K) {
        const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((ix->K + 255) / 256, uint64_t(ix->sms) * 8));
        k_dim_ranges<<<blocks, 256, 0, ix->stream>>>(ix->keys.p, ix->K, ix->dim_range.p);
        GENIE_CUDA(cudaGetLastError());
        // token maps for gapped dims whose token span is at most 8x their key
        // count (C2: 1M-word vocabulary with gaps -> one 4 MB map); a point
        // item then resolves with one map load instead of a 20-step search.
        // Planned on the device (one CTA scans the 65536 dims); only the
        // total comes back to size the map.
        DevBuf<unsigned long long> total_d;
        total_d.reserve(1);
        k_tokmap_plan<<<1, 1024, 0, ix->stream>>>(ix->dim_range.p, total_d.p);
        unsigned long long total = 0;
        GENIE_CUDA(cudaMemcpyAsync(&total, total_d.p, 8, cudaMemcpyDeviceToHost, ix->stream));
        GENIE_CUDA(cudaStreamSynchronize(ix->stream));
        if (total) {
            ix->tokmap.reserve(total);
            GENIE_CUDA(cudaMemsetAsync(ix->tokmap.p, 0, total * 4, ix->stream));
            k_tokmap<<<blocks, 256, 0, ix->stream>>>(ix->keys.p, ix->K, ix->dim_range.p, ix->tokmap.p);
            GENIE_CUDA(cudaGetLastError());
        }
    }
    const double dens = dense_density(ix);
    ix->bitmap_words = ((ix->n + 31) / 32 + 3) & ~3u;  // 16-byte rows
    // key_dense[j]: word offset of key j's bitmap row in `bitmaps`, or -1.
    // k_scan adds it to a per-thread pointer as a 32-bit index (one IMAD per
    // row load), so the rows span at most 2^31 words (8 GB): beyond that the
    // longest lists keep their bitmaps and the rest stay posting lists.
    std::vector<int32_t> slot(ix->K, -1);
    std::vector<uint64_t> dense_keys;
    if (dens > 0.0 && ix->n >= 1024) {
        for (uint64_t j = 0; j < ix->K; ++j)
            if (double(h_off[j + 1] - h_off[j]) >= dens * double(ix->n)) dense_keys.push_back(j);
        const uint64_t max_rows = ((1ull << 31) - 1) / ix->bitmap_words;
        if (dense_keys.size() > max_rows) {
            std::stable_sort(dense_keys.begin(), dense_keys.end(), [&](uint64_t a, uint64_t b) {
                return h_off[a + 1] - h_off[a] > h_off[b + 1] - h_off[b];
            });
            dense_keys.resize(max_rows);
            std::sort(dense_keys.begin(), dense_keys.end());
        }
        for (size_t d = 0; d < dense_keys.size(); ++d)
            slot[dense_keys[d]] = static_cast<int32_t>(d * ix->bitmap_words);
    }
    ix->n_dense = static_cast<uint32_t>(dense_keys.size());
    ix->key_dense.reserve(ix->K + 1);
    if (ix->K)
        GENIE_CUDA(cudaMemcpy(ix->key_dense.p, slot.data(), ix->K * sizeof(int32_t), cudaMemcpyHostToDevice));
    ix->bitmaps.reserve(std::max<size_t>(size_t(ix->n_dense) * ix->bitmap_words, 4));
    if (!ix->n_dense) return;
    GENIE_CUDA(cudaMemsetAsync(ix->bitmaps.p, 0, size_t(ix->n_dense) * ix->bitmap_words * 4, ix->stream));
    for (uint32_t d = 0; d < ix->n_dense; ++d) {
        const uint64_t j = dense_keys[d], b = h_off[j], e = h_off[j + 1];
        const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((e - b + 255) / 256, uint64_t(ix->sms) * 8));
        k_build_bitmap<<<blocks, 256, 0, ix->stream>>>(ix->postings.p, b, e,
                                                        ix->bitmaps.p + size_t(d) * ix->bitmap_words);
    }
    GENIE_CUDA(cudaStreamSynchronize(ix->stream));
    GENIE_CUDA(cudaGetLastError());
}

static void validate_csr(uint32_t n, uint64_t K, const uint64_t* keys, const uint64_t* off,
                         const uint32_t* post) {
    if (K >= (1ull << 32)) throw Error(GENIE_ERR_DATA, "index: too many keywords");
    if (off[0] != 0) throw Error(GENIE_ERR_DATA, "index: key_off[0] must be 0");
    for (uint64_t j = 0; j < K; ++j) {
        if (j && keys[j] <= keys[j - 1])
            throw Error(GENIE_ERR_DATA, "index: keywords must be strictly ascending");
        if ((keys[j] >> 32) > 0xffffu) throw Error(GENIE_ERR_DATA, "index: dim exceeds 16 bits");
        if (off[j + 1] < off[j]) throw Error(GENIE_ERR_DATA, "index: key_off must be non-decreasing");
    }
    const uint64_t P = off[K];
    // postings: ascending per key, < n (index_io.hpp:136-150 validation rules)
    const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    std::vector<int> bad(T, 0);
    for (unsigned t = 0; t < T; ++t) {
        pool.emplace_back([&, t] {
            for (uint64_t j = t; j < K; j += T) {
                for (uint64_t p = off[j]; p < off[j + 1]; ++p) {
                    if (post[p] >= n) { bad[t] = 1; return; }
                    if (p > off[j] && post[p] <= post[p - 1]) { bad[t] = 2; return; }
                }
            }
        });
    }
    for (auto& th : pool) th.join();
    for (int b : bad) {
        if (b == 1) throw Error(GENIE_ERR_DATA, "index: object id out of range");
        if (b == 2) throw Error(GENIE_ERR_DATA, "index: postings must be strictly ascending per keyword");
    }
    (void)P;
}

// ---- device build (build_index, index.hpp:190-250): one (packed keyword,
// object id) pair per object keyword, emitted in object order, so the stable
// radix sort by keyword leaves each list's ids ascending.
__global__ void k_obj_pairs(const uint64_t* obj_off, uint32_t n, const uint16_t* dims, const uint32_t* tokens,
                            uint64_t* keys, uint32_t* ids) {
    for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
        for (uint64_t i = obj_off[o]; i < obj_off[o + 1]; ++i) {
            keys[i] = (uint64_t(dims[i]) << 32) | tokens[i];
            ids[i] = o;
        }
    }
}

// a keyword repeated inside one object (ObjectRecord rejects it, model.hpp:57-62):
// the smallest such position of the sorted pairs
__global__ void k_dup_pairs(const uint64_t* keys, const uint32_t* ids, uint64_t total, unsigned long long* first) {
    for (uint64_t i = 1 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x)
        if (keys[i] == keys[i - 1] && ids[i] == ids[i - 1]) atomicMin(first, static_cast<unsigned long long>(i));
}

static genie_index* upload(uint32_t n, uint64_t K, const uint64_t* keys, const uint64_t* off,
                           const uint32_t* post, const uint32_t* dim_mult, uint32_t id_offset,
                           int device) {
    ensure_device(device);
    auto* ix = new genie_index;
    try {
        ix->device = device;
        ix->n = n;
        ix->K = K;
        ix->P = off[K];
        ix->id_offset = id_offset;
        ix->sms = sm_count(device);
        GENIE_CUDA(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
        for (auto& e : ix->ev) GENIE_CUDA(cudaEventCreate(&e));
        ix->keys.reserve(K + 1);
        ix->key_off.reserve(K + 1);
        // +64 padding: 16-byte tail loads of the scan may read past a list end
        ix->postings.reserve(ix->P + 64);
        ix->dim_mult.reserve(65536);
        if (K) GENIE_CUDA(cudaMemcpy(ix->keys.p, keys, K * sizeof(uint64_t), cudaMemcpyHostToDevice));
        GENIE_CUDA(cudaMemcpy(ix->key_off.p, off, (K + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice));
        GENIE_CUDA(cudaMemset(ix->postings.p, 0, (ix->P + 64) * sizeof(uint32_t)));
        if (ix->P)
            GENIE_CUDA(cudaMemcpy(ix->postings.p, post, ix->P * sizeof(uint32_t), cudaMemcpyHostToDevice));
        if (dim_mult) {
            GENIE_CUDA(cudaMemcpy(ix->dim_mult.p, dim_mult, 65536 * sizeof(uint32_t),
                                  cudaMemcpyHostToDevice));
        } else {
            compute_dim_stats(ix, keys, off);
        }
        build_dense_containers(ix, off);
        GENIE_CUDA(cudaDeviceSynchronize());
    } catch (...) {
        genie_index_destroy(ix);
        throw;
    }
    return ix;
}

}  // namespace genie

using namespace genie;

extern "C" {

genie_config genie_config_default(void) {
    genie_config c{};
    c.selector = GENIE_SELECT_CPQ;
    c.span_chunk = 4 * kDefaultUnit;  // 4096, engine.hpp:40
    c.max_spans_per_task = 2;
    c.tile_bytes = 0;
    c.ctas_per_sm = 0;
    c.flags = 0;
    return c;
}

int genie_index_create(uint32_t num_objects, uint64_t num_keys, const uint64_t* keys,
                       const uint64_t* key_off, const uint32_t* postings,
                       const uint32_t* dim_max_mult, uint32_t id_offset, int device,
                       genie_index** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!out || !key_off || (num_keys && (!keys)))
            throw Error(GENIE_ERR_CONTRACT, "genie_index_create: null argument");
        validate_csr(num_objects, num_keys, keys, key_off, postings);
        *out = upload(num_objects, num_keys, keys, key_off, postings, dim_max_mult, id_offset, device);
        return GENIE_OK;
    });
}

int genie_index_create_shard(uint32_t num_objects, uint64_t num_keys, const uint64_t* keys,
                             const uint64_t* key_off, const uint32_t* postings, uint32_t id_begin,
                             uint32_t id_end, int device, genie_index** out, char* err,
                             size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!out) throw Error(GENIE_ERR_CONTRACT, "genie_index_create_shard: null argument");
        if (id_begin > id_end || id_end > num_objects)
            throw Error(GENIE_ERR_CONTRACT, "genie_index_create_shard: bad id range");
        validate_csr(num_objects, num_keys, keys, key_off, postings);
        // one part of partition_dataset (index.hpp:263-291): keep ids in
        // [id_begin, id_end), rebase, drop keywords absent from the part
        std::vector<uint64_t> sb(num_keys), se(num_keys);
        for (uint64_t j = 0; j < num_keys; ++j) {
            const uint32_t* a = postings + key_off[j];
            const uint32_t* b = postings + key_off[j + 1];
            sb[j] = std::lower_bound(a, b, id_begin) - postings;
            se[j] = std::lower_bound(a, b, id_end) - postings;
        }
        std::vector<uint64_t> k2, o2{0};
        for (uint64_t j = 0; j < num_keys; ++j)
            if (se[j] > sb[j]) {
                k2.push_back(keys[j]);
                o2.push_back(o2.back() + (se[j] - sb[j]));
            }
        std::vector<uint32_t> p2(o2.back());
        uint64_t w = 0;
        for (uint64_t j = 0; j < num_keys; ++j)
            for (uint64_t p = sb[j]; p < se[j]; ++p) p2[w++] = postings[p] - id_begin;
        *out = upload(id_end - id_begin, k2.size(), k2.data(), o2.data(), p2.data(), nullptr, id_begin,
                      device);
        return GENIE_OK;
    });
}

void genie_index_destroy(genie_index* ix) {
    if (!ix) return;
    cudaSetDevice(ix->device);
    if (ix->stream) cudaStreamSynchronize(ix->stream);
    if (ix->ws.h_status) cudaFreeHost(ix->ws.h_status);
    if (ix->host_graph) cudaGraphExecDestroy(ix->host_graph);
    if (ix->h_bounds) cudaFreeHost(ix->h_bounds);
    for (auto& e : ix->ev)
        if (e) cudaEventDestroy(e);
    if (ix->stream) cudaStreamDestroy(ix->stream);
    delete ix;
}

void genie_index_info(const genie_index* ix, uint32_t* num_objects, uint64_t* num_keys,
                      uint64_t* num_postings, uint32_t* id_offset, int* device) {
    if (num_objects) *num_objects = ix->n;
    if (num_keys) *num_keys = ix->K;
    if (num_postings) *num_postings = ix->P;
    if (id_offset) *id_offset = ix->id_offset;
    if (device) *device = ix->device;
}

int genie_index_dim_stats(genie_index* ix, uint32_t* dim_max_mult, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        ensure_device(ix->device);
        GENIE_CUDA(cudaMemcpy(dim_max_mult, ix->dim_mult.p, 65536 * sizeof(uint32_t),
                              cudaMemcpyDeviceToHost));
        return GENIE_OK;
    });
}

int genie_index_export(genie_index* ix, uint64_t* keys, uint64_t* key_off, uint32_t* postings,
                       char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        ensure_device(ix->device);
        if (ix->K && keys)
            GENIE_CUDA(cudaMemcpy(keys, ix->keys.p, ix->K * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        if (key_off)
            GENIE_CUDA(cudaMemcpy(key_off, ix->key_off.p, (ix->K + 1) * sizeof(uint64_t),
                                  cudaMemcpyDeviceToHost));
        if (ix->P && postings)
            GENIE_CUDA(cudaMemcpy(postings, ix->postings.p, ix->P * sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost));
        return GENIE_OK;
    });
}

int genie_index_build(uint32_t num_objects, const uint64_t* obj_off, const uint16_t* dims, const uint32_t* tokens,
                      int device, genie_index** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        if (!out || !obj_off) throw Error(GENIE_ERR_CONTRACT, "genie_index_build: null argument");
        const uint64_t total = obj_off[num_objects];
        if (obj_off[0] != 0) throw Error(GENIE_ERR_CONTRACT, "genie_index_build: obj_off[0] must be 0");
        for (uint32_t o = 0; o < num_objects; ++o)
            if (obj_off[o + 1] < obj_off[o]) throw Error(GENIE_ERR_CONTRACT, "genie_index_build: obj_off not monotone");
        if (total && (!dims || !tokens)) throw Error(GENIE_ERR_CONTRACT, "genie_index_build: null argument");
        ensure_device(device);
        auto* ix = new genie_index;
        try {
            ix->device = device;
            ix->n = num_objects;
            ix->sms = sm_count(device);
            GENIE_CUDA(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
            for (auto& e : ix->ev) GENIE_CUDA(cudaEventCreate(&e));
            cudaStream_t s = ix->stream;
            DevBuf<uint64_t> d_off, k1, k2, uk;
            DevBuf<uint16_t> d_dims;
            DevBuf<uint32_t> d_tok, v1, runs;
            DevBuf<unsigned long long> first;
            DevBuf<int64_t> nruns;
            d_off.reserve(uint64_t(num_objects) + 1);
            d_dims.reserve(total);
            d_tok.reserve(total);
            k1.reserve(total);
            k2.reserve(total);
            v1.reserve(total);
            first.reserve(1);
            nruns.reserve(1);
            ix->postings.reserve(total + 64);
            GENIE_CUDA(cudaMemsetAsync(ix->postings.p, 0, (total + 64) * 4, s));
            GENIE_CUDA(cudaMemcpyAsync(d_off.p, obj_off, (uint64_t(num_objects) + 1) * 8, cudaMemcpyHostToDevice, s));
            if (total) {
                GENIE_CUDA(cudaMemcpyAsync(d_dims.p, dims, total * 2, cudaMemcpyHostToDevice, s));
                GENIE_CUDA(cudaMemcpyAsync(d_tok.p, tokens, total * 4, cudaMemcpyHostToDevice, s));
            }
            const unsigned grid = std::max(1u, std::min<unsigned>((num_objects + 255) / 256, ix->sms * 16));
            if (num_objects) k_obj_pairs<<<grid, 256, 0, s>>>(d_off.p, num_objects, d_dims.p, d_tok.p, k1.p, v1.p);
            cub::DoubleBuffer<uint64_t> dk(k1.p, k2.p);
            cub::DoubleBuffer<uint32_t> dv(v1.p, ix->postings.p);
            std::vector<uint64_t> hkeys, hoff{0};
            if (total) {
                size_t tmp = 0;
                GENIE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, static_cast<int64_t>(total), 0, 48, s));
                DevBuf<unsigned char> t;
                t.reserve(tmp);
                GENIE_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, dk, dv, static_cast<int64_t>(total), 0, 48, s));
                if (dv.Current() != ix->postings.p)
                    GENIE_CUDA(cudaMemcpyAsync(ix->postings.p, dv.Current(), total * 4, cudaMemcpyDeviceToDevice, s));
                GENIE_CUDA(cudaMemsetAsync(first.p, 0xff, 8, s));
                const unsigned g2 = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, uint64_t(ix->sms) * 16));
                k_dup_pairs<<<std::max(1u, g2), 256, 0, s>>>(dk.Current(), ix->postings.p, total, first.p);
                unsigned long long h_first = 0;
                GENIE_CUDA(cudaMemcpyAsync(&h_first, first.p, 8, cudaMemcpyDeviceToHost, s));
                GENIE_CUDA(cudaStreamSynchronize(s));
                if (h_first != ~0ull) {
                    uint64_t key = 0;
                    uint32_t id = 0;
                    GENIE_CUDA(cudaMemcpy(&key, dk.Current() + h_first, 8, cudaMemcpyDeviceToHost));
                    GENIE_CUDA(cudaMemcpy(&id, ix->postings.p + h_first, 4, cudaMemcpyDeviceToHost));
                    throw Error(GENIE_ERR_CONTRACT, "ObjectRecord " + std::to_string(id) + ": duplicate keyword (dim=" +
                                                        std::to_string(key >> 32) + ", token=" +
                                                        std::to_string(key & 0xffffffffull) + ")");
                }
                // list boundaries: run-length encode of the sorted keywords
                uk.reserve(total);
                runs.reserve(total);
                size_t tmp2 = 0;
                GENIE_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tmp2, dk.Current(), uk.p, runs.p, nruns.p,
                                                              static_cast<int64_t>(total), s));
                DevBuf<unsigned char> t2;
                t2.reserve(tmp2);
                GENIE_CUDA(cub::DeviceRunLengthEncode::Encode(t2.p, tmp2, dk.Current(), uk.p, runs.p, nruns.p,
                                                              static_cast<int64_t>(total), s));
                int64_t K = 0;
                GENIE_CUDA(cudaMemcpyAsync(&K, nruns.p, 8, cudaMemcpyDeviceToHost, s));
                GENIE_CUDA(cudaStreamSynchronize(s));
                hkeys.resize(K);
                std::vector<uint32_t> hruns(K);
                GENIE_CUDA(cudaMemcpy(hkeys.data(), uk.p, K * 8, cudaMemcpyDeviceToHost));
                GENIE_CUDA(cudaMemcpy(hruns.data(), runs.p, K * 4, cudaMemcpyDeviceToHost));
                hoff.resize(K + 1);
                for (int64_t j = 0; j < K; ++j) hoff[j + 1] = hoff[j] + hruns[j];
            }
            ix->K = hkeys.size();
            ix->P = total;
            ix->keys.reserve(ix->K + 1);
            ix->key_off.reserve(ix->K + 1);
            if (ix->K) GENIE_CUDA(cudaMemcpy(ix->keys.p, hkeys.data(), ix->K * 8, cudaMemcpyHostToDevice));
            GENIE_CUDA(cudaMemcpy(ix->key_off.p, hoff.data(), (ix->K + 1) * 8, cudaMemcpyHostToDevice));
            ix->dim_mult.reserve(65536);
            compute_dim_stats(ix, hkeys.data(), hoff.data());
            build_dense_containers(ix, hoff.data());
            GENIE_CUDA(cudaDeviceSynchronize());
        } catch (...) {
            genie_index_destroy(ix);
            throw;
        }
        *out = ix;
        return GENIE_OK;
    });
}

}  // extern "C"
