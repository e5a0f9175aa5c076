// Batched match-count query pipeline for B200 (sm_100a).
//
// Replaces mcx::execute_batch (engine.hpp:184-304) with Selector::cpq:
//
//   k_resolve   lookup_into + max_count_bound per query (index.hpp:86-133),
//               one warp per query, binary search over the packed keys.
//   k_plan      per-query prefix sums, counter width W = width_for(bound)
//               (cpq.hpp:63-68) and the object-tile decomposition.
//   k_worklist  tile-major (query, object tile) work list.
//   k_cut       per (query, span): positions of the object-tile boundaries
//               inside the ascending posting list (long lists are thereby
//               split into tile-aligned sub-lists).
//   k_scan      persistent CTAs over (query, tile) items: packed 4/8/16-bit
//               counters for the tile's objects live in shared memory
//               (BitmapCounter, cpq.hpp:53-120); 128-bit streaming posting
//               loads; every increment returns the new count, which feeds
//               the Count Priority Queue gate (ZipperArray + AuditThreshold,
//               cpq.hpp:294-301, 374-389) and the lock-free modified Robin
//               Hood table in shared memory (cpq.hpp:149-204).  At the end
//               of the item the CTA extracts the tile's exact top-k
//               (cpq.hpp:307-339: entries above AT-1 from the table, ties at
//               AT-1 by ascending id from the counters).
//   k_merge     per query: merge_topk over its tiles (engine.hpp:158-177);
//               exact by the partition lemma that makes execute_partitioned
//               equal execute_batch.
//
// Counters never touch HBM; every posting id of every matched span is read
// exactly once per query (the algorithmic traffic).
#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "block.cuh"
#include "internal.cuh"

namespace genie {

// ------------------------------------------------------------------ params

// Everything k_scan needs about a query, one 80-byte record (k_plan; nd is
// counted by k_cut): warp 0 prefetches it with five 16-byte asynchronous
// copies one item ahead, so preparing an item starts with it in shared memory.
struct __align__(16) QueryPlan {
    uint64_t cut_base, span_base, out_base, item0;
    uint32_t S, nt, W, k, bound, tile_base, cap, nd, nitems, pad[3];
};
static_assert(sizeof(QueryPlan) == 80, "five 16-byte copies");

struct BatchParams {
    // index
    const uint64_t* keys;
    const uint64_t* key_off;
    const uint32_t* postings;
    const uint32_t* dim_mult;
    const int32_t* key_dense;  // [K] word offset of the key's bitmap row, or -1 (< 2^31 words)
    const DimRange* dim_range; // [65536] each dim's key range
    const uint32_t* tokmap;    // token maps of gapped dims (DimRange::map_*)
    const uint32_t* keycut[kClasses]; // per work class: precomputed tile cuts of every key (or null)
    const uint32_t* bitmaps;   // [n_dense][bitmap_words]
    uint32_t bitmap_words, n_dense;
    uint32_t dense_inv[3];  // per width class W = 4, 8, 16: use a bitmap iff len * inv >= n (0: always)
    uint64_t K;
    uint32_t n;
    uint32_t id_offset;
    // queries
    uint32_t Q;
    const uint32_t* k;
    const uint64_t* item_off;
    const uint16_t* dim;
    const uint32_t* lo;
    const uint32_t* hi;
    // plan
    uint32_t tile_bits;       // counter tile allocated per CTA (bits)
    uint32_t tile_bits_w[kClasses];  // tile of class c = tile_bits_w[c] / (4 << c) objects (W = 4, 8, 16:
                                     // <= tile_bits; hashed class: hash_sub_T x GENIE_HASH_TILES)
    // hashed sparse class (class 3; hash_slots == 0: off)
    uint32_t hash_slots;  // open-addressing table slots (power of two) in the counter area
    uint32_t hash_fill;   // an item takes the table path iff its postings <= hash_fill
    uint32_t hash_pmax;   // a query joins the class iff P x T / n <= hash_pmax (expected postings per tile)
    uint32_t hash_sub_T;  // objects of one 8-bit counter sub-tile (the overflow path)
    uint32_t hash_dmax;   // ... and iff P x (W = 8 tile) / n <= hash_dmax (dense items would be overhead-bound)
    uint32_t hash_min_items;  // the class runs only with at least this many items (k_plan), else its
                              // queries go back to their dense width
    uint32_t hash_launch;     // k_scan<kHashW> is launched in this batch (else every query is folded back)
    uint32_t unit;
    uint32_t selector;
    // workspace
    uint64_t *q_bound, *q_P, *q_span_base, *q_cut_base, *q_out_base;
    uint32_t *q_S, *q_W, *q_ntiles, *q_cap, *q_tile_base, *q_rank, *q_big, *q_floor;
    uint32_t* tile_rec;  // [work items][kRecWords]: what each finished tile emitted (see gate_start)
    QueryPlan* plan;     // [Q]
    uint32_t ht_slots;
    uint32_t *it_kb, *it_nk, *it_sbase;
    uint64_t* span_beg;
    int32_t* span_dense;  // [spans] word offset of the bitmap row used for the span's list, or -1
    uint32_t* cuts;
    uint32_t *work_q, *work_t;
    uint32_t* tile_len;
    genie_entry* tile_out;
    unsigned long long* st;
    uint64_t cap_spans, cap_cuts, cap_work, cap_tout;
    // output
    uint32_t out_stride;
    genie_entry* out;
    uint32_t* out_len;
    uint32_t* out_thr;
};

__device__ __forceinline__ uint32_t wclass(uint32_t W) { return W == 4 ? 0 : (W == 8 ? 1 : (W == 16 ? 2 : 3)); }

__device__ __forceinline__ uint32_t tile_objs(const BatchParams& p, uint32_t W) {
    return p.tile_bits_w[wclass(W)] / W;
}

__device__ __forceinline__ uint32_t ntiles_for(uint32_t n, uint32_t tile_bits, uint32_t W) {
    const uint32_t T = tile_bits / W;
    return (n + T - 1) / T;
}

// ------------------------------------------------------------------ init

__global__ void k_init_status(unsigned long long* st) {
    const int i = threadIdx.x;
    if (i < ST_WORDS) {
        st[i] = (i == ST_BAD_INPUT || i == ST_BAD_BOUND || i == ST_MERGE_DUP) ? ~0ull : 0ull;
    }
}

// ---------------------------------------------------------------- resolve

// One warp per query: items -> keyword ranges (lookup_into, index.hpp:86-96),
// span counts, postings P_q and max_count_bound (index.hpp:118-133).
__global__ void __launch_bounds__(256) k_resolve(BatchParams p) {
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= p.Q) return;
    const uint64_t i0 = p.item_off[q], i1 = p.item_off[q + 1];
    const uint32_t kq = p.k[q];
    uint32_t bad = 0;
    bool lohi_bad = false;
    uint64_t bound = 0, P = 0;
    uint32_t carry = 0;
    for (uint64_t base = i0; base < i1; base += 32) {
        const uint64_t i = base + lane;
        uint32_t nk = 0, kb = 0, b = 0;
        uint64_t pp = 0;
        if (i < i1) {
            const uint32_t d = p.dim[i], l = p.lo[i], h = p.hi[i];
            if (l > h) {
                lohi_bad = true;
            } else {
                const uint64_t kl = (uint64_t(d) << 32) | l;
                // search only the dim's keys; a dim whose tokens are contiguous
                // resolves by arithmetic (LSH dims, categorical domains)
                const DimRange r = p.dim_range[d];
                const uint32_t cnt = r.count & ~kDimDenseFlag;
                uint64_t a, e;
                if (r.count & kDimDenseFlag) {
                    const uint64_t lo_off = l > r.tok0 ? uint64_t(l) - r.tok0 : 0;
                    const uint64_t hi_end = h >= r.tok0 ? uint64_t(h) - r.tok0 + 1 : 0;
                    a = r.first + (lo_off < cnt ? lo_off : cnt);
                    e = r.first + (hi_end < cnt ? hi_end : cnt);
                    if (e < a) e = a;
                } else if (r.map_span) {  // gapped dim with a token map: #keys below a token
                    const uint64_t lo_off = l > r.tok0 ? uint64_t(l) - r.tok0 : 0;
                    const uint64_t hi_end = h >= r.tok0 ? uint64_t(h) - r.tok0 + 1 : 0;
                    a = r.first + p.tokmap[r.map_off + (lo_off < r.map_span ? lo_off : r.map_span)];
                    e = l == h ? a + (a < r.first + cnt && p.keys[a] == kl)
                               : r.first + p.tokmap[r.map_off + (hi_end < r.map_span ? hi_end : r.map_span)];
                    if (e < a) e = a;
                } else {
                    const uint64_t* dk = p.keys + r.first;
                    a = r.first + lower_bound_dev(dk, cnt, kl);
                    // single-token items (the common case) need no second search:
                    // keys are unique, so the range is [a, a + (keys[a] == key))
                    e = l == h ? a + (a < r.first + cnt && p.keys[a] == kl)
                               : r.first + upper_bound_dev(dk, cnt, (uint64_t(d) << 32) | h);
                }
                kb = static_cast<uint32_t>(a);
                nk = static_cast<uint32_t>(e - a);
                pp = p.key_off[e] - p.key_off[a];
                b = min(nk, p.dim_mult[d]);
            }
        }
        const uint32_t incl = warp_inclusive_scan(nk);
        if (i < i1) {
            p.it_kb[i] = kb;
            p.it_nk[i] = nk;
            p.it_sbase[i] = carry + incl - nk;
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
        bound += warp_sum(static_cast<uint64_t>(b));
        P += warp_sum(pp);
    }
    lohi_bad = __any_sync(0xffffffffu, lohi_bad);
    if (lane != 0) return;
    if (lohi_bad) bad = 3;
    else if (i1 <= i0) bad = 1;
    else if (kq == 0) bad = 2;
    uint32_t W = 0, nt = 0;
    if (bad) {
        atomicMin(&p.st[ST_BAD_INPUT], (static_cast<unsigned long long>(q) << 8) | bad);
    } else {
        const uint64_t bnd = bound < 1 ? 1 : bound;  // engine.hpp:228
        if (bnd > 0xffffu) {                          // engine.hpp:230-233
            atomicMin(&p.st[ST_BAD_BOUND], static_cast<unsigned long long>(q));
        } else {
            W = width_for(bnd);
            // hashed sparse class: counts fit 8 bits, the spans one staging
            // batch, the W = 8 path would cut the objects into several tiles
            // that each get few postings (expected <= hash_dmax: such items
            // are bound by their fixed per-item work), and the query's
            // postings are few for a hashed tile's objects (expected per tile
            // <= hash_pmax; a tile that still gets more than the table takes
            // takes the sub-tile path in k_scan)
            if (W <= 8 && p.hash_slots && p.selector == GENIE_SELECT_CPQ && P > 0 && carry <= kSpanBatch &&
                i1 - i0 <= kSpanBatch && p.n > tile_objs(p, 8) &&
                P * tile_objs(p, 8) <= uint64_t(p.hash_dmax) * p.n &&
                P * (p.tile_bits_w[3] / kHashW) <= uint64_t(p.hash_pmax) * p.n)
                W = kHashW;
            nt = (P == 0 || p.n == 0) ? 0 : ntiles_for(p.n, p.tile_bits_w[wclass(W)], W);
        }
    }
    p.q_bound[q] = bound;
    p.q_S[q] = carry;
    p.q_P[q] = P;
    p.q_floor[q] = 0;
    p.q_W[q] = W;
    p.q_ntiles[q] = nt;
    if (nt) atomicAdd(&p.st[ST_TOTAL_POSTINGS], static_cast<unsigned long long>(P));
}

// ------------------------------------------------------------------- plan

// Single CTA: exclusive prefix sums over queries and the width classes.
__global__ void __launch_bounds__(1024) k_plan(BatchParams p) {
    __shared__ unsigned long long sums[32];
    __shared__ uint32_t s_hash_items;
    unsigned long long c_span = 0, c_cut = 0, c_tile = 0, c_out = 0, c_cls = 0, c_cls3 = 0;
    uint32_t max_nt = 0;
    // The hashed class is its own k_scan launch after the dense classes: with
    // too few items to occupy the GPU it would only add a tail (a handful of
    // sparse queries in a dense batch), so its queries then go back to their
    // dense width (results do not depend on the class)
    if (threadIdx.x == 0) s_hash_items = 0;
    __syncthreads();
    if (p.hash_slots) {
        uint32_t mine = 0;
        for (uint32_t q = threadIdx.x; q < p.Q; q += blockDim.x)
            if (p.q_W[q] == kHashW) mine += p.q_ntiles[q];
        mine = warp_sum(mine);
        if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_hash_items, mine);
    }
    __syncthreads();
    const bool want = s_hash_items && s_hash_items >= p.hash_min_items;
    const bool demote = !(want && p.hash_launch);
    if (threadIdx.x == 0) p.st[ST_HASH_WANT] = want ? 1ull : 0ull;
    for (uint32_t base = 0; base < p.Q; base += blockDim.x) {
        const uint32_t q = base + threadIdx.x;
        unsigned long long v_span = 0, v_cut = 0, v_tile = 0, v_out = 0, v_cls = 0, v_cls3 = 0;
        uint32_t cap = 0, W = 0, nt = 0;
        if (q < p.Q) {
            nt = p.q_ntiles[q];
            W = p.q_W[q];
            if (W == kHashW && demote) {
                const uint64_t qb = p.q_bound[q];
                W = width_for(qb < 1 ? 1 : qb);
                nt = ntiles_for(p.n, p.tile_bits_w[wclass(W)], W);
                p.q_W[q] = W;
                p.q_ntiles[q] = nt;
            }
            if (nt) {
                const uint32_t T = tile_objs(p, W);
                const uint32_t kq = p.k[q];
                // a hashed tile whose postings overflow the table emits the
                // top-k of each of its 8-bit sub-tiles (k_scan): up to
                // ceil(T / hash_sub_T) x k entries
                cap = W == kHashW ? min(uint32_t(min(uint64_t(kq) * ((T + p.hash_sub_T - 1) / p.hash_sub_T),
                                                     uint64_t(0xffffffffu))), T)
                                  : min(kq, T);
                // single-tile queries read each item's contiguous keyword
                // range directly (no per-keyword spans / cuts)
                v_span = nt > 1 ? p.q_S[q] : 0u;
                v_cut = nt > 1 ? static_cast<unsigned long long>(p.q_S[q]) * (nt + 1) : 0ull;
                v_tile = nt;
                v_out = static_cast<unsigned long long>(nt) * cap;
                if (W == kHashW) v_cls3 = 1;
                else v_cls = 1ull << (21 * wclass(W));
            }
            max_nt = max(max_nt, nt);
        }
        unsigned long long t_span, t_cut, t_tile, t_out, t_cls, t_cls3;
        const unsigned long long e_span = block_exclusive_scan(v_span, sums, t_span);
        const unsigned long long e_cut = block_exclusive_scan(v_cut, sums, t_cut);
        const unsigned long long e_tile = block_exclusive_scan(v_tile, sums, t_tile);
        const unsigned long long e_out = block_exclusive_scan(v_out, sums, t_out);
        const unsigned long long e_cls = block_exclusive_scan(v_cls, sums, t_cls);
        const unsigned long long e_cls3 = block_exclusive_scan(v_cls3, sums, t_cls3);
        if (q < p.Q) {
            p.q_span_base[q] = c_span + e_span;
            p.q_cut_base[q] = c_cut + e_cut;
            p.q_tile_base[q] = static_cast<uint32_t>(c_tile + e_tile);
            p.q_out_base[q] = c_out + e_out;
            p.q_cap[q] = cap;
            const unsigned long long r = c_cls + e_cls;
            p.q_rank[q] = !nt ? 0u
                          : W == kHashW ? static_cast<uint32_t>(c_cls3 + e_cls3)
                                        : static_cast<uint32_t>((r >> (21 * wclass(W))) & 0x1fffffull);
            QueryPlan pl;
            pl.cut_base = c_cut + e_cut;
            pl.span_base = c_span + e_span;
            pl.out_base = c_out + e_out;
            pl.item0 = p.item_off[q];
            pl.S = p.q_S[q];
            pl.nt = nt;
            pl.W = W;
            pl.k = p.k[q];
            const uint64_t qb = p.q_bound[q];
            pl.bound = qb < 1 ? 1u : (qb > 0xffffffffull ? 0xffffffffu : static_cast<uint32_t>(qb));
            pl.tile_base = static_cast<uint32_t>(c_tile + e_tile);
            pl.cap = cap;
            pl.nd = 0;  // k_cut counts the query's dense spans
            pl.nitems = static_cast<uint32_t>(p.item_off[q + 1] - pl.item0);
            pl.pad[0] = pl.pad[1] = pl.pad[2] = 0;
            p.plan[q] = pl;
        }
        c_span += t_span;
        c_cut += t_cut;
        c_tile += t_tile;
        c_out += t_out;
        c_cls += t_cls;
        c_cls3 += t_cls3;
    }
    if (threadIdx.x == 0) {
        p.st[ST_TOTAL_SPANS] = c_span;
        p.st[ST_TOTAL_CUTS] = c_cut;
        p.st[ST_TOTAL_WORK] = c_tile;
        p.st[ST_TOTAL_TOUT] = c_out;
        p.st[ST_CLASS0] = c_cls & 0x1fffffull;
        p.st[ST_CLASS1] = (c_cls >> 21) & 0x1fffffull;
        p.st[ST_CLASS2] = (c_cls >> 42) & 0x1fffffull;
        p.st[ST_CLASS3] = c_cls3;
        if (c_span > p.cap_spans || c_cut > p.cap_cuts || c_tile > p.cap_work ||
            c_out > p.cap_tout)
            p.st[ST_OVERFLOW] = 1;
    }
}

// --------------------------------------------------------------- worklist

// Class-major, then tile-major order: the width classes follow each other
// (one k_scan launch each); within a class all queries' tile 0, then tile 1,
// ..., queries in request order.  Items of the same tile read the same slice
// of every hot list, so the hot slice of the index stays L2-resident while
// the batch sweeps it.
__global__ void __launch_bounds__(256) k_worklist(BatchParams p) {
    // one warp per query, lanes over its tiles
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (q >= p.Q || p.st[ST_OVERFLOW]) return;
    const uint32_t nt = p.q_ntiles[q];
    if (!nt) return;
    const uint32_t c = wclass(p.q_W[q]);
    uint64_t cnt[kClasses], ntc[kClasses];
    for (int i = 0; i < kClasses; ++i) {
        cnt[i] = p.st[class_st(i)];
        ntc[i] = p.n ? ntiles_for(p.n, p.tile_bits_w[i], 4u << i) : 0;
    }
    const uint32_t rank = p.q_rank[q];
    const uint32_t tbase = p.q_tile_base[q];
    uint64_t cbase = 0;  // items of the lower width classes
    for (uint32_t i = 0; i < c; ++i) cbase += cnt[i] * ntc[i];
    for (uint32_t t = lane; t < nt; t += 32) {
        const uint64_t item = cbase + uint64_t(t) * cnt[c] + rank;
        p.work_q[item] = q;
        p.work_t[item] = t;
        uint4* rec = reinterpret_cast<uint4*>(p.tile_rec + uint64_t(tbase + t) * kRecWords);
#pragma unroll
        for (uint32_t j = 0; j < kRecWords / 4; ++j) rec[j] = make_uint4(0, 0, 0, 0);
    }
}

// -------------------------------------------------------------------- cut

// One warp per group of G (query, span)s: lane l < G resolves span l of the
// group (its query, keyword list and dense slot -- a chain of dependent
// loads), then the warp's lanes run over the group's flattened (span, tile
// boundary) pairs: the position of every object-tile boundary inside each
// list (lower_bound on the ascending ids).  G grows with the span count so
// batches of many short spans (C4: 128 per query) overlap their header
// chains instead of resolving one span per warp; G = 1 when spans are few.
__global__ void __launch_bounds__(256) k_cut(BatchParams p) {
    if (p.st[ST_OVERFLOW]) return;
    const uint64_t total = p.st[ST_TOTAL_SPANS];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t per = (total * GENIE_CUT_GROUP_MUL + nwarps - 1) / nwarps;
    const uint32_t G = per < 1 ? 1u : (per > 32 ? 32u : static_cast<uint32_t>(per));
    for (uint64_t g0 = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * G; g0 < total;
         g0 += nwarps * G) {
        const uint64_t g = g0 + lane;
        uint32_t npair = 0, len = 0, nt = 0, T = 0, cst = 0;
        uint64_t beg = 0, cbase = 0, krow = 0;  // krow: address of the key's row of the cut table (0: none)
        if (lane < G && g < total) {
            // query owning global span g (last q with span_base <= g)
            const uint32_t q = static_cast<uint32_t>(upper_bound_dev(p.q_span_base, p.Q, g) - 1);
            const uint32_t s = static_cast<uint32_t>(g - p.q_span_base[q]);
            const uint64_t i0 = p.item_off[q], i1 = p.item_off[q + 1];
            const uint64_t it = i0 + upper_bound_dev(p.it_sbase + i0, i1 - i0, s) - 1;
            const uint64_t j = p.it_kb[it] + (s - p.it_sbase[it]);
            beg = p.key_off[j];
            len = static_cast<uint32_t>(p.key_off[j + 1] - beg);
            // the list's bitmap replaces its posting scan when the list is dense
            // enough for this query's counter width (bit-sliced / lane-wise adds
            // per 32 objects vs. an atomic per posting)
            const uint32_t cls = wclass(p.q_W[q]);  // the hashed class never uses bitmaps
            int32_t ds = p.n_dense && cls < 3 ? p.key_dense[j] : -1;
            const uint32_t inv = p.dense_inv[cls < 3 ? cls : 0];
            if (ds >= 0 && inv && uint64_t(len) * inv < p.n) ds = -1;
            p.span_beg[g] = beg;
            p.span_dense[g] = ds;
            if (ds >= 0) atomicAdd(&p.plan[q].nd, 1u);  // dense spans per query
            // k_scan uses the bitmaps when all of the query's spans fit one
            // staging batch; then this list needs no tile cuts
            if (!(ds >= 0 && p.q_S[q] <= kSpanBatch)) {
                nt = p.q_ntiles[q];
                T = tile_objs(p, p.q_W[q]);
                // boundary-major: boundary b of span s at q_cut_base + b * S + s,
                // so an item (q, t) stages rows t and t + 1 with coalesced loads
                cst = p.q_S[q];
                cbase = p.q_cut_base[q] + s;
                npair = nt + 1;
                if (const uint32_t* kc = p.keycut[wclass(p.q_W[q])]) krow = reinterpret_cast<uint64_t>(kc + j * (nt + 1));
            }
        }
        // Short lists: the whole warp streams the list once (coalesced) and a
        // tile boundary is cut where consecutive postings change tile --
        // ceil(len / 32) loads instead of nt - 1 binary searches (C4: ~244
        // postings, 21 boundaries per list).
        uint32_t lin = __ballot_sync(0xffffffffu, npair && len <= kCutLinearMax);
        if (lin & (1u << lane)) npair = 0;
        while (lin) {
            const int o = __ffs(lin) - 1;
            lin &= lin - 1;
            const uint32_t o_len = __shfl_sync(0xffffffffu, len, o), o_nt = __shfl_sync(0xffffffffu, nt, o);
            const uint32_t o_T = __shfl_sync(0xffffffffu, T, o), o_st = __shfl_sync(0xffffffffu, cst, o);
            const uint64_t o_beg = __shfl_sync(0xffffffffu, beg, o), o_cb = __shfl_sync(0xffffffffu, cbase, o);
            uint32_t* cut = p.cuts + o_cb;
            if (lane == 0) {
                cut[0] = 0;
                cut[uint64_t(o_nt) * o_st] = o_len;
            }
            uint32_t carry = 0;  // tile of the posting before this chunk (0 before the first)
            for (uint32_t c0 = 0; c0 < o_len; c0 += 32 * kCutLinearUnroll) {
                // every load of the chunk in flight at once
                uint32_t v[kCutLinearUnroll];
#pragma unroll
                for (uint32_t u = 0; u < kCutLinearUnroll; ++u) {
                    const uint32_t i = c0 + u * 32 + lane;
                    v[u] = i < o_len ? __ldg(p.postings + o_beg + i) : 0u;
                }
#pragma unroll
                for (uint32_t u = 0; u < kCutLinearUnroll; ++u) {
                    const uint32_t b0 = c0 + u * 32;
                    if (b0 >= o_len) break;  // warp-uniform
                    const uint32_t i = b0 + lane;
                    const uint32_t ti = i < o_len ? v[u] / o_T : 0xffffffffu;
                    uint32_t tp = __shfl_up_sync(0xffffffffu, ti, 1);
                    if (lane == 0) tp = carry;
                    // boundaries b in (tp, ti] start at posting i (b < nt; b = nt is the end)
                    if (i < o_len)
                        for (uint32_t b = tp + 1; b <= ti && b < o_nt; ++b) cut[uint64_t(b) * o_st] = i;
                    carry = __shfl_sync(0xffffffffu, ti, min(31u, o_len - 1 - b0));
                }
            }
            // boundaries past the last posting's tile: all postings precede them
            for (uint32_t b = carry + 1 + lane; b < o_nt; b += 32) cut[uint64_t(b) * o_st] = o_len;
        }
        const uint32_t incl = warp_inclusive_scan(npair);
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t r = 0; r < tot; r += 32) {
            const uint32_t idx = r + lane;
            // owning lane: the number of lanes whose pairs all precede idx
            uint32_t o = 0;
#pragma unroll
            for (uint32_t step = 16; step; step >>= 1)
                if (__shfl_sync(0xffffffffu, incl, o + step - 1) <= idx) o += step;
            const uint32_t o_incl = __shfl_sync(0xffffffffu, incl, o & 31);
            const uint32_t o_np = __shfl_sync(0xffffffffu, npair, o & 31);
            const uint32_t o_len = __shfl_sync(0xffffffffu, len, o & 31);
            const uint32_t o_nt = __shfl_sync(0xffffffffu, nt, o & 31);
            const uint32_t o_T = __shfl_sync(0xffffffffu, T, o & 31);
            const uint64_t o_beg = __shfl_sync(0xffffffffu, beg, o & 31);
            const uint64_t o_cb = __shfl_sync(0xffffffffu, cbase, o & 31);
            const uint32_t o_st = __shfl_sync(0xffffffffu, cst, o & 31);
            const uint64_t o_krow = __shfl_sync(0xffffffffu, krow, o & 31);
            if (idx < tot) {
                const uint32_t b = idx - (o_incl - o_np);
                uint32_t v;
                if (b == 0) v = 0;
                else if (b == o_nt) v = o_len;
                else if (o_krow) v = reinterpret_cast<const uint32_t*>(o_krow)[b];
                else v = static_cast<uint32_t>(lower_bound_dev(p.postings + o_beg, o_len, b * o_T));
                p.cuts[o_cb + uint64_t(b) * o_st] = v;
            }
        }
    }
}

// ------------------------------------------------------------------- scan

// Staged slices of one item (double-buffered: warp 0 stages item i + 1 while
// the other warps scan item i).
struct StageBuf {
    uint8_t* base;
    // slice start (absolute posting position)
    __device__ __forceinline__ uint64_t* beg() const { return reinterpret_cast<uint64_t*>(base); }
    // postings before each slice (kSpanBatch + 1 entries): slice i has
    // ppref[i + 1] - ppref[i] postings (0 for dense spans)
    __device__ __forceinline__ uint32_t* ppref() const { return reinterpret_cast<uint32_t*>(base + kSpanBatch * 8); }
    // rank of the slice's first 128-posting group
    __device__ __forceinline__ uint32_t* upref() const {
        return reinterpret_cast<uint32_t*>(base + kSpanBatch * 12 + 16);
    }
    // dense-container slots of the staged spans, in span order
    __device__ __forceinline__ uint32_t* dense() const {
        return reinterpret_cast<uint32_t*>(base + kSpanBatch * 16 + 16);
    }
};

// One work item as prepared by warp 0 (prepare_item); 64 bytes.
struct ItemDesc {
    uint32_t valid, q, t, kq, bound, W, cap, nt, S, nd, G, a0;
    uint64_t out_base;
    uint32_t tile_slot;  // q_tile_base[q] + t: the item's tile_len / tile_rec slot
    uint32_t ptot;       // postings of the first staged batch
};

// Shared memory of a scan CTA.  Everything but the counters sits at a fixed
// offset from the dynamic shared base (compile-time addresses, no pointer
// registers); the counter tile comes last because its size is a knob.
struct ScanSmem {
    uint32_t* cnt;             // packed counters of the tile
    uint64_t* ht;              // Robin Hood table / histogram scratch
    uint32_t* za;              // ZipperArray, levels [0, bound]
    unsigned long long* sums;  // block scan scratch (32)
    uint32_t* scal;            // scalars
    ItemDesc* desc;            // [2]
    QueryPlan* plan;           // prefetched plan of the query prepare_item works on next
    uint8_t* stage;            // 2 x StageBuf
    __device__ __forceinline__ StageBuf sb(uint32_t b) const { return StageBuf{stage + b * (kSpanBatch * 20 + 16)}; }
};

enum ScalarSlot {
    SC_AT = 1,          // live AuditThreshold
    SC_OVF = 2,         // table overflow -> histogram fallback
    SC_NOUT = 3,        // entries emitted by the item
    SC_UCTR = 4,        // guided-scheduling cursor
    SC_T = 7,           // hist_select scratch
    SC_HTHR = 5,        // hashed items: AT - 1, entries above it, the tie cut (bin, rank in bin, id)
    SC_HABOVE = 6,
    SC_HBIN = 8,
    SC_HNEED = 9,
    SC_HCUT = 11,
    SC_FLOOR = 10,      // gate start of the item
    SC_PF_ITEM = 13,    // the item the next prepare_item prepares (claimed and resolved), its query and tile
    SC_PF_Q = 14,
    SC_PF_T = 15,
    SC_CLAIM = 28,      // the item after it: claimed, not yet resolved to (query, tile)
    SC_LVL = 16,        // dense-phase level counts (kLvl <= 8)
    SC_ADM_CALLS = 24,  // instrumented builds only
    SC_ADM_PASS = 25,
    SC_WMAX = 26,       // instrumented builds: slowest / fastest scan warp of the item
    SC_WMIN = 27,
    SC_WORDS = 31
};
static_assert(SC_WORDS <= 32, "scalar area");

namespace smem_off {
constexpr uint32_t kScal = 0;                                  // SC_WORDS u32 (<= 32)
constexpr uint32_t kSums = 128;                                // 32 u64
constexpr uint32_t kDesc = kSums + 256;                        // 2 x ItemDesc
#if GENIE_PLAN_AT_END  // the QueryPlan slot after the tile (carve); the fixed area keeps round 1's offsets
constexpr uint32_t kZa = kDesc + 2 * sizeof(ItemDesc);         // kZaMax u32
#else
constexpr uint32_t kPlan = kDesc + 2 * sizeof(ItemDesc);       // QueryPlan of the next item's query
constexpr uint32_t kZa = kPlan + sizeof(QueryPlan);            // kZaMax u32
#endif
constexpr uint32_t kStage = kZa + kZaMax * 4;                  // 2 x StageBuf
constexpr uint32_t kStageBytes = kSpanBatch * (8 + 4 + 4 + 4) + 16;
// ht_slots u64, then the counter tile (start aligned to GENIE_HT_ALIGN bytes)
constexpr uint32_t kHt = (kStage + 2 * kStageBytes + GENIE_HT_ALIGN - 1) / GENIE_HT_ALIGN * GENIE_HT_ALIGN;
static_assert(kHt % 16 == 0, "16-byte aligned table");
}  // namespace smem_off

__device__ __forceinline__ ScanSmem carve(uint8_t* base, uint32_t ht_slots, uint32_t tile_bytes) {
    using namespace smem_off;
    ScanSmem s;
    s.scal = reinterpret_cast<uint32_t*>(base + kScal);
    s.sums = reinterpret_cast<unsigned long long*>(base + kSums);
    s.desc = reinterpret_cast<ItemDesc*>(base + kDesc);
#if GENIE_PLAN_AT_END
    s.plan = reinterpret_cast<QueryPlan*>(base + kHt + size_t(ht_slots) * 8 + tile_bytes);
#else
    s.plan = reinterpret_cast<QueryPlan*>(base + kPlan);
    (void)tile_bytes;
#endif
    s.za = reinterpret_cast<uint32_t*>(base + kZa);
    s.stage = base + kStage;
    static_assert(kStageBytes == kSpanBatch * 20 + 16, "stage buffer layout");
    s.cnt = reinterpret_cast<uint32_t*>(base + kHt);
    s.ht = nullptr;  // per item: right after the item's counters (process_item)
    (void)ht_slots;
    return s;
}

inline size_t scan_smem_bytes(uint32_t tile_bytes, uint32_t ht_slots) {
    return smem_off::kHt + size_t(ht_slots) * 8 + tile_bytes + (GENIE_PLAN_AT_END ? sizeof(QueryPlan) : 0);
}

__device__ __forceinline__ uint32_t ht_home(uint32_t id, uint32_t mask) {
    return static_cast<uint32_t>(mix64(id)) & mask;
}

__device__ __forceinline__ uint64_t pack_slot(uint32_t id, uint32_t v, uint32_t age) {
    return (uint64_t(id) << 32) | (uint64_t(v & 0xffffu) << 16) | uint64_t(age & 0xffffu);
}

// Lock-free modified Robin Hood insert in shared memory; the same protocol
// as CountHashTable::insert (cpq.hpp:149-204): empty -> claim, same id ->
// raise value keeping age, dead resident (value + 1 < AT) -> overwrite,
// younger resident -> displace and keep probing with it.  Returns false when
// the table is full (the caller falls back to an exact histogram select).
__device__ __forceinline__ bool ht_insert(uint64_t* ht, uint32_t cap, uint32_t id, uint32_t value,
                          uint32_t cur_at) {
    const uint32_t mask = cap - 1;
    uint64_t carried = pack_slot(id, value, 0);
    uint32_t slot = ht_home(id, mask);
    for (uint32_t probes = 0; probes <= cap; ++probes) {
        unsigned long long* addr = reinterpret_cast<unsigned long long*>(&ht[slot]);
        uint64_t res = *reinterpret_cast<volatile uint64_t*>(&ht[slot]);
        bool advance = false;
        while (!advance) {
            if (res == kEmptySlot) {
                const uint64_t prev = atomicCAS(addr, kEmptySlot, carried);
                if (prev == kEmptySlot) return true;
                res = prev;
                continue;
            }
            const uint32_t rid = uint32_t(res >> 32), rv = uint32_t(res >> 16) & 0xffffu,
                           rage = uint32_t(res) & 0xffffu;
            const uint32_t cid = uint32_t(carried >> 32), cv = uint32_t(carried >> 16) & 0xffffu,
                           cage = uint32_t(carried) & 0xffffu;
            if (rid == cid) {
                if (rv >= cv) return true;
                const uint64_t merged = pack_slot(rid, cv, rage);
                const uint64_t prev = atomicCAS(addr, res, merged);
                if (prev == res) return true;
                res = prev;
                continue;
            }
            if (uint64_t(rv) + 1 < cur_at) {  // dead: cannot reach top-k any more
                const uint64_t prev = atomicCAS(addr, res, carried);
                if (prev == res) return true;
                res = prev;
                continue;
            }
            if (rage < cage) {  // Robin Hood displacement
                const uint64_t prev = atomicCAS(addr, res, carried);
                if (prev == res) {
                    carried = res;
                    advance = true;
                    continue;
                }
                res = prev;
                continue;
            }
            advance = true;
        }
        slot = (slot + 1) & mask;
        const uint32_t age = uint32_t(carried) & 0xffffu;
        if (age >= 0xffffu) break;
        carried += 1;
    }
    return false;
}

// ---------------------------------------------------------------- layouts

// Counter layouts of a tile (x = object id relative to the tile origin, which
// is a multiple of 32).  Both pack 32/W counters per 32-bit word and 32
// objects per W words:
//   linear       word x / kPer, lane x % kPer (ids ascend inside a word): the
//                cheapest address arithmetic for the posting scan;
//   interleaved  word (x / 32) * W + x % W, lane (x % 32) / W: bit j of a
//                dense bitmap word lands in word j % W at lane j / W, so a
//                dense list adds into a 32-object block with W shift-and-mask
//                steps (no bit spreading), and the counters equal to T of a
//                block gather into one id-ordered 32-bit mask with W shifts.
// Items of a query with dense containers use the interleaved layout.
template <int W, bool IL>
struct Lay {
    static constexpr uint32_t kPer = 32 / W;
    static constexpr uint32_t kLogW = W == 4 ? 2 : (W == 8 ? 3 : 4);
    static constexpr uint32_t kLogPer = 5 - kLogW;
    static constexpr uint32_t kMask = (1u << W) - 1u;
    __device__ static __forceinline__ uint32_t word(uint32_t x) {
        if constexpr (IL) return ((x >> 5) << kLogW) | (x & (W - 1));
        else return x >> kLogPer;
    }
    __device__ static __forceinline__ uint32_t lane(uint32_t x) {
        if constexpr (IL) return (x >> kLogW) & (kPer - 1);
        else return x & (kPer - 1);
    }
    __device__ static __forceinline__ uint32_t obj(uint32_t wi, uint32_t l) {
        if constexpr (IL) return ((wi >> kLogW) << 5) | (l << kLogW) | (wi & (W - 1));
        else return wi * kPer + l;
    }
    __device__ static __forceinline__ uint32_t get(const uint32_t* cnt, uint32_t x) {
        return (cnt[word(x)] >> (lane(x) * W)) & kMask;
    }
};

// Lane-wise SWAR compares of packed W-bit counters: the top bit of every lane
// whose counter equals / is at least v (1 <= v < 2^W).
template <int W>
struct Swar {
    static constexpr uint32_t kOnes = W == 4 ? 0x11111111u : (W == 8 ? 0x01010101u : 0x00010001u);
    static constexpr uint32_t kHigh = kOnes << (W - 1);
    static constexpr uint32_t kLow = ~kHigh;
    __device__ static __forceinline__ uint32_t eq(uint32_t x, uint32_t v) {
        const uint32_t y = x ^ (v * kOnes);
        return ~(((y & kLow) + kLow) | y | kLow);
    }
    __device__ static __forceinline__ uint32_t ge(uint32_t x, uint32_t v) {
        const uint32_t y = v * kOnes;
        const uint32_t d = (x | kHigh) - (y & kLow);  // lane top bit: low(x) >= low(y)
        return ((x & ~y) | (~(x ^ y) & d)) & kHigh;
    }
};

struct ItemCtx {
    uint32_t q, t, kq, bound, tile_lo, tile_n, words, ht_cap, cap, slot;
    uint32_t rec_b;  // base level of the tile's record (every emitted entry counts >= rec_b)
    uint64_t out_base;
    bool gate;   // Selector::cpq semantics: tile records, query floor
    bool admit;  // ... and the scan-time c-PQ gate (admissions); else the tile's exact histogram select
};

// The c-PQ admission path (cpq.hpp:294-301): the new value passed the
// register copy of the gate, so re-check against the live AuditThreshold,
// insert into the table, bump ZA[val] and advance AT while ZA[AT] >= k
// (cpq.hpp:374-389).  Rare once AT has climbed; kept out of line so the scan
// loop stays small.  Returns the refreshed gate comparand.
template <int W>
__device__ __noinline__ uint32_t cpq_admit(uint64_t* ht, uint32_t* za, uint32_t* scal, uint32_t ht_cap,
                                           uint32_t bound, uint32_t kq, uint32_t local, uint32_t old,
                                           uint32_t sh) {
    constexpr uint32_t kMask = (W == 32) ? 0xffffffffu : ((1u << W) - 1u);
    const uint32_t val = ((old >> sh) & kMask) + 1;
    volatile uint32_t* s_at = scal + SC_AT;
    uint32_t a = *s_at;
#ifdef GENIE_PHASE_TIMERS
    atomicAdd(&scal[SC_ADM_CALLS], 1u);
    if (val >= a) atomicAdd(&scal[SC_ADM_PASS], 1u);
#endif
    if (val >= a) {
        if (!ht_insert(ht, ht_cap, local, val, a)) scal[SC_OVF] = 1;
        atomicAdd(&za[val], 1u);
        a = *s_at;
        while (a <= bound && reinterpret_cast<volatile uint32_t*>(za)[a] >= kq) {
            atomicCAS(scal + SC_AT, a, a + 1);
            a = *s_at;
        }
    }
    return (a - 1) << (32 - W);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Shared-memory atomic add on a 32-bit shared-window address (no memory
// clobber: the counters are only read after a __syncthreads()).
__device__ __forceinline__ uint32_t atom_add_shared(uint32_t addr, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v));
    return old;
}

__device__ __forceinline__ void emit(const BatchParams& p, const ItemCtx& it, const ScanSmem& sm,
                                     uint32_t local, uint32_t count) {
    const uint32_t pos = atomicAdd(&sm.scal[SC_NOUT], 1u);
    if (it.gate) {  // the tile's record: #emitted entries counting >= rec_b + j
        uint32_t* rec = p.tile_rec + uint64_t(it.slot) * kRecWords;
#pragma unroll
        for (int j = 0; j < kRecLevels; ++j)
            if (count >= it.rec_b + j) atomicAdd(rec + 1 + j, 1u);
    }
    genie_entry e;
    e.id = local + it.tile_lo;
    e.count = count;
    p.tile_out[it.out_base + pos] = e;
}

// Id-ordered mask of the counters equal to T in the 32-object block whose
// W words are w[0..W) (interleaved layout: object j sits in word j % W at
// lane j / W, and Swar::eq flags bit lane * W + W - 1).
template <int W>
__device__ __forceinline__ uint32_t block_eq_mask_il(const uint32_t* w, uint32_t T) {
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < W; ++j) m |= Swar<W>::eq(w[j], T) >> (W - 1 - j);
    return m;
}

// Ties at T in ascending local id, the first `need` of them
// (cpq.hpp:330-336).  Ordered block scan over the counter words; stops as
// soon as enough ties were seen.
template <int W, bool IL>
__device__ void emit_ties(const BatchParams& p, const ItemCtx& it, const ScanSmem& sm, uint32_t T,
                          uint32_t need) {
    unsigned long long seen = 0;
    if constexpr (IL) {
        // one 32-object block (W words) per thread per step
        const uint32_t nblk = it.words / W;
        for (uint32_t g0 = 0; g0 < nblk; g0 += blockDim.x) {
            const uint32_t gi = g0 + threadIdx.x;
            uint32_t m = 0;
            if (gi < nblk) {
                uint32_t w[W];
                const uint4* c4 = reinterpret_cast<const uint4*>(sm.cnt + gi * W);
#pragma unroll
                for (int j = 0; j < W / 4; ++j) {
                    const uint4 x = c4[j];
                    w[4 * j] = x.x;
                    w[4 * j + 1] = x.y;
                    w[4 * j + 2] = x.z;
                    w[4 * j + 3] = x.w;
                }
                m = block_eq_mask_il<W>(w, T);
            }
            unsigned long long total;
            unsigned long long r = seen + block_exclusive_scan<unsigned long long>(__popc(m), sm.sums, total);
            while (m && r < need) {
                const uint32_t bit = __ffs(m) - 1;
                m &= m - 1;
                emit(p, it, sm, gi * 32 + bit, T);
                ++r;
            }
            seen += total;
            if (seen >= need) break;  // uniform: total is block-wide
        }
    } else {
        using Sw = Swar<W>;
        constexpr uint32_t kPer = 32 / W;
        constexpr uint32_t WPT = 4;  // counter words per thread per step (one 16-byte load)
        const uint4* c4 = reinterpret_cast<const uint4*>(sm.cnt);
        const uint32_t w4 = it.words / 4;
        for (uint32_t g0 = 0; g0 < w4; g0 += blockDim.x) {
            const uint32_t gi = g0 + threadIdx.x;
            uint32_t m[WPT] = {0, 0, 0, 0};
            if (gi < w4) {
                const uint4 x = c4[gi];
                m[0] = Sw::eq(x.x, T);
                m[1] = Sw::eq(x.y, T);
                m[2] = Sw::eq(x.z, T);
                m[3] = Sw::eq(x.w, T);
            }
            const uint32_t c = __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
            unsigned long long total;
            unsigned long long r = seen + block_exclusive_scan<unsigned long long>(c, sm.sums, total);
#pragma unroll
            for (uint32_t j = 0; j < WPT; ++j) {
                while (m[j] && r < need) {
                    const uint32_t bit = __ffs(m[j]) - 1;
                    m[j] &= m[j] - 1;
                    emit(p, it, sm, (gi * WPT + j) * kPer + bit / W, T);
                    ++r;
                }
            }
            seen += total;
            if (seen >= need) break;  // uniform: total is block-wide
        }
    }
}

// Exact histogram k-selection over the tile counters (GEN-SPQ ablation and
// the fallback when the table overflowed): T = k-th largest count in the
// tile, zeros included (0 if fewer than k non-zero), then every count > T
// and the first ties at T in ascending id.
template <int W, bool IL>
__device__ uint32_t hist_select(const BatchParams& p, const ItemCtx& it0, const ScanSmem& sm) {
    ItemCtx it = it0;  // rec_b is set once T is known
    using L = Lay<W, IL>;
    constexpr uint32_t kPer = 32 / W;
    const int nsub = static_cast<int>(it.ht_cap * 8 / 1024);  // 256-bin sub-histograms in the table's space
    const int warp = (threadIdx.x >> 5) % nsub;
    const int nwarps = nsub;
    uint32_t* h = reinterpret_cast<uint32_t*>(sm.ht);
    // level 1: high byte of the count (W == 16) or the count itself (W <= 8)
    constexpr uint32_t kShift1 = W == 16 ? 8 : 0;
    uint32_t T = 0, above = 0;
    uint32_t hi_sel = 0;
    unsigned long long cum_above = 0;
    for (int level = 0; level < (W == 16 ? 2 : 1); ++level) {
        for (uint32_t i = threadIdx.x; i < uint32_t(nwarps) * 256; i += blockDim.x) h[i] = 0;
        __syncthreads();
        for (uint32_t wi = threadIdx.x; wi < it.words; wi += blockDim.x) {
            const uint32_t x = sm.cnt[wi];
            if (!x) continue;
#pragma unroll
            for (uint32_t j = 0; j < kPer; ++j) {
                const uint32_t c = (x >> (j * W)) & L::kMask;
                if (!c) continue;
                if (level == 0) {
                    atomicAdd(&h[warp * 256 + (c >> kShift1)], 1u);
                } else if ((c >> 8) == hi_sel) {
                    atomicAdd(&h[warp * 256 + (c & 0xffu)], 1u);
                }
            }
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x) {
            uint32_t s = 0;
            for (int w = 0; w < nwarps; ++w) s += h[w * 256 + b];
            h[b] = s;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            // walk bins from the top until k objects are covered
            unsigned long long cum = cum_above;
            uint32_t sel = 0;
            bool found = false;
            for (int b = 255; b >= 0; --b) {
                if (level == 0 && W != 16 && b == 0) break;  // count 0 is not a level
                if (level == 1 && hi_sel == 0 && b == 0) break;
                const unsigned long long nb = cum + h[b];
                if (nb >= it.kq) {
                    sel = b;
                    found = true;
                    break;
                }
                cum = nb;
            }
            sm.scal[SC_T] = found ? sel : 0xffffffffu;
            reinterpret_cast<unsigned long long*>(sm.sums)[31] = cum;
        }
        __syncthreads();
        const uint32_t sel = sm.scal[SC_T];
        const unsigned long long cum = reinterpret_cast<unsigned long long*>(sm.sums)[31];
        __syncthreads();
        if (sel == 0xffffffffu) {  // fewer than k non-zero objects at this level
            if (level == 0 || W != 16) {
                T = 0;
                above = 0;
                break;
            }
            // level 1 with hi_sel chosen: cannot happen (level 0 found >= k)
            T = hi_sel << 8;
            break;
        }
        if (W == 16 && level == 0) {
            hi_sel = sel;
            cum_above = cum;
            continue;
        }
        T = (W == 16) ? ((hi_sel << 8) | sel) : sel;
        above = static_cast<uint32_t>(cum);
    }
    it.rec_b = max(T, 1u);
    if (it.gate && threadIdx.x == 0) p.tile_rec[uint64_t(it.slot) * kRecWords] = it.rec_b;
    // emit: every count > T, then ties at T (T > 0) in ascending id; one
    // 32-object block per thread per step (both layouts keep a block in W
    // consecutive words)
    const uint32_t need = T ? it.kq - above : 0;
    const uint32_t nblk = it.words / W;
    unsigned long long seen = 0;
    for (uint32_t b0 = 0; b0 < nblk; b0 += blockDim.x) {
        const uint32_t bi = b0 + threadIdx.x;
        uint32_t tie_mask = 0;
        if (bi < nblk) {
#pragma unroll 4
            for (uint32_t j = 0; j < 32; ++j) {
                const uint32_t c = L::get(sm.cnt, bi * 32 + j);
                if (c > T) emit(p, it, sm, bi * 32 + j, c);
                else if (T && c == T) tie_mask |= 1u << j;
            }
        }
        unsigned long long total;
        unsigned long long r =
            seen + block_exclusive_scan<unsigned long long>(__popc(tie_mask), sm.sums, total);
        while (tie_mask && r < need) {
            const uint32_t j = __ffs(tie_mask) - 1;
            tie_mask &= tie_mask - 1;
            emit(p, it, sm, bi * 32 + j, T);
            ++r;
        }
        seen += total;
    }
    return T;
}

// Carry-save adder: l = a ^ b ^ c (sum), h = majority (carry); two LOP3s.
__device__ __forceinline__ void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t u = a ^ b;
    h = (a & b) | (u & c);
    l = u ^ c;
}

// Dense phase (interleaved layout): every thread owns whole 32-object blocks
// and initialises their counters as the sum of the query's dense bitmaps
// (plain 16-byte stores, no atomics, no zeroing pass).  The bitmaps of a
// block are first summed into bit planes of the count (plane i = bit i of
// every object's count): up to three lists by a full adder lane by lane
// (dense_lanes); more by carry-save adders, a Harley-Seal tree over 8 lists
// at a time (dense_planes).  The planes become counter words through a
// masked-swap transpose (planes_to_words).  With the gate on, the same
// planes count, in registers, the objects reaching each level v in
// [at0, at0 + kLvl) for the c-PQ catch-up (dense_gate).

__host__ __device__ constexpr uint32_t swap_mask(int s) {
    return s == 0 ? 0x55555555u : (s == 1 ? 0x33333333u : (s == 2 ? 0x0f0f0f0fu : 0x00ff00ffu));
}

// (a & m) | (b & ~m) as one LOP3 (the mask an immediate)
__device__ __forceinline__ uint32_t bitsel(uint32_t a, uint32_t b, uint32_t m) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "r"(m));
    return d;
}

// Bit b of plane i (bit i of the count of object b of a 32-object block) ->
// field j of word m (the counter of object j * W + m: the interleaved
// layout).  log2(W) levels of masked swaps between words 2^s apart; a pair
// costs two shifts and two LOP3s, and planes known to be zero (i >= NP) fold.
template <int W, int NP, bool LOP = true>
__device__ __forceinline__ void planes_to_words(const uint32_t (&P)[NP], uint32_t (&X)[W]) {
#pragma unroll
    for (int i = 0; i < W; ++i) X[i] = i < NP ? P[i < NP ? i : 0] : 0u;
#pragma unroll
    for (int s = 0; (1 << s) < W; ++s) {
        const int f = 1 << s;
        const uint32_t m = swap_mask(s);
#pragma unroll
        for (int i = 0; i < W; ++i) {
            if (i & f) continue;
            const uint32_t a = X[i], b = X[i + f];
            if constexpr (LOP) {
                X[i] = bitsel(a, b << f, m);
                X[i + f] = bitsel(a >> f, b, m);
            } else {
                X[i] = (a & m) | ((b << f) & ~m);
                X[i + f] = ((a >> f) & m) | (b & ~m);
            }
        }
    }
}

// consecutive 32-object blocks per thread in the many-list dense path (one
// G-word bitmap load per list); dense_gate re-reads the same ownership
template <int W>
__host__ __device__ constexpr int csa_blocks() {
    return W == 8 ? (GENIE_CSA_QUAD ? 4 : (GENIE_CSA_PAIR ? 2 : 1)) : (W == 4 ? GENIE_CSA_BLOCKS_W4 : 1);
}

// objects of the block whose count (NP planes) is >= v
template <int NP>
__device__ __forceinline__ uint32_t planes_ge(const uint32_t (&P)[NP], uint32_t v) {
    if (v >> NP) return 0u;
    uint32_t ge = 0, eq = 0xffffffffu;
#pragma unroll
    for (int i = NP - 1; i >= 0; --i) {
        if ((v >> i) & 1u) {
            eq &= P[i];
        } else {
            ge |= eq & P[i];
            eq &= ~P[i];
        }
    }
    return ge | eq;
}

// adds c (weight 2^i0) into planes i0.. (ripple carry; a carry out of the top
// plane cannot happen: counts stay below 2^NP)
template <int NP>
__device__ __forceinline__ void plane_add(uint32_t (&P)[NP], uint32_t c, int i0) {
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        if (i < i0) continue;
        const uint32_t t = P[i] & c;
        P[i] ^= c;
        c = t;
    }
}

template <int G>
__device__ __forceinline__ void ldg_words(const uint32_t* src, uint32_t (&x)[G]) {
    if constexpr (G == 1) {
        x[0] = __ldg(src);
    } else if constexpr (G == 2) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(src));
        x[0] = v.x;
        x[1] = v.y;
    } else {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src));
        x[0] = v.x;
        x[1] = v.y;
        x[2] = v.z;
        x[3] = v.w;
    }
}

// G bitmap words of each of N lists whose row offsets sit at slot[0..N)
// (16-byte shared loads of the offsets measured no faster)
template <int N, int G>
__device__ __forceinline__ void ldg_lists(const uint32_t* col, const uint32_t* slot, uint32_t (&a)[N][G]) {
#pragma unroll
    for (int u = 0; u < N; ++u) ldg_words<G>(col + slot[u], a[u]);
}

// 16 lists into planes 0..3 (ones, twos, fours, eights accumulate there);
// the weight-16 carry is returned in s16 for the caller to place.
template <int NP, int G>
__device__ __forceinline__ void hs16(uint32_t (&P)[G][NP], const uint32_t* col, const uint32_t* slot,
                                     uint32_t (&s16)[G]) {
    uint32_t eA[G];
    {
        uint32_t a[8][G];
        ldg_lists<8, G>(col, slot, a);
#pragma unroll
        for (int h = 0; h < G; ++h) {
            uint32_t twosA, twosB, foursA, foursB;
            csa(twosA, P[h][0], P[h][0], a[0][h], a[1][h]);
            csa(twosB, P[h][0], P[h][0], a[2][h], a[3][h]);
            csa(foursA, P[h][1], P[h][1], twosA, twosB);
            csa(twosA, P[h][0], P[h][0], a[4][h], a[5][h]);
            csa(twosB, P[h][0], P[h][0], a[6][h], a[7][h]);
            csa(foursB, P[h][1], P[h][1], twosA, twosB);
            csa(eA[h], P[h][2], P[h][2], foursA, foursB);
        }
    }
    uint32_t a[8][G];
    ldg_lists<8, G>(col, slot + 8, a);
#pragma unroll
    for (int h = 0; h < G; ++h) {
        uint32_t twosA, twosB, foursA, foursB, eB;
        csa(twosA, P[h][0], P[h][0], a[0][h], a[1][h]);
        csa(twosB, P[h][0], P[h][0], a[2][h], a[3][h]);
        csa(foursA, P[h][1], P[h][1], twosA, twosB);
        csa(twosA, P[h][0], P[h][0], a[4][h], a[5][h]);
        csa(twosB, P[h][0], P[h][0], a[6][h], a[7][h]);
        csa(foursB, P[h][1], P[h][1], twosA, twosB);
        csa(eB, P[h][2], P[h][2], foursA, foursB);
        csa(s16[h], P[h][3], P[h][3], eA[h], eB);
    }
}

// 32 lists into planes 0..4; the weight-32 carry is returned in s32.
template <int NP, int G>
__device__ __forceinline__ void hs32(uint32_t (&P)[G][NP], const uint32_t* col, const uint32_t* slot,
                                     uint32_t (&s32)[G]) {
    uint32_t sA[G], sB[G];
    hs16<NP, G>(P, col, slot, sA);
    hs16<NP, G>(P, col, slot + 16, sB);
#pragma unroll
    for (int h = 0; h < G; ++h) csa(s32[h], P[h][4], P[h][4], sA[h], sB[h]);
}

template <int W>
__device__ __forceinline__ void store_block(const ScanSmem& sm, uint32_t blk, const uint32_t (&acc)[W]) {
    uint4* dst = reinterpret_cast<uint4*>(sm.cnt + blk * W);
#pragma unroll
    for (int j = 0; j < W; j += 4) dst[j / 4] = make_uint4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
}

// Many lists (nd > 3, W <= 8): G consecutive blocks per thread (one G-word
// bitmap load per list), NP planes (NP = W, or fewer when nd < 2^NP).
template <int W, int NP, int G>
__device__ __forceinline__ void dense_planes(const BatchParams& p, const ScanSmem& sm, const StageBuf& sb,
                                             uint32_t bw0, uint32_t nblk, uint32_t nd, uint32_t at0, uint32_t nlv,
                                             uint32_t (&lv)[kLvl]) {
    const uint32_t* dslot = sb.dense();
    for (uint32_t blk = G * threadIdx.x; blk < nblk; blk += G * blockDim.x) {
        const uint32_t* col = p.bitmaps + bw0 + blk;
        uint32_t P[G][NP];
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
            for (int i = 0; i < NP; ++i) P[h][i] = 0;
        uint32_t d = 0;
#if GENIE_CSA16
        if constexpr (NP >= 7 && GENIE_CSA64) {
            // 64 lists: two 32-list trees whose weight-32 carries meet plane 5
            for (; d + 64 <= nd; d += 64) {
                uint32_t sA[G], sB[G];
                hs32<NP, G>(P, col, dslot + d, sA);
                hs32<NP, G>(P, col, dslot + d + 32, sB);
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    uint32_t t64;
                    csa(t64, P[h][5], P[h][5], sA[h], sB[h]);
                    plane_add<NP>(P[h], t64, 6);  // weight 64
                }
            }
        }
        if constexpr (NP >= 6 && GENIE_CSA32) {
            // 32 lists: two 16-list trees whose weight-16 carries meet plane 4
            for (; d + 32 <= nd; d += 32) {
                uint32_t s32[G];
                hs32<NP, G>(P, col, dslot + d, s32);
#pragma unroll
                for (int h = 0; h < G; ++h) plane_add<NP>(P[h], s32[h], 5);  // weight 32
            }
        }
        if constexpr (NP >= 5) {
            // Harley-Seal over 16 lists: two 8-list halves whose weight-8
            // carries meet plane 3 in one more CSA, so only the weight-16
            // carry ripples (planes 4..NP-1) -- 38 logic ops per 16 lists and
            // block instead of 2 x 24
            for (; d + 16 <= nd; d += 16) {
                uint32_t s16[G];
                hs16<NP, G>(P, col, dslot + d, s16);
#pragma unroll
                for (int h = 0; h < G; ++h) plane_add<NP>(P[h], s16[h], 4);  // weight 16
            }
        }
#endif
        if constexpr (NP >= 4) {
            for (; d + 8 <= nd; d += 8) {
                uint32_t a[8][G];
                ldg_lists<8, G>(col, dslot + d, a);
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    uint32_t twosA, twosB, foursA, foursB, eights;
                    csa(twosA, P[h][0], P[h][0], a[0][h], a[1][h]);
                    csa(twosB, P[h][0], P[h][0], a[2][h], a[3][h]);
                    csa(foursA, P[h][1], P[h][1], twosA, twosB);
                    csa(twosA, P[h][0], P[h][0], a[4][h], a[5][h]);
                    csa(twosB, P[h][0], P[h][0], a[6][h], a[7][h]);
                    csa(foursB, P[h][1], P[h][1], twosA, twosB);
                    csa(eights, P[h][2], P[h][2], foursA, foursB);
                    plane_add<NP>(P[h], eights, 3);  // weight 8
                }
            }
        }
        if constexpr (NP >= 3) {
            for (; d + 4 <= nd; d += 4) {
                uint32_t a[4][G];
                ldg_lists<4, G>(col, dslot + d, a);
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    uint32_t twosA, twosB, fours;
                    csa(twosA, P[h][0], P[h][0], a[0][h], a[1][h]);
                    csa(twosB, P[h][0], P[h][0], a[2][h], a[3][h]);
                    csa(fours, P[h][1], P[h][1], twosA, twosB);
                    plane_add<NP>(P[h], fours, 2);  // weight 4
                }
            }
        }
        for (; d < nd; ++d) {
            uint32_t a[G];
            ldg_words<G>(col + dslot[d], a);
#pragma unroll
            for (int h = 0; h < G; ++h) plane_add<NP>(P[h], a[h], 0);
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
            if (blk + h >= nblk) break;
            if (nlv) {
#pragma unroll
                for (uint32_t l = 0; l < kLvl; ++l)
                    if (l < nlv) lv[l] += __popc(planes_ge<NP>(P[h], at0 + l));
            }
            uint32_t acc[W];
            planes_to_words<W, NP, GENIE_PLANES_LOP>(P[h], acc);
            store_block<W>(sm, blk + h, acc);
        }
    }
}

// One to three lists (most C2 items): lane-wise, a warp step covers 32 * BPT
// consecutive blocks and lane l owns blocks base + 32 i (i < BPT), so every
// bitmap load (one word per lane) and every 16-byte counter store of the warp
// is contiguous.  Two planes: the lists' sum (XOR) and carry (majority); the
// level counts are OR (>= 1), the carry (>= 2) and AND (>= 3), picked by
// per-level masks set once per item.  Full steps run without bounds checks;
// only the last warp step of the tile may be partial.
template <int W, int ND, bool LV, bool FULL>
__device__ __forceinline__ void dense_lane_step(const uint32_t* const (&r)[ND], uint4* dst, uint32_t base,
                                                uint32_t nblk, const uint32_t (&msel)[kLvl][3],
                                                uint32_t (&lv)[kLvl]) {
    constexpr uint32_t BPT = W == 4 ? 4 : (W == 8 ? 2 : 1);
    constexpr int NP = ND == 1 ? 1 : 2;
    uint32_t b[ND][BPT];
#pragma unroll
    for (int u = 0; u < ND; ++u)
#pragma unroll
        for (uint32_t i = 0; i < BPT; ++i) b[u][i] = (FULL || base + 32 * i < nblk) ? __ldg(r[u] + 32 * i) : 0u;
#pragma unroll
    for (uint32_t i = 0; i < BPT; ++i) {
        uint32_t P[NP];
        uint32_t ge1, ge3 = 0;
        if constexpr (ND == 1) {
            P[0] = ge1 = b[0][i];
        } else if constexpr (ND == 2) {
            P[0] = b[0][i] ^ b[1][i];
            P[1] = b[0][i] & b[1][i];
            ge1 = b[0][i] | b[1][i];
        } else {
            const uint32_t x = b[0][i], y = b[1][i], z = b[2][i];
            P[0] = x ^ y ^ z;
            P[1] = (x & y) | (x & z) | (y & z);
            ge1 = x | y | z;
            ge3 = x & y & z;
        }
        if (FULL || base + 32 * i < nblk) {
            uint32_t acc[W];
            planes_to_words<W, NP>(P, acc);
#pragma unroll
            for (int j = 0; j < W; j += 4) dst[i * 32 * (W / 4) + j / 4] = make_uint4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        }
        if constexpr (LV) {
            const uint32_t ge2 = NP > 1 ? P[NP - 1] : 0u;
#pragma unroll
            for (uint32_t l = 0; l < kLvl; ++l)
                lv[l] += __popc((ge1 & msel[l][0]) | (ge2 & msel[l][1]) | (ge3 & msel[l][2]));
        }
    }
}

template <int W, int ND, bool LV>
__device__ __forceinline__ void dense_lanes(const BatchParams& p, const ScanSmem& sm, const StageBuf& sb,
                                            uint32_t bw0, uint32_t nblk, uint32_t at0, uint32_t nlv,
                                            uint32_t (&lv)[kLvl]) {
    constexpr uint32_t BPT = W == 4 ? 4 : (W == 8 ? 2 : 1);
    constexpr uint32_t STEP = 32 * BPT;  // blocks per warp step
    const uint32_t lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    uint32_t msel[kLvl][3];
#pragma unroll
    for (uint32_t l = 0; l < kLvl; ++l)
#pragma unroll
        for (uint32_t c = 0; c < 3; ++c) msel[l][c] = (l < nlv && at0 + l == c + 1) ? ~0u : 0u;
    uint32_t wt = threadIdx.x >> 5;
    const uint32_t* r[ND];
#pragma unroll
    for (int u = 0; u < ND; ++u) r[u] = p.bitmaps + bw0 + sb.dense()[u] + wt * STEP + lane;
    uint4* dst = reinterpret_cast<uint4*>(sm.cnt) + (wt * STEP + lane) * (W / 4);
    const uint32_t nfull = nblk / STEP;
    for (; wt < nfull; wt += nwarps) {
        dense_lane_step<W, ND, LV, true>(r, dst, 0, 0, msel, lv);
#pragma unroll
        for (int u = 0; u < ND; ++u) r[u] += nwarps * STEP;
        dst += nwarps * STEP * (W / 4);
    }
    if (wt * STEP < nblk) dense_lane_step<W, ND, LV, false>(r, dst, wt * STEP + lane, nblk, msel, lv);
}

template <int W>
GENIE_DENSE_FN uint32_t dense_init(const BatchParams& p, const ItemCtx& it, const ScanSmem& sm, const StageBuf& sb,
                               uint32_t nd, uint32_t at0, uint32_t nlv, bool& csa_path, long long* t_work = nullptr) {
    using Sw = Swar<W>;
    constexpr uint32_t BPT = W == 4 ? 4 : (W == 8 ? 2 : 1);  // blocks per lane per warp step
    constexpr uint32_t NW = BPT * W;
    const uint32_t bw0 = it.tile_lo >> 5;
    const uint32_t nblk = it.words / W;
    uint32_t lv[kLvl] = {};
    csa_path = false;
    if constexpr (W <= 8) {
        if (nd > GENIE_LANES_MAX) {
            csa_path = true;
            constexpr int G = csa_blocks<W>();
            if (nd >= 2 * W) dense_planes<W, W, G>(p, sm, sb, bw0, nblk, nd, at0, nlv, lv);
#if GENIE_LANES_MAX < 3  // ablation: few-list items through the planes path too (C2 -13 %)
            else if (nd <= 3) dense_planes<W, 2, G>(p, sm, sb, bw0, nblk, nd, at0, nlv, lv);
#endif
            else dense_planes<W, W == 4 ? 3 : 4, G>(p, sm, sb, bw0, nblk, nd, at0, nlv, lv);
            nd = 0;
        }
    }
    if (!(W == 4 && kLanesLvSplit) || nlv) {  // W >= 8: one variant (measured faster: C3 / C5 +2 %)
        if (nd == 1) dense_lanes<W, 1, true>(p, sm, sb, bw0, nblk, at0, nlv, lv);
        else if (nd == 2) dense_lanes<W, 2, true>(p, sm, sb, bw0, nblk, at0, nlv, lv);
        else if (nd == 3) dense_lanes<W, 3, true>(p, sm, sb, bw0, nblk, at0, nlv, lv);
    } else {
        if (nd == 1) dense_lanes<W, 1, false>(p, sm, sb, bw0, nblk, at0, nlv, lv);
        else if (nd == 2) dense_lanes<W, 2, false>(p, sm, sb, bw0, nblk, at0, nlv, lv);
        else if (nd == 3) dense_lanes<W, 3, false>(p, sm, sb, bw0, nblk, at0, nlv, lv);
    }
    if (nd <= 3) nd = 0;
    // W = 16 with more than three lists: per-lane adds (counts < 2^15, no carries)
    if constexpr (W > 8) {
    const uint32_t lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (uint32_t wt = threadIdx.x >> 5; nd && wt * 32 * BPT < nblk; wt += nwarps) {
        const uint32_t base = wt * 32 * BPT + lane;
        uint32_t acc[NW];
#pragma unroll
        for (uint32_t j = 0; j < NW; ++j) acc[j] = 0;
        const uint32_t* col = p.bitmaps + bw0 + base;
        uint32_t d = 0;
        for (; d + 4 <= nd; d += 4) {  // four lists' loads in flight
            uint32_t b[4][BPT];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t* src = col + sb.dense()[d + u];
#pragma unroll
                for (uint32_t i = 0; i < BPT; ++i) b[u][i] = base + 32 * i < nblk ? __ldg(src + 32 * i) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (uint32_t i = 0; i < BPT; ++i)
#pragma unroll
                    for (uint32_t m = 0; m < W; ++m) acc[i * W + m] += (b[u][i] >> m) & Sw::kOnes;
        }
        for (; d < nd; ++d) {
            const uint32_t* src = col + sb.dense()[d];
            uint32_t b[BPT];
#pragma unroll
            for (uint32_t i = 0; i < BPT; ++i) b[i] = base + 32 * i < nblk ? __ldg(src + 32 * i) : 0u;
#pragma unroll
            for (uint32_t i = 0; i < BPT; ++i)
#pragma unroll
                for (uint32_t m = 0; m < W; ++m) acc[i * W + m] += (b[i] >> m) & Sw::kOnes;
        }
#pragma unroll
        for (uint32_t i = 0; i < BPT; ++i) {
            if (base + 32 * i < nblk) {
                uint4* dst = reinterpret_cast<uint4*>(sm.cnt + (base + 32 * i) * W);
#pragma unroll
                for (uint32_t j = 0; j < W; j += 4)
                    dst[j / 4] = make_uint4(acc[i * W + j], acc[i * W + j + 1], acc[i * W + j + 2], acc[i * W + j + 3]);
            }
        }
        if (nlv) {  // counts <= nd < 2W < 2^(W-1): one add and one mask per level
#pragma unroll
            for (uint32_t l = 0; l < kLvl; ++l) {
                if (l < nlv) {
                    const uint32_t bias = Sw::kHigh - (at0 + l) * Sw::kOnes;
#pragma unroll
                    for (uint32_t j = 0; j < NW; ++j) lv[l] += __popc((acc[j] + bias) & Sw::kHigh);
                }
            }
        }
    }
    }
    uint32_t reach = 0;  // levels at0 + l (l < reach) that some object of this thread's blocks reaches
#pragma unroll
    for (uint32_t l = 0; l < kLvl; ++l) reach += (l < nlv && lv[l]) ? 1u : 0u;
    if (nlv) {
#pragma unroll
        for (uint32_t l = 0; l < kLvl; ++l) {
            if (l < nlv) {
                const uint32_t c = warp_sum(lv[l]);
                if ((threadIdx.x & 31) == 0 && c) atomicAdd(&sm.scal[SC_LVL + l], c);
            }
        }
    }
    if (t_work) *t_work = clock64();
    __syncthreads();
    return reach;
}

// Brings the c-PQ state to what one gated update per (dense list, member
// object) yields (cpq.hpp:294-301, 374-389): AT advances to the smallest
// level v >= at0 that fewer than k objects reach (ZA below AT is never read
// again); every object at or above the new AT -- fewer than k -- enters the
// table and adds one to ZA[v] for each level v in [AT, count].
template <int W>
GENIE_DENSE_FN void dense_gate(const ItemCtx& it, const ScanSmem& sm, uint32_t at0, uint32_t dmax, uint32_t nlv,
                           uint32_t reach, bool csa_path) {
    using Sw = Swar<W>;
    using L = Lay<W, true>;
    uint32_t j = 0;
    while (j < nlv && sm.scal[SC_LVL + j] >= it.kq) ++j;
    uint32_t a = at0 + j;
    if (j == nlv && a <= dmax) {
        // beyond the register levels: binary search for the smallest v in
        // [a, dmax + 1] with #(count >= v) < k (block-uniform)
        uint32_t lo = a, hi = dmax + 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            unsigned long long c = 0;
            for (uint32_t wi = threadIdx.x * 4; wi < it.words; wi += blockDim.x * 4) {
                const uint4 x = *reinterpret_cast<const uint4*>(sm.cnt + wi);
                c += __popc(Sw::ge(x.x, mid)) + __popc(Sw::ge(x.y, mid)) + __popc(Sw::ge(x.z, mid)) +
                     __popc(Sw::ge(x.w, mid));
            }
            const unsigned long long tot = block_sum<unsigned long long>(c, sm.sums);
            if (tot >= it.kq) lo = mid + 1;
            else hi = mid;
        }
        a = lo;
    }
    if (threadIdx.x == 0) sm.scal[SC_AT] = a;
    // A thread re-reads only its own dense_init blocks, and only when they
    // may hold an object at or above a (its level counts say so, or do not
    // reach that high): the fewer than k objects sit in a few blocks.
    if (a <= dmax && (a - at0 < reach || reach == nlv)) {
        constexpr uint32_t BPT = W == 4 ? 4 : (W == 8 ? 2 : 1);
        const uint32_t nblk = it.words / W;
        // blocks of this thread: csa path blk = tid + k * blockDim; lane-wise
        // path blk = (warp + k * nwarps) * 32 * BPT + lane + 32 i
        const uint32_t lane = threadIdx.x & 31;
        constexpr uint32_t kGrp = csa_blocks<W>();  // csa blocks per thread
        const bool pair = kGrp > 1 && csa_path;
        const uint32_t first = pair ? kGrp * threadIdx.x : (csa_path ? threadIdx.x : (threadIdx.x >> 5) * 32 * BPT + lane);
        const uint32_t stride = pair ? kGrp * blockDim.x : (csa_path ? blockDim.x : (blockDim.x >> 5) * 32 * BPT);
        const uint32_t per = pair ? kGrp : (csa_path ? 1u : BPT);
        const uint32_t step = pair ? 1u : 32u;
        for (uint32_t b0 = first; b0 < nblk; b0 += stride) {
            for (uint32_t i = 0; i < per && b0 + step * i < nblk; ++i) {
                const uint32_t blk = b0 + step * i;
                for (uint32_t wi = blk * W; wi < blk * W + W; ++wi) {
                    const uint32_t x = sm.cnt[wi];
                    uint32_t m = Sw::ge(x, a);
                    while (m) {
                        const uint32_t l = (__ffs(m) - 1) / W;
                        m &= m - 1;
                        const uint32_t c = (x >> (l * W)) & L::kMask;
                        if (!ht_insert(sm.ht, it.ht_cap, L::obj(wi, l), c, a)) sm.scal[SC_OVF] = 1;
                        for (uint32_t v = a; v <= c; ++v) atomicAdd(&sm.za[v], 1u);
                    }
                }
            }
        }
    }
    __syncthreads();
}

// Count the postings of one warp's groups [g0, g1) of the staged slices into
// the tile's shared counters; with the gate on, feed the c-PQ with each new
// value.  A group is an absolute 128-posting (512-byte) block of the postings
// array intersected with its slice; lane l owns the 16 bytes at 4l.  Up to
// kScanUnroll groups are loaded before any of them is counted, so a warp's
// share costs one memory round trip per pass whatever slices it spans.
//
// Per posting: one shared atomicAdd of 1 << shift on the packed word (exact:
// the query's max_count_bound keeps every counter below 2^W, so no carry
// crosses lanes -- the reference's CAS loop, cpq.hpp:70-88, is not needed).
// Addresses are 32-bit shared-window offsets with the tile origin folded into
// the base (the tile origin is a multiple of 32 objects, so both layouts map
// absolute ids linearly across 32-object blocks).  The gate test "old value
// >= AT - 1" is done on the word shifted so the counter sits in the top W
// bits, as one max over the four postings of a lane's group and one compare.
template <int W, bool GATE, bool IL>
__device__ __forceinline__ void scan_warp_groups(const uint32_t* __restrict__ postings, const ItemCtx& it,
                                                 const ScanSmem& sm, const StageBuf& sb, uint32_t nsb, uint32_t G,
                                                 uint32_t g0, uint32_t g1, uint32_t stride) {
    using L = Lay<W, IL>;
    constexpr uint32_t kPer = 32 / W, kTop = 32 - W;
    constexpr int UNR = kScanUnroll;
    if (g0 >= g1) return;
    const uint32_t lane = threadIdx.x & 31;
    // byte address of the word holding absolute id x: cbase + word(x) * 4 (mod 2^32)
    const uint32_t cbase = smem_u32(sm.cnt) - (L::word(it.tile_lo) << 2);
    const uint32_t word0 = smem_u32(sm.cnt) + lane * 4;  // private target of masked-off lanes
    volatile uint32_t* s_at = sm.scal + SC_AT;
    // slice holding group g0: last si with upref[si] <= g0 (empty slices share
    // the next slice's prefix, so this is the non-empty one)
    uint32_t si;
    {
        uint32_t lo = 0, hi = nsb;
        while (lo < hi) {
            const uint32_t m = (lo + hi) >> 1;
            if (sb.upref()[m] <= g0) lo = m + 1;
            else hi = m;
        }
        si = lo - 1;
    }
    uint64_t s_beg = sb.beg()[si];
    uint64_t s_end = s_beg + (sb.ppref()[si + 1] - sb.ppref()[si]);
    uint64_t s_blk = (s_beg >> 7) - sb.upref()[si];  // absolute block of group g: s_blk + g
    uint32_t s_next = si + 1 < nsb ? sb.upref()[si + 1] : G;
    uint32_t gate = 0;
    if constexpr (GATE) gate = (*s_at - 1) << kTop;
    for (uint32_t gb = g0; gb < g1; gb += UNR * stride) {
        uint4 v[UNR];
        uint32_t msk = 0;  // 4 bits per group: the lane's positions inside the slice
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t g = gb + u * stride;
            v[u] = make_uint4(0, 0, 0, 0);
            if (g < g1) {
                while (g >= s_next) {  // warp-uniform slice advance
                    ++si;
                    s_beg = sb.beg()[si];
                    s_end = s_beg + (sb.ppref()[si + 1] - sb.ppref()[si]);
                    s_blk = (s_beg >> 7) - sb.upref()[si];
                    s_next = si + 1 < nsb ? sb.upref()[si + 1] : G;
                }
                const uint64_t pos = ((s_blk + g) << 7) + lane * 4;
                if (pos + 4 > s_beg && pos < s_end) {
                    v[u] = ldg_stream_v4(postings + pos);
                    const uint32_t lo_n = s_beg > pos ? static_cast<uint32_t>(s_beg - pos) : 0u;
                    const uint32_t hi_n = s_end - pos < 4 ? static_cast<uint32_t>(s_end - pos) : 4u;
                    msk |= (((1u << hi_n) - 1u) & ~((1u << lo_n) - 1u)) << (4 * u);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t m = (msk >> (4 * u)) & 0xfu;
            if (!m) continue;
            const uint32_t x[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
            uint32_t old[4];
            uint32_t top = 0;
            if (m == 0xfu) {  // whole 16 bytes inside the slice: unconditional atomics
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    // r = kTop - shift: the counter's distance from the top of the word
                    const uint32_t r = ((~L::lane(x[e])) & (kPer - 1)) * W;
                    old[e] = atom_add_shared(cbase + (L::word(x[e]) << 2), (1u << kTop) >> r);
                    if constexpr (GATE) top = max(top, old[e] << r);
                }
            } else {  // slice edge: masked-off positions add 0 to a private word
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t r = ((~L::lane(x[e])) & (kPer - 1)) * W;
                    const bool ok = (m >> e) & 1u;
                    old[e] = atom_add_shared(ok ? cbase + (L::word(x[e]) << 2) : word0,
                                             ok ? (1u << kTop) >> r : 0u);
                    if constexpr (GATE) top = max(top, ok ? old[e] << r : 0u);
                }
            }
            if constexpr (GATE) {
                if (top >= gate) {  // some new value may pass: check each
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t r = ((~L::lane(x[e])) & (kPer - 1)) * W;
                        if ((m & (1u << e)) && (old[e] << r) >= gate)
                            gate = cpq_admit<W>(sm.ht, sm.za, sm.scal, it.ht_cap, it.bound, it.kq,
                                                x[e] - it.tile_lo, old[e], kTop - r);
                    }
                }
                gate = (*s_at - 1) << kTop;
            }
        }
    }
}


// Compact mode for tiles whose slices are short (average 128-posting group
// less than half full, e.g. minHash: ~10 postings per list per tile): the
// warp's share is a contiguous run [r0, r1) of the item's postings counted
// across its slices; lane l takes postings r0 + l + 32 j, one 4-byte id each,
// so every shared atomic instruction carries 32 real postings.  Each lane
// tracks the slice of its position (ppref: postings before each slice).
template <int W, bool GATE, bool IL>
__device__ __forceinline__ void scan_compact(const uint32_t* __restrict__ postings, const ItemCtx& it,
                                             const ScanSmem& sm, const StageBuf& sb, uint32_t nsb, uint32_t r0,
                                             uint32_t r1) {
    using L = Lay<W, IL>;
    constexpr uint32_t kPer = 32 / W, kTop = 32 - W;
    constexpr int UNR = 4;
    if (r0 >= r1) return;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t cbase = smem_u32(sm.cnt) - (L::word(it.tile_lo) << 2);
    volatile uint32_t* s_at = sm.scal + SC_AT;
    const uint32_t* pp = sb.ppref();
    // slice of this lane's first position: last si with ppref[si] <= r
    uint32_t si;
    {
        const uint32_t r = min(r0 + lane, r1 - 1);
        uint32_t lo = 0, hi = nsb;
        while (lo < hi) {
            const uint32_t m = (lo + hi) >> 1;
            if (pp[m] <= r) lo = m + 1;
            else hi = m;
        }
        si = lo - 1;
    }
    uint32_t gate = 0;
    if constexpr (GATE) gate = (*s_at - 1) << kTop;
    for (uint32_t base = r0; base < r1; base += 32 * UNR) {
        uint32_t x[UNR];
        uint32_t ok = 0;
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t r = base + u * 32 + lane;
            x[u] = 0;
            if (r < r1) {
                while (pp[si + 1] <= r) ++si;  // the slices ahead (empty ones skipped)
                x[u] = __ldg(postings + sb.beg()[si] + (r - pp[si]));
                ok |= 1u << u;
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if (!((ok >> u) & 1u)) continue;
            const uint32_t r = ((~L::lane(x[u])) & (kPer - 1)) * W;
            const uint32_t old = atom_add_shared(cbase + (L::word(x[u]) << 2), (1u << kTop) >> r);
            if constexpr (GATE) {
                if ((old << r) >= gate) {
                    gate = cpq_admit<W>(sm.ht, sm.za, sm.scal, it.ht_cap, it.bound, it.kq, x[u] - it.tile_lo, old,
                                        kTop - r);
                }
                gate = (*s_at - 1) << kTop;
            }
        }
    }
}

// One warp's share [g0, g1) of the staged slices' 128-posting groups.
template <int W, bool IL>
__device__ __forceinline__ void scan_group_range(const BatchParams& p, const ItemCtx& it, const ScanSmem& sm,
                                                 const StageBuf& sb, uint32_t nsb, uint32_t G, uint32_t g0,
                                                 uint32_t g1, uint32_t stride = 1) {
    if (it.admit) scan_warp_groups<W, true, IL>(p.postings, it, sm, sb, nsb, G, g0, g1, stride);
    else scan_warp_groups<W, false, IL>(p.postings, it, sm, sb, nsb, G, g0, g1, stride);
}

// The sparse (posting-list) part of the tile.  Few groups per warp: a static
// contiguous split (no claiming); many: guided self-scheduling of runs of
// groups (chunks shrink as the tile drains, so the warps reach the
// end-of-tile barrier together).
template <int W, bool IL>
__device__ void scan_groups(const BatchParams& p, const ItemCtx& it, const ScanSmem& sm, const StageBuf& sb,
                            uint32_t nsb, uint32_t G, uint32_t unit, uint32_t wfirst, uint32_t ptot = 0) {
    // warps [wfirst, nwarps) scan
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (threadIdx.x >> 5) - wfirst;
    const uint32_t nwarps = (blockDim.x >> 5) - wfirst;
    if (ptot && uint64_t(ptot) * kCompactFillInv < uint64_t(G) * 128) {  // short slices: compact mode
        // contiguous shares of ceil(ptot / nwarps) (32-bit arithmetic)
        const uint32_t share = (ptot + nwarps - 1) / nwarps;
        const uint32_t r0 = min(ptot, warp * share), r1 = min(ptot, r0 + share);
        if (it.admit) scan_compact<W, true, IL>(p.postings, it, sm, sb, nsb, r0, r1);
        else scan_compact<W, false, IL>(p.postings, it, sm, sb, nsb, r0, r1);
        return;
    }
    if (G <= kStaticGroups * nwarps) {
#if GENIE_SCAN_STRIDED
        // round-robin groups: every warp's share mixes hot (L2) and cold lists
        scan_group_range<W, IL>(p, it, sm, sb, nsb, G, warp, G, nwarps);
#else
        // G <= kStaticGroups * nwarps: the products stay far below 2^32
        const uint32_t g0 = G * warp / nwarps, g1 = G * (warp + 1) / nwarps;
        scan_group_range<W, IL>(p, it, sm, sb, nsb, G, g0, g1);
#endif
        return;
    }
    const uint32_t max_chunk = max(1u, unit >> 7);
    for (;;) {
        uint32_t g0 = 0, chunk = 0;
        if (lane == 0) {
            const uint32_t cur = *reinterpret_cast<volatile uint32_t*>(&sm.scal[SC_UCTR]);
            const uint32_t rem = cur < G ? G - cur : 0u;
            chunk = min(max_chunk, max(1u, rem / (2 * nwarps)));
            g0 = rem ? atomicAdd(&sm.scal[SC_UCTR], chunk) : G;
        }
        g0 = __shfl_sync(0xffffffffu, g0, 0);
        chunk = __shfl_sync(0xffffffffu, chunk, 0);
        if (g0 >= G) break;
        scan_group_range<W, IL>(p, it, sm, sb, nsb, G, g0, min(G, g0 + chunk));
    }
}

// Stages spans [s0, s0 + nsb) of item (q, t): the slice of each list inside
// the tile (s_beg, s_len), its first 128-posting group's rank (s_upref) and,
// for dense spans, the bitmap slot (s_dense, in span order; the slice is then
// empty).  Returns the number of groups.  Warp-only variant for nsb <= 32
// (called by warp 0 alone, no barrier); block variant otherwise (every thread,
// ends with a barrier).
struct StageArgs {
    bool item_mode, dense;
    uint64_t i0, cb, sbq;
    uint32_t nt, S;  // tiles of the query; its spans (the length of a cut row)
};

__device__ __forceinline__ void stage_one(const BatchParams& p, const StageArgs& a, uint32_t t, uint32_t s,
                                          uint64_t& beg, uint32_t& len, int32_t& dslot) {
    dslot = -1;
    if (a.item_mode) {
        const uint64_t it_i = a.i0 + s, kb = p.it_kb[it_i];
        beg = p.key_off[kb];
        len = static_cast<uint32_t>(p.key_off[kb + p.it_nk[it_i]] - beg);
    } else {
        if (a.dense) {
            dslot = p.span_dense[a.sbq + s];
            if (dslot >= 0) {  // the list's bitmap covers this tile: no posting scan (and no cuts)
                beg = 0;
                len = 0;
                return;
            }
        }
        const uint32_t* c = p.cuts + a.cb + uint64_t(t) * a.S + s;
        beg = p.span_beg[a.sbq + s] + c[0];
        len = c[a.S] - c[0];
    }
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Bulk L2 prefetch (TMA unit) of the 16-byte-aligned cover of ids[0, n).
__device__ __forceinline__ void prefetch_l2(const uint32_t* ids, uint32_t n) {
    const uint64_t a = reinterpret_cast<uint64_t>(ids), e = a + uint64_t(n) * 4;
    const uint64_t a16 = a & ~15ull, bytes = ((e + 15) & ~15ull) - a16;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a16), "r"(static_cast<uint32_t>(bytes))
                 : "memory");
}

// Warp variant, first half: the raw words of spans [s0, s0 + nsb) of a
// multi-tile item -- span start, its cut at tile t and t + 1, dense slot --
// go straight from global memory into the stage buffer with asynchronous
// copies (no registers held), all in flight at once; the rows of the
// boundary-major cut table make them coalesced.  Item-mode spans (one-tile
// queries) are read by stage_warp_finish.
__device__ __forceinline__ void stage_warp_issue(const BatchParams& p, const StageArgs& a, const StageBuf& sb,
                                                 uint32_t t, uint32_t s0, uint32_t nsb) {
    if (a.item_mode) return;
    const uint32_t* c0 = p.cuts + a.cb + uint64_t(t) * a.S + s0;
    for (uint32_t i = threadIdx.x & 31; i < nsb; i += 32) {
        cp_async8(sb.beg() + i, p.span_beg + a.sbq + s0 + i);
        cp_async4(sb.ppref() + i, c0 + i);
        cp_async4(sb.upref() + i, c0 + a.S + i);
        if (a.dense) cp_async4(sb.dense() + i, p.span_dense + a.sbq + s0 + i);
    }
}

// Second half: slices (start, length) from the raw words, then group ranks,
// posting prefix and the compacted dense slots, 32 spans at a time, written
// over the raw words in place.  Returns the number of 128-posting groups.
__device__ __forceinline__ uint32_t stage_warp_finish(const BatchParams& p, const StageArgs& a, const StageBuf& sb,
                                                      uint32_t t, uint32_t s0, uint32_t nsb, uint32_t W = 0) {
    const uint32_t lane = threadIdx.x & 31;
#if GENIE_BITMAP_PREFETCH
    // the item's object tile, for the bitmap-row prefetch
    const uint32_t T = W ? tile_objs(p, W) : 0u, tile_lo = t * T;
    const uint32_t tile_n = T ? min(T, p.n - min(p.n, tile_lo)) : 0u;
    const uint32_t tile_word0 = tile_lo >> 5, tile_bytes = (tile_n + 7) / 8;
#endif
    if (!a.item_mode) {
        cp_async_wait_all();
        __syncwarp();
    }
    uint32_t carry = 0, dcarry = 0, pcarry = 0;
    for (uint32_t c0 = 0; c0 < nsb; c0 += 32) {
        const uint32_t i = c0 + lane;
        uint64_t beg = 0;
        uint32_t len = 0, groups = 0;
        int32_t dslot = -1;
        if (i < nsb) {
            if (a.item_mode) {
                stage_one(p, a, t, s0 + i, beg, len, dslot);
            } else {
                dslot = a.dense ? static_cast<int32_t>(sb.dense()[i]) : -1;
                if (dslot < 0) {  // the list's bitmap (dslot >= 0) covers the tile: no slice
                    const uint32_t lo = sb.ppref()[i];
                    beg = sb.beg()[i] + lo;
                    len = sb.upref()[i] - lo;
                }
            }
            groups = len ? static_cast<uint32_t>(((beg + len - 1) >> 7) - (beg >> 7) + 1) : 0u;
            // the slice streams into L2 while the current item is scanned, so
            // this item's posting loads hit L2 instead of waiting on DRAM
#if GENIE_SPAN_PREFETCH == 1
            if (len) prefetch_l2(p.postings + beg, len);
#elif GENIE_SPAN_PREFETCH == 2
            // the slice's first two 128-byte lines into L2 (per-lane prefetch;
            // minHash slices are ~12 postings)
            if (len) {
                // up to GENIE_PREFETCH_LINES 128-byte lines of the slice
                const char* a = reinterpret_cast<const char*>(p.postings + beg);
                const char* line = reinterpret_cast<const char*>(reinterpret_cast<uint64_t>(a) & ~127ull);
                const char* end = a + uint64_t(len) * 4;
                for (uint32_t l = 0; l < GENIE_PREFETCH_LINES && line < end; ++l, line += 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(line));
            }
#endif
        }
        __syncwarp();  // every lane has read its raw words before any result overwrites them
        const uint32_t incl = warp_inclusive_scan(groups);
        const uint32_t pincl = warp_inclusive_scan(len);
        const uint32_t dm = __ballot_sync(0xffffffffu, dslot >= 0);
#if GENIE_BITMAP_PREFETCH
        // the tile's slice of every dense list's bitmap row into L2, its 128-byte
        // lines spread over the warp (C3: 64 lines per list, C2: 184)
        if (dm && tile_bytes) {
            for (uint32_t m = dm; m;) {
                const int o = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t slot = __shfl_sync(0xffffffffu, static_cast<uint32_t>(dslot), o);
                const char* row = reinterpret_cast<const char*>(p.bitmaps + slot + tile_word0);
                for (uint32_t off = lane * 128; off < tile_bytes; off += 32 * 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(row + off));
            }
        }
#endif
        if (i < nsb) {
            sb.beg()[i] = beg;
            sb.upref()[i] = carry + incl - groups;
            sb.ppref()[i] = pcarry + pincl - len;
            // compacted slot index <= i: never a raw word still to be read
            if (dslot >= 0) sb.dense()[dcarry + __popc(dm & ((1u << lane) - 1u))] = static_cast<uint32_t>(dslot);
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
        pcarry += __shfl_sync(0xffffffffu, pincl, 31);
        dcarry += __popc(dm);
    }
    if (lane == 0) sb.ppref()[nsb] = pcarry;  // postings of the batch
    __syncwarp();
    return carry;
}

// Block variant (every thread; ends with a barrier): the further batches of
// queries with more than kSpanBatch spans.
__device__ __forceinline__ uint32_t stage_block(const BatchParams& p, const StageArgs& a, const ScanSmem& sm,
                                                const StageBuf& sb, uint32_t t, uint32_t s0, uint32_t nsb) {
    uint64_t beg = 0;
    uint32_t len = 0, groups = 0;
    int32_t dslot = -1;
    if (threadIdx.x < nsb) {
        stage_one(p, a, t, s0 + threadIdx.x, beg, len, dslot);
        groups = len ? static_cast<uint32_t>(((beg + len - 1) >> 7) - (beg >> 7) + 1) : 0u;
    }
    // one scan of (dense flag << 40 | groups): group ranks and dense slots;
    // one of the lengths: posting prefix
    const unsigned long long v = (static_cast<unsigned long long>(dslot >= 0) << 40) | groups;
    unsigned long long total, ptotal;
    const unsigned long long ex = block_exclusive_scan<unsigned long long>(v, sm.sums, total);
    const unsigned long long pex = block_exclusive_scan<unsigned long long>(len, sm.sums, ptotal);
    if (threadIdx.x == 0) sb.ppref()[nsb] = static_cast<uint32_t>(ptotal);
    if (threadIdx.x < nsb) {
        sb.beg()[threadIdx.x] = beg;
        sb.ppref()[threadIdx.x] = static_cast<uint32_t>(pex);
        sb.upref()[threadIdx.x] = static_cast<uint32_t>(ex & ((1ull << 40) - 1));
        if (dslot >= 0) sb.dense()[ex >> 40] = static_cast<uint32_t>(dslot);
    }
    if (threadIdx.x == 0) sm.scal[SC_UCTR] = 0;
    __syncthreads();
    return static_cast<uint32_t>(total & ((1ull << 40) - 1));
}

// The rest of an item once its counters hold the dense part (or zeros):
// posting scan, then the tile's exact top-k.
__device__ __forceinline__ StageArgs stage_args(const BatchParams& p, const QueryPlan& pl, uint32_t& S) {
    StageArgs sa;
    sa.nt = pl.nt;
    // one tile: the slices are the items' keyword ranges, contiguous in the
    // postings array (keys of one dim are adjacent); several tiles: one slice
    // per keyword list, cut at the tile boundaries by k_cut
    sa.item_mode = sa.nt == 1;
    sa.i0 = pl.item0;
    sa.cb = pl.cut_base;
    sa.sbq = pl.span_base;
    sa.S = pl.S;
    S = sa.item_mode ? pl.nitems : sa.S;
    // dense containers apply when all spans of the query fit one staging batch
    sa.dense = p.n_dense && !sa.item_mode && S <= kSpanBatch;
    return sa;
}

// warps that prepare the next item in the W kernel (GENIE_PREP_WARPS_W8 for W >= 8)
template <int W>
__device__ __host__ constexpr uint32_t prep_warps() {
    return W == kHashW ? GENIE_HASH_PW : (W >= 8 ? GENIE_PREP_WARPS_W8 : 1u);
}
struct WorkQueue {  // one width class's items [base, end) of the work list, claimed via st[ctr]
    uint32_t base, end, ctr;
};
template <int PW>
GENIE_PREP_FN void prepare_item(const BatchParams& p, const ScanSmem& sm, uint32_t buf, const WorkQueue& total);

template <int W, bool IL>
__device__ void scan_and_select(const BatchParams& p, const ItemCtx& it, const ScanSmem& sm, uint32_t b,
                                uint32_t S, uint32_t nsb, uint32_t G, uint32_t ptot, const WorkQueue& total) {
    using L = Lay<W, IL>;
#ifdef GENIE_PHASE_TIMERS
    const long long t_setup = clock64();
#endif
    // warps PW.. scan this item's postings while warps 0..PW-1 prepare the next item
    constexpr uint32_t kScanWarp0 = prep_warps<W>();
#ifdef GENIE_PHASE_TIMERS
    if (threadIdx.x < 32 * kScanWarp0) {
        prepare_item<kScanWarp0>(p, sm, b ^ 1u, total);
        if (threadIdx.x == 0) atomicAdd(&p.st[ST_T_PREP], static_cast<unsigned long long>(clock64() - t_setup));
    } else {
        scan_groups<W, IL>(p, it, sm, sm.sb(b), nsb, G, p.unit, kScanWarp0, ptot);
        const uint32_t dt = static_cast<uint32_t>(clock64() - t_setup);
        if (threadIdx.x == 32) atomicAdd(&p.st[ST_T_WARP1], static_cast<unsigned long long>(dt));
        if ((threadIdx.x & 31) == 0) {
            atomicMax(&sm.scal[SC_WMAX], dt);
            atomicMin(&sm.scal[SC_WMIN], dt);
        }
    }
#else
    if (threadIdx.x < 32 * kScanWarp0) prepare_item<kScanWarp0>(p, sm, b ^ 1u, total);
    else scan_groups<W, IL>(p, it, sm, sm.sb(b), nsb, G, p.unit, kScanWarp0, ptot);
#endif
    __syncthreads();
    for (uint32_t s0 = kSpanBatch; s0 < S; s0 += kSpanBatch) {  // long queries: further batches
        uint32_t S_;
        const StageArgs sa = stage_args(p, p.plan[it.q], S_);
        const uint32_t nb = min(kSpanBatch, S - s0);
        const uint32_t g = stage_block(p, sa, sm, sm.sb(b), it.t, s0, nb);
        scan_groups<W, IL>(p, it, sm, sm.sb(b), nb, g, p.unit, 0);
        __syncthreads();
    }
#ifdef GENIE_PHASE_TIMERS
    const long long t_scanned = clock64();
    if (threadIdx.x == 0) {
        atomicAdd(&p.st[ST_T_WMAX], static_cast<unsigned long long>(sm.scal[SC_WMAX]));
        atomicAdd(&p.st[ST_T_WMIN], static_cast<unsigned long long>(sm.scal[SC_WMIN]));
        sm.scal[SC_WMAX] = 0;
        sm.scal[SC_WMIN] = 0xffffffffu;
    }
#endif
    // ---- select: the tile's exact top-k
    if (it.admit && !sm.scal[SC_OVF]) {
        uint32_t a = sm.scal[SC_AT];  // every thread finishes AT (cpq.hpp:383-389)
        while (a <= it.bound && sm.za[a] >= it.kq) ++a;
        const uint32_t thr = a - 1;  // cpq.hpp:310-311
        const uint32_t floor = sm.scal[SC_FLOOR];
        // The tile's record for the later tiles of its query (gate_start):
        // base level b and, counted by emit(), n[j] = #emitted entries
        // counting >= b + j (any prefix of those adds is a valid under-count)
        ItemCtx itr = it;
        itr.rec_b = max((thr > 0 && thr >= floor) ? thr : floor, 1u);
        if (threadIdx.x == 0) p.tile_rec[uint64_t(it.slot) * kRecWords] = itr.rec_b;
        // table entries above the threshold (all touched ids when thr == 0);
        // an id may own a stale slot -- only the slot holding its final
        // count is reported (cpq.hpp:212-222, 391-406)
        const uint4* ht4 = reinterpret_cast<const uint4*>(sm.ht);
        for (uint32_t s = threadIdx.x; s < it.ht_cap / 2; s += blockDim.x) {
            const uint4 w2 = ht4[s];
            const uint64_t ws[2] = {(uint64_t(w2.y) << 32) | w2.x, (uint64_t(w2.w) << 32) | w2.z};
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint64_t w = ws[e];
                if (w == kEmptySlot) continue;
                const uint32_t id = uint32_t(w >> 32), v = uint32_t(w >> 16) & 0xffffu;
                const uint32_t c = L::get(sm.cnt, id);
                if (v == c && c > thr) emit(p, itr, sm, id, c);
            }
        }
        __syncthreads();
        const uint32_t n_above = sm.scal[SC_NOUT];
        // thr >= floor: thr is the tile's true k-th count -> tie fill and
        // publish it as the query's new floor.  thr < floor (AT never left
        // the floor): fewer than k objects reach the floor here; they are all
        // in the table and nothing below the floor can make the global top-k.
        if (thr > 0 && thr >= floor) {
#ifdef GENIE_PHASE_TIMERS
            const long long tt0 = clock64();
            if (n_above < it.kq) emit_ties<W, IL>(p, itr, sm, thr, it.kq - n_above);
            if (threadIdx.x == 0) {
                atomicAdd(&p.st[ST_T_GATE], 1ull);
                atomicAdd(&p.st[ST_T_STAGE], static_cast<unsigned long long>(clock64() - tt0));
            }
#else
            if (n_above < it.kq) emit_ties<W, IL>(p, itr, sm, thr, it.kq - n_above);
#endif
            if (threadIdx.x == 0) atomicMax(&p.q_floor[it.q], thr);
        }
    } else {
        if (it.admit && threadIdx.x == 0) atomicAdd(&p.st[ST_FALLBACK], 1ull);
        const uint32_t T_t = hist_select<W, IL>(p, it, sm);
        if (it.gate && T_t > 0 && threadIdx.x == 0) atomicMax(&p.q_floor[it.q], T_t);
    }
    __syncthreads();
    if (threadIdx.x == 0) p.tile_len[it.slot] = sm.scal[SC_NOUT];
#ifdef GENIE_PHASE_TIMERS
    if (threadIdx.x == 0) {
        const long long t_end = clock64();
        atomicAdd(&p.st[ST_T_SCAN], static_cast<unsigned long long>(t_scanned - t_setup));
        atomicAdd(&p.st[ST_T_EXTRACT], static_cast<unsigned long long>(t_end - t_scanned));
        atomicAdd(&p.st[ST_ADMIT_CALLS], static_cast<unsigned long long>(sm.scal[SC_ADM_CALLS]));
        atomicAdd(&p.st[ST_ADMIT_PASS], static_cast<unsigned long long>(sm.scal[SC_ADM_PASS]));
        sm.scal[SC_ADM_CALLS] = 0;
        sm.scal[SC_ADM_PASS] = 0;
    }
#endif
}

// Where the c-PQ gate of tile t of query q starts (its AuditThreshold floor).
// Two valid lower limits for the count an object of this tile needs to make
// the merged top-k:
//  * F = the query's published floor: the largest k-th count of a finished
//    tile (q_floor) -- the global k-th count (Appendix A rule 2) is at least F;
//  * c_low + 1, where k objects of LOWER tiles (smaller ids) are known to
//    count >= c_low: an object here counting <= c_low loses to all of them
//    (count desc, id asc -- cpq.hpp:37-40), so it cannot enter.
// The lower tiles' knowledge comes from their records (b, n[j] = #emitted
// entries counting >= b + j): emitted entries are distinct objects with their
// final counts, and a record read half-written or still zero only
// under-counts.  Called by one whole warp.  Returns max(F, c_low + 1).
__device__ __forceinline__ uint32_t gate_start(const BatchParams& p, uint32_t q, uint32_t t, uint32_t kq,
                                               uint32_t bound, uint32_t tbase) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t F = __ldcg(p.q_floor + q);
    uint32_t tot[kRecLevels];  // entries of lower tiles counting >= F + j
#pragma unroll
    for (int j = 0; j < kRecLevels; ++j) tot[j] = 0;
    const uint32_t* base = p.tile_rec + uint64_t(tbase) * kRecWords;
    for (uint32_t l = lane; l < t; l += 32) {
        const uint4* r4 = reinterpret_cast<const uint4*>(base + uint64_t(l) * kRecWords);
        uint32_t r[kRecWords];
#pragma unroll
        for (int j = 0; j < int(kRecWords / 4); ++j) {
            const uint4 x = __ldcg(r4 + j);
            r[4 * j] = x.x, r[4 * j + 1] = x.y, r[4 * j + 2] = x.z, r[4 * j + 3] = x.w;
        }
        const uint32_t b = r[0];
#pragma unroll
        for (int j = 0; j < kRecLevels; ++j) {
            const uint32_t c = F + j;  // level whose lower-tile population is summed
            uint32_t n = 0;
            if (c <= b) n = r[1];
#pragma unroll
            for (int i = 1; i < kRecLevels; ++i)
                if (c == b + i) n = r[1 + i];
            tot[j] += n;
        }
    }
    uint32_t start = F;
#pragma unroll
    for (int j = 0; j < kRecLevels; ++j) {
        const uint32_t s = warp_sum(tot[j]);
        if (s >= kq && F + j >= 1) start = max(start, F + j + 1);
    }
    return min(start, bound + 1);
}

__device__ __forceinline__ uint32_t fetch_item(const BatchParams& p, const WorkQueue& wq) {
    const unsigned long long i = wq.base + atomicAdd(&p.st[wq.ctr], 1ull);
    return i < wq.end ? static_cast<uint32_t>(i) : 0xffffffffu;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Warp 0: prepares the CTA's next work item into desc[buf] / stage buffer
// `buf` while the other warps scan the current one (valid = 0 when the queue
// is empty).  A two-deep pipeline keeps this to ONE memory round trip per
// item: on entry the item (query q, tile t) is known and q's plan already sits
// in shared memory (copied asynchronously by the previous call), and the item
// after it has been claimed.  This call issues at once the span words of its
// item (asynchronous copies), the lower tiles' records (gate start), the
// (query, tile) of the claimed item and the next claim; then it finishes the
// staging and starts the copy of the claimed item's plan.
__device__ __forceinline__ void named_barrier(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// PW = 1: warp 0 does everything below.  PW = 2 (the W >= 8 kernels: C3-C5,
// whose items stage up to 237 short slices): warp 1 stages the slices while
// warp 0 claims, reads the records for the gate start and writes the
// descriptor -- the two halves of the round trip run side by side (two
// named barriers: the plan is in shared memory / warp 1 is done with it).
template <int PW>
GENIE_PREP_FN void prepare_item(const BatchParams& p, const ScanSmem& sm, uint32_t buf, const WorkQueue& total) {
    const uint32_t lane = threadIdx.x & 31, pw = threadIdx.x >> 5;  // pw < PW
    ItemDesc* d = sm.desc + buf;
    const uint32_t item = sm.scal[SC_PF_ITEM];
    if (item == 0xffffffffu) {
        if (threadIdx.x == 0) d->valid = 0;
        return;
    }
    const uint32_t q = sm.scal[SC_PF_Q], t = sm.scal[SC_PF_T], claim = sm.scal[SC_CLAIM];
    constexpr uint32_t kStager = PW - 1;  // the warp that stages the slices
#ifdef GENIE_PHASE_TIMERS
    const long long pt0 = clock64();
#endif
#if GENIE_PLAN_ASYNC
    if (pw == 0) cp_async_wait_all();  // q's plan (issued by warp 0 in the previous call)
    if constexpr (PW > 1) named_barrier(1, 32 * PW);
    else __syncwarp();
    const QueryPlan pl = *sm.plan;
#else
    const QueryPlan pl = p.plan[q];
#endif
#ifdef GENIE_PHASE_TIMERS
    const long long pt1 = clock64();
#endif
    uint32_t S;
    const StageArgs sa = stage_args(p, pl, S);
    const uint32_t nsb = min(kSpanBatch, S);
    if (pw == kStager) stage_warp_issue(p, sa, sm.sb(buf), t, 0, nsb);
    uint32_t nq = 0, ntile = 0, a0 = 0;
    unsigned long long raw_claim = ~0ull;
    const bool gate = (p.selector == GENIE_SELECT_CPQ) && (pl.W <= 8 || pl.W == kHashW);
#ifdef GENIE_PHASE_TIMERS
    long long pt2 = 0, pt3 = 0;
#endif
    if (pw == 0) {
        if (claim != 0xffffffffu) {
            nq = p.work_q[claim];
            ntile = p.work_t[claim];
        }
        // the next claim: the raw counter value is range-checked only at the
        // end, so nothing waits on the atomic's round trip before then
        if (lane == 0 && claim != 0xffffffffu) raw_claim = atomicAdd(&p.st[total.ctr], 1ull);
#ifdef GENIE_PHASE_TIMERS
        pt2 = clock64();
#endif
        a0 = gate ? gate_start(p, q, t, pl.k, pl.bound, pl.tile_base) : 0u;
#ifdef GENIE_PHASE_TIMERS
        pt3 = clock64();
#endif
    }
    uint32_t G = 0;
    if (pw == kStager) {
        G = stage_warp_finish(p, sa, sm.sb(buf), t, 0, nsb, pl.W);
        if (lane == 0) {
            d->G = G;
            d->ptot = sm.sb(buf).ppref()[nsb];
        }
    }
    if constexpr (PW > 1) named_barrier(2, 32 * PW);  // staging done, warp 1 no longer reads sm.plan
#ifdef GENIE_PHASE_TIMERS
    const long long pt4 = clock64();
    if (threadIdx.x == 0) {  // prepare split: plan wait / issue / gate start / staging finish
        atomicAdd(&p.st[ST_P_WAIT], static_cast<unsigned long long>(pt1 - pt0));
        atomicAdd(&p.st[ST_P_ISSUE], static_cast<unsigned long long>(pt2 - pt1));
        atomicAdd(&p.st[ST_P_GATE], static_cast<unsigned long long>(pt3 - pt2));
        atomicAdd(&p.st[ST_P_STAGE], static_cast<unsigned long long>(pt4 - pt3));
    }
#endif
    if (pw != 0) return;
    if (claim != 0xffffffffu && lane < sizeof(QueryPlan) / 16)
        if (GENIE_PLAN_ASYNC)
            cp_async16(reinterpret_cast<uint4*>(sm.plan) + lane, reinterpret_cast<const uint4*>(p.plan + nq) + lane);
    raw_claim = __shfl_sync(0xffffffffu, raw_claim, 0);
    const uint32_t nclaim = raw_claim != ~0ull && total.base + raw_claim < total.end
                                ? static_cast<uint32_t>(total.base + raw_claim)
                                : 0xffffffffu;
    if (lane == 0) {
        d->q = q;
        d->t = t;
        d->kq = pl.k;
        d->bound = pl.bound;
        d->W = pl.W;
        d->cap = pl.cap;
        d->nt = sa.nt;
        d->S = S;
        d->nd = sa.dense ? pl.nd : 0u;
        d->a0 = a0;
        d->out_base = pl.out_base + uint64_t(t) * pl.cap;
        d->tile_slot = pl.tile_base + t;
        d->valid = 1;
        sm.scal[SC_PF_ITEM] = claim;
        sm.scal[SC_PF_Q] = nq;
        sm.scal[SC_PF_T] = ntile;
        sm.scal[SC_CLAIM] = nclaim;
    }
    __syncwarp();
}

template <int W, bool FH>
__device__ void process_item(const BatchParams& p, const ScanSmem& sm0, uint32_t b, const WorkQueue& total) {
#ifdef GENIE_PHASE_TIMERS
    const long long t_begin = clock64();
#endif
    ScanSmem sm = sm0;
    const ItemDesc& d = sm.desc[b];
    ItemCtx it;
    it.q = d.q;
    it.t = d.t;
    it.kq = d.kq;
    it.bound = d.bound;
    const uint32_t T = tile_objs(p, W);
    it.tile_lo = it.t * T;
    it.tile_n = min(T, p.n - it.tile_lo);
    it.words = ((it.tile_n + 31) >> 5) * W;  // whole 32-object blocks
    it.cap = d.cap;
    it.slot = d.tile_slot;
    it.out_base = d.out_base;
    it.gate = (p.selector == GENIE_SELECT_CPQ) && W <= 8;
    // An item whose gate starts at zero (a query's first tile: no floor, no
    // lower-tile records) admits in bulk until AT climbs; on a small tile
    // (<= kFirstHistWords counter words, e.g. C1's one-tile queries) it is
    // cheaper to count without the gate and take the exact histogram select
    // (records and floor as usual: C1 1.38 M -> 2.0 M q/s); on large tiles
    // the histogram's pass over every counter costs more (C2 -21 %)
    // (FH: the k_scan<4> instance launched for indexes of at most kFirstHistWords
    // x 32 / 4 objects; every other instance keeps the gate: admit == gate)
    it.admit = FH ? it.gate && !(d.a0 <= 1 && it.words <= kFirstHistWords) : it.gate;
    // The table sits right after the item's counters (whole 16-word steps of
    // dense_init): p.ht_slots slots, or -- for a query's first tile, whose
    // gate starts low without lower-tile records and admits in bulk (one-tile
    // queries, C1) -- all the room up to kHtMaxSlots.  The reference sizes it
    // bit_ceil(2 k bound) (cpq.hpp:137-138, 283; that figure is kept for
    // MemoryStats); concurrent admissions arrive in bursts of up to one per
    // thread before AT can move, and spare capacity absorbs them without the
    // exact-histogram fallback.  Results do not depend on the capacity.
    {
        const uint32_t cnt_bytes = ((it.words + 15) & ~15u) * 4;
        const uint32_t room = (p.tile_bits / 8 + p.ht_slots * 8 - cnt_bytes) / 8;
        it.ht_cap = it.t == 0 ? min(kHtMaxSlots, 1u << (31 - __clz(room))) : p.ht_slots;
        sm.ht = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sm.cnt) + cnt_bytes);
    }
    const uint32_t S = d.S, nd = d.nd, G = d.G, ptot = d.ptot;
    const uint32_t nsb = min(kSpanBatch, S);

    // setup (cpq.hpp:281-292): empty table and ZA, AT at the gate start
    // (gate_start); counters zeroed unless the dense phase writes them
    if (it.admit) {
        uint4* ht4 = reinterpret_cast<uint4*>(sm.ht);
        for (uint32_t i = threadIdx.x; i < it.ht_cap / 2; i += blockDim.x) ht4[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
        for (uint32_t i = threadIdx.x; i <= it.bound; i += blockDim.x) sm.za[i] = 0;
    }
    if (!nd) {
        uint4* c4 = reinterpret_cast<uint4*>(sm.cnt);
        // four 16-byte stores per loop trip (the zeroing is a fixed cost of
        // every sparse item: C4 spends ~8 % of its instructions here)
        const uint32_t n4 = it.words / 4;
        uint32_t i = threadIdx.x;
        for (; i + 3 * kScanThreads < n4; i += 4 * kScanThreads) {
            c4[i] = make_uint4(0, 0, 0, 0);
            c4[i + kScanThreads] = make_uint4(0, 0, 0, 0);
            c4[i + 2 * kScanThreads] = make_uint4(0, 0, 0, 0);
            c4[i + 3 * kScanThreads] = make_uint4(0, 0, 0, 0);
        }
        for (; i < n4; i += kScanThreads) c4[i] = make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) {
        const uint32_t floor = it.gate ? d.a0 : 0u;
        sm.scal[SC_AT] = floor > 1 ? floor : 1;
        sm.scal[SC_FLOOR] = floor;
        sm.scal[SC_OVF] = 0;
        sm.scal[SC_NOUT] = 0;
        sm.scal[SC_UCTR] = 0;
#pragma unroll
        for (int l = 0; l < 8; ++l) sm.scal[SC_LVL + l] = 0;
    }
    __syncthreads();
#ifdef GENIE_PHASE_TIMERS
    if (threadIdx.x == 0) atomicAdd(&p.st[ST_T_SETUP], static_cast<unsigned long long>(clock64() - t_begin));
#endif
    if (nd) {
        const uint32_t at0 = sm.scal[SC_AT];
        const uint32_t dmax = min(nd, it.bound);
        const uint32_t nlv = (it.admit && at0 <= dmax) ? min(dmax - at0 + 1, kLvl) : 0u;
#ifdef GENIE_PHASE_TIMERS
        const long long t_d = clock64();
#endif
        bool csa_path;
#ifdef GENIE_PHASE_TIMERS
        long long t_di = 0;
        const uint32_t reach = dense_init<W>(p, it, sm, sm.sb(b), nd, at0, nlv, csa_path, &t_di);
        const long long t_db = clock64();
#else
        const uint32_t reach = dense_init<W>(p, it, sm, sm.sb(b), nd, at0, nlv, csa_path);
#endif
        if (it.admit && at0 <= dmax) dense_gate<W>(it, sm, at0, dmax, nlv, reach, csa_path);
#ifdef GENIE_PHASE_TIMERS
        if (threadIdx.x == 0) {
            atomicAdd(&p.st[ST_T_DENSE], static_cast<unsigned long long>(clock64() - t_d));
            atomicAdd(&p.st[ST_DENSE_ND],
                      static_cast<unsigned long long>(nd) | (1ull << 32) | (csa_path ? (1ull << 48) : 0ull));
            atomicAdd(&p.st[ST_T_LAT], static_cast<unsigned long long>(t_di - t_d));
            atomicAdd(&p.st[ST_T_LATN], static_cast<unsigned long long>(t_db - t_d));
        }
#endif
        scan_and_select<W, true>(p, it, sm, b, S, nsb, G, ptot, total);
    } else {
        scan_and_select<W, false>(p, it, sm, b, S, nsb, G, ptot, total);
    }
}

// ------------------------------------------------------ hashed sparse class
//
// A query whose postings are few for the objects they spread over (tens to a
// few hundred postings per 94 K-object W = 8 tile: sparse sets over tens of
// millions of objects) spends almost all of a dense item on fixed per-item
// work -- the prepare chain, zeroing the counter tile, the extract scans,
// barriers.  The hashed class (k_resolve, GENIE_HASH_DENSE_MAX) gives such a
// query tiles of GENIE_HASH_TILES x the W = 8 tile (2^20 objects) and counts into
// an open-addressing table in the counter area instead: one 32-bit slot per
// touched object, (local id << 8) | count, linear probing; a posting costs one
// shared CAS (first touch) or CAS + add.  The Count Priority Queue state is
// then read off the final counts: ZA[v] = #objects counting >= v is a suffix
// sum of the count histogram, so AT = the first level >= the gate start that
// fewer than k objects reach (cpq.hpp:374-389), thr = AT - 1, and the tile
// emits exactly what extract() does (cpq.hpp:307-339): every count > thr,
// then the first k - above ties at thr in ascending id -- found by a two-level
// radix selection on the tie ids.  Records and the query floor as in
// scan_and_select.  An item whose postings exceed the table's fill limit
// (skewed ids) counts its tile as 8-bit dense sub-tiles of hash_sub_T objects
// instead and emits each sub-tile's exact top-k (hist_select).
constexpr uint32_t kEmptyHash = 0xffffffffu;
constexpr uint32_t kTieBins = 1024;
static_assert((kScanThreads / 32) * 256 * 4 + kTieBins * 4 <= kHashScratch, "hashed-item scratch");

__device__ __forceinline__ uint32_t atom_cas_shared(uint32_t addr, uint32_t cmp, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(addr), "r"(cmp), "r"(v));
    return old;
}
__device__ __forceinline__ void red_add_shared(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

// One posting: count object `local` in the table at shared address `tab`.
__device__ __forceinline__ void hash_count(uint32_t tab, uint32_t hmask, uint32_t hshift, uint32_t local) {
    const uint32_t key = local << 8;
    uint32_t h = (local * 0x9E3779B1u) >> hshift;
    for (;;) {
        const uint32_t a = tab + h * 4;
        const uint32_t old = atom_cas_shared(a, kEmptyHash, key | 1u);
        if (old == kEmptyHash) return;
        if ((old & ~0xffu) == key) {
            red_add_shared(a, 1u);
            return;
        }
        h = (h + 1) & hmask;
    }
}

// A warp's contiguous run [r0, r1) of the item's staged postings (across its
// slices, as scan_compact), lane l taking r0 + l + 32 j.  SUB = false: count
// into the table; SUB = true: 8-bit dense counters of the objects
// [lo, lo + n) (linear layout), other ids skipped.
template <bool SUB>
__device__ __forceinline__ void hashed_scan(const uint32_t* __restrict__ postings, const StageBuf& sb, uint32_t nsb,
                                            uint32_t r0, uint32_t r1, uint32_t lo, uint32_t n, uint32_t base,
                                            uint32_t hmask, uint32_t hshift) {
    constexpr int UNR = GENIE_HASH_UNR;
    if (r0 >= r1) return;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t* pp = sb.ppref();
    uint32_t si;
    {
        const uint32_t r = min(r0 + lane, r1 - 1);
        uint32_t a = 0, b = nsb;
        while (a < b) {
            const uint32_t m = (a + b) >> 1;
            if (pp[m] <= r) a = m + 1;
            else b = m;
        }
        si = a - 1;
    }
    for (uint32_t r00 = r0; r00 < r1; r00 += 32 * UNR) {
        uint32_t x[UNR];
        uint32_t ok = 0;
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t r = r00 + u * 32 + lane;
            x[u] = 0;
            if (r < r1) {
                while (pp[si + 1] <= r) ++si;
                x[u] = __ldg(postings + sb.beg()[si] + (r - pp[si]));
                ok |= 1u << u;
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if (!((ok >> u) & 1u)) continue;
            const uint32_t d = x[u] - lo;
            if constexpr (SUB) {
                if (d < n) red_add_shared(base + (d >> 2) * 4, 1u << ((d & 3u) * 8));
            } else {
                hash_count(base, hmask, hshift, d);
            }
        }
    }
}

// The tile's exact top-k from the table (see above).
__device__ void hashed_select(const BatchParams& p, const ItemCtx& it, const ScanSmem& sm, uint32_t H) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t* tab = sm.cnt;
    uint32_t* hsub = sm.cnt + H;                       // per-warp 256-bin count histograms
    uint32_t* tbin = hsub + (kScanThreads / 32) * 256;  // tie bins
    const uint4* t4 = reinterpret_cast<const uint4*>(tab);
#ifdef GENIE_PHASE_TIMERS
    const long long hs0 = clock64();
#endif
    // 1. count histogram (counts 1..3, the bulk, tallied in registers)
    {
        uint32_t n1 = 0, n2 = 0, n3 = 0;
        uint32_t* hw = hsub + warp * 256;
        for (uint32_t i = threadIdx.x; i < H / 4; i += kScanThreads) {
            const uint4 v = t4[i];
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (w[e] == kEmptyHash) continue;
                const uint32_t c = w[e] & 0xffu;
                n1 += c == 1;
                n2 += c == 2;
                n3 += c == 3;
                if (c > 3) atomicAdd(&hw[c], 1u);
            }
        }
        n1 = warp_sum(n1);
        n2 = warp_sum(n2);
        n3 = warp_sum(n3);
        if (lane == 0) {
            hw[1] += n1;
            hw[2] += n2;
            hw[3] += n3;
        }
    }
    __syncthreads();
#ifdef GENIE_PHASE_TIMERS
    const long long hs1 = clock64();
#endif
    // 2. ZA[v] = #objects counting >= v, the histogram's suffix sums (threads
    // 0..255: bin 255 - t, warp scans + the lower warps' totals), then AT =
    // the first level >= the gate start that fewer than k objects reach
    {
        const uint32_t t = threadIdx.x;
        uint32_t v = 0;
        if (t < 256)
            for (uint32_t w = 0; w < kScanThreads / 32; ++w) v += hsub[w * 256 + (255 - t)];
        const uint32_t incl = warp_inclusive_scan(v);
        if (lane == 31) sm.sums[warp] = incl;
        __syncthreads();
        if (t < 256) {
            uint32_t add = 0;
            for (uint32_t w = 0; w < warp; ++w) add += static_cast<uint32_t>(sm.sums[w]);
            sm.za[255 - t] = incl + add;
        }
        __syncthreads();
        const uint32_t floor = sm.scal[SC_FLOOR], a0 = floor > 1 ? floor : 1u;
        if (t < 256 && t >= a0 && (t > it.bound || sm.za[t] < it.kq)) atomicMin(&sm.scal[SC_HTHR], t);
        __syncthreads();
        if (t == 0) {
            const uint32_t at = min(sm.scal[SC_HTHR], it.bound + 1);
            sm.scal[SC_HTHR] = at - 1;
            sm.scal[SC_HABOVE] = at <= 255 ? sm.za[at] : 0u;
        }
    }
    __syncthreads();
#ifdef GENIE_PHASE_TIMERS
    const long long ht1 = clock64();
    if (threadIdx.x == 0) {
        atomicAdd(&p.st[ST_P_WAIT], static_cast<unsigned long long>(hs1 - hs0));
        atomicAdd(&p.st[ST_P_ISSUE], static_cast<unsigned long long>(ht1 - hs1));
    }
#endif
    const uint32_t thr = sm.scal[SC_HTHR], above = sm.scal[SC_HABOVE], floor = sm.scal[SC_FLOOR];
    ItemCtx itr = it;
    itr.rec_b = max((thr > 0 && thr >= floor) ? thr : floor, 1u);
    if (threadIdx.x == 0) p.tile_rec[uint64_t(it.slot) * kRecWords] = itr.rec_b;
    const bool ties = thr > 0 && thr >= floor;  // then ZA[thr] >= k > above: ties fill the rest
    const uint32_t need = ties ? it.kq - above : 0u;
    const uint32_t lbits = 32 - __clz(max(it.tile_n - 1, 1u));  // <= 20 bits (host caps the tile)
    const uint32_t shift = lbits > 10 ? lbits - 10 : 0u;
    // 3. counts > thr out; tie bins by the high id bits
    for (uint32_t i = threadIdx.x; i < H / 4; i += kScanThreads) {
        const uint4 v = t4[i];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (w[e] == kEmptyHash) continue;
            const uint32_t c = w[e] & 0xffu;
            if (c > thr) emit(p, itr, sm, w[e] >> 8, c);
            else if (ties && c == thr) atomicAdd(&tbin[(w[e] >> 8) >> shift], 1u);
        }
    }
    __syncthreads();
#ifdef GENIE_PHASE_TIMERS
    const long long ht2 = clock64();
    if (threadIdx.x == 0) atomicAdd(&p.st[ST_T_DENSE], static_cast<unsigned long long>(ht2 - ht1));
#endif
    if (!ties) return;
    // 4. the bin holding the need-th smallest tie id, and the rank inside it
    auto find_rank = [&](uint32_t want, uint32_t slot_bin, uint32_t slot_rank) {
        if (warp == 0) {
            uint32_t s = 0;  // lane l: bins 32 l .. 32 l + 31, read rotated (no bank conflicts)
            for (uint32_t j = 0; j < kTieBins / 32; ++j) s += tbin[lane * (kTieBins / 32) + ((j + lane) & 31)];
            const uint32_t incl = warp_inclusive_scan(s);
            uint32_t cum = incl - s;
            if (cum < want && want <= incl) {
                for (uint32_t j = 0; j < kTieBins / 32; ++j) {
                    const uint32_t v = tbin[lane * (kTieBins / 32) + j];
                    if (cum + v >= want) {
                        sm.scal[slot_bin] = lane * (kTieBins / 32) + j;
                        sm.scal[slot_rank] = want - cum;
                        break;
                    }
                    cum += v;
                }
            }
        }
        __syncthreads();
    };
    find_rank(need, SC_HBIN, SC_HNEED);
    const uint32_t B = sm.scal[SC_HBIN];
    uint32_t cut = B << shift;  // the need-th smallest tie id
    if (shift) {
        // 5. ids are distinct: flag the low parts of bin B's ties, pick the rank
        const uint32_t need2 = sm.scal[SC_HNEED];
        for (uint32_t i = threadIdx.x; i < kTieBins; i += kScanThreads) tbin[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < H / 4; i += kScanThreads) {
            const uint4 v = t4[i];
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (w[e] != kEmptyHash && (w[e] & 0xffu) == thr && ((w[e] >> 8) >> shift) == B)
                    tbin[(w[e] >> 8) & ((1u << shift) - 1u)] = 1u;
        }
        __syncthreads();
        find_rank(need2, SC_HCUT, SC_HNEED);
        cut |= sm.scal[SC_HCUT];
    }
    // 6. ties with id <= cut: exactly `need` of them
    for (uint32_t i = threadIdx.x; i < H / 4; i += kScanThreads) {
        const uint4 v = t4[i];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (w[e] != kEmptyHash && (w[e] & 0xffu) == thr && (w[e] >> 8) <= cut) emit(p, itr, sm, w[e] >> 8, thr);
    }
    if (threadIdx.x == 0) atomicMax(&p.q_floor[it.q], thr);
#ifdef GENIE_PHASE_TIMERS
    if (threadIdx.x == 0) {
        atomicAdd(&p.st[ST_T_GATE], 1ull);
        atomicAdd(&p.st[ST_T_STAGE], static_cast<unsigned long long>(clock64() - ht2));
    }
#endif
}

// Overflow path: the tile as 8-bit dense sub-tiles, each one's exact top-k
// (up to ceil(T / hash_sub_T) x k entries: the class's tile capacity).
__device__ void hashed_sub_tiles(const BatchParams& p, const ItemCtx& it, const ScanSmem& sm0, const StageBuf& sb,
                                 uint32_t nsb, uint32_t ptot) {
    ScanSmem sm = sm0;
    const uint32_t nwarps = kScanThreads / 32, warp = threadIdx.x >> 5;
    const uint32_t share = (ptot + nwarps - 1) / nwarps;
    const uint32_t r0 = min(ptot, warp * share), r1 = min(ptot, r0 + share);
    for (uint32_t lo = 0; lo < it.tile_n; lo += p.hash_sub_T) {
        ItemCtx is = it;
        is.tile_lo = it.tile_lo + lo;
        is.tile_n = min(p.hash_sub_T, it.tile_n - lo);
        is.words = ((is.tile_n + 31) >> 5) * 8;
        is.gate = false;
        is.ht_cap = kHtSlots;
        sm.ht = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sm.cnt) + ((is.words + 15) & ~15u) * 4);
        uint4* c4 = reinterpret_cast<uint4*>(sm.cnt);
        for (uint32_t i = threadIdx.x; i < (is.words + 3) / 4; i += kScanThreads) c4[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        hashed_scan<true>(p.postings, sb, nsb, r0, r1, is.tile_lo, is.tile_n, smem_u32(sm.cnt), 0, 0);
        __syncthreads();
        hist_select<8, false>(p, is, sm);
        __syncthreads();
    }
    if (threadIdx.x == 0) atomicAdd(&p.st[ST_FALLBACK], 1ull);
}

__device__ void process_item_hashed(const BatchParams& p, const ScanSmem& sm, uint32_t b, const WorkQueue& total) {
    constexpr uint32_t PW = prep_warps<kHashW>();
    const ItemDesc& d = sm.desc[b];
    ItemCtx it;
    it.q = d.q;
    it.t = d.t;
    it.kq = d.kq;
    it.bound = d.bound;
    const uint32_t T = tile_objs(p, kHashW);
    it.tile_lo = it.t * T;
    it.tile_n = min(T, p.n - it.tile_lo);
    it.words = 0;
    it.cap = d.cap;
    it.slot = d.tile_slot;
    it.out_base = d.out_base;
    it.gate = true;
    it.admit = false;
    it.ht_cap = 0;
    const uint32_t nsb = min(kSpanBatch, d.S), ptot = d.ptot;
    const uint32_t H = p.hash_slots;
    const bool fast = ptot <= p.hash_fill;  // block-uniform
#ifdef GENIE_PHASE_TIMERS
    const long long t0 = clock64();
#endif
    if (fast) {
        uint4* t4 = reinterpret_cast<uint4*>(sm.cnt);
        for (uint32_t i = threadIdx.x; i < H / 4; i += kScanThreads) t4[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
        uint4* h4 = reinterpret_cast<uint4*>(sm.cnt + H);
        for (uint32_t i = threadIdx.x; i < ((kScanThreads / 32) * 256 + kTieBins) / 4; i += kScanThreads)
            h4[i] = make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) {
        sm.scal[SC_FLOOR] = d.a0;
        sm.scal[SC_NOUT] = 0;
        sm.scal[SC_HTHR] = 0xffffffffu;
    }
    __syncthreads();
#ifdef GENIE_PHASE_TIMERS
    const long long t1 = clock64();
#endif
    // warps 0 .. PW-1 prepare the next item while the others count this one
    if (threadIdx.x < 32 * PW) {
        prepare_item<PW>(p, sm, b ^ 1u, total);
    } else if (fast) {
        const uint32_t nwarps = kScanThreads / 32 - PW, warp = (threadIdx.x >> 5) - PW;
        const uint32_t share = (ptot + nwarps - 1) / nwarps;
        const uint32_t r0 = min(ptot, warp * share), r1 = min(ptot, r0 + share);
        hashed_scan<false>(p.postings, sm.sb(b), nsb, r0, r1, it.tile_lo, 0, smem_u32(sm.cnt), H - 1,
                           1u + __clz(H));
    }
    __syncthreads();
#ifdef GENIE_PHASE_TIMERS
    const long long t2 = clock64();
#endif
#if GENIE_HASH_NOSELECT  // timing experiment only: results are not produced
    if (false) hashed_select(p, it, sm, H);
#else
    if (fast) hashed_select(p, it, sm, H);
#endif
    else if (!fast) hashed_sub_tiles(p, it, sm, sm.sb(b), nsb, ptot);
    __syncthreads();
    if (threadIdx.x == 0) p.tile_len[it.slot] = sm.scal[SC_NOUT];
#ifdef GENIE_PHASE_TIMERS
    if (threadIdx.x == 0) {
        atomicAdd(&p.st[ST_T_SETUP], static_cast<unsigned long long>(t1 - t0));
        atomicAdd(&p.st[ST_T_SCAN], static_cast<unsigned long long>(t2 - t1));
        atomicAdd(&p.st[ST_T_EXTRACT], static_cast<unsigned long long>(clock64() - t2));
        atomicAdd(&p.st[ST_T_WMAX], static_cast<unsigned long long>(ptot));
    }
#endif
}

// One persistent kernel per counter width W (its own register allocation):
// the CTAs drain the W class's slice of the work list (k_worklist orders the
// list class-major), a launch per class.
template <int W, bool FH = false>
__global__ void __launch_bounds__(kScanThreads, kScanCtasPerSm)
    k_scan(BatchParams p, uint32_t tile_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    const ScanSmem sm = carve(smem, p.ht_slots, tile_bytes);
    if (p.st[ST_OVERFLOW]) return;
    constexpr uint32_t c = W == 4 ? 0 : (W == 8 ? 1 : (W == 16 ? 2 : 3));
    WorkQueue total{0, 0, kWorkCtr[c]};
    for (uint32_t i = 0; i <= c; ++i) {
        const uint32_t items = static_cast<uint32_t>(p.st[class_st(i)]) *
                               (p.n ? ntiles_for(p.n, p.tile_bits_w[i], 4u << i) : 0u);
        total.base = total.end;
        total.end += items;
    }
    if (total.base == total.end) return;
    // item i runs from desc[i & 1]; its scan phase prepares item i + 1 into
    // the other descriptor / stage buffer (prepare_item).  Prime the pipeline:
    // the first item resolved with its plan in shared memory, the second claimed.
    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        uint32_t i0 = 0xffffffffu, i1 = 0xffffffffu;
        if (lane == 0) {
            i0 = fetch_item(p, total);
            if (i0 != 0xffffffffu) i1 = fetch_item(p, total);
        }
        i0 = __shfl_sync(0xffffffffu, i0, 0);
        i1 = __shfl_sync(0xffffffffu, i1, 0);
        uint32_t q0 = 0, t0 = 0;
        if (i0 != 0xffffffffu) {
            q0 = p.work_q[i0];
            t0 = p.work_t[i0];
            if (lane < sizeof(QueryPlan) / 16)
                cp_async16(reinterpret_cast<uint4*>(sm.plan) + lane, reinterpret_cast<const uint4*>(p.plan + q0) + lane);
        }
        if (lane == 0) {
            sm.scal[SC_PF_ITEM] = i0;
            sm.scal[SC_PF_Q] = q0;
            sm.scal[SC_PF_T] = t0;
            sm.scal[SC_CLAIM] = i1;
            sm.scal[SC_ADM_CALLS] = 0;
            sm.scal[SC_ADM_PASS] = 0;
            sm.scal[SC_WMAX] = 0;
            sm.scal[SC_WMIN] = 0xffffffffu;
        }
    }
    __syncthreads();
    if (threadIdx.x < 32 * prep_warps<W>()) prepare_item<prep_warps<W>()>(p, sm, 0, total);
    __syncthreads();
    for (uint32_t iter = 0;; ++iter) {
        const uint32_t b = iter & 1u;
        if (!sm.desc[b].valid) break;
        if constexpr (W == kHashW) process_item_hashed(p, sm, b, total);
        else process_item<W, FH>(p, sm, b, total);
    }
}

// ------------------------------------------------------------------ merge

// Where the candidate lists of query q live.
struct MergeSrc {
    // mode 0: object tiles of this batch; mode 1: explicit lists (multi-GPU)
    int mode;
    // mode 0
    const uint64_t* q_out_base;
    const uint32_t* q_cap;
    const uint32_t* q_tile_base;
    const uint32_t* q_ntiles;
    const uint32_t* tile_len;
    const genie_entry* tile_out;
    const uint32_t* q_floor;  // per-query floor (tile mode) or null
    int sorted_lists;         // mode 1: every list is ordered by (count desc, id asc) (list floors apply)
    // mode 1: list l of query q at in + q * in_q + l * in_l, length in_len[q * len_q + l * len_l]
    uint32_t L;
    const genie_entry* in;
    const uint32_t* in_len;
    uint64_t in_q, in_l, len_q, len_l;
    // common
    const uint32_t* k;
    uint32_t Q;
    uint32_t id_offset;
    uint32_t* q_big;
    unsigned long long* st;
    uint32_t out_stride;
    genie_entry* out;
    uint32_t* out_len;
    uint32_t* out_thr;
};

__device__ __forceinline__ void list_of(const MergeSrc& m, uint32_t q, uint32_t l,
                                        const genie_entry*& base, uint32_t& len) {
    if (m.mode == 0) {
        base = m.tile_out + m.q_out_base[q] + uint64_t(l) * m.q_cap[q];
        len = m.tile_len[m.q_tile_base[q] + l];
    } else {
        base = m.in + q * m.in_q + l * m.in_l;
        len = m.in_len[q * m.len_q + l * m.len_l];
    }
}

__device__ __forceinline__ uint32_t nlists_of(const MergeSrc& m, uint32_t q) {
    return m.mode == 0 ? m.q_ntiles[q] : m.L;
}

// merge_topk (engine.hpp:158-177) for unions of at most kSortCap entries:
// concatenate, bitonic sort by (count desc, id asc), truncate to k,
// threshold = k-th count if at least k entries else 0.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_merge(MergeSrc m, uint32_t cap) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
    __shared__ unsigned long long sums[32];
    __shared__ uint32_t s_flag, s_pos, s_lfloor, s_total;
    __shared__ uint32_t s_scratch[256 + 8];
    // a workspace overflow skipped k_worklist..k_scan: tile_len / tile_out
    // hold nothing of this batch (the host grows the workspace and retries)
    if (m.st[ST_OVERFLOW]) return;
    // list merges: the duplicate-id set lives in the upper half of the buffer
    uint32_t* dset = reinterpret_cast<uint32_t*>(keys + cap / 2);
    const uint32_t dslots = cap;  // u32 slots in cap / 2 keys (a power of two)
    for (uint32_t q = blockIdx.x; q < m.Q; q += gridDim.x) {
        const uint32_t L = nlists_of(m, q);
        const uint32_t kq = m.k[q];
        // Gather the union, dropping entries below the query's floor: the
        // floor is the k-th count of some tile, so at least k entries sit at
        // or above it and nothing below can make the merged top-k.
        uint32_t floor = m.q_floor ? m.q_floor[q] : 0u;
        // List merges (rows of partitions / shards, each sorted by count desc,
        // id asc): the floor is the largest k-th count over the rows, by the
        // same argument; every id still goes through the duplicate-id set, so
        // the ContractError verdict covers the whole union (engine.hpp:165-172)
        bool lset = false;
        if (m.mode == 1) {
            if (threadIdx.x == 0) s_lfloor = 0, s_total = 0, s_flag = 0;
            __syncthreads();
            for (uint32_t l = threadIdx.x; l < L; l += blockDim.x) {
                const genie_entry* bb;
                uint32_t ll;
                list_of(m, q, l, bb, ll);
                atomicAdd(&s_total, ll);
                if (kq && ll >= kq) atomicMax(&s_lfloor, bb[kq - 1].count);
            }
            for (uint32_t i = threadIdx.x; i < dslots; i += blockDim.x) dset[i] = 0xffffffffu;
            __syncthreads();
            lset = 2 * s_total <= dslots;  // block-uniform
            if (lset && m.sorted_lists) floor = s_lfloor;
        }
        if (threadIdx.x == 0) s_pos = 0;
        __syncthreads();
        {
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            for (uint32_t l = warp; l < L; l += blockDim.x >> 5) {
                const genie_entry* bb;
                uint32_t ll;
                list_of(m, q, l, bb, ll);
                for (uint32_t e0 = 0; e0 < ll; e0 += 32) {
                    const uint32_t e = e0 + lane;
                    genie_entry x{0, 0};
                    if (e < ll) x = bb[e];
                    if (lset && e < ll) {  // duplicate-id set (list merges)
                        uint32_t h = (x.id * 0x9E3779B1u) & (dslots - 1);
                        for (;;) {
                            const uint32_t old = atomicCAS(&dset[h], 0xffffffffu, x.id);
                            if (old == 0xffffffffu) break;
                            if (old == x.id) {
                                s_flag = 1;
                                break;
                            }
                            h = (h + 1) & (dslots - 1);
                        }
                    }
                    const bool keep = e < ll && x.count >= floor;
                    const uint32_t mask = __ballot_sync(0xffffffffu, keep);
                    uint32_t base = 0;
                    if (lane == 0 && mask) base = atomicAdd(&s_pos, static_cast<uint32_t>(__popc(mask)));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    const uint32_t pos = base + __popc(mask & ((1u << lane) - 1u));
                    if (keep && pos < (lset ? cap / 2 : cap)) keys[pos] = order_key(x.id, x.count);
                }
            }
        }
        __syncthreads();
        const uint32_t filled = s_pos;
        if (lset) {
            if (s_flag && threadIdx.x == 0) atomicMin(&m.st[ST_MERGE_DUP], (unsigned long long)q);
        }
        if (filled > (lset ? cap / 2 : cap)) {  // large union: radix selection path (k_merge_big)
            if (threadIdx.x == 0) {
                m.q_big[q] = 1;
                atomicAdd(&m.st[ST_MERGE_BIG], 1ull);
            }
            __syncthreads();
            continue;
        }
        if (threadIdx.x == 0) m.q_big[q] = 0;
        uint32_t N = 1;
        while (N < filled) N <<= 1;
        for (uint32_t i = filled + threadIdx.x; i < N; i += blockDim.x) keys[i] = ~0ull;
        __syncthreads();
        uint32_t H = 1;  // slots of the duplicate-id set (list merges)
        while (H < 2 * filled) H <<= 1;
        if (lset) {
            // checked while gathering
        } else if (m.mode == 1 && filled > 1 && N + H / 2 <= cap) {
            // duplicate ids across lists are a ContractError (engine.hpp:165-172):
            // every id goes into an open-addressing set in the shared memory
            // after the union (>= 2 slots per entry), a second insert of an id
            // is the duplicate -- the same verdict as the reference's sort by id
            uint32_t* set = reinterpret_cast<uint32_t*>(keys + N);
            for (uint32_t i = threadIdx.x; i < H; i += blockDim.x) set[i] = 0xffffffffu;
            if (threadIdx.x == 0) s_flag = 0;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < filled; i += blockDim.x) {
                const uint32_t id = key_id(keys[i]);
                uint32_t h = (id * 0x9E3779B1u) & (H - 1);
                for (;;) {
                    const uint32_t old = atomicCAS(&set[h], 0xffffffffu, id);
                    if (old == 0xffffffffu) break;
                    if (old == id) {
                        s_flag = 1;
                        break;
                    }
                    h = (h + 1) & (H - 1);
                }
            }
            __syncthreads();
            if (s_flag && threadIdx.x == 0) atomicMin(&m.st[ST_MERGE_DUP], (unsigned long long)q);
            __syncthreads();
        } else if (m.mode == 1 && filled > 1) {
            // duplicate ids across lists are a ContractError (engine.hpp:165-172)
            for (uint32_t i = threadIdx.x; i < filled; i += blockDim.x) {
                const uint64_t k0 = keys[i];
                keys[i] = (uint64_t(key_id(k0)) << 32) | key_count(k0);
            }
            __syncthreads();
            bitonic_sort_smem(keys, N);
            if (threadIdx.x == 0) s_flag = 0;
            __syncthreads();
            for (uint32_t i = threadIdx.x + 1; i < filled; i += blockDim.x)
                if ((keys[i] >> 32) == (keys[i - 1] >> 32)) s_flag = 1;
            __syncthreads();
            if (s_flag && threadIdx.x == 0) atomicMin(&m.st[ST_MERGE_DUP], (unsigned long long)q);
            for (uint32_t i = threadIdx.x; i < filled; i += blockDim.x) {
                const uint64_t k0 = keys[i];
                keys[i] = order_key(uint32_t(k0 >> 32), uint32_t(k0));
            }
            __syncthreads();
        }
        select_k_smallest(keys, filled, kq, s_scratch);
        const uint32_t outn = kq < filled ? kq : filled;
        genie_entry* row = m.out + uint64_t(q) * m.out_stride;
        for (uint32_t e = threadIdx.x; e < outn; e += blockDim.x) {
            genie_entry x;
            x.id = key_id(keys[e]) + m.id_offset;
            x.count = key_count(keys[e]);
            row[e] = x;
        }
        if (threadIdx.x == 0) {
            m.out_len[q] = outn;
            m.out_thr[q] = filled >= kq ? key_count(keys[kq - 1]) : 0;  // engine.hpp:175
        }
        __syncthreads();
    }
}

// Large unions (> kSortCap entries): exact selection by radix histograms in
// global memory, then a shared-memory sort of the k winners (k <= kSortCap)
// or a device segmented sort for longer rows.
__global__ void __launch_bounds__(kMergeThreads) k_merge_big(MergeSrc m) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
    __shared__ uint32_t hist[256];
    __shared__ unsigned long long sums[32];
    __shared__ uint32_t s_sel;
    __shared__ unsigned long long s_cum;
    __shared__ uint32_t s_pos;
    __shared__ uint32_t s_dup;
    if (m.st[ST_OVERFLOW]) return;  // see k_merge
    for (uint32_t q = blockIdx.x; q < m.Q; q += gridDim.x) {
        if (!m.q_big[q]) continue;
        const uint32_t L = nlists_of(m, q);
        const uint32_t kq = m.k[q];
        unsigned long long M = 0;
        for (uint32_t l = 0; l < L; ++l) {
            const genie_entry* b;
            uint32_t len;
            list_of(m, q, l, b, len);
            M += len;
        }
        // --- threshold count T: 2 x 8-bit radix passes over the 16-bit counts
        uint32_t T = 0;
        unsigned long long n_above = 0;
        const bool all = M <= kq;
        if (!all) {
            uint32_t prefix = 0;
            unsigned long long cum_above = 0;
            for (int pass = 0; pass < 2; ++pass) {
                for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
                __syncthreads();
                for (uint32_t l = 0; l < L; ++l) {
                    const genie_entry* b;
                    uint32_t len;
                    list_of(m, q, l, b, len);
                    for (uint32_t e = threadIdx.x; e < len; e += blockDim.x) {
                        const uint32_t c = b[e].count;
                        if (pass == 0) atomicAdd(&hist[(c >> 8) & 0xffu], 1u);
                        else if ((c >> 8) == prefix) atomicAdd(&hist[c & 0xffu], 1u);
                    }
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    unsigned long long cum = cum_above;
                    uint32_t sel = 0;
                    for (int b = 255; b >= 0; --b) {
                        if (cum + hist[b] >= kq) {
                            sel = b;
                            break;
                        }
                        cum += hist[b];
                    }
                    s_sel = sel;
                    s_cum = cum;
                }
                __syncthreads();
                if (pass == 0) {
                    prefix = s_sel;
                    cum_above = s_cum;
                } else {
                    T = (prefix << 8) | s_sel;
                    n_above = s_cum;
                }
                __syncthreads();
            }
        }
        // --- tie cutoff: the need-th smallest id among count == T (4 radix passes)
        const unsigned long long need = all ? 0 : kq - n_above;
        uint32_t id_cut = 0xffffffffu;
        if (!all) {
            uint32_t idp = 0;
            unsigned long long below = 0;
            for (int pass = 0; pass < 4; ++pass) {
                const int sh = 24 - 8 * pass;
                for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
                __syncthreads();
                for (uint32_t l = 0; l < L; ++l) {
                    const genie_entry* b;
                    uint32_t len;
                    list_of(m, q, l, b, len);
                    for (uint32_t e = threadIdx.x; e < len; e += blockDim.x) {
                        const genie_entry x = b[e];
                        if (x.count != T) continue;
                        const uint32_t hi = pass ? (x.id >> (sh + 8)) : 0;
                        if (hi == (pass ? (idp >> (sh + 8)) : 0)) atomicAdd(&hist[(x.id >> sh) & 0xffu], 1u);
                    }
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    unsigned long long cum = below;
                    uint32_t sel = 255;
                    for (uint32_t b = 0; b < 256; ++b) {
                        if (cum + hist[b] >= need) {
                            sel = b;
                            break;
                        }
                        cum += hist[b];
                    }
                    s_sel = sel;
                    s_cum = cum;
                }
                __syncthreads();
                idp |= s_sel << sh;
                below = s_cum;
                __syncthreads();
            }
            id_cut = idp;
        }
        // --- emit the winners into the output row.  Exactly min(k, M)
        // entries pass unless an id repeats across lists (mode 1: a
        // ContractError, engine.hpp:165-172); writes stay inside the row.
        if (threadIdx.x == 0) {
            s_pos = 0;
            s_dup = 0;
        }
        __syncthreads();
        genie_entry* row = m.out + uint64_t(q) * m.out_stride;
        const uint32_t lim = static_cast<uint32_t>(min(all ? M : static_cast<unsigned long long>(kq), static_cast<unsigned long long>(m.out_stride)));
        for (uint32_t l = 0; l < L; ++l) {
            const genie_entry* b;
            uint32_t len;
            list_of(m, q, l, b, len);
            for (uint32_t e = threadIdx.x; e < len; e += blockDim.x) {
                const genie_entry x = b[e];
                if (all || x.count > T || (x.count == T && x.id <= id_cut)) {
                    const uint32_t pos = atomicAdd(&s_pos, 1u);
                    if (pos < lim) row[pos] = x;
                    else s_dup = 1;
                }
            }
        }
        __syncthreads();
        const uint32_t outn = min(s_pos, lim);
        if (m.mode == 1 && outn <= kSortCap) {
            // duplicate ids among the winners (sorted by id, adjacent pairs)
            uint32_t N = 1;
            while (N < outn) N <<= 1;
            for (uint32_t i = threadIdx.x; i < N; i += blockDim.x)
                keys[i] = i < outn ? (uint64_t(row[i].id) << 32) | row[i].count : ~0ull;
            __syncthreads();
            bitonic_sort_smem(keys, N);
            for (uint32_t i = threadIdx.x + 1; i < outn; i += blockDim.x)
                if ((keys[i] >> 32) == (keys[i - 1] >> 32)) s_dup = 1;
            __syncthreads();
        }
        if (m.mode == 1 && s_dup && threadIdx.x == 0) atomicMin(&m.st[ST_MERGE_DUP], (unsigned long long)q);
        if (outn <= kSortCap) {
            uint32_t N = 1;
            while (N < outn) N <<= 1;
            for (uint32_t i = threadIdx.x; i < N; i += blockDim.x)
                keys[i] = i < outn ? order_key(row[i].id, row[i].count) : ~0ull;
            __syncthreads();
            bitonic_sort_smem(keys, N);
            for (uint32_t e = threadIdx.x; e < outn; e += blockDim.x) {
                genie_entry x;
                x.id = key_id(keys[e]) + m.id_offset;
                x.count = key_count(keys[e]);
                row[e] = x;
            }
        } else {
            // leave unsorted (local ids); the segmented sort finishes the row
            if (threadIdx.x == 0) atomicAdd(&m.st[ST_SORT_BIG], 1ull);
        }
        if (threadIdx.x == 0) {
            m.out_len[q] = outn;
            // threshold: the k-th count when at least k entries (engine.hpp:175)
            m.out_thr[q] = (!all || M >= kq) ? (all ? 0u : T) : 0u;
            if (all && M == kq) {
                uint32_t mn = 0xffffffffu;
                for (uint32_t e = 0; e < outn; ++e) mn = min(mn, row[e].count);
                m.out_thr[q] = mn;
            }
        }
        __syncthreads();
    }
}

// Rows longer than kSortCap: to order keys, segmented radix sort, back.
__global__ void k_rows_to_keys(const genie_entry* out, const uint32_t* out_len, uint32_t stride,
                               uint32_t Q, uint64_t* keys, uint64_t* seg_b, uint64_t* seg_e) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t total = uint64_t(Q) * stride;
    if (i < Q) {
        seg_b[i] = uint64_t(i) * stride;
        seg_e[i] = uint64_t(i) * stride + (out_len[i] > kSortCap ? out_len[i] : 0);
    }
    if (i >= total) return;
    const uint32_t q = static_cast<uint32_t>(i / stride), e = static_cast<uint32_t>(i % stride);
    keys[i] = (out_len[q] > kSortCap && e < out_len[q]) ? order_key(out[i].id, out[i].count) : ~0ull;
}

__global__ void k_keys_to_rows(genie_entry* out, const uint32_t* out_len, uint32_t stride,
                               uint32_t Q, const uint64_t* keys, uint32_t id_offset) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= uint64_t(Q) * stride) return;
    const uint32_t q = static_cast<uint32_t>(i / stride), e = static_cast<uint32_t>(i % stride);
    if (out_len[q] > kSortCap && e < out_len[q]) {
        genie_entry x;
        x.id = key_id(keys[i]) + id_offset;
        x.count = key_count(keys[i]);
        out[i] = x;
    }
}

// ------------------------------------------------------------ key cut table

// keycut[j * (nt + 1) + b] = number of key j's postings below object b * T
// (b = 0 .. nt): the tile-aligned slices of every list, searched once per
// index and tile size instead of once per (query, span) in every batch.
__global__ void k_keycut(const uint64_t* key_off, const uint32_t* postings, uint64_t K, uint32_t nt, uint32_t T,
                         uint32_t* out) {
    const uint64_t total = K * (nt + 1);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t j = i / (nt + 1);
        const uint32_t b = static_cast<uint32_t>(i - j * (nt + 1));
        const uint64_t beg = key_off[j];
        const uint32_t len = static_cast<uint32_t>(key_off[j + 1] - beg);
        out[i] = b == 0 ? 0u : (b == nt ? len : static_cast<uint32_t>(lower_bound_dev(postings + beg, len, b * T)));
    }
}

// Builds the table of every width class the index has been queried with
// (class_seen, from the previous batches' status) at the batch's tile sizes.
static void ensure_keycuts(genie_index* ix, const uint32_t (&tile_bits_w)[kClasses], cudaStream_t s) {
    if (!ix->K || !ix->n) return;
    for (int c = 0; c < kClasses; ++c) {
        const uint32_t T = tile_bits_w[c] / (4u << c);
        if (!ix->class_seen[c] || ix->keycut_T[c] == T) continue;
        const uint32_t nt = (ix->n + T - 1) / T;
        const uint64_t total = ix->K * uint64_t(nt + 1);
        if (total > (1ull << 31)) continue;  // bound the cache (~8 GB); such indexes keep searching
        ix->keycut[c].reserve(total);
        const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, uint64_t(ix->sms) * 32));
        k_keycut<<<blocks, 256, 0, s>>>(ix->key_off.p, ix->postings.p, ix->K, nt, T, ix->keycut[c].p);
        GENIE_CUDA(cudaGetLastError());
        ix->keycut_T[c] = T;
    }
}

// ------------------------------------------------------------ CUDA graphs

// What a captured batch depends on: replayed only while all of it is equal.
struct GraphKey {
    BatchParams p;
    MergeSrc m;
    cudaStream_t s;
    uint32_t Q, tile_bytes, per_sm;
    size_t smem;
    bool timed;
};

struct GraphCache {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    uint32_t launches = 0;
    uint64_t captures = 0;
    ~GraphCache() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

static GraphCache& graph_cache(genie_index* ix) {
    if (!ix->graph) ix->graph = std::shared_ptr<void>(new GraphCache(), [](void* g) { delete static_cast<GraphCache*>(g); });
    return *static_cast<GraphCache*>(ix->graph.get());
}

uint64_t graph_captures(const genie_index* ix) {
    return ix->graph ? static_cast<const GraphCache*>(ix->graph.get())->captures : 0;
}

// ------------------------------------------------------------ orchestration

int sm_count(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    return v > 0 ? v : 148;
}

void ensure_device(int device) { GENIE_CUDA(cudaSetDevice(device)); }

// Per-device launch attributes already applied (cudaFuncSetAttribute is
// per device context).  Guarded by the handle's single-controlling-thread
// contract; distinct handles on one device set the same values.
struct DeviceAttrCache {
    size_t scan_smem = 0;
    int scan_occ = 0;             // resident k_scan CTAs per SM at scan_occ_smem bytes
    size_t scan_occ_smem = 0;
    bool merge_set = false;       // k_merge (batch) and k_merge_big
    bool list_merge_set = false;  // k_merge (list merge) and k_merge_big
};
static DeviceAttrCache& attr_cache(int device) {
    static DeviceAttrCache caches[kMaxDevices];
    return caches[device >= 0 && device < kMaxDevices ? device : 0];
}

static void reserve_workspace(genie_index* ix, uint32_t Q, uint32_t items, uint32_t max_k,
                              uint32_t out_stride, uint32_t tile_bits) {
    Workspace& w = ix->ws;
    if (!w.status.p) {
        w.status.reserve(ST_WORDS);
        GENIE_CUDA(cudaMallocHost(&w.h_status, ST_WORDS * sizeof(unsigned long long)));
    }
    const size_t q = Q + 1;
    if (q > w.cap_q) {
        const size_t c = std::max(q, w.cap_q * 2);
        w.q_bound.reserve(c);
        w.q_P.reserve(c);
        w.q_span_base.reserve(c);
        w.q_cut_base.reserve(c);
        w.q_out_base.reserve(c);
        w.q_S.reserve(c);
        w.q_W.reserve(c);
        w.q_ntiles.reserve(c);
        w.q_cap.reserve(c);
        w.q_tile_base.reserve(c);
        w.q_rank.reserve(c);
        w.q_big.reserve(c);
        w.q_floor.reserve(c);
        w.q_plan.reserve(c * (sizeof(QueryPlan) / 16));
        w.cap_q = c;
    }
    if (items > w.cap_items || !w.it_kb.p) {
        const size_t c = std::max<size_t>(std::max<size_t>(items, 1024), w.cap_items * 2);
        w.it_kb.reserve(c);
        w.it_nk.reserve(c);
        w.it_sbase.reserve(c);
        w.cap_items = c;
    }
    // first-guess capacities; the device plan verifies them and the batch is
    // retried with exact sizes on overflow
    const uint64_t nt16 = ix->n ? (uint64_t(ix->n) + (tile_bits / 16) - 1) / (tile_bits / 16) : 1;
    const uint64_t want_spans = std::max<uint64_t>(uint64_t(items) * 8, 4096);
    const uint64_t want_work = std::max<uint64_t>(uint64_t(Q) * nt16, 1024);
    const uint64_t want_cuts = std::max<uint64_t>(want_spans * 4, 16384);
    const uint64_t want_tout =
        std::max<uint64_t>(std::min<uint64_t>(uint64_t(Q) * nt16 * std::max<uint32_t>(max_k, 1),
                                              uint64_t(Q) * (uint64_t(ix->n) + nt16)),
                           4096);
    if (want_spans > w.cap_spans) {
        w.span_beg.reserve(want_spans);
        w.span_dense.reserve(want_spans);
        w.cap_spans = want_spans;
    }
    if (want_cuts > w.cap_cuts) {
        w.cuts.reserve(want_cuts);
        w.cap_cuts = want_cuts;
    }
    if (want_work > w.cap_work) {
        w.work_q.reserve(want_work);
        w.work_t.reserve(want_work);
        w.tile_len.reserve(want_work);
        w.tile_rec.reserve(want_work * kRecWords);
        w.cap_work = want_work;
    }
    if (want_tout > w.cap_tout) {
        w.tile_out.reserve(want_tout);
        w.cap_tout = want_tout;
    }
    (void)out_stride;
}

static void grow_from_status(genie_index* ix) {
    Workspace& w = ix->ws;
    const unsigned long long* h = w.h_status;
    if (h[ST_TOTAL_SPANS] > w.cap_spans) {
        w.cap_spans = h[ST_TOTAL_SPANS] + (h[ST_TOTAL_SPANS] >> 2);
        w.span_beg.reserve(w.cap_spans);
        w.span_dense.reserve(w.cap_spans);
    }
    if (h[ST_TOTAL_CUTS] > w.cap_cuts) {
        w.cap_cuts = h[ST_TOTAL_CUTS] + (h[ST_TOTAL_CUTS] >> 2);
        w.cuts.reserve(w.cap_cuts);
    }
    if (h[ST_TOTAL_WORK] > w.cap_work) {
        w.cap_work = h[ST_TOTAL_WORK] + (h[ST_TOTAL_WORK] >> 2);
        w.work_q.reserve(w.cap_work);
        w.work_t.reserve(w.cap_work);
        w.tile_len.reserve(w.cap_work);
        w.tile_rec.reserve(w.cap_work * kRecWords);
    }
    if (h[ST_TOTAL_TOUT] > w.cap_tout) {
        w.cap_tout = h[ST_TOTAL_TOUT] + (h[ST_TOTAL_TOUT] >> 2);
        w.tile_out.reserve(w.cap_tout);
    }
}

// Default tile: the largest counter tile with which two scan CTAs share an SM
// (B200: 2 x 113 KB of shared memory -> ~92 KB of counters, 188K objects at
// W = 4): fewer, larger (query, tile) items amortise the per-item work.
static uint32_t auto_tile_bytes() {
    static thread_local int dev_cached = -1;
    static thread_local uint32_t tb_cached = 0;
    int dev = 0;
    GENIE_CUDA(cudaGetDevice(&dev));
    if (dev != dev_cached) {
        int smem_sm = 0, reserved = 0;
        GENIE_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
        GENIE_CUDA(cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev));
        const int per_cta = smem_sm / static_cast<int>(kScanCtasPerSm) - reserved - static_cast<int>(smem_off::kHt) -
                            static_cast<int>(kHtSlots * 8) - (GENIE_PLAN_AT_END ? int(sizeof(QueryPlan)) : 0);
        tb_cached = per_cta > 4096 ? static_cast<uint32_t>(per_cta) : 4096u;
        dev_cached = dev;
    }
    return tb_cached;
}

static uint32_t tile_bits_of(const genie_config& cfg) {
    uint32_t tb = cfg.tile_bytes ? cfg.tile_bytes : auto_tile_bytes();
    tb = std::max<uint32_t>(4096, std::min<uint32_t>(tb, 160u << 10));
    tb &= ~127u;  // tiles of whole 32-object blocks in 16-byte bitmap steps for every W
    return tb * 8;
}

// Counter tile allocation and per-width tiles.  Auto mode caps the tile so
// that one tile's slice of the index (postings + bitmaps: bytes per object x
// objects, at W = 8) fits ~90 % of L2 with 10 % slack: the tile-major sweep
// then reads each slice from DRAM about once per batch, and the shared memory
// left unallocated serves as L1 for the bitmap rows consecutive items of a
// tile share.  The cap snaps to 64 / 48 / 32 KB (C3: 64 KB, +23 %; measured
// non-power-of-two sizes lose up to 12 %).  W = 4 tiles hold at most as many
// objects as the cap.  Explicit tile_bytes apply to every class unchanged.
static uint32_t class_tile_bits_dense(const genie_index* ix, const genie_config& cfg, uint32_t tile_bits,
                                      uint32_t (&out)[kClasses]) {
    for (int c = 0; c < 3; ++c) out[c] = tile_bits;
    if (cfg.tile_bytes || ix->n == 0) return tile_bits;
    static thread_local int dev_cached = -1;
    static thread_local int l2_cached = 0;
    if (dev_cached != ix->device) {
        GENIE_CUDA(cudaDeviceGetAttribute(&l2_cached, cudaDevAttrL2CacheSize, ix->device));
        dev_cached = ix->device;
    }
    const double bytes = double(ix->P) * 4.0 + double(ix->n_dense) * ix->bitmap_words * 4.0;
    const double per_obj = bytes / double(ix->n);
    if (per_obj <= 0 || l2_cached <= 0) return tile_bits;
    const double objs = 0.9 * double(l2_cached) / per_obj;  // objects whose index slice fits L2
    uint32_t alloc = tile_bits;
    if (objs * 8.0 < 1.1 * double(tile_bits)) {  // the W = 8 tile would overflow L2
        alloc = 32u << 13;                        // 32 KB floor
        for (const uint32_t kb : {64u, 48u})
            if (double(kb << 13) <= 1.1 * objs * 8.0 && (kb << 13) <= tile_bits) {
                alloc = kb << 13;
                break;
            }
    }
    out[0] = std::min<uint32_t>(alloc, static_cast<uint32_t>(std::max(objs * 4.0, double(alloc) / 2)) & ~1023u);
    out[1] = alloc;
    out[2] = alloc;
    return alloc;
}

static uint32_t env_u32(const char* name, uint32_t dflt) {
    const char* v = std::getenv(name);
    return v && *v ? static_cast<uint32_t>(std::strtoul(v, nullptr, 10)) : dflt;
}

// Hashed sparse class (k_scan<kHashW>): the table takes the largest power of
// two of slots the counter area holds next to its scratch; the class's tile
// is GENIE_HASH_TILES 8-bit sub-tiles of the allocation (<= 2^20 objects: the
// tie selection's id radix).  Knobs (read per batch): GENIE_HASH_TILES (0: the
// class is off), GENIE_HASH_DENSE_MAX, GENIE_HASH_LOAD_PCT, GENIE_HASH_FILL_PCT.
// Results do not depend on them.
struct HashPlan {
    uint32_t slots = 0, fill = 0, pmax = 0, sub_T = 0, dmax = 0, tile_objs = 1024;
};
static HashPlan hash_plan(uint32_t tile_bits) {
    HashPlan h;
    const uint32_t tile_bytes = tile_bits / 8;
    const uint32_t nsub = env_u32("GENIE_HASH_TILES", GENIE_HASH_TILES);
    h.sub_T = tile_bytes & ~1023u;
    if (nsub == 0 || tile_bytes < kHashScratch + 4096 * 4 || h.sub_T == 0) return h;
    const uint32_t room = (tile_bytes - kHashScratch) / 4;
    h.slots = 1u << (31 - __builtin_clz(room));
    h.fill = static_cast<uint32_t>(uint64_t(h.slots) * std::min<uint32_t>(env_u32("GENIE_HASH_FILL_PCT", GENIE_HASH_FILL_PCT), 90) / 100);
    h.pmax = static_cast<uint32_t>(uint64_t(h.slots) * env_u32("GENIE_HASH_LOAD_PCT", GENIE_HASH_LOAD_PCT) / 100);
    h.dmax = env_u32("GENIE_HASH_DENSE_MAX", GENIE_HASH_DENSE_MAX);
    h.tile_objs = static_cast<uint32_t>(std::min<uint64_t>(uint64_t(nsub) * h.sub_T, 1u << 20));
    return h;
}

static uint32_t class_tile_bits(const genie_index* ix, const genie_config& cfg, uint32_t tile_bits,
                                uint32_t (&out)[kClasses], HashPlan* hp = nullptr) {
    const uint32_t alloc = class_tile_bits_dense(ix, cfg, tile_bits, out);
    const HashPlan h = hash_plan(alloc);
    out[3] = h.tile_objs * kHashW;
    if (hp) *hp = h;
    return alloc;
}

static MergeSrc tile_merge_src(genie_index* ix, uint32_t Q, const uint32_t* d_k, uint32_t stride,
                               genie_entry* out, uint32_t* out_len, uint32_t* out_thr, uint32_t id_offset) {
    Workspace& w = ix->ws;
    MergeSrc m{};
    m.mode = 0;
    m.q_out_base = w.q_out_base.p;
    m.q_cap = w.q_cap.p;
    m.q_tile_base = w.q_tile_base.p;
    m.q_ntiles = w.q_ntiles.p;
    m.tile_len = w.tile_len.p;
    m.tile_out = w.tile_out.p;
    m.q_floor = w.q_floor.p;
    m.k = d_k;
    m.Q = Q;
    m.id_offset = id_offset;
    m.q_big = w.q_big.p;
    m.st = w.status.p;
    m.out_stride = stride;
    m.out = out;
    m.out_len = out_len;
    m.out_thr = out_thr;
    return m;
}

static void segmented_sort_rows(genie_index* ix, uint32_t Q, uint32_t stride, genie_entry* out,
                                uint32_t* out_len, uint32_t id_offset, cudaStream_t s) {
    Workspace& w = ix->ws;
    const uint64_t total = uint64_t(Q) * stride;
    w.sort_keys.reserve(total);
    w.sort_keys_alt.reserve(total);
    w.sort_seg_begin.reserve(Q);
    w.sort_seg_end.reserve(Q);
    const uint32_t thr = 256;
    const uint64_t blocks = (std::max<uint64_t>(total, Q) + thr - 1) / thr;
    k_rows_to_keys<<<static_cast<unsigned>(blocks), thr, 0, s>>>(
        out, out_len, stride, Q, w.sort_keys.p, w.sort_seg_begin.p, w.sort_seg_end.p);
    size_t tmp = 0;
    cub::DoubleBuffer<uint64_t> db(w.sort_keys.p, w.sort_keys_alt.p);
    GENIE_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tmp, db, static_cast<int>(total),
                                                       static_cast<int>(Q), w.sort_seg_begin.p,
                                                       w.sort_seg_end.p, 0, 64, s));
    w.sort_tmp.reserve(tmp);
    GENIE_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(w.sort_tmp.p, tmp, db, static_cast<int>(total),
                                                       static_cast<int>(Q), w.sort_seg_begin.p,
                                                       w.sort_seg_end.p, 0, 64, s));
    k_keys_to_rows<<<static_cast<unsigned>((total + thr - 1) / thr), thr, 0, s>>>(
        out, out_len, stride, Q, db.Current(), id_offset);
}

uint64_t prepare_batch(genie_index* ix, const genie_config& cfg, uint32_t Q, uint32_t total_items, uint32_t max_k,
                       uint32_t out_stride, cudaStream_t s) {
    uint32_t tile_bits_w[kClasses];
    HashPlan hp;
    class_tile_bits(ix, cfg, tile_bits_of(cfg), tile_bits_w, &hp);
    reserve_workspace(ix, Q, total_items, max_k, out_stride,
                      std::min({tile_bits_w[0] * 4, tile_bits_w[1] * 2, tile_bits_w[2]}));
    ensure_keycuts(ix, tile_bits_w, s);
    // signature of every device buffer and capacity the batch will use
    const Workspace& w = ix->ws;
    uint64_t h = 0x9e3779b97f4a7c15ull;
    auto mixin = [&h](uint64_t v) { h = mix64(h ^ v); };
    for (const void* ptr : {(const void*)w.q_bound.p, (const void*)w.q_P.p, (const void*)w.q_span_base.p,
                            (const void*)w.q_cut_base.p, (const void*)w.q_out_base.p, (const void*)w.q_S.p,
                            (const void*)w.q_W.p, (const void*)w.q_ntiles.p, (const void*)w.q_cap.p,
                            (const void*)w.q_tile_base.p, (const void*)w.q_rank.p, (const void*)w.q_big.p,
                            (const void*)w.q_floor.p, (const void*)w.q_plan.p, (const void*)w.it_kb.p,
                            (const void*)w.it_nk.p, (const void*)w.it_sbase.p, (const void*)w.span_beg.p,
                            (const void*)w.span_dense.p, (const void*)w.cuts.p, (const void*)w.work_q.p,
                            (const void*)w.work_t.p, (const void*)w.tile_len.p, (const void*)w.tile_rec.p,
                            (const void*)w.tile_out.p, (const void*)w.status.p, (const void*)w.d_qid.p,
                            (const void*)w.d_k.p, (const void*)w.d_item_off.p, (const void*)w.d_dim.p,
                            (const void*)w.d_lo.p, (const void*)w.d_hi.p, (const void*)w.d_out.p,
                            (const void*)w.d_out_len.p, (const void*)w.d_out_thr.p, (const void*)ix->keycut[0].p,
                            (const void*)ix->keycut[1].p, (const void*)ix->keycut[2].p, (const void*)ix->keycut[3].p})
        mixin(reinterpret_cast<uint64_t>(ptr));
    for (uint64_t v : {uint64_t(w.cap_spans), uint64_t(w.cap_cuts), uint64_t(w.cap_work), uint64_t(w.cap_tout),
                       uint64_t(ix->keycut_T[0]), uint64_t(ix->keycut_T[1]), uint64_t(ix->keycut_T[2]),
                       uint64_t(ix->keycut_T[3]), uint64_t(tile_bits_w[3]), uint64_t(hp.slots), uint64_t(hp.fill),
                       uint64_t(hp.pmax), uint64_t(hp.sub_T), uint64_t(hp.dmax)})
        mixin(v);
    return h;
}

void launch_batch(genie_index* ix, const genie_config& cfg, uint32_t Q, const uint32_t* d_qid,
                  const uint32_t* d_k, const uint64_t* d_item_off, const uint16_t* d_dim,
                  const uint32_t* d_lo, const uint32_t* d_hi, uint32_t total_items,
                  uint32_t max_k, uint32_t out_stride, genie_entry* d_out, uint32_t* d_out_len,
                  uint32_t* d_out_thr, cudaStream_t s, bool timed, uint32_t extra_offset) {
    (void)d_qid;
    const uint32_t id_offset = ix->id_offset + extra_offset;  // reported ids are local + id_offset
    uint32_t tile_bits_w[kClasses];
    HashPlan hp;
    const uint32_t tile_bits = class_tile_bits(ix, cfg, tile_bits_of(cfg), tile_bits_w, &hp);
    const uint32_t tile_bytes = tile_bits / 8;
    reserve_workspace(ix, Q, total_items, max_k, out_stride,
                      std::min({tile_bits_w[0] * 4, tile_bits_w[1] * 2, tile_bits_w[2]}));
    ensure_keycuts(ix, tile_bits_w, s);
    Workspace& w = ix->ws;
    ix->last_Q = Q;
    ix->last_cfg = cfg;
    ix->last_timed = timed;
    uint32_t launches = 0;

    BatchParams p{};
    p.keys = ix->keys.p;
    p.key_off = ix->key_off.p;
    p.postings = ix->postings.p;
    p.dim_mult = ix->dim_mult.p;
    p.K = ix->K;
    p.n = ix->n;
    p.id_offset = id_offset;
    p.Q = Q;
    p.k = d_k;
    p.item_off = d_item_off;
    p.dim = d_dim;
    p.lo = d_lo;
    p.hi = d_hi;
    p.tile_bits = tile_bits;
    for (int c = 0; c < kClasses; ++c) p.tile_bits_w[c] = tile_bits_w[c];
    p.hash_slots = hp.slots;
    p.hash_fill = hp.fill;
    p.hash_pmax = hp.pmax;
    p.hash_sub_T = hp.sub_T;
    p.hash_dmax = hp.dmax;
    p.hash_min_items = 0;  // set with the scan grid below
    // span_chunk is the reference's chunk (ids per task chunk, engine.hpp:40);
    // a scan warp claims a quarter of one at a time (guided self-scheduling)
    uint32_t unit = cfg.span_chunk ? cfg.span_chunk / 4 : kDefaultUnit;
    unit = std::min<uint32_t>(std::max<uint32_t>((unit + 127) & ~127u, 128), 1u << 16);
    p.unit = unit;
    p.selector = cfg.selector;
    p.q_bound = w.q_bound.p;
    p.q_P = w.q_P.p;
    p.q_span_base = w.q_span_base.p;
    p.q_cut_base = w.q_cut_base.p;
    p.q_out_base = w.q_out_base.p;
    p.q_S = w.q_S.p;
    p.q_W = w.q_W.p;
    p.q_ntiles = w.q_ntiles.p;
    p.q_cap = w.q_cap.p;
    p.q_tile_base = w.q_tile_base.p;
    p.q_rank = w.q_rank.p;
    p.q_big = w.q_big.p;
    p.q_floor = w.q_floor.p;
    p.plan = reinterpret_cast<QueryPlan*>(w.q_plan.p);
    p.tile_rec = w.tile_rec.p;
    p.it_kb = w.it_kb.p;
    p.it_nk = w.it_nk.p;
    p.it_sbase = w.it_sbase.p;
    p.span_beg = w.span_beg.p;
    p.span_dense = w.span_dense.p;
    p.key_dense = ix->key_dense.p;
    p.dim_range = ix->dim_range.p;
    p.tokmap = ix->tokmap.p;
    for (int c = 0; c < kClasses; ++c)
        p.keycut[c] = ix->keycut_T[c] == tile_bits_w[c] / (4u << c) ? ix->keycut[c].p : nullptr;
    p.bitmaps = ix->bitmaps.p;
    p.bitmap_words = ix->bitmap_words;
    p.n_dense = ix->n_dense;
    for (int c = 0; c < 3; ++c) p.dense_inv[c] = ix->dense_inv[c];
    p.cuts = w.cuts.p;
    p.work_q = w.work_q.p;
    p.work_t = w.work_t.p;
    p.tile_len = w.tile_len.p;
    p.tile_out = w.tile_out.p;
    p.st = w.status.p;
    p.cap_spans = w.cap_spans;
    p.cap_cuts = w.cap_cuts;
    p.cap_work = w.cap_work;
    p.cap_tout = w.cap_tout;
    p.out_stride = out_stride;
    p.out = d_out;
    p.out_len = d_out_len;
    p.out_thr = d_out_thr;

    // host-side set-up first (launch attributes, occupancy): the enqueue
    // below issues stream work only, so it can be captured into a graph
    const int sms = ix->sms;
    p.ht_slots = kHtSlots;
    const size_t smem = scan_smem_bytes(tile_bytes, p.ht_slots);
    const size_t msmem = kSortCap * sizeof(uint64_t);
    // cudaFuncSetAttribute applies per device context: cached per device
    // (one host thread may drive several devices, genie_group_*)
    DeviceAttrCache& ac = attr_cache(ix->device);
    if (ac.scan_smem < smem) {
        GENIE_CUDA(cudaFuncSetAttribute(k_scan<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        GENIE_CUDA(cudaFuncSetAttribute(k_scan<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        GENIE_CUDA(cudaFuncSetAttribute(k_scan<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        GENIE_CUDA(cudaFuncSetAttribute(k_scan<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        GENIE_CUDA(cudaFuncSetAttribute(k_scan<kHashW>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        ac.scan_smem = smem;
    }
    if (!ac.merge_set) {
        GENIE_CUDA(cudaFuncSetAttribute(k_merge<kMergeSmallThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kMergeSmallCap * sizeof(uint64_t))));
        GENIE_CUDA(cudaFuncSetAttribute(k_merge_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(msmem)));
        ac.merge_set = true;
    }
    uint32_t per_sm = cfg.ctas_per_sm ? cfg.ctas_per_sm : 0;
    if (!per_sm) {
        if (!ac.scan_occ || ac.scan_occ_smem != smem) {
            int occ = 0;
            GENIE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scan<8>, kScanThreads, smem));
            ac.scan_occ = std::max(1, occ);
            ac.scan_occ_smem = smem;
        }
        per_sm = ac.scan_occ;
    }
    // two items per scan CTA at least, or the hashed class is folded back (k_plan;
    // GENIE_HASH_MIN_ITEMS overrides)
    p.hash_min_items = env_u32("GENIE_HASH_MIN_ITEMS", 2 * static_cast<uint32_t>(sms) * per_sm);
    // launched when the previous batch on this index wanted it (a dense batch
    // pays no empty launch; GENIE_HASH_LAUNCH=1 forces it)
    p.hash_launch = hp.slots && (ix->hash_wanted || env_u32("GENIE_HASH_LAUNCH", 0)) ? 1u : 0u;
    const MergeSrc m = tile_merge_src(ix, Q, d_k, out_stride, d_out, d_out_len, d_out_thr, id_offset);
    const bool big_rows = max_k > kSortCap;  // CUB segmented sort (allocates): never captured

    // stage events are recorded as external event nodes when captured, so a
    // replayed graph still records them (cudaEventRecordExternal)
    auto enqueue = [&](bool capturing) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (!capturing) GENIE_CUDA(cudaStreamIsCapturing(s, &cs));  // an enclosing capture (host-buffer graphs)
        const bool external = capturing || cs == cudaStreamCaptureStatusActive;
        auto record = [&](int e) {
            GENIE_CUDA(external ? cudaEventRecordWithFlags(ix->ev[e], s, cudaEventRecordExternal)
                                : cudaEventRecord(ix->ev[e], s));
        };
        if (timed) record(0);
        k_init_status<<<1, 64, 0, s>>>(w.status.p);
        ++launches;
        if (Q) {
            k_resolve<<<(Q * 32 + kLookupThreads - 1) / kLookupThreads, kLookupThreads, 0, s>>>(p);
            k_plan<<<1, 1024, 0, s>>>(p);
            k_worklist<<<(Q * 32 + 255) / 256, 256, 0, s>>>(p);
            k_cut<<<sms * kCutCtasPerSm, kLookupThreads, 0, s>>>(p);
            launches += 4;
            if (timed) record(1);
            // one launch per width class (an empty class's CTAs exit at once)
            // small indexes (one W = 4 tile of <= kFirstHistWords counter words):
            // the instance whose gate-less first tiles take the histogram select
            if (uint64_t(ix->n) * 4 <= uint64_t(kFirstHistWords) * 32)
                k_scan<4, true><<<sms * per_sm, kScanThreads, smem, s>>>(p, tile_bytes);
            else
                k_scan<4><<<sms * per_sm, kScanThreads, smem, s>>>(p, tile_bytes);
            k_scan<8><<<sms * per_sm, kScanThreads, smem, s>>>(p, tile_bytes);
            k_scan<16><<<sms * per_sm, kScanThreads, smem, s>>>(p, tile_bytes);
            launches += 3;
            if (p.hash_launch) {  // the hashed sparse class (GENIE_HASH_TILES; see hash_wanted)
                k_scan<kHashW><<<sms * per_sm, kScanThreads, smem, s>>>(p, tile_bytes);
                ++launches;
            }
            if (timed) record(2);
            // one small CTA per query: after the floors prune them, unions are a
            // few k entries, so all queries merge concurrently; larger unions
            // are left to k_merge_big
            k_merge<kMergeSmallThreads><<<Q, kMergeSmallThreads, kMergeSmallCap * sizeof(uint64_t), s>>>(
                m, kMergeSmallCap);
            k_merge_big<<<std::min<uint32_t>(Q, sms * 4), kMergeThreads, msmem, s>>>(m);
            launches += 2;
            if (big_rows) {
                segmented_sort_rows(ix, Q, out_stride, d_out, d_out_len, id_offset, s);
                launches += 3;
            }
            if (timed) record(3);
        } else if (timed) {
            record(1);
            record(2);
            record(3);
        }
        GENIE_CUDA(cudaMemcpyAsync(w.h_status, w.status.p, ST_WORDS * sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, s));
    };

    const bool graph = (cfg.flags & GENIE_FLAG_GRAPH) && !big_rows && s != nullptr &&
                       s != cudaStreamLegacy && s != cudaStreamPerThread;
    if (!graph) {
        enqueue(false);
    } else {
        // CUDA graph per batch shape: the whole pipeline (11 launches, events,
        // status read-back) replays with one cudaGraphLaunch while nothing it
        // captured -- parameters, workspace, buffers, stream -- has changed
        GraphKey key;
        std::memset(&key, 0, sizeof(key));
        key.p = p;
        key.m = m;
        key.s = s;
        key.Q = Q;
        key.tile_bytes = tile_bytes;
        key.per_sm = per_sm;
        key.smem = smem;
        key.timed = timed;
        GraphCache& gc = graph_cache(ix);
        if (!gc.exec || std::memcmp(&gc.key, &key, sizeof(key)) != 0) {
            cudaGraph_t g = nullptr;
            GENIE_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            try {
                enqueue(true);
            } catch (...) {
                cudaStreamEndCapture(s, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            GENIE_CUDA(cudaStreamEndCapture(s, &g));
            bool updated = false;
            if (gc.exec) {
                cudaGraphExecUpdateResultInfo info{};
                updated = cudaGraphExecUpdate(gc.exec, g, &info) == cudaSuccess;
                if (!updated) {
                    cudaGetLastError();
                    cudaGraphExecDestroy(gc.exec);
                    gc.exec = nullptr;
                }
            }
            if (!updated) GENIE_CUDA(cudaGraphInstantiate(&gc.exec, g, 0));
            cudaGraphDestroy(g);
            gc.key = key;
            gc.launches = launches;
            ++gc.captures;
        }
        launches = gc.launches;
        GENIE_CUDA(cudaGraphLaunch(gc.exec, s));
    }
    GENIE_CUDA(cudaGetLastError());
    ix->last_launches = launches;
}

int finish_batch(genie_index* ix, genie_batch_stats* stats, std::string& msg,
                 const uint32_t* h_qid) {
    GENIE_CUDA(cudaStreamSynchronize(ix->stream));
    GENIE_CUDA(cudaGetLastError());
    const unsigned long long* h = ix->ws.h_status;
    for (int c = 0; c < kClasses; ++c)
        if (h[class_st(c)]) ix->class_seen[c] = true;  // its cut table is built before the next batch
    if (!h[ST_OVERFLOW]) ix->hash_wanted = h[ST_HASH_WANT] != 0;
    if (stats) {
        stats->postings = h[ST_TOTAL_POSTINGS];
        stats->work_items = h[ST_TOTAL_WORK];
        stats->fallback_tiles = h[ST_FALLBACK];
    }
    if (h[ST_OVERFLOW]) {
        grow_from_status(ix);
        msg = "workspace grown; re-issue the batch";
        return GENIE_RETRY;
    }
    auto qname = [&](unsigned long long q) {
        return std::to_string(h_qid ? h_qid[q] : static_cast<uint32_t>(q));
    };
    if (h[ST_BAD_INPUT] != ~0ull) {
        const unsigned long long q = h[ST_BAD_INPUT] >> 8;
        const unsigned kind = h[ST_BAD_INPUT] & 0xff;
        msg = "Query " + qname(q) +
              (kind == 1 ? ": no items" : kind == 2 ? ": k must be >= 1" : ": QueryItem lo > hi");
        return GENIE_ERR_CONTRACT;
    }
    if (h[ST_BAD_BOUND] != ~0ull) {
        const unsigned long long q = h[ST_BAD_BOUND];
        uint64_t bound = 0;
        GENIE_CUDA(cudaMemcpy(&bound, ix->ws.q_bound.p + q, sizeof(bound), cudaMemcpyDeviceToHost));
        msg = "query " + qname(q) + " (setup): match-count bound " + std::to_string(bound) +
              " exceeds the counter range";
        return GENIE_ERR_CONTRACT;
    }
    if (h[ST_MERGE_DUP] != ~0ull) {
        msg = "merge_topk: an object was reported by more than one partition (query " +
              qname(h[ST_MERGE_DUP]) + ")";
        return GENIE_ERR_CONTRACT;
    }
    return GENIE_OK;
}

// ------------------------------------------------------------ merge (multi-GPU)

void launch_list_merge(genie_index* ix, uint32_t Q, uint32_t L, const genie_entry* d_in,
                       const uint32_t* d_in_len, uint32_t in_stride, const uint32_t* d_k,
                       uint32_t out_stride, genie_entry* d_out, uint32_t* d_out_len,
                       uint32_t* d_out_thr, uint32_t max_k, cudaStream_t s, bool list_major, bool sorted_lists) {
    Workspace& w = ix->ws;
    if (!w.status.p) {
        w.status.reserve(ST_WORDS);
        GENIE_CUDA(cudaMallocHost(&w.h_status, ST_WORDS * sizeof(unsigned long long)));
    }
    if (Q + 1 > w.cap_q) {
        w.q_big.reserve(Q + 1);
    }
    w.q_big.reserve(std::max<size_t>(Q + 1, w.q_big.n));
    MergeSrc m{};
    m.mode = 1;
    m.L = L;
    m.in = d_in;
    m.in_len = d_in_len;
    // query-major [Q][L][in_stride] (merge_topk callers) or list-major
    // [L][Q][in_stride] (the order an all-gather of per-shard rows produces)
    m.in_q = list_major ? in_stride : uint64_t(L) * in_stride;
    m.in_l = list_major ? uint64_t(Q) * in_stride : in_stride;
    m.len_q = list_major ? 1 : L;
    m.len_l = list_major ? Q : 1;
    m.sorted_lists = sorted_lists ? 1 : 0;
    m.k = d_k;
    m.Q = Q;
    m.id_offset = 0;
    m.q_big = w.q_big.p;
    m.st = w.status.p;
    m.out_stride = out_stride;
    m.out = d_out;
    m.out_len = d_out_len;
    m.out_thr = d_out_thr;
    k_init_status<<<1, 64, 0, s>>>(w.status.p);
    const size_t msmem = kSortCap * sizeof(uint64_t);
    DeviceAttrCache& ac = attr_cache(ix->device);
    if (!ac.list_merge_set) {
        GENIE_CUDA(cudaFuncSetAttribute(k_merge<kMergeThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(msmem)));
        GENIE_CUDA(cudaFuncSetAttribute(k_merge_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(msmem)));
        ac.list_merge_set = true;
    }
    const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(Q, ix->sms * 4));
    if (Q) {
        // unions that fit the small merge (the per-shard rows of a multi-GPU
        // batch: L x k entries) take one 128-thread CTA per query, as the
        // batch's tile merge does; larger ones the 512-thread CTAs
        if (uint64_t(L) * std::max<uint32_t>(max_k, 1) <= kMergeSmallCap)
            k_merge<kMergeSmallThreads><<<Q, kMergeSmallThreads, kMergeSmallCap * sizeof(uint64_t), s>>>(
                m, kMergeSmallCap);
        else
            k_merge<kMergeThreads><<<grid, kMergeThreads, msmem, s>>>(m, kSortCap);
        k_merge_big<<<grid, kMergeThreads, msmem, s>>>(m);
        if (max_k > kSortCap) segmented_sort_rows(ix, Q, out_stride, d_out, d_out_len, 0, s);
    }
    GENIE_CUDA(cudaMemcpyAsync(w.h_status, w.status.p, ST_WORDS * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s));
    GENIE_CUDA(cudaGetLastError());
    ix->last_launches = 3;
}

}  // namespace genie
