// Internal structures shared by the libgenie_b200 translation units.
#pragma once

#include <algorithm>
#include <memory>

#include "common.cuh"

namespace genie {

// Tunables (result-invariant).  The GENIE_SCAN_* macros exist for variant
// builds (make variant V=<name> X="-D...") used by tools/ sweeps.
#ifndef GENIE_SCAN_THREADS
#define GENIE_SCAN_THREADS 512
#endif
#ifndef GENIE_SCAN_UNROLL
#define GENIE_SCAN_UNROLL 2
#endif
#ifndef GENIE_SCAN_CTAS
#define GENIE_SCAN_CTAS (1024 / GENIE_SCAN_THREADS)
#endif
constexpr uint32_t kScanThreads = GENIE_SCAN_THREADS;  // threads per scan CTA
constexpr uint32_t kScanCtasPerSm = GENIE_SCAN_CTAS;   // resident scan CTAs per SM (registers, tile size)
constexpr uint32_t kSpanBatch = 256;          // spans staged in shared memory per pass (x2 buffers)
#ifndef GENIE_HT_MIN
#define GENIE_HT_MIN 1024
#endif
constexpr uint32_t kHtSlots = GENIE_HT_MIN;           // shared-memory Robin Hood table, minimum (8 KB; >= 4 x 256-bin histograms)
constexpr uint32_t kHtMaxSlots = 4096;        // ... and maximum (items whose counters leave room)
#ifndef GENIE_REC_LEVELS
#define GENIE_REC_LEVELS 3
#endif
constexpr int kRecLevels = GENIE_REC_LEVELS;   // levels in a tile's record (gate_start)
constexpr uint32_t kRecWords = (1 + kRecLevels + 3) & ~3u;  // record: base level + kRecLevels counts, 16-B padded
constexpr uint32_t kZaMax = 256;              // ZipperArray levels held in shared memory (W <= 8)
#ifndef GENIE_LOOKUP_THREADS
#define GENIE_LOOKUP_THREADS 256
#endif
#ifndef GENIE_CUT_GROUP_MUL  // k_cut spans per warp = clamp(mul x spans / warps, 1, 32)
#define GENIE_CUT_GROUP_MUL 2
#endif
#ifndef GENIE_CUT_CTAS
#define GENIE_CUT_CTAS 32
#endif
#ifndef GENIE_CUT_LINEAR_MAX  // k_cut: lists up to this many postings are cut by one linear pass
#define GENIE_CUT_LINEAR_MAX 0  // measured slower than the binary searches on C4 (0.37 vs 0.28 ms lookup)
#endif
constexpr uint32_t kCutLinearMax = GENIE_CUT_LINEAR_MAX;
constexpr uint32_t kCutLinearUnroll = 8;  // posting loads per lane in flight in the linear pass
constexpr uint32_t kLookupThreads = GENIE_LOOKUP_THREADS;  // k_resolve / k_cut block size
constexpr uint32_t kCutCtasPerSm = GENIE_CUT_CTAS;         // k_cut grid: CTAs per SM
constexpr uint32_t kMergeThreads = 512;
#ifndef GENIE_MERGE_THREADS
#define GENIE_MERGE_THREADS 128
#endif
constexpr uint32_t kMergeSmallThreads = GENIE_MERGE_THREADS;  // per-query merge CTAs of a batch
constexpr uint32_t kMergeSmallCap = 16 * kMergeSmallThreads;  // their key capacity (<= 16 x threads)
constexpr uint32_t kSortCap = 8192;           // merge entries sorted in shared memory
constexpr uint32_t kDefaultUnit = 1024;       // postings per warp work unit (guided scheduling)
#ifndef GENIE_DENSE_LEVELS
#define GENIE_DENSE_LEVELS 2
#endif
constexpr uint32_t kLvl = GENIE_DENSE_LEVELS;  // dense-phase c-PQ levels counted in registers
#ifndef GENIE_SCAN_STRIDED
#define GENIE_SCAN_STRIDED 0
#endif
#ifndef GENIE_COMPACT_FILL_INV
#define GENIE_COMPACT_FILL_INV 2
#endif
// compact posting scan when the staged slices fill their 128-posting groups
// less than 1/kCompactFillInv on average
constexpr uint32_t kCompactFillInv = GENIE_COMPACT_FILL_INV;
#ifndef GENIE_PLAN_ASYNC  // query plans prefetched into shared memory one item ahead (1) or loaded in place (0)
#define GENIE_PLAN_ASYNC 1
#endif
#ifndef GENIE_PLAN_AT_END  // the prefetched QueryPlan after the counter tile instead of in the fixed area
#define GENIE_PLAN_AT_END 0
#endif
#ifndef GENIE_HT_ALIGN  // alignment of the table + counter-tile start in the scan CTA's shared memory
#define GENIE_HT_ALIGN 16
#endif
#ifndef GENIE_DENSE_NOINLINE  // dense phase as out-of-line calls (own register allocation)
#define GENIE_DENSE_NOINLINE 0
#endif
#if GENIE_DENSE_NOINLINE
#define GENIE_DENSE_FN __device__ __noinline__
#else
#define GENIE_DENSE_FN __device__
#endif
#ifndef GENIE_PREP_WARPS_W8  // warps preparing the next item in the W >= 8 kernels (1 or 2)
#define GENIE_PREP_WARPS_W8 2
#endif
#ifndef GENIE_PREP_NOINLINE  // warp 0's prepare_item as an out-of-line call
#define GENIE_PREP_NOINLINE 0
#endif
#if GENIE_PREP_NOINLINE
#define GENIE_PREP_FN __device__ __noinline__
#else
#define GENIE_PREP_FN __device__
#endif
#ifndef GENIE_BITMAP_PREFETCH  // also prefetch the next item's bitmap-row slices into L2
#define GENIE_BITMAP_PREFETCH 0
#endif
#ifndef GENIE_PREFETCH_LINES  // 128-byte lines prefetched per posting slice (GENIE_SPAN_PREFETCH = 2)
#define GENIE_PREFETCH_LINES 2
#endif
#ifndef GENIE_SPAN_PREFETCH  // L2 prefetch of the next item's posting slices: 0 off, 1 bulk (UBLKPF), 2 per-lane lines
#define GENIE_SPAN_PREFETCH 2
#endif
#ifndef GENIE_STATIC_GROUPS  // <= this many 128-posting groups per scan warp: static split, else guided
#define GENIE_STATIC_GROUPS 64
#endif
#ifndef GENIE_PLANES_LOP  // many-list dense path: transpose through explicit LOP3 selects
#define GENIE_PLANES_LOP 1
#endif
#ifndef GENIE_LANES_LV_SPLIT  // few-list dense path: separate code for items without gate levels (W = 4 / W >= 8)
#define GENIE_LANES_LV_SPLIT 1
#endif
#ifndef GENIE_CSA_BLOCKS_W4  // W = 4 many-list dense path: blocks per thread
#define GENIE_CSA_BLOCKS_W4 2
#endif
#ifndef GENIE_LANES_MAX  // dense lists per item up to which the lane-wise path runs (W <= 8)
#define GENIE_LANES_MAX 3
#endif
#ifndef GENIE_HASH_TILES  // hashed sparse class: object tile = this many W = 8 counter tiles, <= 2^20 objects (0: off)
#define GENIE_HASH_TILES 11
#endif
#ifndef GENIE_HASH_DENSE_MAX  // ... taken by queries with at most this many expected postings per W = 8 tile
#define GENIE_HASH_DENSE_MAX 512  // (C4: ~1 500, dense tiles faster; 30-400: hashed 1.4-4.3x faster)
#endif
#ifndef GENIE_HASH_LOAD_PCT  // ... admits a query whose expected postings per tile fill <= this % of the table
#define GENIE_HASH_LOAD_PCT 50
#endif
#ifndef GENIE_HASH_FILL_PCT  // ... an item takes the table path while its postings fill <= this % of it
#define GENIE_HASH_FILL_PCT 75
#endif
#ifndef GENIE_HASH_PW  // ... warps preparing the next item (1 or 2)
#define GENIE_HASH_PW 2
#endif
#ifndef GENIE_HASH_UNR  // ... posting loads per lane in flight
#define GENIE_HASH_UNR 4
#endif
constexpr uint32_t kHashScratch = 20u << 10;  // per-warp count histograms + tie bins after the table
#ifndef GENIE_CSA16  // many-list dense path (>= 5 planes): 16-list Harley-Seal steps before the 8-list ones
#define GENIE_CSA16 1
#endif
#ifndef GENIE_CSA32  // ... and (>= 6 planes) 32-list steps before those
#define GENIE_CSA32 1
#endif
#ifndef GENIE_CSA64  // ... and (>= 7 planes) 64-list steps before those
#define GENIE_CSA64 1
#endif
#ifndef GENIE_FIRST_HIST_WORDS  // items whose c-PQ gate starts at zero, on tiles of at most this many
#define GENIE_FIRST_HIST_WORDS 8192  // counter words: no admissions, exact histogram select (0: never)
#endif
constexpr uint32_t kFirstHistWords = GENIE_FIRST_HIST_WORDS;
#ifndef GENIE_CSA_QUAD
#define GENIE_CSA_QUAD 0
#endif
#ifndef GENIE_CSA_PAIR
#define GENIE_CSA_PAIR 1
#endif
constexpr int kScanUnroll = GENIE_SCAN_UNROLL;               // 128-posting groups loaded per warp pass
constexpr bool kLanesLvSplit = GENIE_LANES_LV_SPLIT;
constexpr uint32_t kStaticGroups = GENIE_STATIC_GROUPS;        // <= this many 128-posting groups per warp: static split
constexpr uint64_t kEmptySlot = ~0ull;
constexpr int kMaxDevices = 64;              // per-device host caches (launch attributes)

// Status block words (u64) written by the device pipeline.
enum StatusWord : int {
    ST_BAD_INPUT = 0,   // min (q << 8 | kind): 1 empty query, 2 k == 0, 3 lo > hi
    ST_BAD_BOUND = 1,   // min q whose max_count_bound > 0xffff
    ST_TOTAL_SPANS = 2,
    ST_TOTAL_CUTS = 3,
    ST_TOTAL_WORK = 4,
    ST_TOTAL_TOUT = 5,
    ST_TOTAL_POSTINGS = 6,
    ST_OVERFLOW = 7,    // workspace too small
    ST_WORK_CTR = 8,    // persistent scan queue cursor
    ST_FALLBACK = 9,    // tiles that fell back to histogram select
    ST_MERGE_BIG = 10,  // queries merged by the large-union path
    ST_MERGE_DUP = 11,  // min q with a duplicate id across merge lists
    ST_CLASS0 = 12,     // queries per counter-width class (W = 4, 8, 16)
    ST_CLASS1 = 13,
    ST_CLASS2 = 14,
    ST_CUT_CTR = 15,
    ST_SORT_BIG = 16,   // rows longer than kSortCap left for the segmented sort
    ST_T_SETUP = 20,    // GENIE_PHASE_TIMERS builds: k_scan cycles per phase (thread 0 of each CTA)
    ST_T_SCAN = 21,
    ST_T_EXTRACT = 22,
    ST_T_DENSE = 23,
    ST_ADMIT_CALLS = 24,  // GENIE_PHASE_TIMERS builds: c-PQ admit path entries / passes
    ST_ADMIT_PASS = 25,
    ST_T_PREP = 26,     // warp 0's prepare_item / warp 1's scan share, cycles
    ST_T_WARP1 = 27,
    ST_T_LAT = 28,      // latency of one dependent global load in prepare_item (cycles, count)
    ST_T_LATN = 29,
    ST_T_GATE = 30,     // instrumented: items that tie-fill / cycles of their tie fill
    ST_T_STAGE = 31,
    ST_DENSE_ND = 17,   // instrumented: sum of dense lists per dense item | bit-sliced items << 40
    ST_T_WMAX = 18,     // instrumented: sum over items of the slowest / fastest scan warp (cycles)
    ST_T_WMIN = 19,
    ST_WORK_CTR1 = 32,  // scan queue cursors of the W = 8 / W = 16 classes (ST_WORK_CTR: W = 4)
    ST_WORK_CTR2 = 33,
    ST_P_WAIT = 34,     // instrumented: prepare_item split (cycles): plan wait, issue, gate start, staging
    ST_P_ISSUE = 35,
    ST_P_GATE = 36,
    ST_P_STAGE = 37,
    ST_CLASS3 = 38,     // queries of the hashed sparse class (kHashW)
    ST_WORK_CTR3 = 39,  // its scan queue cursor
    ST_HASH_WANT = 40,  // the batch had enough hashed-class items to launch the class (next batch's hint)
    ST_WORDS = 41
};
// Work classes: counter widths W = 4, 8, 16 (dense counter tiles) and the
// hashed sparse class (class 3, pseudo-width kHashW = 32: a query whose
// postings are few for the object range counts into a shared-memory
// open-addressing table instead of a dense counter tile).  W = 4 << class.
constexpr int kClasses = 4;
constexpr uint32_t kHashW = 32;
constexpr uint32_t kWorkCtr[kClasses] = {ST_WORK_CTR, ST_WORK_CTR1, ST_WORK_CTR2, ST_WORK_CTR3};
// status word holding the number of queries of class c
__host__ __device__ constexpr uint32_t class_st(int c) { return c < 3 ? ST_CLASS0 + c : ST_CLASS3; }

// Per-batch device scratch, grown on demand (never shrinks).
struct Workspace {
    // per query
    DevBuf<uint64_t> q_bound, q_P, q_span_base, q_cut_base, q_out_base;
    DevBuf<uint32_t> q_S, q_W, q_ntiles, q_cap, q_tile_base, q_rank, q_big, q_floor;
    DevBuf<uint4> q_plan;  // QueryPlan records (80 B each, genie_query.cu)
    // per item
    DevBuf<uint32_t> it_kb, it_nk, it_sbase;
    // spans / cuts / work / tiles
    DevBuf<uint64_t> span_beg;
    DevBuf<int32_t> span_dense;
    DevBuf<uint32_t> cuts;
    DevBuf<uint32_t> work_q, work_t;
    DevBuf<uint32_t> tile_len;
    DevBuf<uint32_t> tile_rec;  // [work items][kRecWords]
    DevBuf<genie_entry> tile_out;
    // status
    DevBuf<unsigned long long> status;
    unsigned long long* h_status = nullptr;  // pinned mirror
    // host-API staging (device copies of caller buffers)
    DevBuf<uint32_t> d_qid, d_k, d_lo, d_hi;
    DevBuf<uint64_t> d_item_off;
    DevBuf<uint16_t> d_dim;
    DevBuf<genie_entry> d_out;
    DevBuf<uint32_t> d_out_len, d_out_thr;
    // segmented-sort scratch for rows longer than kSortCap
    DevBuf<uint64_t> sort_keys, sort_keys_alt;
    DevBuf<uint64_t> sort_seg_begin, sort_seg_end;
    DevBuf<unsigned char> sort_tmp;

    size_t cap_q = 0, cap_items = 0, cap_spans = 0, cap_cuts = 0, cap_work = 0, cap_tout = 0;
};

// Keywords of one dim (k_dim_ranges): keys[first, first + (count & ~flag));
// kDimDenseFlag set when its tokens are tok0 .. tok0 + count - 1.
struct __align__(16) DimRange {
    uint64_t first;
    uint32_t count;
    uint32_t tok0;
    // token map of a dim whose tokens have gaps (map_span > 0): the dim's
    // tokmap[map_off + x] = #keys with token < tok0 + x, x in [0, map_span]
    uint64_t map_off;
    uint32_t map_span;
    uint32_t pad;
};
constexpr uint32_t kDimDenseFlag = 0x80000000u;

}  // namespace genie

struct genie_index {
    int device = 0;
    uint32_t n = 0;
    uint64_t K = 0, P = 0;
    uint32_t id_offset = 0;
    int sms = 148;
    genie::DevBuf<uint64_t> keys, key_off;
    genie::DevBuf<uint32_t> postings;  // padded for aligned 16-byte tail loads
    genie::DevBuf<uint32_t> dim_mult;  // 65536
    genie::DevBuf<genie::DimRange> dim_range;  // 65536: each dim's key range (k_resolve)
    genie::DevBuf<uint32_t> tokmap;            // token -> key-rank maps of gapped dims (DimRange::map_*)
    // per width class: every key's position of each object-tile boundary
    // (keycut[c][j * (nt + 1) + b], tiles of keycut_T[c] objects), built once
    // the class has been queried; k_cut then reads cuts instead of searching
    genie::DevBuf<uint32_t> keycut[genie::kClasses];
    uint32_t keycut_T[genie::kClasses] = {0, 0, 0, 0};
    bool class_seen[genie::kClasses] = {false, false, false, false};
    // the last batch had enough hashed-class items: launch k_scan<kHashW> in
    // the next one (until then its queries run on dense tiles; results equal)
    bool hash_wanted = false;
    // dense containers: keys whose list covers >= dense_density of the
    // objects also carry a bitmap of n bits (Roaring-style bitmap container)
    genie::DevBuf<int32_t> key_dense;   // [K] word offset of the key's row in `bitmaps`, or -1
    genie::DevBuf<uint32_t> bitmaps;    // [n_dense][bitmap_words]
    uint32_t n_dense = 0, bitmap_words = 0;
    uint32_t dense_inv[3] = {0, 0, 0};  // query-time density rule per counter width (W = 4, 8, 16)
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[6] = {};
    genie::Workspace ws;
    // last device batch
    uint32_t last_Q = 0;
    uint32_t last_launches = 0;
    bool last_timed = false;
    genie_config last_cfg{};
    std::shared_ptr<void> graph;  // captured batch pipeline (GENIE_FLAG_GRAPH), genie_query.cu
    // captured host-buffer batch (genie_query_batch with GENIE_FLAG_GRAPH): H2D, pipeline, D2H
    cudaGraphExec_t host_graph = nullptr;
    uint64_t host_graph_key[16] = {};
    uint64_t host_graph_captures = 0;
    uint64_t* h_bounds = nullptr;  // pinned staging of the per-query bounds (graph path)
    uint32_t h_bounds_cap = 0;
};

namespace genie {

// Launches the whole device pipeline for a batch already resident on the
// device.  Does not synchronise.  Implemented in genie_query.cu.
void launch_batch(genie_index* ix, const genie_config& cfg, uint32_t Q, const uint32_t* d_qid,
                  const uint32_t* d_k, const uint64_t* d_item_off, const uint16_t* d_dim,
                  const uint32_t* d_lo, const uint32_t* d_hi, uint32_t total_items,
                  uint32_t max_k, uint32_t out_stride, genie_entry* d_out, uint32_t* d_out_len,
                  uint32_t* d_out_thr, cudaStream_t stream, bool timed, uint32_t extra_offset = 0);

// merge_topk over explicit candidate lists (engine.hpp:158-177), on the
// device: query-major [Q][L][in_stride] or list-major [L][Q][in_stride].
void launch_list_merge(genie_index* ix, uint32_t Q, uint32_t L, const genie_entry* d_in,
                       const uint32_t* d_in_len, uint32_t in_stride, const uint32_t* d_k,
                       uint32_t out_stride, genie_entry* d_out, uint32_t* d_out_len,
                       uint32_t* d_out_thr, uint32_t max_k, cudaStream_t s, bool list_major, bool sorted_lists = true);

// Host-side set-up of a batch (tile sizes, workspace, cut tables) without any
// stream work, so the launch that follows can be captured; returns a digest of
// every device buffer / capacity the batch will use (a graph key).
uint64_t prepare_batch(genie_index* ix, const genie_config& cfg, uint32_t Q, uint32_t total_items, uint32_t max_k,
                       uint32_t out_stride, cudaStream_t s);

// Reads the status block (synchronises) and converts it to a status code +
// message.  Grows the workspace and returns GENIE_RETRY on overflow.
int finish_batch(genie_index* ix, genie_batch_stats* stats, std::string& msg,
                 const uint32_t* h_qid /* optional, for messages */);

void ensure_device(int device);

// CUDA-graph captures made for this index (GENIE_FLAG_GRAPH batches).
uint64_t graph_captures(const genie_index* ix);

// ---- host-side helpers shared by the C-ABI translation units

// engine.hpp:186-188 and model.hpp:80-85, 97-101: the reference raises these
// before any work happens.
inline void validate_config(const genie_config& c) {
    if (c.span_chunk == 0 || c.max_spans_per_task == 0)
        throw Error(GENIE_ERR_CONTRACT, "span_chunk and max_spans_per_task must be positive");
    if (c.selector > GENIE_SELECT_SORT) throw Error(GENIE_ERR_CONTRACT, "unknown selector");
}

// The O(Q) part of the checks (sizes): the per-item / per-query contract
// checks run on the device (k_resolve) and, only when it reports a bad
// input, validate_queries re-derives the reference's exact message.
inline void validate_offsets(uint32_t Q, const uint64_t* item_off) {
    if (Q >= (1u << 21)) throw Error(GENIE_ERR_CONTRACT, "batch exceeds 2^21 queries");
    for (uint32_t q = 0; q < Q; ++q)
        if (item_off[q + 1] < item_off[q]) throw Error(GENIE_ERR_CONTRACT, "item_off must be non-decreasing");
}

inline void validate_queries(uint32_t Q, const uint32_t* qid, const uint32_t* k,
                             const uint64_t* item_off, const uint16_t* dim, const uint32_t* lo,
                             const uint32_t* hi) {
    if (Q >= (1u << 21)) throw Error(GENIE_ERR_CONTRACT, "batch exceeds 2^21 queries");
    for (uint32_t q = 0; q < Q; ++q) {
        if (item_off[q + 1] < item_off[q]) throw Error(GENIE_ERR_CONTRACT, "item_off must be non-decreasing");
        for (uint64_t i = item_off[q]; i < item_off[q + 1]; ++i)
            if (lo[i] > hi[i])
                throw Error(GENIE_ERR_CONTRACT, "QueryItem: lo " + std::to_string(lo[i]) + " > hi " +
                                                    std::to_string(hi[i]) + " on dim " +
                                                    std::to_string(dim[i]));
        if (item_off[q + 1] == item_off[q])
            throw Error(GENIE_ERR_CONTRACT, "Query " + std::to_string(qid[q]) + ": no items");
        if (k[q] == 0) throw Error(GENIE_ERR_CONTRACT, "Query " + std::to_string(qid[q]) + ": k must be >= 1");
    }
}

template <typename T>
inline void h2d(DevBuf<T>& b, const T* src, size_t n, cudaStream_t s) {
    b.reserve(n);
    if (n) GENIE_CUDA(cudaMemcpyAsync(b.p, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

// Reference accounting of MemoryStats (engine.hpp:239-241; cpq.hpp:103-106,
// 243, 283, 359-362), from the per-query bounds.
inline void memory_stats(uint32_t n, uint32_t Q, const uint32_t* k, const uint64_t* bounds,
                         genie_batch_stats* st) {
    st->counter_bytes = st->gate_bytes = st->table_bytes = 0;
    for (uint32_t q = 0; q < Q; ++q) {
        const uint64_t b = std::max<uint64_t>(bounds[q], 1);
        const uint64_t w = width_for(b);
        st->counter_bytes += (uint64_t(n) * w + 7) / 8;
        st->gate_bytes += (b + 1) * 4 + 4;
        st->table_bytes += 8 * bit_ceil64(std::max<uint64_t>(2ull * k[q] * b, 2));
    }
}

}  // namespace genie
