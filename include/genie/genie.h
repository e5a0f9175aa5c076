/*
 * genie.h -- the C-ABI drop-in boundary of the B200-native GENIE match-count
 * engine (libgenie_b200.so, sm_100a).
 *
 * The reference (mcx, /root/reference/proj/include) has no FFI layer: its
 * hot path is inline C++ in namespace mcx.  These entry points are exactly
 * what a binding of that path needs; the C++ mirror in the include/mcx headers
 * (same names and semantics as the reference) and the Python mirror
 * (paper_1603_08390_b200.mcx) are thin hosts over them.  Each function names
 * the reference interface it replaces.
 *
 * Conventions
 *  - plain pointers and sizes only; no torch / CUDA types in signatures
 *    (streams are passed as void*).
 *  - every call returns a genie_status; on failure a NUL-terminated message
 *    is written to err[errlen] (may be NULL).  Messages that concern one
 *    query carry the reference prefix "query N (stage): " (engine.hpp:127-135).
 *  - the index handle owns its device memory and one CUDA stream; it is not
 *    re-entrant (one controlling thread per handle).
 *  - results are written into caller-owned host buffers (or device buffers
 *    for the *_device variants).
 */
#ifndef GENIE_GENIE_H
#define GENIE_GENIE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error taxonomy mirrors mcx/error.hpp:24-41 and the CLI exit codes
 * (mcx_cli.cpp:682-694). */
typedef enum {
    GENIE_OK = 0,
    GENIE_ERR_CONTRACT = 1,  /* mcx::ContractError (std::invalid_argument) */
    GENIE_ERR_DATA = 2,      /* mcx::DataError (std::runtime_error) */
    GENIE_ERR_INVARIANT = 3, /* mcx::InvariantError (std::logic_error) */
    GENIE_ERR_CUDA = 4,      /* CUDA runtime / device failure */
    GENIE_ERR_NCCL = 5,
    GENIE_RETRY = 6          /* device batch outgrew the workspace: it was grown, re-issue the batch */
} genie_status;

/* mcx::Selector (engine.hpp:33).  All selectors return identical results.
 *  CPQ    : Count Priority Queue per object tile -- AuditThreshold gate,
 *           ZipperArray and a lock-free Robin Hood table in shared memory.
 *  BUCKET : histogram k-selection over the tile counters (GEN-SPQ ablation,
 *           stands in for bucket_kselect select.hpp:62-120).
 *  SORT   : same device path as BUCKET (sort_topk select.hpp:40-51 semantics). */
typedef enum { GENIE_SELECT_CPQ = 0, GENIE_SELECT_BUCKET = 1, GENIE_SELECT_SORT = 2 } genie_selector;

/* mcx::TopKEntry (cpq.hpp:31-41): result order is count desc, id asc. */
typedef struct {
    uint32_t id;
    uint32_t count;
} genie_entry;

/* mcx::EngineConfig (engine.hpp:36-42) plus device knobs.  Every field is
 * result-invariant; zero means "default" except span_chunk /
 * max_spans_per_task, where 0 is a ContractError exactly as in
 * engine.hpp:186-188 (use genie_config_default()). */
typedef struct {
    uint32_t selector;           /* genie_selector */
    uint32_t span_chunk;         /* ids per chunk (engine.hpp:40, default 4096); a scan warp claims
                                    span_chunk / 4 postings at a time (rounded up to 128) */
    uint32_t max_spans_per_task; /* accepted for API parity; must be > 0 */
    uint32_t tile_bytes;         /* shared-memory counter bytes per object tile (0: default) */
    uint32_t ctas_per_sm;        /* persistent scan CTAs per SM (0: default) */
    uint32_t flags;              /* GENIE_FLAG_* */
} genie_config;

/* genie_config.flags: record CUDA events around the device stages on the
 * launching stream (read back with genie_last_stage_ns after synchronising). */
#define GENIE_FLAG_STAGE_EVENTS 1u
/* genie_config.flags: genie_query_batch_device replays the batch pipeline as
 * one CUDA graph, captured on first use and re-captured whenever the batch
 * shape, buffers, stream or workspace change (ignored for the legacy default
 * stream and for k > 8192).  genie_query_batch does the same with the uploads
 * and read-backs inside the graph when every host buffer is page-locked
 * (cudaHostAlloc / pinned) and item_off[0] == 0; otherwise it launches
 * directly. */
#define GENIE_FLAG_GRAPH 2u

/* mcx::StageTimings (engine.hpp:44-50), measured with CUDA events on the
 * handle's stream (device stages) and the host clock (total). */
typedef struct {
    uint64_t lookup_ns;
    uint64_t match_ns;
    uint64_t select_ns;
    uint64_t merge_ns;
    uint64_t total_ns;
} genie_stage_ns;

/* mcx::MemoryStats (engine.hpp:52-56) with the reference accounting
 * (cpq.hpp:103-106, 359-362), plus device-side facts. */
typedef struct {
    uint64_t counter_bytes;  /* sum_q ceil(n * W_q / 8) */
    uint64_t gate_bytes;     /* sum_q ((bound_q + 1) * 4 + 4) */
    uint64_t table_bytes;    /* sum_q 8 * bit_ceil(max(2 k_q bound_q, 2)) */
    uint64_t postings;       /* sum_q P_q: posting ids scanned (algorithmic work) */
    uint64_t work_items;     /* (query, object tile) items processed */
    uint64_t fallback_tiles; /* tiles whose table overflowed -> exact histogram select */
} genie_batch_stats;

genie_config genie_config_default(void);

/* Build-side ------------------------------------------------------------- */

typedef struct genie_index genie_index;

/* Uploads a CSR inverted index to `device` (replaces mcx::build_index's
 * product, index.hpp:190-250, and InvertedIndex, index.hpp:41-182).
 *   keys[K]      packed dim<<32|token (Keyword::packed, model.hpp:43-45),
 *                strictly ascending
 *   key_off[K+1] postings offsets; key j owns postings[key_off[j], key_off[j+1])
 *   postings[P]  object ids, strictly ascending within each key, < num_objects
 *   dim_max_mult optional [65536]: InvertedIndex::max_multiplicity per dim
 *                (index.hpp:110-113); NULL computes it on the device
 * id_offset is added to every reported id (IndexPartition::id_offset,
 * index.hpp:254-259) -- used for object-range shards.
 * Validation failures (order, range) are GENIE_ERR_DATA. */
int genie_index_create(uint32_t num_objects, uint64_t num_keys, const uint64_t* keys,
                       const uint64_t* key_off, const uint32_t* postings,
                       const uint32_t* dim_max_mult, uint32_t id_offset, int device,
                       genie_index** out, char* err, size_t errlen);

/* Same as genie_index_create but keeps only object ids in [id_begin, id_end)
 * of a full CSR (rebased to local ids, id_offset = id_begin): one GPU's slice
 * of partition_dataset (index.hpp:263-291) without materialising parts. */
int genie_index_create_shard(uint32_t num_objects, uint64_t num_keys, const uint64_t* keys,
                             const uint64_t* key_off, const uint32_t* postings,
                             uint32_t id_begin, uint32_t id_end, int device, genie_index** out,
                             char* err, size_t errlen);

/* MCIX index files (the reference's on-disk format, index_io.hpp:27-154).
 * genie_mcix_parse: validates an image exactly as deserialize_index does
 * (index_io.hpp:84-146; failures are GENIE_ERR_DATA with its messages) and
 * returns it as CSR -- call once with null arrays for the sizes, then with
 * keys[K], key_off[K+1], postings[P].
 * genie_index_load_mcix: parse + genie_index_create (load_index's product
 * straight into device memory, index_io.hpp:148-154).
 * genie_mcix_serialize: the image serialize_index (index_io.hpp:63-82) writes
 * for the index build_index makes from this CSR with split threshold `split`
 * (0 = no splitting; index.hpp:229-238); *size in/out (null out: size only). */
int genie_mcix_parse(const uint8_t* data, uint64_t size, uint32_t* num_objects, uint64_t* num_keys,
                     uint64_t* num_postings, uint64_t* keys, uint64_t* key_off, uint32_t* postings,
                     char* err, size_t errlen);
int genie_index_load_mcix(const uint8_t* data, uint64_t size, int device, genie_index** out, char* err,
                          size_t errlen);
int genie_mcix_serialize(uint32_t num_objects, uint64_t num_keys, const uint64_t* keys, const uint64_t* key_off,
                         const uint32_t* postings, uint32_t split, uint8_t* out, uint64_t* size, char* err,
                         size_t errlen);

/* The span structure of an image (InvertedIndex::entries()/spans(),
 * index.hpp:41-73) for hosts that keep it (mcx::deserialize_index, which
 * re-serializes byte-identically, test_index.cpp:222-236): validates like
 * genie_mcix_parse; shape call with null arrays gives *num_spans, the fill call
 * writes span_count[K] and span_bounds[2 * num_spans] (begin, end pairs). */
int genie_mcix_parse_spans(const uint8_t* data, uint64_t size, uint64_t* num_spans, uint16_t* span_count,
                           uint64_t* span_bounds, char* err, size_t errlen);
/* serialize_index (index_io.hpp:63-82) of an index with explicit spans:
 * keyword j owns span_count[j] consecutive (begin, end) pairs of span_bounds. */
int genie_mcix_serialize_spans(uint32_t num_objects, uint64_t num_keys, const uint64_t* keys,
                               const uint16_t* span_count, const uint64_t* span_bounds, uint64_t num_postings,
                               const uint32_t* postings, uint8_t* out, uint64_t* size, char* err, size_t errlen);

/* build_index (index.hpp:190-250) on the device: object o owns keywords
 * [obj_off[o], obj_off[o+1]) of dims / tokens (host arrays; ids dense 0..n-1).
 * A keyword repeated inside one object is a ContractError (ObjectRecord,
 * model.hpp:57-62).  The CSR is identical to the host build (tested). */
int genie_index_build(uint32_t num_objects, const uint64_t* obj_off, const uint16_t* dims, const uint32_t* tokens,
                      int device, genie_index** out, char* err, size_t errlen);

void genie_index_destroy(genie_index* ix);

/* Index facts: num_objects, keys, postings, id_offset, device. */
void genie_index_info(const genie_index* ix, uint32_t* num_objects, uint64_t* num_keys,
                      uint64_t* num_postings, uint32_t* id_offset, int* device);

/* max_multiplicity per dim as held by the device index (65536 entries). */
int genie_index_dim_stats(genie_index* ix, uint32_t* dim_max_mult, char* err, size_t errlen);

/* Query-side ------------------------------------------------------------- */

/* mcx::execute_batch (engine.hpp:184-304) with host buffers.
 * Queries (mcx::Query, model.hpp:91-102): query q has items
 * [item_off[q], item_off[q+1]) with dims / inclusive [lo, hi] ranges, asks
 * for k[q] >= 1 results and reports query_id qid[q].
 * Output row q (stride out_stride >= max k) receives out_len[q] entries in
 * (count desc, id asc) order and out_threshold[q] (TopKResult, cpq.hpp:43-47).
 * out_bound (optional, Q) receives max_count_bound per query.
 * Errors: k == 0, empty query, lo > hi -> CONTRACT ("Query N: ..."), bound >
 * 0xffff -> CONTRACT "query N (setup): ...", table overflow never surfaces
 * (exact fallback), CUDA failures -> CUDA.
 * Counter range: the device counters are 4/8/16-bit for EVERY selector, so
 * the bound > 0xffff ContractError (engine.hpp:230-233) also applies to
 * GENIE_SELECT_BUCKET / GENIE_SELECT_SORT, whose reference counterparts use
 * 32-bit counters and would answer such a query (a divergence only for
 * queries matching one object more than 65 535 times). */
int genie_query_batch(genie_index* ix, const genie_config* cfg, uint32_t num_queries,
                      const uint32_t* qid, const uint32_t* k, const uint64_t* item_off,
                      const uint16_t* item_dim, const uint32_t* item_lo, const uint32_t* item_hi,
                      uint32_t out_stride, genie_entry* out, uint32_t* out_len,
                      uint32_t* out_threshold, uint64_t* out_bound, genie_stage_ns* timings,
                      genie_batch_stats* stats, char* err, size_t errlen);

/* Device-resident variant: every array is a device pointer on the index's
 * device; work is enqueued on `stream` (a cudaStream_t, NULL = the handle's
 * stream) and the call returns without synchronising.  Validation and
 * counter-range checks happen on the device; call genie_query_status() after
 * synchronising to surface them.  out_len/out_threshold/out_bound are device
 * arrays.  No host<->device copies are issued. */
int genie_query_batch_device(genie_index* ix, const genie_config* cfg, uint32_t num_queries,
                             const uint32_t* d_qid, const uint32_t* d_k,
                             const uint64_t* d_item_off, const uint16_t* d_item_dim,
                             const uint32_t* d_item_lo, const uint32_t* d_item_hi,
                             uint32_t max_k, uint32_t total_items, uint32_t out_stride,
                             genie_entry* d_out, uint32_t* d_out_len, uint32_t* d_out_threshold,
                             void* stream, char* err, size_t errlen);

/* Status of the last genie_query_batch_device call (synchronises the
 * handle's stream).  Fills stats if non-NULL. */
int genie_query_status(genie_index* ix, genie_batch_stats* stats, char* err, size_t errlen);

/* Raw device status words of the last batch (diagnostics; words 20-22 hold
 * per-phase k_scan cycle sums in GENIE_PHASE_TIMERS builds).  Synchronises. */
int genie_debug_status(genie_index* ix, uint64_t* words, uint32_t n_words, char* err, size_t errlen);

/* Kernels launched by the last batch (for launch accounting). */
uint32_t genie_last_launch_count(const genie_index* ix);
/* CUDA graphs captured for this index so far (GENIE_FLAG_GRAPH). */
uint64_t genie_graph_captures(const genie_index* ix);

/* Device stage times of the last batch launched with GENIE_FLAG_STAGE_EVENTS
 * (or through genie_query_batch with timings): lookup = resolve + plan + cut,
 * match = the fused scan / c-PQ / tile-select kernel, merge = the per-query
 * merge kernels.  total_ns = sum of the device stages.  Synchronises. */
int genie_last_stage_ns(genie_index* ix, genie_stage_ns* out, char* err, size_t errlen);

/* mcx::merge_topk (engine.hpp:158-177) over device-resident candidate lists,
 * batched over queries: list l of query q is d_in[(q*L + l)*in_stride ...]
 * with d_in_len[q*L + l] valid entries, each list ordered by (count desc, id
 * asc) and lists holding disjoint ascending id ranges in list order (the
 * per-GPU top-k of id-range shards).  Output as genie_query_batch_device.
 * Duplicate ids across lists are a ContractError (reported by
 * genie_query_status). */
int genie_merge_topk_device(genie_index* ix, uint32_t num_queries, uint32_t num_lists,
                            const genie_entry* d_in, const uint32_t* d_in_len, uint32_t in_stride,
                            const uint32_t* d_k, uint32_t out_stride, genie_entry* d_out,
                            uint32_t* d_out_len, uint32_t* d_out_threshold, void* stream,
                            char* err, size_t errlen);
/* Same with the lists in list-major order when list_major != 0: list l of
 * query q at d_in[(l*Q + q)*in_stride ...], length d_in_len[l*Q + q] -- the
 * layout an all-gather of per-shard [Q][in_stride] rows produces, merged in
 * place without a transpose. */
int genie_merge_topk_device_layout(genie_index* ix, uint32_t num_queries, uint32_t num_lists,
                                   const genie_entry* d_in, const uint32_t* d_in_len, uint32_t in_stride,
                                   uint32_t list_major, const uint32_t* d_k, uint32_t out_stride,
                                   genie_entry* d_out, uint32_t* d_out_len, uint32_t* d_out_threshold,
                                   void* stream, char* err, size_t errlen);

/* Host variant of the batched merge (runs on `device`). */
int genie_merge_topk(int device, uint32_t num_queries, uint32_t num_lists, const genie_entry* in,
                     const uint32_t* in_len, uint32_t in_stride, const uint32_t* k,
                     uint32_t out_stride, genie_entry* out, uint32_t* out_len,
                     uint32_t* out_threshold, char* err, size_t errlen);

/* hash_results (engine.hpp:141-153): the byte-exact parity digest (host). */
uint64_t genie_hash_results(uint32_t num_queries, const uint32_t* qid, const uint32_t* threshold,
                            const uint32_t* len, uint32_t stride, const genie_entry* entries);

/* Device groups ------------------------------------------- *
 * Object-id-range shards of one index on several GPUs driven by ONE host
 * thread: the concurrent form of execute_partitioned (engine.hpp:308-347).
 * Shard p owns ids [p n / G, (p + 1) n / G) and lives on devices[p]; every
 * shard's batch runs at once, the per-shard top-k rows (global ids) are
 * exchanged -- an NCCL all-gather over NVLink when the shards sit on distinct
 * devices (libnccl.so.2 loaded at run time), device-to-device / peer copies
 * otherwise -- and merged on devices[0] with merge_topk's rule
 * (engine.hpp:158-177).  Results equal genie_query_batch on the whole index. */
typedef struct genie_group genie_group;
enum genie_exchange {
    GENIE_EXCHANGE_AUTO = 0, /* NCCL when possible, else peer copies */
    GENIE_EXCHANGE_NCCL = 1, /* NCCL all-gather (ContractError if unavailable) */
    GENIE_EXCHANGE_PEER = 2  /* peer / device-to-device copies into the root */
};
int genie_group_create(uint32_t num_objects, uint64_t num_keys, const uint64_t* keys, const uint64_t* key_off,
                       const uint32_t* postings, uint32_t num_shards, const int* devices, int exchange,
                       genie_group** out, char* err, size_t errlen);
/* A group over existing indexes (borrowed, not destroyed with the group):
 * part p reports local ids + id_offsets[p] (IndexPartition::id_offset,
 * index.hpp:254-259); parts must be disjoint id ranges. */
int genie_group_from_indexes(genie_index* const* indexes, const uint32_t* id_offsets, uint32_t num_shards,
                             int exchange, genie_group** out, char* err, size_t errlen);
void genie_group_destroy(genie_group* g);
/* num_shards, the exchange in use (genie_exchange), total objects */
int genie_group_info(const genie_group* g, uint32_t* num_shards, int* exchange, uint32_t* num_objects);
/* genie_query_batch over the group (host buffers, same contract); timings:
 * lookup / match = the slowest shard, merge = the root merge; stats: work
 * summed, memory accounting the per-shard maximum (engine.hpp:330-333). */
int genie_group_query_batch(genie_group* g, const genie_config* cfg, uint32_t num_queries, const uint32_t* query_id,
                            const uint32_t* k, const uint64_t* item_off, const uint16_t* item_dim,
                            const uint32_t* item_lo, const uint32_t* item_hi, uint32_t out_stride, genie_entry* out,
                            uint32_t* out_len, uint32_t* out_threshold, genie_stage_ns* timings,
                            genie_batch_stats* stats, char* err, size_t errlen);

/* Sequence verification (SequenceSearcher, sa.hpp:127-162, 298-336,
 * 419-512) ---------------------------------------------------------------- *
 * A device-resident corpus of byte strings: sequence i is
 * bytes[off[i], off[i+1]).  genie_seqset_distances: Levenshtein distance
 * (unit costs) of `query` to sequences ids[0..count) -- or to sequences
 * 0..count-1 when ids is NULL (the exhaustive scan) -- with
 * edit_distance_bounded's contract: the exact distance when <= cap, else
 * cap + 1 (cap = UINT32_MAX: always exact).  Bit-parallel (Myers/Hyyro) on
 * the GPU, one thread per pair; out[count] host buffer. */
typedef struct genie_seqset genie_seqset;
int genie_seqset_create(const uint8_t* bytes, const uint64_t* off, uint64_t num_sequences, int device,
                        genie_seqset** out, char* err, size_t errlen);
void genie_seqset_destroy(genie_seqset* s);
void genie_seqset_info(const genie_seqset* s, uint64_t* num_sequences, uint64_t* total_bytes, int* device);
int genie_seqset_distances(genie_seqset* s, const uint8_t* query, uint64_t query_len, const uint32_t* ids,
                           uint64_t count, uint32_t cap, uint32_t* out, char* err, size_t errlen);

/* LSH / minHash transforms ------------------------------------------------- */

/* mcx::LshFamily (lsh.hpp:130) plus minHash (new). */
typedef enum { GENIE_LSH_PSTABLE = 0, GENIE_LSH_RBH = 1, GENIE_LSH_MINHASH = 2 } genie_lsh_family;

/* mcx::LshEncoderConfig (lsh.hpp:132-145). */
typedef struct {
    uint32_t family; /* genie_lsh_family */
    uint32_t m;      /* hash functions == keyword dims */
    uint32_t dims;   /* point dimensionality (unused for minHash) */
    uint32_t rehash_domain;
    uint64_t seed;
    double w;
    uint32_t bucket_count;
    int32_t rehash_pstable;
    int64_t bucket_min;
    double sigma;
    uint32_t precision; /* GENIE_LSH_FP64 (default: bit-exact with the reference) or GENIE_LSH_FP32 (opt-in fast
                           mode: fp32 FMA arithmetic; tokens at bucket boundaries may differ -- counted by
                           tests/test_gpu_lsh.py and reported by bench.py) */
    uint32_t reserved;
} genie_lsh_config;
enum { GENIE_LSH_FP64 = 0, GENIE_LSH_FP32 = 1 };

genie_lsh_config genie_lsh_config_default(void);

/* Host-side parameter sampling exactly as LshEncoder::create (lsh.hpp:151-166).
 * p-stable: a[m*dims], b[m]; RBH: a = pitch[m*dims], b = shift[m*dims];
 * minHash: hash_seed[m] (a, b unused).  rehash_seed[m] always. */
int genie_lsh_sample(const genie_lsh_config* cfg, double* a, double* b, uint64_t* hash_seed,
                     uint64_t* rehash_seed, char* err, size_t errlen);

typedef struct genie_encoder genie_encoder;

/* Samples parameters on the host and uploads them to `device`. */
int genie_encoder_create(const genie_lsh_config* cfg, int device, genie_encoder** out, char* err,
                         size_t errlen);
void genie_encoder_destroy(genie_encoder* enc);

/* LshEncoder::encode_point / encode_query_point (lsh.hpp:176-195), batched:
 * tokens[n_points * m], token of function i for point p at [p*m + i]
 * (Keyword{dim=i, token}).  Host buffers.  fp64 with IEEE mul/add/div in the
 * reference order (no contraction): bit-exact with the reference. */
int genie_lsh_encode(genie_encoder* enc, const float* points, uint64_t n_points,
                     uint32_t* tokens, char* err, size_t errlen);
int genie_lsh_encode_device(genie_encoder* enc, const float* d_points, uint64_t n_points,
                            uint32_t* d_tokens, void* stream, char* err, size_t errlen);

/* minHash over sets of u64 elements: set s = elems[set_off[s], set_off[s+1]). */
int genie_minhash_encode(genie_encoder* enc, const uint64_t* set_off, const uint64_t* elems,
                         uint64_t n_sets, uint32_t* tokens, char* err, size_t errlen);
int genie_minhash_encode_device(genie_encoder* enc, const uint64_t* d_set_off,
                                const uint64_t* d_elems, uint64_t n_sets, uint32_t* d_tokens,
                                void* stream, char* err, size_t errlen);

/* LshEncoder::encode_query_point + execute_batch in one call on the GPU (the
 * query path of a vector / set index): host points (n x dims f32) or sets
 * (minHash encoders: set_off[n+1], elems) are uploaded, encoded on the device
 * into one point item per hash function (Keyword{i, f_i(p)}, lsh.hpp:186-195),
 * queried with k results each (query_id = first_id + row) and the results read
 * back -- the tokens never leave the device.  Same output contract as
 * genie_query_batch. */
int genie_lsh_query_batch(genie_encoder* enc, genie_index* ix, const genie_config* cfg, const float* points,
                          const uint64_t* set_off, const uint64_t* elems, uint64_t n, uint32_t k, uint32_t first_id,
                          uint32_t out_stride, genie_entry* out, uint32_t* out_len, uint32_t* out_threshold,
                          genie_batch_stats* stats, char* err, size_t errlen);

/* Builds a device index directly from device tokens (n_points x m, dim = function
 * index): the GPU counterpart of encode_dataset + build_index for LSH data.
 * Postings per key are ascending ids (stable counting sort). */
int genie_index_from_tokens_device(const uint32_t* d_tokens, uint32_t n_points, uint32_t m,
                                   uint32_t token_domain, uint32_t id_offset, int device,
                                   genie_index** out, char* err, size_t errlen);

/* Copies the device CSR back (for parity checks): keys[K], key_off[K+1], postings[P]. */
int genie_index_export(genie_index* ix, uint64_t* keys, uint64_t* key_off, uint32_t* postings,
                       char* err, size_t errlen);

#ifdef __cplusplus
}
#endif

#endif /* GENIE_GENIE_H */
