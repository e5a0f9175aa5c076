/*
 * genie_synth.h -- seeded synthetic workloads of the five BASELINE.json
 * configs, generated natively on the host (libgenie_synth.so).
 * This is input preparation, not the engine: it produces the same objects /
 * queries for the GPU path, the C oracle and the reference shim.
 *
 * Relational and bag-of-words configs come out as a CSR inverted index
 * (keys ascending, ids ascending per key) plus a query batch.  Vector and
 * set configs come out as raw points / sets (the LSH transforms run on the
 * GPU or in the oracle).
 */
#ifndef GENIE_SYNTH_H
#define GENIE_SYNTH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct genie_dataset genie_dataset;

/* C1: Adult-shaped relational table, 14 attributes (6 numeric x 1024 bins,
 * 8 categorical {9,16,7,15,6,5,2,42}); queries are sampled rows with +-50
 * windows on the numeric attributes (clamped, model.hpp:167-188). */
int genie_synth_adult(uint32_t n, uint32_t num_queries, uint32_t k, uint64_t seed,
                      genie_dataset** out);

/* C2: Tweets-shaped bag of words: `words` distinct Zipf(1) ranks over a
 * `vocab` vocabulary per document, keyword (0, rank); queries are fresh
 * documents (point items). */
int genie_synth_tweets(uint32_t n, uint32_t vocab, uint32_t words, uint32_t num_queries, uint32_t k,
                       uint64_t seed, genie_dataset** out);

/* C3: SIFT-shaped centred 64-component Gaussian mixture in `dims` dims. */
int genie_synth_sift(uint32_t n, uint32_t dims, uint32_t num_queries, uint64_t seed,
                     genie_dataset** out);

/* C5: OCR-shaped 10-class mixture in [0,1]^dims; labels kept. */
int genie_synth_ocr(uint32_t n, uint32_t dims, uint32_t num_queries, uint64_t seed,
                    genie_dataset** out);

/* C4: sets of u64 elements, sizes U[32,256], 20% near-duplicates; queries are
 * copies of indexed sets with 10% of the elements replaced. */
int genie_synth_sets(uint32_t n, uint32_t num_queries, uint64_t seed, genie_dataset** out);

/* Random small instance in the style of the reference unit tests
 * (test_engine.cpp:34-60): dims in [0,dims), tokens in [0,tokens), up to
 * max_kw keywords per object, 1..max_items range items per query, k in
 * [1,max_k]. */
int genie_synth_random(uint32_t n, uint32_t dims, uint32_t tokens, uint32_t max_kw,
                       uint32_t num_queries, uint32_t max_items, uint32_t max_span, uint32_t max_k,
                       uint64_t seed, genie_dataset** out);

void genie_dataset_free(genie_dataset* ds);

/* Views (pointers stay valid until genie_dataset_free).  Absent parts report 0. */
void genie_dataset_csr(const genie_dataset* ds, uint32_t* n, uint64_t* num_keys,
                       const uint64_t** keys, const uint64_t** key_off, const uint32_t** postings);
void genie_dataset_queries(const genie_dataset* ds, uint32_t* num_queries, const uint32_t** qid,
                           const uint32_t** k, const uint64_t** item_off, const uint16_t** dim,
                           const uint32_t** lo, const uint32_t** hi);
void genie_dataset_points(const genie_dataset* ds, uint32_t* n, uint32_t* dims, const float** points,
                          uint32_t* num_queries, const float** query_points, const uint32_t** labels,
                          const uint32_t** query_labels);
void genie_dataset_sets(const genie_dataset* ds, uint32_t* n, const uint64_t** set_off,
                        const uint64_t** elems, uint32_t* num_queries, const uint64_t** query_off,
                        const uint64_t** query_elems);

/* CSR from per-object keyword lists (object i owns [obj_off[i], obj_off[i+1])),
 * i.e. build_index (index.hpp:190-250) on the host without splitting.  Keys
 * of one object must be distinct.  Returns a dataset holding only the CSR. */
int genie_synth_csr_from_objects(uint32_t n, const uint64_t* obj_off, const uint16_t* dims,
                                 const uint32_t* tokens, genie_dataset** out, char* err,
                                 size_t errlen);

#ifdef __cplusplus
}
#endif

#endif
