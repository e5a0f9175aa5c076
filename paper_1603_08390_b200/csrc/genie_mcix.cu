// MCIX index files (the reference's on-disk format, index_io.hpp:27-154)
// read straight into the device CSR and written from a CSR.
//
// Layout (little-endian): "MCIX", u32 version = 1, u32 num_objects,
// u32 num_keywords, then per keyword {u16 dim, u32 token, u16 span_count,
// span_count x {u64 begin, u64 end}}, then the list array (u32 ids).  The
// spans of the keywords tile the list array in keyword order, so a keyword's
// postings are one contiguous range -- exactly a CSR row -- and the list array
// is the CSR postings array as it lies in the file.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

namespace genie {
namespace {

struct Reader {
    const uint8_t* d;
    uint64_t n, pos = 0;
    uint64_t take(int bytes) {
        if (pos + uint64_t(bytes) > n)
            throw Error(GENIE_ERR_DATA, "index file truncated at offset " + std::to_string(pos));
        uint64_t v = 0;
        for (int i = 0; i < bytes; ++i) v |= uint64_t(d[pos + i]) << (8 * i);
        pos += uint64_t(bytes);
        return v;
    }
};

// Parses and validates an image the way deserialize_index does
// (index_io.hpp:84-146): magic, version, keyword order, spans present, in
// order and tiling the list array, list size, id range, ascending ids per
// keyword.  Fills the CSR arrays when they are non-null.
void parse(const uint8_t* data, uint64_t size, uint32_t& num_objects, uint64_t& K, uint64_t& P,
           uint64_t* keys, uint64_t* key_off, uint32_t* postings, uint64_t* num_spans = nullptr,
           uint16_t* span_count = nullptr, uint64_t* span_bounds = nullptr) {
    if (!data && size) throw Error(GENIE_ERR_CONTRACT, "genie_mcix_parse: null data");
    Reader in{data, size};
    if (in.take(1) != 'M' || in.take(1) != 'C' || in.take(1) != 'I' || in.take(1) != 'X')
        throw Error(GENIE_ERR_DATA, "not an MCIX index file (bad magic)");
    const uint64_t version = in.take(4);
    if (version != 1) throw Error(GENIE_ERR_DATA, "unsupported index version " + std::to_string(version));
    num_objects = static_cast<uint32_t>(in.take(4));
    K = in.take(4);
    uint64_t total = 0, prev_key = 0, nspan = 0;
    for (uint64_t j = 0; j < K; ++j) {
        const uint64_t dim = in.take(2), token = in.take(4), spans = in.take(2);
        const uint64_t key = (dim << 32) | token;
        if (j && !(prev_key < key)) throw Error(GENIE_ERR_DATA, "index keywords out of order");
        if (spans == 0) throw Error(GENIE_ERR_DATA, "keyword with no postings spans");
        if (keys) keys[j] = key;
        if (key_off) key_off[j] = total;
        if (span_count) span_count[j] = static_cast<uint16_t>(spans);
        for (uint64_t s = 0; s < spans; ++s) {
            const uint64_t b = in.take(8), e = in.take(8);
            if (b > e) throw Error(GENIE_ERR_DATA, "span with begin > end");
            if (b != total) throw Error(GENIE_ERR_DATA, "spans do not tile the list array");
            if (span_bounds) {
                span_bounds[2 * nspan] = b;
                span_bounds[2 * nspan + 1] = e;
            }
            ++nspan;
            total = e;
        }
        prev_key = key;
    }
    if (num_spans) *num_spans = nspan;
    if (key_off) key_off[K] = total;
    const uint64_t rest = in.n - in.pos;
    if (rest != total * 4)
        throw Error(GENIE_ERR_DATA, "list array size mismatch: spans cover " + std::to_string(total) +
                                        " ids, file holds " + std::to_string(rest / 4));
    P = total;
    if (!postings) return;
    const uint8_t* ids = data + in.pos;
    for (uint64_t i = 0; i < total; ++i) {
        uint32_t v;
        std::memcpy(&v, ids + 4 * i, 4);  // little-endian host (x86-64 / aarch64)
        if (v >= num_objects) throw Error(GENIE_ERR_DATA, "object id " + std::to_string(v) + " out of range");
        postings[i] = v;
    }
    // per keyword, its postings strictly ascending
    for (uint64_t j = 0; j < K; ++j)
        for (uint64_t i = key_off[j] + 1; i < key_off[j + 1]; ++i)
            if (postings[i] <= postings[i - 1])
                throw Error(GENIE_ERR_DATA, "postings of one keyword not strictly ascending");
}

void put(std::vector<uint8_t>& out, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) out.push_back(static_cast<uint8_t>((v >> (8 * i)) & 0xff));
}

// The keyword table of an image (everything before the list array); span s of
// keyword j is [bound(j, s, 0), bound(j, s, 1)).
template <class Spans, class Bound>
std::vector<uint8_t> image_head(uint32_t num_objects, uint64_t K, const uint64_t* keys, Spans spans_of,
                                Bound bound) {
    std::vector<uint8_t> img;
    img.insert(img.end(), {'M', 'C', 'I', 'X'});
    put(img, 1, 4);
    put(img, num_objects, 4);
    put(img, K, 4);
    for (uint64_t j = 0; j < K; ++j) {
        const uint64_t spans = spans_of(j);
        if (spans == 0) throw Error(GENIE_ERR_DATA, "keyword with no postings");
        if (spans > 0xffff) throw Error(GENIE_ERR_DATA, "keyword has too many sub-lists (" + std::to_string(spans) + ")");
        put(img, keys[j] >> 32, 2);
        put(img, keys[j] & 0xffffffffull, 4);
        put(img, spans, 2);
        for (uint64_t s = 0; s < spans; ++s) {
            put(img, bound(j, s, 0), 8);
            put(img, bound(j, s, 1), 8);
        }
    }
    return img;
}

void write_image(const std::vector<uint8_t>& head, uint64_t P, const uint32_t* postings, uint8_t* out,
                 uint64_t* size) {
    const uint64_t need = head.size() + 4 * P;
    if (out) {
        if (*size < need) throw Error(GENIE_ERR_CONTRACT, "genie_mcix_serialize: output buffer too small");
        std::memcpy(out, head.data(), head.size());
        for (uint64_t i = 0; i < P; ++i) {
            const uint32_t v = postings[i];
            std::memcpy(out + head.size() + 4 * i, &v, 4);
        }
    }
    *size = need;
}

}  // namespace
}  // namespace genie

using namespace genie;

int genie_mcix_parse(const uint8_t* data, uint64_t size, uint32_t* num_objects, uint64_t* num_keys,
                     uint64_t* num_postings, uint64_t* keys, uint64_t* key_off, uint32_t* postings, char* err,
                     size_t errlen) {
    return guarded(err, errlen, [&] {
        uint32_t n = 0;
        uint64_t K = 0, P = 0;
        // shape call: null arrays; fill call: keys, key_off and postings sized by it
        if ((keys || key_off || postings) && !(keys && key_off && postings))
            throw Error(GENIE_ERR_CONTRACT, "genie_mcix_parse: keys, key_off and postings go together");
        parse(data, size, n, K, P, keys, key_off, postings);
        if (num_objects) *num_objects = n;
        if (num_keys) *num_keys = K;
        if (num_postings) *num_postings = P;
        return GENIE_OK;
    });
}

int genie_index_load_mcix(const uint8_t* data, uint64_t size, int device, genie_index** out, char* err,
                          size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        if (!out) throw Error(GENIE_ERR_CONTRACT, "genie_index_load_mcix: null argument");
        uint32_t n = 0;
        uint64_t K = 0, P = 0;
        parse(data, size, n, K, P, nullptr, nullptr, nullptr);
        std::vector<uint64_t> keys(K), off(K + 1);
        std::vector<uint32_t> post(P);
        parse(data, size, n, K, P, keys.data(), off.data(), post.data());
        return genie_index_create(n, K, keys.data(), off.data(), post.data(), nullptr, 0, device, out, err, errlen);
    });
}

int genie_mcix_serialize(uint32_t num_objects, uint64_t num_keys, const uint64_t* keys, const uint64_t* key_off,
                         const uint32_t* postings, uint32_t split, uint8_t* out, uint64_t* size, char* err,
                         size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!size || (num_keys && (!keys || !key_off))) throw Error(GENIE_ERR_CONTRACT, "genie_mcix_serialize: null argument");
        if (num_keys > 0xffffffffull) throw Error(GENIE_ERR_CONTRACT, "genie_mcix_serialize: too many keywords");
        // serialize_index (index_io.hpp:63-82) of the index build_index makes
        // with this split threshold (index.hpp:229-238): every list cut into
        // consecutive spans of `split` ids (the last one shorter), 0 = whole
        auto limit = [&](uint64_t j) {
            const uint64_t len = key_off[j + 1] - key_off[j];
            return split ? uint64_t(split) : (len ? len : 1);
        };
        const auto head = image_head(
            num_objects, num_keys, keys,
            [&](uint64_t j) { return (key_off[j + 1] - key_off[j] + limit(j) - 1) / limit(j); },
            [&](uint64_t j, uint64_t s, int end) {
                const uint64_t b = key_off[j] + s * limit(j);
                return end ? std::min(b + limit(j), key_off[j + 1]) : b;
            });
        write_image(head, num_keys ? key_off[num_keys] : 0, postings, out, size);
        return GENIE_OK;
    });
}

int genie_mcix_parse_spans(const uint8_t* data, uint64_t size, uint64_t* num_spans, uint16_t* span_count,
                           uint64_t* span_bounds, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!num_spans) throw Error(GENIE_ERR_CONTRACT, "genie_mcix_parse_spans: null argument");
        uint32_t n = 0;
        uint64_t K = 0, P = 0;
        parse(data, size, n, K, P, nullptr, nullptr, nullptr, num_spans, span_count, span_bounds);
        return GENIE_OK;
    });
}

int genie_mcix_serialize_spans(uint32_t num_objects, uint64_t num_keys, const uint64_t* keys,
                               const uint16_t* span_count, const uint64_t* span_bounds, uint64_t num_postings,
                               const uint32_t* postings, uint8_t* out, uint64_t* size, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!size || (num_keys && (!keys || !span_count || !span_bounds)) || (num_postings && !postings))
            throw Error(GENIE_ERR_CONTRACT, "genie_mcix_serialize_spans: null argument");
        if (num_keys > 0xffffffffull) throw Error(GENIE_ERR_CONTRACT, "genie_mcix_serialize: too many keywords");
        std::vector<uint64_t> first(num_keys + 1, 0);
        for (uint64_t j = 0; j < num_keys; ++j) first[j + 1] = first[j] + span_count[j];
        const auto head = image_head(
            num_objects, num_keys, keys, [&](uint64_t j) { return uint64_t(span_count[j]); },
            [&](uint64_t j, uint64_t s, int end) { return span_bounds[2 * (first[j] + s) + end]; });
        write_image(head, num_postings, postings, out, size);
        return GENIE_OK;
    });
}
