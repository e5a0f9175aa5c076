// Sequence verification for SequenceSearcher (sa.hpp:127-162, 298-336,
// 419-512): Levenshtein distances of one query to many corpus sequences on
// the GPU, one thread per (query, sequence) pair, with the bit-parallel
// block algorithm of Myers (1999) in Hyyrö's formulation: the DP column of
// each text character is advanced 64 query rows per word operation, so a
// ~100-byte pair costs ~200 word steps instead of ~10 000 cells.
//
// The corpus lives on the device (genie_seqset: concatenated bytes +
// offsets).  Per query, a small kernel builds the match-mask table
// Peq[c][w] (bit r of word w set when query[64 w + r] == c); the distance
// kernel then streams each sequence's bytes.  Results follow
// edit_distance_bounded's contract (sa.hpp:127-162): the exact distance when
// it is <= cap, cap + 1 otherwise -- a thread stops as soon as the distance
// is provably above the cap (the last row can fall by at most one per
// remaining text byte).
#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace genie {
namespace {

constexpr int kSeqThreads = 128;
constexpr uint32_t kRegWords = 4;  // queries up to 256 bytes keep the DP state in registers

__global__ void k_peq(const uint8_t* __restrict__ q, uint32_t m, uint32_t W, unsigned long long* __restrict__ peq) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // (c, w)
    if (i >= 256u * W) return;
    const uint32_t c = i / W, w = i % W;
    unsigned long long bits = 0;
    for (uint32_t r = 0; r < 64; ++r) {
        const uint32_t pos = w * 64 + r;
        if (pos < m && q[pos] == c) bits |= 1ull << r;
    }
    peq[i] = bits;
}

// One block of 64 DP rows advanced by one text byte (Myers 1999, Sec. 4):
// hin is the horizontal delta entering the block's top row (-1, 0, +1);
// returns the delta leaving its row `out_bit`.
__device__ __forceinline__ int advance_block(unsigned long long& Pv, unsigned long long& Mv, unsigned long long Eq,
                                             int hin, uint32_t out_bit) {
    const unsigned long long hneg = hin < 0 ? 1ull : 0ull;
    const unsigned long long Xv = Eq | Mv;
    Eq |= hneg;
    const unsigned long long Xh = (((Eq & Pv) + Pv) ^ Pv) | Eq;
    unsigned long long Ph = Mv | ~(Xh | Pv);
    unsigned long long Mh = Pv & Xh;
    const int hout = int((Ph >> out_bit) & 1ull) - int((Mh >> out_bit) & 1ull);
    Ph = (Ph << 1) | (hin > 0 ? 1ull : 0ull);
    Mh = (Mh << 1) | hneg;
    Pv = Mh | ~(Xv | Ph);
    Mv = Ph & Xv;
    return hout;
}

// State in registers (W <= kRegWords) or in a per-thread global slice.
template <bool REG>
__global__ void __launch_bounds__(kSeqThreads)
    k_edit_distance(const uint8_t* __restrict__ bytes, const uint64_t* __restrict__ off,
                    const uint32_t* __restrict__ ids, uint64_t count, const unsigned long long* __restrict__ peq,
                    uint32_t m, uint32_t W, uint32_t cap, unsigned long long* __restrict__ scratch,
                    uint32_t* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t sid = ids ? ids[i] : static_cast<uint32_t>(i);
    const uint64_t b = off[sid], n = off[sid + 1] - b;
    const uint8_t* t = bytes + b;
    const uint64_t inf = uint64_t(cap) + 1;
    // |m - n| is a lower bound (the band of edit_distance_bounded)
    const uint64_t diff = n > m ? n - m : m - n;
    if (diff > cap) {
        out[i] = static_cast<uint32_t>(inf);
        return;
    }
    if (m == 0 || n == 0) {  // the other length
        out[i] = static_cast<uint32_t>(m + n < inf ? m + n : inf);
        return;
    }
    unsigned long long regP[REG ? kRegWords : 1], regM[REG ? kRegWords : 1];
    unsigned long long* gP = REG ? nullptr : scratch + i * 2 * W;
    unsigned long long* gM = REG ? nullptr : gP + W;
    for (uint32_t w = 0; w < W; ++w) {
        if constexpr (REG) {
            regP[w] = ~0ull;  // D[r][0] = r: vertical deltas +1
            regM[w] = 0;
        } else {
            gP[w] = ~0ull;
            gM[w] = 0;
        }
    }
    const uint32_t last_bit = (m - 1) & 63u;
    int64_t score = m;  // D[m][0]
    for (uint64_t j = 0; j < n; ++j) {
        const unsigned long long* eq = peq + uint32_t(t[j]) * W;
        int h = 1;  // D[0][j+1] - D[0][j] = +1 (global distance)
        if constexpr (REG) {
#pragma unroll
            for (uint32_t w = 0; w < kRegWords; ++w)
                if (w < W) h = advance_block(regP[w], regM[w], eq[w], h, w + 1 == W ? last_bit : 63u);
        } else {
            for (uint32_t w = 0; w < W; ++w) {
                unsigned long long P = gP[w], M = gM[w];
                h = advance_block(P, M, eq[w], h, w + 1 == W ? last_bit : 63u);
                gP[w] = P;
                gM[w] = M;
            }
        }
        score += h;
        // the last row falls by at most one per remaining byte
        if (score - int64_t(n - j - 1) > int64_t(cap)) {
            out[i] = static_cast<uint32_t>(inf);
            return;
        }
    }
    out[i] = static_cast<uint32_t>(uint64_t(score) < inf ? uint64_t(score) : inf);
}

}  // namespace
}  // namespace genie

struct genie_seqset {
    int device = 0;
    uint64_t n = 0, total = 0;
    cudaStream_t stream = nullptr;
    genie::DevBuf<uint8_t> bytes, query;
    genie::DevBuf<uint64_t> off;
    genie::DevBuf<unsigned long long> peq, scratch;
    genie::DevBuf<uint32_t> ids, out;
};

using namespace genie;

extern "C" {

int genie_seqset_create(const uint8_t* bytes, const uint64_t* off, uint64_t n, int device, genie_seqset** out,
                        char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        if (!out || !off || (off[n] && !bytes)) throw Error(GENIE_ERR_CONTRACT, "genie_seqset_create: null argument");
        for (uint64_t i = 0; i < n; ++i)
            if (off[i + 1] < off[i]) throw Error(GENIE_ERR_CONTRACT, "genie_seqset_create: offsets not monotone");
        if (off[0] != 0) throw Error(GENIE_ERR_CONTRACT, "genie_seqset_create: off[0] must be 0");
        ensure_device(device);
        auto* s = new genie_seqset;
        try {
            s->device = device;
            s->n = n;
            s->total = off[n];
            GENIE_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
            s->bytes.reserve(s->total + 16);
            s->off.reserve(n + 1);
            if (s->total)
                GENIE_CUDA(cudaMemcpyAsync(s->bytes.p, bytes, s->total, cudaMemcpyHostToDevice, s->stream));
            GENIE_CUDA(cudaMemcpyAsync(s->off.p, off, (n + 1) * 8, cudaMemcpyHostToDevice, s->stream));
            GENIE_CUDA(cudaStreamSynchronize(s->stream));
        } catch (...) {
            genie_seqset_destroy(s);
            throw;
        }
        *out = s;
        return GENIE_OK;
    });
}

void genie_seqset_destroy(genie_seqset* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    s->bytes.release();
    s->query.release();
    s->off.release();
    s->peq.release();
    s->scratch.release();
    s->ids.release();
    s->out.release();
    if (s->stream) cudaStreamDestroy(s->stream);
    delete s;
}

int genie_seqset_distances(genie_seqset* s, const uint8_t* query, uint64_t qlen, const uint32_t* ids, uint64_t count,
                           uint32_t cap, uint32_t* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        if (!s || (count && !out) || (qlen && !query)) throw Error(GENIE_ERR_CONTRACT, "genie_seqset_distances: null argument");
        if (qlen >= (1ull << 31)) throw Error(GENIE_ERR_CONTRACT, "genie_seqset_distances: query too long");
        if (ids) {
            for (uint64_t i = 0; i < count; ++i)
                if (ids[i] >= s->n) throw Error(GENIE_ERR_CONTRACT, "genie_seqset_distances: sequence id out of range");
        } else if (count > s->n) {
            throw Error(GENIE_ERR_CONTRACT, "genie_seqset_distances: count exceeds the set");
        }
        if (!count) return GENIE_OK;
        ensure_device(s->device);
        cudaStream_t st = s->stream;
        const uint32_t m = static_cast<uint32_t>(qlen);
        const uint32_t W = std::max<uint32_t>(1, (m + 63) / 64);
        s->query.reserve(std::max<uint64_t>(qlen, 1));
        s->peq.reserve(256ull * W);
        if (qlen) GENIE_CUDA(cudaMemcpyAsync(s->query.p, query, qlen, cudaMemcpyHostToDevice, st));
        k_peq<<<(256 * W + 255) / 256, 256, 0, st>>>(s->query.p, m, W, s->peq.p);
        const uint32_t* d_ids = nullptr;
        if (ids) {
            s->ids.reserve(count);
            GENIE_CUDA(cudaMemcpyAsync(s->ids.p, ids, count * 4, cudaMemcpyHostToDevice, st));
            d_ids = s->ids.p;
        }
        s->out.reserve(count);
        const unsigned grid = static_cast<unsigned>((count + kSeqThreads - 1) / kSeqThreads);
        if (W <= kRegWords) {
            k_edit_distance<true><<<grid, kSeqThreads, 0, st>>>(s->bytes.p, s->off.p, d_ids, count, s->peq.p, m, W,
                                                                cap, nullptr, s->out.p);
        } else {
            s->scratch.reserve(count * 2 * W);
            k_edit_distance<false><<<grid, kSeqThreads, 0, st>>>(s->bytes.p, s->off.p, d_ids, count, s->peq.p, m, W,
                                                                 cap, s->scratch.p, s->out.p);
        }
        GENIE_CUDA(cudaGetLastError());
        GENIE_CUDA(cudaMemcpyAsync(out, s->out.p, count * 4, cudaMemcpyDeviceToHost, st));
        GENIE_CUDA(cudaStreamSynchronize(st));
        return GENIE_OK;
    });
}

void genie_seqset_info(const genie_seqset* s, uint64_t* num_sequences, uint64_t* total_bytes, int* device) {
    if (!s) return;
    if (num_sequences) *num_sequences = s->n;
    if (total_bytes) *total_bytes = s->total;
    if (device) *device = s->device;
}

}  // extern "C"
