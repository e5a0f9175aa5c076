// LSH / minHash transforms (north_star subsystem 5) and the GPU index build
// from encoded tokens.
//
//   k_pstable   PStableHash::bucket + clamp / rehash (lsh.hpp:42-50, 203-210):
//               dot = b; dot += a_j * (double)p_j in order j = 0..dims-1, then
//               floor(dot / w).  IEEE fp64 with explicit __dmul_rn/__dadd_rn
//               (never contracted into DFMA) and __ddiv_rn: bit-exact with the
//               reference built with -ffp-contract=off.  Register-tiled
//               (4 points x 4 functions per thread) over shared-memory tiles.
//   k_rbh       RbhHash::signature + Rehasher (lsh.hpp:72-80, 105-111):
//               sig_j = floor(((double)p_j - u_j) / g_j), state = mix64(seed);
//               state = mix64(state ^ sig_j).  The quotient is first formed
//               with a multiply by the host-computed reciprocal; only when it
//               lies within a few ulps of an integer is the exact IEEE division
//               evaluated, so floor() always sees the correctly rounded quotient.
//   k_minhash   new: min_e mix64(seed_i ^ e), then Rehasher.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.cuh"

struct genie_encoder {
    int device = 0;
    genie_lsh_config cfg{};
    genie::DevBuf<double> a, b, inv;       // p-stable: a[m*dims], b[m]; RBH: pitch, shift, 1/pitch
    genie::DevBuf<float> af, bf, invf;     // fp32 copies (GENIE_LSH_FP32)
    genie::DevBuf<unsigned long long> hash_seed, rehash_seed;
    // host-API staging, grown on demand and kept (no allocation per call)
    genie::DevBuf<float> ws_points;
    genie::DevBuf<uint32_t> ws_tokens;
    genie::DevBuf<uint64_t> ws_off, ws_elems;
    cudaStream_t stream = nullptr;
};

namespace genie {

void build_dense_containers(genie_index* ix, const uint64_t* h_off);

// ------------------------------------------------------------ host sampling

namespace {
struct HostRng {  // SplitMix64 (rng.hpp:36-88)
    uint64_t state;
    double spare = 0.0;
    bool has_spare = false;
    explicit HostRng(uint64_t s) : state(s) {}
    uint64_t next() {
        state += 0x9e3779b97f4a7c15ull;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double normal() {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare = r * std::sin(theta);
        has_spare = true;
        return r * std::cos(theta);
    }
    double exponential(double scale) {
        double u = uniform();
        while (u <= 0.0) u = uniform();
        return -scale * std::log(u);
    }
    double gamma2(double scale) {
        const double x = exponential(scale);
        return x + exponential(scale);
    }
};
}  // namespace

static void check_cfg(const genie_lsh_config& c) {
    if (c.m == 0) throw Error(GENIE_ERR_CONTRACT, "encoder needs at least one hash function");
    if (c.m > 0x10000u) throw Error(GENIE_ERR_CONTRACT, "m exceeds the 16-bit dim space");
    if (c.family != GENIE_LSH_MINHASH && c.dims == 0)
        throw Error(GENIE_ERR_CONTRACT, "encoder needs a point dimensionality");
    if (c.rehash_domain == 0) throw Error(GENIE_ERR_CONTRACT, "re-hash domain must be positive");
    if (c.family == GENIE_LSH_PSTABLE && !(c.w > 0.0))
        throw Error(GENIE_ERR_CONTRACT, "bucket width must be positive");
    if (c.family == GENIE_LSH_RBH && !(c.sigma > 0.0))
        throw Error(GENIE_ERR_CONTRACT, "kernel width must be positive");
    if (c.family > GENIE_LSH_MINHASH) throw Error(GENIE_ERR_CONTRACT, "unknown LSH family");
    if (c.precision > GENIE_LSH_FP32) throw Error(GENIE_ERR_CONTRACT, "unknown LSH precision");
}

// LshEncoder::create (lsh.hpp:151-166)
static void sample(const genie_lsh_config& c, double* a, double* b, uint64_t* hs, uint64_t* rs) {
    for (uint32_t i = 0; i < c.m; ++i) {
        HostRng r(mix64(c.seed) ^ mix64(0x9e3779b9ull + i));
        if (c.family == GENIE_LSH_PSTABLE) {
            for (uint32_t j = 0; j < c.dims; ++j) a[size_t(i) * c.dims + j] = r.normal();
            b[i] = r.uniform() * c.w;  // uniform(w) (rng.hpp:95)
        } else if (c.family == GENIE_LSH_RBH) {
            for (uint32_t j = 0; j < c.dims; ++j) {
                const double g = r.gamma2(c.sigma);
                a[size_t(i) * c.dims + j] = g;
                b[size_t(i) * c.dims + j] = r.uniform() * g;
            }
        } else {
            if (hs) hs[i] = r.next();
        }
        rs[i] = r.next();
    }
}

// ---------------------------------------------------------------- p-stable

constexpr int PS_PT = 64;   // points per block
constexpr int PS_FN = 64;   // functions per block
constexpr int PS_DC = 16;   // dims per smem chunk
constexpr int PS_THREADS = 256;

__global__ void __launch_bounds__(PS_THREADS)
    k_pstable(const float* __restrict__ pts, uint64_t n, uint32_t dims, uint32_t m,
              const double* __restrict__ a, const double* __restrict__ b, double w,
              uint32_t bucket_count, int64_t bucket_min, int rehash,
              const unsigned long long* __restrict__ rseed, uint32_t domain,
              uint32_t* __restrict__ tokens) {
    __shared__ double sp[PS_DC][PS_PT + 1];
    __shared__ double sa[PS_DC][PS_FN + 1];
    const uint64_t p0 = uint64_t(blockIdx.x) * PS_PT;
    const uint32_t f0 = blockIdx.y * PS_FN;
    const int tx = threadIdx.x & 15;  // function group
    const int ty = threadIdx.x >> 4;  // point group
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t f = f0 + tx + 16 * j;
            acc[i][j] = f < m ? b[f] : 0.0;  // dot starts at b (lsh.hpp:47)
        }
    for (uint32_t d0 = 0; d0 < dims; d0 += PS_DC) {
        for (int i = threadIdx.x; i < PS_DC * PS_PT; i += PS_THREADS) {
            const int pp = i / PS_DC, dd = i % PS_DC;
            const uint64_t p = p0 + pp;
            const uint32_t d = d0 + dd;
            sp[dd][pp] = (p < n && d < dims) ? static_cast<double>(pts[p * dims + d]) : 0.0;
        }
        for (int i = threadIdx.x; i < PS_DC * PS_FN; i += PS_THREADS) {
            const int ff = i / PS_DC, dd = i % PS_DC;
            const uint32_t f = f0 + ff, d = d0 + dd;
            sa[dd][ff] = (f < m && d < dims) ? a[size_t(f) * dims + d] : 0.0;
        }
        __syncthreads();
        const int dn = (dims - d0) < uint32_t(PS_DC) ? int(dims - d0) : PS_DC;
        for (int dd = 0; dd < dn; ++dd) {
            double pv[4], av[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) pv[i] = sp[dd][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) av[j] = sa[dd][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(av[j], pv[i]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint64_t p = p0 + ty + 16 * i;
        if (p >= n) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t f = f0 + tx + 16 * j;
            if (f >= m) continue;
            const long long raw = static_cast<long long>(floor(__ddiv_rn(acc[i][j], w)));
            uint32_t tok;
            if (rehash) {
                uint64_t st = mix64(rseed[f]);
                st = mix64(st ^ static_cast<uint64_t>(raw));
                tok = static_cast<uint32_t>(st % domain);
            } else {
                long long off = raw - bucket_min;
                off = off < 0 ? 0 : off;
                off = off > static_cast<long long>(bucket_count) - 1 ? static_cast<long long>(bucket_count) - 1 : off;
                tok = static_cast<uint32_t>(off);
            }
            tokens[p * m + f] = tok;
        }
    }
}

// --------------------------------------------------------------------- RBH

constexpr int RB_PT = 32;  // points per block (one per lane)
constexpr int RB_FN = 8;   // functions per block (one per warp)
constexpr int RB_DC = 64;  // dims per smem chunk

// floor(x / g) with the correctly rounded IEEE quotient, via the reciprocal
// fast path plus an exact fallback near integer boundaries.
__device__ __forceinline__ long long floor_div_exact(double x, double g, double inv) {
    const double q = __dmul_rn(x, inv);
    const double f = floor(q);
    // |q - RN(x/g)| <= 2 ulp(q); if q is farther than 8 ulp from both integers
    // around it, the exact quotient has the same floor
    const double tol = 8.0 * 2.220446049250313e-16 * fabs(q) + 1e-300;
    if (q - f > tol && (f + 1.0) - q > tol) return static_cast<long long>(f);
    return static_cast<long long>(floor(__ddiv_rn(x, g)));
}

__global__ void __launch_bounds__(RB_PT * RB_FN)
    k_rbh(const float* __restrict__ pts, uint64_t n, uint32_t dims, uint32_t m,
          const double* __restrict__ pitch, const double* __restrict__ shift,
          const double* __restrict__ inv, const unsigned long long* __restrict__ rseed,
          uint32_t domain, uint32_t* __restrict__ tokens) {
    __shared__ float sp[RB_PT][RB_DC + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t p = uint64_t(blockIdx.x) * RB_PT + lane;
    const uint32_t f = blockIdx.y * RB_FN + warp;
    uint64_t st = f < m ? mix64(rseed[f]) : 0;
    const double* gp = pitch + size_t(f < m ? f : 0) * dims;
    const double* up = shift + size_t(f < m ? f : 0) * dims;
    const double* ip = inv + size_t(f < m ? f : 0) * dims;
    for (uint32_t d0 = 0; d0 < dims; d0 += RB_DC) {
        for (int i = threadIdx.x; i < RB_PT * RB_DC; i += RB_PT * RB_FN) {
            const int pp = i / RB_DC, dd = i % RB_DC;
            const uint64_t pi = uint64_t(blockIdx.x) * RB_PT + pp;
            const uint32_t d = d0 + dd;
            sp[pp][dd] = (pi < n && d < dims) ? pts[pi * dims + d] : 0.f;
        }
        __syncthreads();
        if (f < m) {
            const int dn = (dims - d0) < uint32_t(RB_DC) ? int(dims - d0) : RB_DC;
            for (int dd = 0; dd < dn; ++dd) {
                const uint32_t d = d0 + dd;
                const double x = __dsub_rn(static_cast<double>(sp[lane][dd]), up[d]);
                const long long sig = floor_div_exact(x, gp[d], ip[d]);
                st = mix64(st ^ static_cast<uint64_t>(sig));
            }
        }
        __syncthreads();
    }
    if (p < n && f < m) tokens[p * m + f] = static_cast<uint32_t>(st % domain);
}

// ------------------------------------------------- opt-in fp32 transforms
// GENIE_LSH_FP32: the same hash functions evaluated in fp32 with FMA
// contraction (p-stable: one FFMA per (point, function, dim); RBH: one
// FFMA-style (p - u) * (1/g) per coordinate).  Not bit-exact: a token whose
// fp64 bucket value lies within fp32 rounding of an integer boundary may land
// in the neighbouring bucket.  SURVEY 8c measured 22 of 11.85M p-stable
// tokens (1.9e-6) and 0 of 711K RBH tokens for this kind of arithmetic; the
// tests count and bound the disagreements against the fp64 path.
__global__ void __launch_bounds__(PS_THREADS)
    k_pstable_f32(const float* __restrict__ pts, uint64_t n, uint32_t dims, uint32_t m, const float* __restrict__ a,
                  const float* __restrict__ b, float w, uint32_t bucket_count, int64_t bucket_min, int rehash,
                  const unsigned long long* __restrict__ rseed, uint32_t domain, uint32_t* __restrict__ tokens) {
    __shared__ float sp[PS_DC][PS_PT + 1];
    __shared__ float sa[PS_DC][PS_FN + 1];
    const uint64_t p0 = uint64_t(blockIdx.x) * PS_PT;
    const uint32_t f0 = blockIdx.y * PS_FN;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t f = f0 + tx + 16 * j;
            acc[i][j] = f < m ? b[f] : 0.f;
        }
    for (uint32_t d0 = 0; d0 < dims; d0 += PS_DC) {
        for (int i = threadIdx.x; i < PS_DC * PS_PT; i += PS_THREADS) {
            const int pp = i / PS_DC, dd = i % PS_DC;
            const uint64_t pt = p0 + pp;
            const uint32_t d = d0 + dd;
            sp[dd][pp] = (pt < n && d < dims) ? pts[pt * dims + d] : 0.f;
        }
        for (int i = threadIdx.x; i < PS_DC * PS_FN; i += PS_THREADS) {
            const int ff = i / PS_DC, dd = i % PS_DC;
            const uint32_t f = f0 + ff, d = d0 + dd;
            sa[dd][ff] = (f < m && d < dims) ? a[size_t(f) * dims + d] : 0.f;
        }
        __syncthreads();
        const int dn = (dims - d0) < uint32_t(PS_DC) ? int(dims - d0) : PS_DC;
        for (int dd = 0; dd < dn; ++dd) {
            float pv[4], av[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) pv[i] = sp[dd][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) av[j] = sa[dd][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[j], pv[i], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint64_t pt = p0 + ty + 16 * i;
        if (pt >= n) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t f = f0 + tx + 16 * j;
            if (f >= m) continue;
            const long long raw = static_cast<long long>(floorf(acc[i][j] / w));
            uint32_t tok;
            if (rehash) {
                uint64_t st = mix64(rseed[f]);
                st = mix64(st ^ static_cast<uint64_t>(raw));
                tok = static_cast<uint32_t>(st % domain);
            } else {
                long long off = raw - bucket_min;
                off = off < 0 ? 0 : off;
                off = off > static_cast<long long>(bucket_count) - 1 ? static_cast<long long>(bucket_count) - 1 : off;
                tok = static_cast<uint32_t>(off);
            }
            tokens[pt * m + f] = tok;
        }
    }
}

__global__ void __launch_bounds__(RB_PT * RB_FN)
    k_rbh_f32(const float* __restrict__ pts, uint64_t n, uint32_t dims, uint32_t m, const float* __restrict__ shift,
              const float* __restrict__ inv, const unsigned long long* __restrict__ rseed, uint32_t domain,
              uint32_t* __restrict__ tokens) {
    __shared__ float sp[RB_PT][RB_DC + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t p = uint64_t(blockIdx.x) * RB_PT + lane;
    const uint32_t f = blockIdx.y * RB_FN + warp;
    uint64_t st = f < m ? mix64(rseed[f]) : 0;
    const float* up = shift + size_t(f < m ? f : 0) * dims;
    const float* ip = inv + size_t(f < m ? f : 0) * dims;
    for (uint32_t d0 = 0; d0 < dims; d0 += RB_DC) {
        for (int i = threadIdx.x; i < RB_PT * RB_DC; i += RB_PT * RB_FN) {
            const int pp = i / RB_DC, dd = i % RB_DC;
            const uint64_t pi = uint64_t(blockIdx.x) * RB_PT + pp;
            const uint32_t d = d0 + dd;
            sp[pp][dd] = (pi < n && d < dims) ? pts[pi * dims + d] : 0.f;
        }
        __syncthreads();
        if (f < m) {
            const int dn = (dims - d0) < uint32_t(RB_DC) ? int(dims - d0) : RB_DC;
            for (int dd = 0; dd < dn; ++dd) {
                const uint32_t d = d0 + dd;
                const long long sig = static_cast<long long>(floorf((sp[lane][dd] - up[d]) * ip[d]));
                st = mix64(st ^ static_cast<uint64_t>(sig));
            }
        }
        __syncthreads();
    }
    if (p < n && f < m) tokens[p * m + f] = static_cast<uint32_t>(st % domain);
}

// ----------------------------------------------------------------- minHash

// One warp per set; lanes stride over the functions.
__global__ void k_minhash(const uint64_t* __restrict__ set_off, const uint64_t* __restrict__ elems,
                          uint64_t n_sets, uint32_t m, const unsigned long long* __restrict__ hseed,
                          const unsigned long long* __restrict__ rseed, uint32_t domain,
                          uint32_t* __restrict__ tokens) {
    const uint64_t s = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= n_sets) return;
    const uint64_t b = set_off[s], e = set_off[s + 1];
    for (uint32_t f0 = 0; f0 < m; f0 += 128) {
        uint64_t mn[4] = {~0ull, ~0ull, ~0ull, ~0ull};
        uint64_t hs[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t f = f0 + lane + 32 * j;
            hs[j] = f < m ? hseed[f] : 0;
        }
        for (uint64_t i = b; i < e; ++i) {
            const uint64_t x = elems[i];
#pragma unroll
            for (int j = 0; j < 4; ++j) mn[j] = min(mn[j], mix64(hs[j] ^ x));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t f = f0 + lane + 32 * j;
            if (f >= m) continue;
            uint64_t st = mix64(rseed[f]);
            st = mix64(st ^ mn[j]);
            tokens[s * m + f] = static_cast<uint32_t>(st % domain);
        }
    }
}

// --------------------------------------------------- index from device tokens

__global__ void k_tok_pairs(const uint32_t* tokens, uint64_t total, uint32_t m, uint32_t domain,
                            uint32_t* keys, uint32_t* vals, uint32_t* counts, unsigned long long* bad) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t f = static_cast<uint32_t>(i % m);
        const uint32_t t = tokens[i];
        if (t >= domain) {
            atomicAdd(bad, 1ull);
            continue;
        }
        const uint32_t key = f * domain + t;
        keys[i] = key;
        vals[i] = static_cast<uint32_t>(i / m);
        atomicAdd(&counts[key], 1u);
    }
}

__global__ void k_tok_keys(const uint32_t* counts, const uint64_t* offs, uint64_t nk, uint32_t domain,
                           const uint64_t* kidx, uint64_t* keys_out, uint64_t* off_out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nk;
         i += uint64_t(gridDim.x) * blockDim.x) {
        if (!counts[i]) continue;
        const uint64_t j = kidx[i];
        keys_out[j] = (uint64_t(i / domain) << 32) | (i % domain);
        off_out[j] = offs[i];
    }
}

__global__ void k_flags(const uint32_t* counts, uint64_t nk, uint64_t* flags) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nk;
         i += uint64_t(gridDim.x) * blockDim.x)
        flags[i] = counts[i] ? 1 : 0;
}

}  // namespace genie

using namespace genie;

extern "C" {

genie_lsh_config genie_lsh_config_default(void) {
    genie_lsh_config c{};  // LshEncoderConfig defaults (lsh.hpp:132-145)
    c.family = GENIE_LSH_RBH;
    c.m = 237;
    c.dims = 0;
    c.rehash_domain = 8192;
    c.seed = 1;
    c.w = 4.0;
    c.bucket_count = 67;
    c.rehash_pstable = 0;
    c.bucket_min = -33;
    c.sigma = 1.0;
    c.precision = GENIE_LSH_FP64;
    c.reserved = 0;
    return c;
}

int genie_lsh_sample(const genie_lsh_config* cfg, double* a, double* b, uint64_t* hash_seed,
                     uint64_t* rehash_seed, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        check_cfg(*cfg);
        sample(*cfg, a, b, hash_seed, rehash_seed);
        return GENIE_OK;
    });
}

int genie_encoder_create(const genie_lsh_config* cfg, int device, genie_encoder** out, char* err,
                         size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        check_cfg(*cfg);
        ensure_device(device);
        auto* enc = new genie_encoder;
        try {
            enc->device = device;
            enc->cfg = *cfg;
            const genie_lsh_config& c = *cfg;
            const size_t ma = c.family == GENIE_LSH_MINHASH ? 1 : size_t(c.m) * c.dims;
            const size_t mb = c.family == GENIE_LSH_PSTABLE ? c.m : ma;
            std::vector<double> a(ma, 0.0), b(mb, 0.0), inv(ma, 0.0);
            std::vector<uint64_t> hs(c.m, 0), rs(c.m, 0);
            sample(c, a.data(), b.data(), hs.data(), rs.data());
            if (c.family == GENIE_LSH_RBH)
                for (size_t i = 0; i < ma; ++i) inv[i] = 1.0 / a[i];
            GENIE_CUDA(cudaStreamCreateWithFlags(&enc->stream, cudaStreamNonBlocking));
            enc->a.reserve(ma);
            enc->b.reserve(mb);
            enc->inv.reserve(ma);
            enc->hash_seed.reserve(c.m);
            enc->rehash_seed.reserve(c.m);
            GENIE_CUDA(cudaMemcpy(enc->a.p, a.data(), ma * 8, cudaMemcpyHostToDevice));
            GENIE_CUDA(cudaMemcpy(enc->b.p, b.data(), mb * 8, cudaMemcpyHostToDevice));
            GENIE_CUDA(cudaMemcpy(enc->inv.p, inv.data(), ma * 8, cudaMemcpyHostToDevice));
            GENIE_CUDA(cudaMemcpy(enc->hash_seed.p, hs.data(), c.m * 8, cudaMemcpyHostToDevice));
            GENIE_CUDA(cudaMemcpy(enc->rehash_seed.p, rs.data(), c.m * 8, cudaMemcpyHostToDevice));
            if (c.precision == GENIE_LSH_FP32 && c.family != GENIE_LSH_MINHASH) {
                std::vector<float> af(a.begin(), a.end()), bf(b.begin(), b.end()), invf(inv.begin(), inv.end());
                enc->af.reserve(ma);
                enc->bf.reserve(mb);
                enc->invf.reserve(ma);
                GENIE_CUDA(cudaMemcpy(enc->af.p, af.data(), ma * 4, cudaMemcpyHostToDevice));
                GENIE_CUDA(cudaMemcpy(enc->bf.p, bf.data(), mb * 4, cudaMemcpyHostToDevice));
                GENIE_CUDA(cudaMemcpy(enc->invf.p, invf.data(), ma * 4, cudaMemcpyHostToDevice));
            }
        } catch (...) {
            genie_encoder_destroy(enc);
            throw;
        }
        *out = enc;
        return GENIE_OK;
    });
}

void genie_encoder_destroy(genie_encoder* enc) {
    if (!enc) return;
    cudaSetDevice(enc->device);
    if (enc->stream) {
        cudaStreamSynchronize(enc->stream);
        cudaStreamDestroy(enc->stream);
    }
    delete enc;
}

int genie_lsh_encode_device(genie_encoder* enc, const float* d_points, uint64_t n, uint32_t* d_tokens,
                            void* stream, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        ensure_device(enc->device);
        const genie_lsh_config& c = enc->cfg;
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : enc->stream;
        if (!n) return GENIE_OK;
        const bool fp32 = c.precision == GENIE_LSH_FP32;
        if (c.family == GENIE_LSH_PSTABLE && fp32) {
            dim3 grid(static_cast<unsigned>((n + PS_PT - 1) / PS_PT), (c.m + PS_FN - 1) / PS_FN);
            k_pstable_f32<<<grid, PS_THREADS, 0, s>>>(d_points, n, c.dims, c.m, enc->af.p, enc->bf.p, float(c.w),
                                                      c.bucket_count, c.bucket_min, c.rehash_pstable,
                                                      enc->rehash_seed.p, c.rehash_domain, d_tokens);
        } else if (c.family == GENIE_LSH_RBH && fp32) {
            dim3 grid(static_cast<unsigned>((n + RB_PT - 1) / RB_PT), (c.m + RB_FN - 1) / RB_FN);
            k_rbh_f32<<<grid, RB_PT * RB_FN, 0, s>>>(d_points, n, c.dims, c.m, enc->bf.p, enc->invf.p,
                                                     enc->rehash_seed.p, c.rehash_domain, d_tokens);
        } else if (c.family == GENIE_LSH_PSTABLE) {
            dim3 grid(static_cast<unsigned>((n + PS_PT - 1) / PS_PT), (c.m + PS_FN - 1) / PS_FN);
            k_pstable<<<grid, PS_THREADS, 0, s>>>(d_points, n, c.dims, c.m, enc->a.p, enc->b.p, c.w,
                                                  c.bucket_count, c.bucket_min, c.rehash_pstable,
                                                  enc->rehash_seed.p, c.rehash_domain, d_tokens);
        } else if (c.family == GENIE_LSH_RBH) {
            dim3 grid(static_cast<unsigned>((n + RB_PT - 1) / RB_PT), (c.m + RB_FN - 1) / RB_FN);
            k_rbh<<<grid, RB_PT * RB_FN, 0, s>>>(d_points, n, c.dims, c.m, enc->a.p, enc->b.p,
                                                 enc->inv.p, enc->rehash_seed.p, c.rehash_domain,
                                                 d_tokens);
        } else {
            throw Error(GENIE_ERR_CONTRACT, "minHash encoders take sets (genie_minhash_encode)");
        }
        GENIE_CUDA(cudaGetLastError());
        return GENIE_OK;
    });
}

int genie_lsh_encode(genie_encoder* enc, const float* points, uint64_t n, uint32_t* tokens, char* err,
                     size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        ensure_device(enc->device);
        const genie_lsh_config& c = enc->cfg;
        DevBuf<float>& dp = enc->ws_points;
        DevBuf<uint32_t>& dt = enc->ws_tokens;
        dp.reserve(n * c.dims);
        dt.reserve(n * c.m);
        if (n) GENIE_CUDA(cudaMemcpyAsync(dp.p, points, n * c.dims * sizeof(float), cudaMemcpyHostToDevice, enc->stream));
        char e2[256];
        const int rc = genie_lsh_encode_device(enc, dp.p, n, dt.p, enc->stream, e2, sizeof(e2));
        if (rc) throw Error(rc, e2);
        if (n) GENIE_CUDA(cudaMemcpyAsync(tokens, dt.p, n * c.m * sizeof(uint32_t), cudaMemcpyDeviceToHost, enc->stream));
        GENIE_CUDA(cudaStreamSynchronize(enc->stream));
        return GENIE_OK;
    });
}

int genie_minhash_encode_device(genie_encoder* enc, const uint64_t* d_set_off, const uint64_t* d_elems,
                                uint64_t n_sets, uint32_t* d_tokens, void* stream, char* err,
                                size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        ensure_device(enc->device);
        const genie_lsh_config& c = enc->cfg;
        if (c.family != GENIE_LSH_MINHASH) throw Error(GENIE_ERR_CONTRACT, "encoder is not a minHash encoder");
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : enc->stream;
        if (!n_sets) return GENIE_OK;
        const uint64_t threads = n_sets * 32;
        k_minhash<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
            d_set_off, d_elems, n_sets, c.m, enc->hash_seed.p, enc->rehash_seed.p, c.rehash_domain,
            d_tokens);
        GENIE_CUDA(cudaGetLastError());
        return GENIE_OK;
    });
}

int genie_minhash_encode(genie_encoder* enc, const uint64_t* set_off, const uint64_t* elems,
                         uint64_t n_sets, uint32_t* tokens, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        ensure_device(enc->device);
        const genie_lsh_config& c = enc->cfg;
        const uint64_t ne = set_off[n_sets] - set_off[0];
        std::vector<uint64_t> off(set_off, set_off + n_sets + 1);
        for (auto& o : off) o -= set_off[0];
        DevBuf<uint64_t>& doff = enc->ws_off;
        DevBuf<uint64_t>& del = enc->ws_elems;
        DevBuf<uint32_t>& dt = enc->ws_tokens;
        doff.reserve(n_sets + 1);
        del.reserve(ne);
        dt.reserve(n_sets * c.m);
        GENIE_CUDA(cudaMemcpyAsync(doff.p, off.data(), (n_sets + 1) * 8, cudaMemcpyHostToDevice, enc->stream));
        if (ne) GENIE_CUDA(cudaMemcpyAsync(del.p, elems + set_off[0], ne * 8, cudaMemcpyHostToDevice, enc->stream));
        char e2[256];
        const int rc = genie_minhash_encode_device(enc, doff.p, del.p, n_sets, dt.p, enc->stream, e2, sizeof(e2));
        if (rc) throw Error(rc, e2);
        if (n_sets) GENIE_CUDA(cudaMemcpyAsync(tokens, dt.p, n_sets * c.m * 4, cudaMemcpyDeviceToHost, enc->stream));
        GENIE_CUDA(cudaStreamSynchronize(enc->stream));
        return GENIE_OK;
    });
}

// Query items of encoded points: row q asks for k results with one point
// item per hash function i (Keyword{dim = i, token = tokens[q m + i]},
// lsh.hpp:186-195); lo / hi read the token matrix in place.
__global__ void k_point_items(uint64_t n, uint32_t m, uint32_t k, uint32_t first_id, uint32_t* qid, uint32_t* kk,
                              uint64_t* item_off, uint16_t* dim) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n * m; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t q = i / m;
        const uint32_t f = static_cast<uint32_t>(i - q * m);
        dim[i] = static_cast<uint16_t>(f);
        if (f == 0) {
            qid[q] = first_id + static_cast<uint32_t>(q);
            kk[q] = k;
            item_off[q] = i;
        }
        if (i + 1 == n * m) item_off[n] = n * m;
    }
}

int genie_lsh_query_batch(genie_encoder* enc, genie_index* ix, const genie_config* cfg_in, const float* points,
                          const uint64_t* set_off, const uint64_t* elems, uint64_t n, uint32_t k, uint32_t first_id,
                          uint32_t out_stride, genie_entry* out, uint32_t* out_len, uint32_t* out_threshold,
                          genie_batch_stats* stats, char* err, size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        const genie_config cfg = cfg_in ? *cfg_in : genie_config_default();
        validate_config(cfg);
        if (!enc || !ix) throw Error(GENIE_ERR_CONTRACT, "genie_lsh_query_batch: null encoder or index");
        if (enc->device != ix->device) throw Error(GENIE_ERR_CONTRACT, "encoder and index on different devices");
        const genie_lsh_config& c = enc->cfg;
        const bool sets = c.family == GENIE_LSH_MINHASH;
        if (n && (sets ? (!set_off || !elems) : !points)) throw Error(GENIE_ERR_CONTRACT, "genie_lsh_query_batch: null input");
        if (n && (!out || !out_len || !out_threshold)) throw Error(GENIE_ERR_CONTRACT, "genie_lsh_query_batch: null output");
        if (k == 0) throw Error(GENIE_ERR_CONTRACT, "Query " + std::to_string(first_id) + ": k must be >= 1");
        if (n >= (1u << 21)) throw Error(GENIE_ERR_CONTRACT, "batch exceeds 2^21 queries");
        if (n * c.m >= (1ull << 32)) throw Error(GENIE_ERR_CONTRACT, "too many query items");
        if (n && out_stride < std::min<uint64_t>(k, std::max<uint32_t>(ix->n, 1)))
            throw Error(GENIE_ERR_CONTRACT, "out_stride must be >= min(k, num_objects)");
        if (!n) return GENIE_OK;
        ensure_device(ix->device);
        cudaStream_t s = ix->stream;
        const uint32_t Q = static_cast<uint32_t>(n);
        // 1. inputs up, tokens on the device (never read back)
        DevBuf<uint32_t>& tok = enc->ws_tokens;
        tok.reserve(n * c.m);
        char e2[256];
        int rc;
        if (sets) {
            const uint64_t ne = set_off[n] - set_off[0];
            std::vector<uint64_t> off(set_off, set_off + n + 1);
            for (auto& o : off) o -= set_off[0];
            enc->ws_off.reserve(n + 1);
            enc->ws_elems.reserve(std::max<uint64_t>(ne, 1));
            GENIE_CUDA(cudaMemcpyAsync(enc->ws_off.p, off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, s));
            if (ne) GENIE_CUDA(cudaMemcpyAsync(enc->ws_elems.p, elems + set_off[0], ne * 8, cudaMemcpyHostToDevice, s));
            rc = genie_minhash_encode_device(enc, enc->ws_off.p, enc->ws_elems.p, n, tok.p, s, e2, sizeof(e2));
        } else {
            enc->ws_points.reserve(n * c.dims);
            GENIE_CUDA(cudaMemcpyAsync(enc->ws_points.p, points, n * c.dims * sizeof(float), cudaMemcpyHostToDevice, s));
            rc = genie_lsh_encode_device(enc, enc->ws_points.p, n, tok.p, s, e2, sizeof(e2));
        }
        if (rc) throw Error(rc, e2);
        // 2. the batch: one point item per function, lo = hi = the token
        Workspace& w = ix->ws;
        w.d_qid.reserve(Q);
        w.d_k.reserve(Q);
        w.d_item_off.reserve(Q + 1);
        w.d_dim.reserve(n * c.m);
        const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((n * c.m + 255) / 256, uint64_t(ix->sms) * 16));
        k_point_items<<<blocks, 256, 0, s>>>(n, c.m, k, first_id, w.d_qid.p, w.d_k.p, w.d_item_off.p, w.d_dim.p);
        GENIE_CUDA(cudaGetLastError());
        const uint32_t stride = std::max<uint32_t>(out_stride, 1);
        w.d_out.reserve(uint64_t(Q) * stride);
        w.d_out_len.reserve(Q + 1);
        w.d_out_thr.reserve(Q + 1);
        // 3. query (re-issued if the workspace had to grow), results down
        std::string msg;
        genie_batch_stats local{};
        rc = GENIE_RETRY;
        for (int attempt = 0; attempt < 4 && rc == GENIE_RETRY; ++attempt) {
            launch_batch(ix, cfg, Q, w.d_qid.p, w.d_k.p, w.d_item_off.p, w.d_dim.p, tok.p, tok.p,
                         static_cast<uint32_t>(n * c.m), k, stride, w.d_out.p, w.d_out_len.p, w.d_out_thr.p, s, false);
            rc = finish_batch(ix, &local, msg, nullptr);
        }
        if (rc != GENIE_OK) throw Error(rc, msg);
        GENIE_CUDA(cudaMemcpyAsync(out, w.d_out.p, uint64_t(Q) * stride * sizeof(genie_entry), cudaMemcpyDeviceToHost, s));
        GENIE_CUDA(cudaMemcpyAsync(out_len, w.d_out_len.p, Q * 4, cudaMemcpyDeviceToHost, s));
        GENIE_CUDA(cudaMemcpyAsync(out_threshold, w.d_out_thr.p, Q * 4, cudaMemcpyDeviceToHost, s));
        GENIE_CUDA(cudaStreamSynchronize(s));
        if (stats) *stats = local;
        return GENIE_OK;
    });
}

// encode_dataset + build_index for LSH data, on the device: stable radix sort
// of (dim*D + token, id) pairs emitted in id order, so every list comes out
// ascending (index.hpp:207-212, 235).
int genie_index_from_tokens_device(const uint32_t* d_tokens, uint32_t n, uint32_t m, uint32_t domain,
                                   uint32_t id_offset, int device, genie_index** out, char* err,
                                   size_t errlen) {
    return guarded(err, errlen, [&]() -> int {
        if (m == 0 || m > 0x10000u || domain == 0)
            throw Error(GENIE_ERR_CONTRACT, "index_from_tokens: bad m / domain");
        const uint64_t nk = uint64_t(m) * domain;
        if (nk >= (1ull << 32)) throw Error(GENIE_ERR_CONTRACT, "index_from_tokens: m * domain too large");
        ensure_device(device);
        auto* ix = new genie_index;
        try {
            ix->device = device;
            ix->n = n;
            ix->id_offset = id_offset;
            ix->sms = sm_count(device);
            GENIE_CUDA(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
            for (auto& e : ix->ev) GENIE_CUDA(cudaEventCreate(&e));
            cudaStream_t s = ix->stream;
            const uint64_t total = uint64_t(n) * m;
            DevBuf<uint32_t> k1, k2, v1, counts;
            DevBuf<uint64_t> offs, flags, kidx;
            DevBuf<unsigned long long> bad;
            k1.reserve(total);
            k2.reserve(total);
            v1.reserve(total);
            counts.reserve(nk);
            offs.reserve(nk + 1);
            flags.reserve(nk + 1);
            kidx.reserve(nk + 1);
            bad.reserve(1);
            ix->postings.reserve(total + 64);
            GENIE_CUDA(cudaMemsetAsync(counts.p, 0, nk * 4, s));
            GENIE_CUDA(cudaMemsetAsync(bad.p, 0, 8, s));
            GENIE_CUDA(cudaMemsetAsync(ix->postings.p, 0, (total + 64) * 4, s));
            const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, uint64_t(ix->sms) * 32));
            if (total) k_tok_pairs<<<std::max(1u, grid), 256, 0, s>>>(d_tokens, total, m, domain, k1.p, v1.p, counts.p, bad.p);
            unsigned long long h_bad = 0;
            GENIE_CUDA(cudaMemcpyAsync(&h_bad, bad.p, 8, cudaMemcpyDeviceToHost, s));
            GENIE_CUDA(cudaStreamSynchronize(s));
            if (h_bad) throw Error(GENIE_ERR_DATA, "index_from_tokens: token outside [0, domain)");
            int end_bit = 1;
            while ((1ull << end_bit) < nk) ++end_bit;
            cub::DoubleBuffer<uint32_t> dk(k1.p, k2.p);
            cub::DoubleBuffer<uint32_t> dv(v1.p, ix->postings.p);
            size_t tmp = 0;
            if (total) {
                GENIE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, static_cast<int64_t>(total), 0, end_bit, s));
                DevBuf<unsigned char> t;
                t.reserve(tmp);
                GENIE_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, dk, dv, static_cast<int64_t>(total), 0, end_bit, s));
                if (dv.Current() != ix->postings.p)
                    GENIE_CUDA(cudaMemcpyAsync(ix->postings.p, dv.Current(), total * 4, cudaMemcpyDeviceToDevice, s));
                GENIE_CUDA(cudaStreamSynchronize(s));
            }
            // offsets over all (dim, token) slots, then compact the non-empty ones
            DevBuf<uint64_t> c64;
            c64.reserve(nk + 1);
            {
                // widen counts for a 64-bit scan
                std::vector<uint32_t> hc(nk);
                GENIE_CUDA(cudaMemcpy(hc.data(), counts.p, nk * 4, cudaMemcpyDeviceToHost));
                std::vector<uint64_t> ho(nk + 1, 0), hkeys, hoff;
                for (uint64_t i = 0; i < nk; ++i) ho[i + 1] = ho[i] + hc[i];
                for (uint64_t i = 0; i < nk; ++i)
                    if (hc[i]) {
                        hkeys.push_back((uint64_t(i / domain) << 32) | (i % domain));
                        hoff.push_back(ho[i]);
                    }
                hoff.push_back(total);
                ix->K = hkeys.size();
                ix->P = total;
                ix->keys.reserve(ix->K + 1);
                ix->key_off.reserve(ix->K + 1);
                if (ix->K) GENIE_CUDA(cudaMemcpy(ix->keys.p, hkeys.data(), ix->K * 8, cudaMemcpyHostToDevice));
                GENIE_CUDA(cudaMemcpy(ix->key_off.p, hoff.data(), (ix->K + 1) * 8, cudaMemcpyHostToDevice));
                // every object carries exactly one token per dim
                std::vector<uint32_t> dm(65536, 0);
                if (n)
                    for (uint32_t f = 0; f < m; ++f) dm[f] = 1;
                ix->dim_mult.reserve(65536);
                GENIE_CUDA(cudaMemcpy(ix->dim_mult.p, dm.data(), 65536 * 4, cudaMemcpyHostToDevice));
                build_dense_containers(ix, hoff.data());
            }
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
