// rng.cu -- the libstdc++ Gaussian stream of randsvd, generated on the GPU.
//
// The reference draws every Gaussian test matrix from one
// std::mt19937_64(seed) + std::normal_distribution<double> pair per randsvd
// call, filled column-major (lowrank.cpp:136-143).  libstdc++ 13 implements
//   u      = double(engine()) / 2^64             (generate_canonical, 1 call)
//   x, y   = 2u1 - 1, 2u2 - 1;  r2 = x*x + y*y  (reject r2 > 1 or r2 == 0)
//   mult   = sqrt(-2 log(r2) / r2);  return y*mult, cache x*mult
// (random.tcc: normal_distribution::operator(), generate_canonical).
//
// GPU design (no sequential 312-word engine walk):
//  * z_k (k >= 0) is the untempered MT19937-64 word sequence (z_0..z_311 the
//    seeded state; output q = temper(z_{312+q})).  Every bit sequence of z
//    obeys the characteristic polynomial phi (deg 19937), found once on the
//    host by Berlekamp-Massey.  For chunk c the window z_{cS..cS+311} is
//    sum_i g_c[i] z_{i..i+311} with g_c = x^{cS} mod phi (GF(2)), so every
//    chunk of S outputs is generated independently by its own CTA (jump-ahead).
//  * Polar rejection pairs never straddle chunks (S even); per-chunk accept
//    counts are prefix-summed, then every accepted pair writes its two
//    deviates at their global stream index -- exactly the column-major Omega
//    of the reference.
//  * The rejection test and mult use round-to-nearest intrinsics
//    (__dmul_rn / __dadd_rn / __ddiv_rn / __dsqrt_rn): no FMA contraction, so
//    accept decisions are bitwise those of the host build; log() may differ
//    from glibc by <= 1 ulp (deviates within a few ulp).
#include <immintrin.h>

#include <cmath>
#include <mutex>

#include "internal.h"

namespace hydot {

namespace mt {
constexpr int NW = 312, MW = 156;
constexpr uint64_t A = 0xB5026F5AA96619E9ULL;
constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
constexpr uint64_t F = 6364136223846793005ULL;
constexpr int L = 19937;              // degree of phi
constexpr int PW = (L + 63) / 64;     // words per polynomial (312)
constexpr int64_t S = 312LL * 1024;   // outputs per chunk (even; one jump per chunk)
constexpr int PREFIX = 312 * 65;      // z_0 .. z_{20279} >= L + 311

__host__ __device__ inline uint64_t mix(uint64_t a, uint64_t b) {
    uint64_t y = (a & UM) | (b & LM);
    return (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
}
__host__ __device__ inline uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}
}  // namespace mt

// ============================================================ host side ====
namespace {

using Poly = std::vector<uint64_t>;

inline int get_bit(const Poly& p, int64_t i) { return int((p[size_t(i >> 6)] >> (i & 63)) & 1ULL); }
inline void flip_bit(Poly& p, int64_t i) { p[size_t(i >> 6)] ^= 1ULL << (i & 63); }

// z sequence on the host (untempered), seeded as std::mt19937_64(seed)
std::vector<uint64_t> host_z(uint64_t seed, int64_t count) {
    std::vector<uint64_t> z(static_cast<size_t>(std::max<int64_t>(count, mt::NW)));
    z[0] = seed;
    for (int i = 1; i < mt::NW; ++i) z[size_t(i)] = mt::F * (z[size_t(i - 1)] ^ (z[size_t(i - 1)] >> 62)) + uint64_t(i);
    for (int64_t k = mt::NW; k < count; ++k)
        z[size_t(k)] = z[size_t(k - mt::MW)] ^ mt::mix(z[size_t(k - mt::NW)], z[size_t(k - mt::NW + 1)]);
    return z;
}

// bits [off, off+64) of bitset R (zero beyond the end)
inline uint64_t window64(const Poly& R, int64_t off) {
    int64_t w = off >> 6;
    int b = int(off & 63);
    uint64_t lo = w < int64_t(R.size()) ? R[size_t(w)] : 0ULL;
    uint64_t hi = (w + 1) < int64_t(R.size()) ? R[size_t(w + 1)] : 0ULL;
    return b ? ((lo >> b) | (hi << (64 - b))) : lo;
}

// Berlekamp-Massey over GF(2) on the bit sequence s_k = LSB(z_{k+1});
// returns phi with phi_i = C_{L-i} (monic, degree L).
Poly berlekamp_massey_phi() {
    const int64_t n = 2 * int64_t(mt::L) + 64;
    std::vector<uint64_t> z = host_z(5489ULL, n + 2);
    const size_t W = size_t((n + 63) / 64 + 2);
    Poly R(W, 0);  // reversed sequence: bit (n-1-k) = s_k
    for (int64_t k = 0; k < n; ++k)
        if (z[size_t(k + 1)] & 1ULL) flip_bit(R, n - 1 - k);
    Poly C(W, 0), B(W, 0), T;
    C[0] = 1;
    B[0] = 1;
    int64_t Ldeg = 0, m = 1;
    for (int64_t k = 0; k < n; ++k) {
        // d = sum_{i=0..L} C_i s_{k-i}; s_{k-i} = bit (n-1-k+i) of R
        const int64_t off = n - 1 - k;
        const int64_t nw = Ldeg / 64 + 1;
        uint64_t acc = 0;
        for (int64_t w = 0; w < nw; ++w) {
            uint64_t cw = C[size_t(w)];
            if (w == nw - 1) {
                int keep = int(Ldeg - 64 * w) + 1;
                if (keep < 64) cw &= (1ULL << keep) - 1;
            }
            acc ^= cw & window64(R, off + 64 * w);
        }
        int d = __builtin_parityll(acc);
        if (d == 0) {
            ++m;
            continue;
        }
        T = C;
        const int64_t ws = m >> 6;
        const int bs = int(m & 63);
        for (int64_t w = int64_t(W) - 1; w >= ws; --w) {
            uint64_t lo = B[size_t(w - ws)];
            uint64_t v = lo << bs;
            if (bs && w - ws - 1 >= 0) v |= B[size_t(w - ws - 1)] >> (64 - bs);
            C[size_t(w)] ^= v;
        }
        if (2 * Ldeg <= k) {
            Ldeg = k + 1 - Ldeg;
            B = T;
            m = 1;
        } else {
            ++m;
        }
    }
    if (Ldeg != mt::L) throw std::runtime_error("MT19937-64 characteristic polynomial degree mismatch");
    Poly phi(size_t(mt::PW) + 1, 0);
    for (int64_t i = 0; i <= mt::L; ++i)
        if (get_bit(C, mt::L - i)) flip_bit(phi, i);
    return phi;
}

inline __m128i clmul(uint64_t a, uint64_t b) {
    return _mm_clmulepi64_si128(_mm_set_epi64x(0, int64_t(a)), _mm_set_epi64x(0, int64_t(b)), 0);
}

struct PolyMod {
    Poly phi;   // PW+1 words, degree L
    uint64_t ft;  // coefficients of degrees L-64 .. L-1

    explicit PolyMod(Poly p) : phi(std::move(p)) {
        ft = 0;
        for (int k = 0; k < 64; ++k)
            if (get_bit(phi, mt::L - 64 + k)) ft |= 1ULL << k;
    }

    // P (any length, degree < 2L) reduced mod phi -> PW words
    Poly reduce(Poly P) const {
        int64_t hi = int64_t(P.size()) * 64 - 1;
        while (hi >= mt::L) {
            int64_t lo = std::max<int64_t>(mt::L, hi - 63);
            int width = int(hi - lo + 1);
            // window bits [lo, lo+width)
            uint64_t w = window64(P, lo);
            if (width < 64) w &= (1ULL << width) - 1;
            if (!w) {
                hi = lo - 1;
                continue;
            }
            uint64_t q = 0;
            for (int b = width - 1; b >= 0; --b) {
                if ((w >> b) & 1ULL) {
                    q |= 1ULL << b;
                    w ^= (1ULL << b) ^ (b ? (ft >> (64 - b)) : 0ULL);
                }
            }
            if (q) {
                // P ^= (q * phi) << (lo - L)
                int64_t sh = lo - mt::L;
                int64_t ws = sh >> 6;
                int bs = int(sh & 63);
                for (size_t i = 0; i < phi.size(); ++i) {
                    __m128i pr = clmul(q, phi[i]);
                    uint64_t p0 = uint64_t(_mm_cvtsi128_si64(pr));
                    uint64_t p1 = uint64_t(_mm_extract_epi64(pr, 1));
                    // 128-bit value at word offset i, shifted by bs
                    uint64_t w0 = p0 << bs;
                    uint64_t w1 = bs ? ((p1 << bs) | (p0 >> (64 - bs))) : p1;
                    uint64_t w2 = bs ? (p1 >> (64 - bs)) : 0;
                    size_t o = size_t(ws) + i;
                    if (o < P.size()) P[o] ^= w0;
                    if (o + 1 < P.size()) P[o + 1] ^= w1;
                    if (o + 2 < P.size()) P[o + 2] ^= w2;
                }
            }
            hi = lo - 1;
        }
        P.resize(size_t(mt::PW));
        // clear bits >= L in the last word
        int rem = mt::L - (mt::PW - 1) * 64;
        P[size_t(mt::PW - 1)] &= (rem == 64) ? ~0ULL : ((1ULL << rem) - 1);
        return P;
    }

    Poly mulmod(const Poly& a, const Poly& b) const {
        Poly P(size_t(2 * mt::PW + 2), 0);
        for (int i = 0; i < mt::PW; ++i) {
            if (!a[size_t(i)]) continue;
            for (int j = 0; j < mt::PW; ++j) {
                __m128i pr = clmul(a[size_t(i)], b[size_t(j)]);
                P[size_t(i + j)] ^= uint64_t(_mm_cvtsi128_si64(pr));
                P[size_t(i + j + 1)] ^= uint64_t(_mm_extract_epi64(pr, 1));
            }
        }
        return reduce(std::move(P));
    }

    Poly xpow(uint64_t e) const {  // x^e mod phi
        Poly r(size_t(mt::PW), 0), base(size_t(mt::PW), 0);
        r[0] = 1;
        base[0] = 2;  // x
        while (e) {
            if (e & 1) r = mulmod(r, base);
            e >>= 1;
            if (e) base = mulmod(base, base);
        }
        return r;
    }
};

// process-wide jump table: g_c = x^{cS} mod phi, c = 0, 1, 2, ...
struct JumpTable {
    std::mutex mu;
    std::unique_ptr<PolyMod> pm;
    Poly g1;
    std::vector<Poly> g;  // g[c]
    const Poly& get(int64_t c) {
        std::lock_guard<std::mutex> lk(mu);
        if (!pm) {
            pm.reset(new PolyMod(berlekamp_massey_phi()));
            g1 = pm->xpow(uint64_t(mt::S));
            Poly one(size_t(mt::PW), 0);
            one[0] = 1;
            g.push_back(one);
        }
        while (int64_t(g.size()) <= c) g.push_back(pm->mulmod(g.back(), g1));
        return g[size_t(c)];
    }
};
JumpTable& jump_table() {
    static JumpTable t;
    return t;
}

}  // namespace

bool rng_selftest_host() {
    // windows of chunk 1 and 2 from the jump polynomials vs sequential z
    const uint64_t seed = 20240811ULL;
    std::vector<uint64_t> z = host_z(seed, 2 * mt::S + mt::PREFIX);
    for (int c = 1; c <= 2; ++c) {
        const Poly& g = jump_table().get(c);
        for (int j = 0; j < mt::NW; ++j) {
            uint64_t acc = 0;
            for (int64_t i = 0; i < mt::L; ++i)
                if (get_bit(g, i)) acc ^= z[size_t(i + j)];
            uint64_t want = z[size_t(c * mt::S + j)];
            if (j == 0) {
                acc &= mt::UM;
                want &= mt::UM;
            }
            if (acc != want) return false;
        }
    }
    return true;
}

// ========================================================== device side ====
namespace {

// seeded state + twist to PREFIX words; one CTA, smem holds all of z
__global__ void rng_prefix_k(uint64_t seed, uint64_t* __restrict__ zout) {
    extern __shared__ uint64_t z[];
    if (threadIdx.x == 0) {
        uint64_t x = seed;
        z[0] = x;
        for (int i = 1; i < mt::NW; ++i) {
            x = mt::F * (x ^ (x >> 62)) + uint64_t(i);
            z[i] = x;
        }
    }
    __syncthreads();
    for (int base = 0; base + 2 * mt::NW <= mt::PREFIX; base += mt::NW) {
        int i = threadIdx.x;
        if (i < mt::MW) z[base + mt::NW + i] = z[base + i + mt::MW] ^ mt::mix(z[base + i], z[base + i + 1]);
        __syncthreads();
        if (i < mt::MW) {
            int k = base + mt::MW + i;
            z[k + mt::NW] = z[k + mt::MW] ^ mt::mix(z[k], z[k + 1]);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < mt::PREFIX; i += blockDim.x) zout[i] = z[i];
}

// window of chunk c: w[j] = xor_{i : g_c[i]} z[i+j].  Branch-free GF(2)
// product: thread (chunk, jj) owns w[4jj .. 4jj+3]; for every 64-bit word of
// g_c it walks the 67 words z[64w + 4jj + b] once and applies all 64 bits as
// masks to the 4 accumulators (no data-dependent loop, 4x reuse of each
// shared-memory load).  One CTA serves JCH chunks from the same prefix.
constexpr int JK = 4;                 // window words per thread
constexpr int JPC = mt::NW / JK;      // threads per chunk (78)
constexpr int JCH = 4;                // chunks per CTA
__global__ void __launch_bounds__(JPC * JCH) rng_jump_k(const uint64_t* __restrict__ zpre,
                                                        const uint64_t* __restrict__ gtab, int64_t c0,
                                                        int64_t nc, uint64_t* __restrict__ windows) {
    extern __shared__ uint64_t z[];
    for (int i = threadIdx.x; i < mt::PREFIX; i += blockDim.x) z[i] = zpre[i];
    __syncthreads();
    const int lc = threadIdx.x / JPC, jj = threadIdx.x % JPC;
    const int64_t ci = int64_t(blockIdx.x) * JCH + lc;  // chunk index within this call
    if (ci >= nc) return;
    const uint64_t* g = gtab + (c0 + ci) * mt::PW;
    const int j0 = jj * JK;
    uint64_t acc[JK] = {0, 0, 0, 0};
    for (int w = 0; w < mt::PW; ++w) {
        const uint64_t bits = __ldg(g + w);
        if (bits == 0) continue;
        const uint64_t* zp = z + 64 * w + j0;
#pragma unroll 16
        for (int b = 0; b < 64; ++b) {
            const uint64_t m = 0ULL - ((bits >> b) & 1ULL);
#pragma unroll
            for (int t = 0; t < JK; ++t) acc[t] ^= zp[b + t] & m;
        }
    }
#pragma unroll
    for (int t = 0; t < JK; ++t) windows[ci * mt::NW + j0 + t] = acc[t];
}

__device__ __forceinline__ bool polar_accept(uint64_t r1, uint64_t r2, double& x, double& y,
                                             double& rr) {
    const double inv = 5.421010862427522e-20;  // 2^-64
    double u1 = __dmul_rn(__ull2double_rn(r1), inv);
    double u2 = __dmul_rn(__ull2double_rn(r2), inv);
    if (u1 >= 1.0) u1 = 0.99999999999999989;  // nextafter(1, 0)
    if (u2 >= 1.0) u2 = 0.99999999999999989;
    x = __dsub_rn(__dmul_rn(2.0, u1), 1.0);
    y = __dsub_rn(__dmul_rn(2.0, u2), 1.0);
    rr = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    return !(rr > 1.0 || rr == 0.0);
}

// one CTA per chunk: run S outputs from the window, write tempered raw
// words, count accepted polar attempts.
__global__ void __launch_bounds__(160) rng_generate_k(const uint64_t* __restrict__ windows,
                                                      uint64_t* __restrict__ raw,
                                                      int* __restrict__ counts) {
    __shared__ uint64_t buf[2][mt::NW + 1];
    __shared__ int wcount[8];
    const int i = threadIdx.x;
    const uint64_t* win = windows + int64_t(blockIdx.x) * mt::NW;
    for (int k = i; k < mt::NW; k += blockDim.x) buf[0][k] = win[k];
    __syncthreads();
    uint64_t* out = raw + int64_t(blockIdx.x) * mt::S;
    int cnt = 0;
    int cur = 0;
    for (int blk = 0; blk < int(mt::S / mt::NW); ++blk) {
        uint64_t* o = buf[cur];
        uint64_t* n = buf[cur ^ 1];
        if (i < mt::MW) n[i] = o[i + mt::MW] ^ mt::mix(o[i], o[i + 1]);
        __syncthreads();
        if (i < mt::MW) {
            int k = mt::MW + i;
            uint64_t nxt = (k + 1 < mt::NW) ? o[k + 1] : n[0];
            n[k] = n[i] ^ mt::mix(o[k], nxt);
        }
        __syncthreads();
        if (i < mt::MW) {
            uint64_t a = mt::temper(n[2 * i]), b = mt::temper(n[2 * i + 1]);
            out[int64_t(blk) * mt::NW + 2 * i] = a;
            out[int64_t(blk) * mt::NW + 2 * i + 1] = b;
            double x, y, rr;
            cnt += polar_accept(a, b, x, y, rr) ? 1 : 0;
        }
        cur ^= 1;
        // next iteration reads buf[cur] (just written) and overwrites the
        // other one, which everybody finished reading before the 2nd sync.
    }
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, off);
    if ((i & 31) == 0) wcount[i >> 5] = cnt;
    __syncthreads();
    if (i == 0) {
        int t = 0;
        for (int w = 0; w < int(blockDim.x + 31) / 32; ++w) t += wcount[w];
        counts[blockIdx.x] = t;
    }
}

// one CTA per chunk: stream-compact accepted attempts into deviates
__global__ void __launch_bounds__(256) rng_normals_k(const uint64_t* __restrict__ raw,
                                                     const int64_t* __restrict__ offsets,
                                                     double* __restrict__ out) {
    __shared__ int wsum[8];
    const uint64_t* r = raw + int64_t(blockIdx.x) * mt::S;
    int64_t pos = offsets[blockIdx.x];  // accepted attempts before this chunk
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t a0 = 0; a0 < mt::S / 2; a0 += blockDim.x) {
        int64_t a = a0 + threadIdx.x;
        bool ok = false;
        double x = 0, y = 0, rr = 0;
        if (a < mt::S / 2) ok = polar_accept(r[2 * a], r[2 * a + 1], x, y, rr);
        unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < 8; ++w) {
            if (w < warp) before += wsum[w];
            total += wsum[w];
        }
        if (ok) {
            int64_t k = pos + before + __popc(bal & ((1u << lane) - 1u));
            double mult = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(rr)), rr));
            out[2 * k] = __dmul_rn(y, mult);
            out[2 * k + 1] = __dmul_rn(x, mult);
        }
        pos += total;
        __syncthreads();
    }
}

// Chunk offsets without a host round trip: one CTA scans the accepted-pair
// counts of this batch of chunks after the running total of the stream
// (device-resident), writes each chunk's first pair index and advances the
// total.  The host only keeps a lower bound of the total (10 sigma below the
// binomial mean); a batch that falls short of it, or overflows the buffer
// sized 10 sigma above, is impossible in practice and traps.
__global__ void __launch_bounds__(1024) rng_scan_k(const int* __restrict__ counts, int nc,
                                                   int64_t* __restrict__ total, int64_t* __restrict__ offs,
                                                   int64_t lower_pairs, int64_t cap_pairs) {
    __shared__ int64_t wsum[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = *total;
    __syncthreads();
    for (int b0 = 0; b0 < nc; b0 += blockDim.x) {
        const int k = b0 + threadIdx.x;
        int64_t v = k < nc ? counts[k] : 0;
        // inclusive warp scan, then across warps
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (lane == 31) wsum[warp] = v;
        __syncthreads();
        if (warp == 0) {
            int64_t w = lane < int(blockDim.x >> 5) ? wsum[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t u = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += u;
            }
            wsum[lane] = w;
        }
        __syncthreads();
        const int64_t incl = v + (warp > 0 ? wsum[warp - 1] : 0);
        const int64_t excl = incl - (k < nc ? counts[k] : 0);
        if (k < nc) offs[k] = carry + excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (carry < lower_pairs || carry > cap_pairs) __trap();  // > 10 sigma off the binomial mean
        *total = carry;
    }
}

// per-ctx device copy of the jump table (grown on demand)
const uint64_t* device_jumps(Ctx& c, int64_t upto) {
    if (c.jump_n < upto) {
        int64_t want = std::max<int64_t>(upto, c.jump_n * 2);
        std::vector<uint64_t> host(static_cast<size_t>(want * mt::PW));
        for (int64_t k = 0; k < want; ++k) {
            const Poly& g = jump_table().get(k);
            std::copy(g.begin(), g.end(), host.begin() + k * mt::PW);
        }
        uint64_t* nb = nullptr;
        HYDOT_CUDA(cudaMalloc(&nb, host.size() * 8));
        HYDOT_CUDA(cudaMemcpyAsync(nb, host.data(), host.size() * 8, cudaMemcpyHostToDevice,
                                   c.stream));
        c.sync();
        if (c.jump_dev) HYDOT_CUDA(cudaFree(c.jump_dev));
        c.jump_dev = nb;
        c.jump_n = want;
    }
    return c.jump_dev;
}

}  // namespace

RngStream::RngStream(Ctx& c, uint64_t seed) : c_(c), seed_(seed) {
    prefix_.alloc(c, size_t(mt::PREFIX) * 8);
    static AttrGate attr;
    attr_once(attr, c.device, [&] {
        HYDOT_CUDA(cudaFuncSetAttribute(rng_prefix_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        mt::PREFIX * 8));
        HYDOT_CUDA(cudaFuncSetAttribute(rng_jump_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        mt::PREFIX * 8));
    });
    rng_prefix_k<<<1, 160, size_t(mt::PREFIX) * 8, c.stream>>>(seed, prefix_.as<uint64_t>());
    c.check_launch();
}

RngStream::~RngStream() = default;

// accepted polar pairs per chunk: S/2 attempts, p = pi/4; the host keeps
// the mean - 10 sigma lower bound, buffers are sized mean + 10 sigma
namespace {
constexpr double kPairs = double(mt::S / 2) * 0.7853981633974483;
inline double pairs_sigma(int64_t nc) {
    return std::sqrt(double(nc) * double(mt::S / 2) * 0.7853981633974483 * (1.0 - 0.7853981633974483));
}
}  // namespace

void RngStream::generate_chunks(int64_t c_end) {
    const int64_t c0 = n_chunks_;
    const int64_t nc = c_end - c0;
    if (nc <= 0) return;
    const uint64_t* jumps = device_jumps(c_, c_end);
    DBuf windows(c_, size_t(nc) * mt::NW * 8);
    DBuf raw(c_, size_t(nc) * size_t(mt::S) * 8);
    DBuf counts(c_, size_t(nc) * sizeof(int));
    DBuf offs(c_, size_t(nc) * sizeof(int64_t));
    if (!total_.bytes()) {
        total_ = DBuf(c_, sizeof(int64_t));
        HYDOT_CUDA(cudaMemsetAsync(total_.as<void>(), 0, sizeof(int64_t), c_.stream));
    }
    rng_jump_k<<<unsigned((nc + JCH - 1) / JCH), JPC * JCH, size_t(mt::PREFIX) * 8, c_.stream>>>(
        prefix_.as<uint64_t>(), jumps, c0, nc, windows.as<uint64_t>());
    c_.check_launch();
    rng_generate_k<<<unsigned(nc), 160, 0, c_.stream>>>(windows.as<uint64_t>(), raw.as<uint64_t>(),
                                                        counts.as<int>());
    c_.check_launch();
    // pair totals after all c_end chunks: lower bound kept on the host, the
    // buffer sized for the upper bound
    const double sd = pairs_sigma(c_end);
    const int64_t lower = int64_t(std::floor(double(c_end) * kPairs - 10.0 * sd));
    const int64_t upper = int64_t(std::ceil(double(c_end) * kPairs + 10.0 * sd));
    rng_scan_k<<<1, 1024, 0, c_.stream>>>(counts.as<int>(), int(nc), total_.as<int64_t>(), offs.as<int64_t>(),
                                          std::max<int64_t>(lower, 0), upper);
    c_.check_launch();
    const int64_t cap = 2 * upper;  // normals
    if (int64_t(normals_.bytes() / 8) < cap) {
        DBuf nb(c_, size_t(std::max<int64_t>(cap, int64_t(normals_.bytes() / 8) * 3 / 2)) * 8);
        if (normals_.bytes())
            HYDOT_CUDA(cudaMemcpyAsync(nb.as<void>(), normals_.as<void>(), normals_.bytes(), cudaMemcpyDeviceToDevice,
                                       c_.stream));
        normals_ = std::move(nb);
    }
    rng_normals_k<<<unsigned(nc), 256, 0, c_.stream>>>(raw.as<uint64_t>(), offs.as<int64_t>(), normals_.d());
    c_.check_launch();
    n_chunks_ = c_end;
    n_normals_ = 2 * std::max<int64_t>(lower, 0);  // normals certainly present
}

void RngStream::ensure_normals(int64_t upto) {
    while (n_normals_ < upto) {
        double per_chunk = double(mt::S) * 0.7853981633974483 * 0.995;  // normals per chunk, with slack
        int64_t extra = int64_t(std::ceil(double(upto - n_normals_) / per_chunk)) + 1;
        extra = std::min<int64_t>(extra, 1024);
        generate_chunks(n_chunks_ + extra);
    }
}

const double* RngStream::take(int64_t count) {
    StageTimer _t(c_, "rng", count, n_chunks_, int64_t(seed_ & 0xffff));
    ensure_normals(consumed_ + count);
    const double* p = normals_.d() + consumed_;
    consumed_ += count;
    return p;
}

void RngStream::fill(int64_t offset, int64_t count, double* out) {
    ensure_normals(offset + count);
    HYDOT_CUDA(cudaMemcpyAsync(out, normals_.d() + offset, size_t(count) * 8,
                               cudaMemcpyDeviceToDevice, c_.stream));
}

void RngStream::raw(int64_t offset, int64_t count, uint64_t* out) {
    if (count <= 0) return;
    int64_t cb = offset / mt::S, ce = (offset + count + mt::S - 1) / mt::S;
    int64_t nc = ce - cb;
    const uint64_t* jumps = device_jumps(c_, ce);
    DBuf windows(c_, size_t(nc) * mt::NW * 8);
    DBuf rawb(c_, size_t(nc) * size_t(mt::S) * 8);
    DBuf counts(c_, size_t(nc) * sizeof(int));
    rng_jump_k<<<unsigned((nc + JCH - 1) / JCH), JPC * JCH, size_t(mt::PREFIX) * 8, c_.stream>>>(
        prefix_.as<uint64_t>(), jumps, cb, nc, windows.as<uint64_t>());
    c_.check_launch();
    rng_generate_k<<<unsigned(nc), 160, 0, c_.stream>>>(windows.as<uint64_t>(),
                                                        rawb.as<uint64_t>(), counts.as<int>());
    c_.check_launch();
    HYDOT_CUDA(cudaMemcpyAsync(out, rawb.as<uint64_t>() + (offset - cb * mt::S),
                               size_t(count) * 8, cudaMemcpyDeviceToDevice, c_.stream));
}

}  // namespace hydot
