// The reference's random start blocks (BlockVector::randomize,
// block_vector.hpp:42-51: std::mt19937_64 feeding libstdc++'s
// std::normal_distribution<double>) generated in parallel, bit-identically.
//
// * mt19937_64 jump-ahead: the untempered word sequence obeys a GF(2) linear
//   recurrence whose minimal polynomial phi (degree 19937) is recovered once
//   with Berlekamp-Massey from output bits; a jump of J outputs applies
//   g(S) = (x^J mod phi)(S) to the 312-word window by Horner's rule.
// * libstdc++'s normal_distribution is the Marsaglia polar method caching the
//   second variate, so the normal stream is [y_0 m_0, x_0 m_0, y_1 m_1, ...]
//   over the ACCEPTED uniform pairs (x, y) = (2u_{2k}-1, 2u_{2k+1}-1); pair
//   acceptance depends only on the pair, so chunks of the uniform stream are
//   transformed independently once their accepted-pair counts are known.
// * log/sqrt/division stay on the host (glibc), keeping every bit.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

#include "capi_common.hpp"

namespace cfd {

namespace {

constexpr int kN = 312, kM = 156;
constexpr uint64_t kA = 0xB5026F5AA96619E9ULL, kUM = 0xFFFFFFFF80000000ULL, kLM = 0x7FFFFFFFULL;
constexpr int kDeg = 19937;
constexpr int kWords = (kDeg + 64) / 64;  // bitset words for polynomials of degree <= kDeg

// 312-word window [x_p .. x_{p+311}] as a circular buffer (logical word j at x[(i+j)%N])
struct Window {
    uint64_t x[kN];
    int i = 0;
    uint64_t next() {  // x_{p+312}; slides the window by one
        const uint64_t a = x[i], b = x[i + 1 == kN ? 0 : i + 1];
        const int m = i + kM >= kN ? i + kM - kN : i + kM;
        const uint64_t y = (a & kUM) | (b & kLM);
        const uint64_t w = x[m] ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
        x[i] = w;
        i = i + 1 == kN ? 0 : i + 1;
        return w;
    }
    // rotate so logical word 0 sits at x[0] (the layout std::mt19937_64 twists in place)
    void normalize() {
        if (i == 0) return;
        uint64_t t[kN];
        for (int j = 0; j < kN; ++j) t[j] = x[i + j >= kN ? i + j - kN : i + j];
        std::memcpy(x, t, sizeof(x));
        i = 0;
    }
    // the next 312 outputs at once (normalized window; == 312 next() calls)
    void twist() {
        auto mix = [](uint64_t a, uint64_t b, uint64_t c) {
            const uint64_t y = (a & kUM) | (b & kLM);
            return c ^ (y >> 1) ^ ((0ULL - (y & 1ULL)) & kA);  // branch-free
        };
        int k = 0;
        for (; k < kN - kM; ++k) x[k] = mix(x[k], x[k + 1], x[k + kM]);
        for (; k < kN - 1; ++k) x[k] = mix(x[k], x[k + 1], x[k + kM - kN]);
        x[kN - 1] = mix(x[kN - 1], x[0], x[kM - 1]);
    }
    void xor_in(const Window& o) {
        // logical word j: x[(i+j)%N] ^= o.x[(o.i+j)%N], in straight segments
        int j = 0;
        while (j < kN) {
            const int a = i + j >= kN ? i + j - kN : i + j;
            const int b = o.i + j >= kN ? o.i + j - kN : o.i + j;
            const int len = std::min({kN - j, kN - a, kN - b});
            uint64_t* __restrict__ dst = x + a;
            const uint64_t* __restrict__ src = o.x + b;
            for (int q = 0; q < len; ++q) dst[q] ^= src[q];
            j += len;
        }
    }
};

inline uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

Window seed_window(uint64_t seed) {  // std::mt19937_64::seed
    Window w;
    w.x[0] = seed;
    for (int k = 1; k < kN; ++k)
        w.x[k] = 6364136223846793005ULL * (w.x[k - 1] ^ (w.x[k - 1] >> 62)) + static_cast<uint64_t>(k);
    w.i = 0;
    return w;
}

using Poly = std::vector<uint64_t>;  // GF(2) polynomial, bit k = coefficient of x^k

inline bool bit(const Poly& p, int k) { return (p[k >> 6] >> (k & 63)) & 1ULL; }
inline void flip(Poly& p, int k) { p[k >> 6] ^= 1ULL << (k & 63); }

// minimal polynomial phi of the mt19937_64 recurrence (monic, degree 19937)
const Poly& min_poly() {
    static Poly phi;
    static std::once_flag once;
    std::call_once(once, [] {
        const int n = 2 * kDeg + 64;
        Window w = seed_window(5489ULL);
        std::vector<uint8_t> s(n);
        for (int k = 0; k < n; ++k) s[k] = static_cast<uint8_t>(w.next() & 1ULL);
        // Berlekamp-Massey over GF(2), bit-packed; rev holds s[t-k] at bit k
        const int W = (n + 64) / 64;
        Poly C(W, 0), B(W, 0), T(W, 0), rev(W, 0);
        C[0] = B[0] = 1ULL;
        int L = 0, m = 1;
        for (int t = 0; t < n; ++t) {
            for (int q = W - 1; q > 0; --q) rev[q] = (rev[q] << 1) | (rev[q - 1] >> 63);
            rev[0] = (rev[0] << 1) | s[t];
            int par = 0;
            const int lw = L / 64 + 1;
            for (int q = 0; q < lw && q < W; ++q) par ^= std::popcount(C[q] & rev[q]) & 1;
            if (!par) {
                ++m;
                continue;
            }
            T = C;
            // C += x^m B
            const int ws = m / 64, bs = m % 64;
            for (int q = W - 1; q >= ws; --q) {
                uint64_t v = B[q - ws] << bs;
                if (bs && q - ws - 1 >= 0) v |= B[q - ws - 1] >> (64 - bs);
                C[q] ^= v;
            }
            if (2 * L <= t) {
                L = t + 1 - L;
                B = T;
                m = 1;
            } else {
                ++m;
            }
        }
        if (L != kDeg) fail(CHEBFD_ERR_RUNTIME, "mt19937_64 jump: unexpected recurrence degree");
        // characteristic polynomial = reciprocal of the connection polynomial
        phi.assign(kWords, 0);
        for (int k = 0; k <= L; ++k)
            if (bit(C, k)) flip(phi, L - k);
    });
    return phi;
}

// r := r mod phi for deg r < 2*kDeg (r has 2*kWords words)
void reduce(Poly& r, const Poly& phi) {
    for (int k = 2 * kDeg; k >= kDeg; --k) {
        if (!bit(r, k)) continue;
        const int sh = k - kDeg;  // r ^= phi * x^sh
        const int ws = sh / 64, bs = sh % 64;
        for (int q = 0; q < kWords; ++q) {
            const uint64_t v = phi[q];
            if (!v) continue;
            r[q + ws] ^= v << bs;
            if (bs && q + ws + 1 < static_cast<int>(r.size())) r[q + ws + 1] ^= v >> (64 - bs);
        }
    }
}

// x^J mod phi
Poly x_pow(uint64_t J) {
    const Poly& phi = min_poly();
    Poly r(2 * kWords + 1, 0);
    r[0] = 1ULL;  // 1
    for (int b = 63; b >= 0; --b) {
        // square: spread bits
        Poly sq(2 * kWords + 1, 0);
        for (int k = 0; k < kDeg; ++k)
            if (bit(r, k)) flip(sq, 2 * k);
        r.swap(sq);
        reduce(r, phi);
        if ((J >> b) & 1ULL) {  // multiply by x
            for (int q = static_cast<int>(r.size()) - 1; q > 0; --q) r[q] = (r[q] << 1) | (r[q - 1] >> 63);
            r[0] <<= 1;
            reduce(r, phi);
        }
    }
    r.resize(kWords);
    return r;
}

// w := g(S) w, S = one step of the recurrence (Horner)
void apply(const Poly& g, Window& w) {
    Window acc;
    std::memset(acc.x, 0, sizeof(acc.x));
    acc.i = 0;
    for (int k = kDeg - 1; k >= 0; --k) {
        acc.next();
        if (bit(g, k)) acc.xor_in(w);
    }
    w = acc;
}

// the jump polynomial for chunks of kChunkOut outputs (cached)
constexpr uint64_t kChunkOut = 1ULL << 23;  // uniforms per chunk (even: whole pairs)
const Poly& chunk_jump() {
    static Poly g;
    static std::once_flag once;
    std::call_once(once, [] { g = x_pow(kChunkOut); });
    return g;
}

// libstdc++ generate_canonical<double, 53>(mt19937_64)
inline double canon(uint64_t u) {
    // / 2^64 == * 2^-64 exactly (power-of-two scaling; the only rounding is the conversion)
    double r = static_cast<double>(u) * 0x1p-64;
    if (r >= 1.0) r = std::nextafter(1.0, 0.0);
    return r;
}

// the chunk's uniform words, 312 per twist (kN is even, so pairs never straddle)
struct Words {
    Window w;
    int pos = kN;
    explicit Words(const Window& start) : w(start) { w.normalize(); }
    uint64_t next() {
        if (pos == kN) {
            w.twist();
            pos = 0;
        }
        return w.x[pos++];
    }
};

// count accepted polar pairs among the chunk's kChunkOut uniforms
int64_t count_pairs(const Window& start) {
    Words src(start);
    int64_t acc = 0;
    for (uint64_t k = 0; k < kChunkOut; k += 2) {
        const double x = 2.0 * canon(temper(src.next())) - 1.0;
        const double y = 2.0 * canon(temper(src.next())) - 1.0;
        const double r2 = x * x + y * y;
        acc += !(r2 > 1.0 || r2 == 0.0);
    }
    return acc;
}

// Write the normals of the chunk's accepted pairs [p0, p1) (chunk-local pair
// index).  Pair j of the stream is normals (2j, 2j+1) = (y m, x m).  Complex
// entries are (re, im) = (normal 2i+1, normal 2i), i.e. pair j lands as
// (x m, y m) at entry j - E0; real normals land at index n - n_begin.
void emit_pairs(const Window& start, int64_t p0, int64_t p1, int64_t pbase, bool cplx,
                int64_t n_begin, int64_t n_end, double* out) {
    Words src(start);
    int64_t pj = 0;
    for (uint64_t k = 0; k < kChunkOut && pj < p1; k += 2) {
        const double x = 2.0 * canon(temper(src.next())) - 1.0;
        const double y = 2.0 * canon(temper(src.next())) - 1.0;
        const double r2 = x * x + y * y;
        if (r2 > 1.0 || r2 == 0.0) continue;
        if (pj >= p0) {
            const double mult = std::sqrt(-2 * std::log(r2) / r2);
            const double n0 = y * mult * 1.0 + 0.0, n1 = x * mult * 1.0 + 0.0;
            const int64_t j = pbase + pj;  // global pair index
            if (cplx) {
                double* e = out + 2 * (j - n_begin / 2);
                e[0] = n1;
                e[1] = n0;
            } else {
                const int64_t a = 2 * j - n_begin;
                if (a >= 0 && 2 * j < n_end) out[a] = n0;
                if (2 * j + 1 >= n_begin && 2 * j + 1 < n_end) out[a + 1] = n1;
            }
        }
        ++pj;
    }
}

// serial path (small blocks): the library's own engine, exactly the reference's
void serial(int kind, uint64_t seed, int64_t first, int64_t count, double* o) {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> dist(0.0, 1.0);
    if (kind == CHEBFD_REAL64) {
        for (int64_t i = 0; i < first; ++i) (void)dist(gen);
        for (int64_t i = 0; i < count; ++i) o[i] = dist(gen);
    } else {
        for (int64_t i = 0; i < 2 * first; ++i) (void)dist(gen);
        for (int64_t i = 0; i < count; ++i) {
            const double im = dist(gen);  // Complex(dist(gen), dist(gen)): GCC evaluates right to left
            const double re = dist(gen);
            o[2 * i] = re;
            o[2 * i + 1] = im;
        }
    }
}

}  // namespace

// Chunk bookkeeping of one seed's stream, extended on demand so a block can be
// generated piecewise in increasing order (pass 1 is never repeated).
struct NormalStream::Impl {
    std::vector<Window> starts;
    std::vector<int64_t> pairs;  // accepted pairs per chunk
    std::vector<int64_t> base{0};
    int64_t total = 0;
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    explicit Impl(uint64_t seed) : starts{seed_window(seed)} {}

    // pass 1: chunk start windows (sequential jumps) and pair counts (parallel)
    void count_to(int64_t P1) {
        const Poly& g = chunk_jump();
        while (total < P1) {
            const int64_t have = static_cast<int64_t>(pairs.size());
            const double est = static_cast<double>(P1 - total) / (0.785 * (kChunkOut / 2));
            const int64_t batch = std::max<int64_t>(static_cast<int64_t>(hw),
                                                    static_cast<int64_t>(std::ceil(est * 1.02)) + 1);
            while (static_cast<int64_t>(starts.size()) < have + batch + 1) {
                Window w = starts.back();
                apply(g, w);
                starts.push_back(w);
            }
            pairs.resize(have + batch);
            std::vector<std::thread> th;
            for (unsigned t = 0; t < hw; ++t)
                th.emplace_back([&, t] {
                    for (int64_t c = have + t; c < have + batch; c += hw)
                        pairs[c] = count_pairs(starts[c]);
                });
            for (auto& x : th) x.join();
            for (int64_t c = have; c < have + batch; ++c) {
                total += pairs[c];
                base.push_back(total);
            }
        }
    }

    // pass 2: emit the normals of pairs [P0, P1) straight into `o` (chunks in parallel)
    void emit(int kind, int64_t first, int64_t count, double* o) {
        const int per = kind == CHEBFD_COMPLEX128 ? 2 : 1;
        const int64_t n_begin = first * per, n_end = (first + count) * per;  // normal indices
        // pairs [P0, P1) hold normals [2 P0, 2 P1) covering [n_begin, n_end)
        const int64_t P0 = n_begin / 2, P1 = (n_end + 1) / 2;
        count_to(P1);
        std::vector<int64_t> todo;
        for (size_t c = 0; c < pairs.size(); ++c)
            if (base[c + 1] > P0 && base[c] < P1) todo.push_back(static_cast<int64_t>(c));
        const bool cplx = kind == CHEBFD_COMPLEX128;
        std::vector<std::thread> th;
        for (unsigned t = 0; t < hw; ++t)
            th.emplace_back([&, t] {
                for (size_t q = t; q < todo.size(); q += hw) {
                    const int64_t c = todo[q];
                    const int64_t lo = std::max(P0, base[c]) - base[c];
                    const int64_t hi = std::min(P1, base[c + 1]) - base[c];
                    emit_pairs(starts[c], lo, hi, base[c], cplx, n_begin, n_end, o);
                }
            });
        for (auto& x : th) x.join();
    }
};

int64_t NormalStream::parallel_piece(int kind) {
    // one RNG chunk per host thread: ~0.785 accepted pairs per uniform pair
    const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t normals = hw * static_cast<int64_t>(0.785 * kChunkOut);
    return normals / (kind == CHEBFD_COMPLEX128 ? 2 : 1);
}

NormalStream::NormalStream(uint64_t seed) : impl_(std::make_unique<Impl>(seed)) {}
NormalStream::~NormalStream() = default;
void NormalStream::emit(int kind, int64_t first, int64_t count, void* out) {
    impl_->emit(kind, first, count, static_cast<double*>(out));
}

// Entries [first, first+count) of the row-major global block's stream.
void host_randomize(int kind, uint64_t seed, int64_t first, int64_t count, void* out) {
    const int per = kind == CHEBFD_COMPLEX128 ? 2 : 1;
    const int64_t n_end = (first + count) * per;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    if (n_end < (int64_t{1} << 23) || hw == 1)
        return serial(kind, seed, first, count, static_cast<double*>(out));
    NormalStream(seed).emit(kind, first, count, out);
}

}  // namespace cfd

extern "C" int chebfd_host_randomize(int kind, uint64_t seed, int64_t first, int64_t count,
                                     void* out) {
    using namespace cfd;
    return guard([&] {
        require(kind == CHEBFD_REAL64 || kind == CHEBFD_COMPLEX128, "bad scalar kind");
        require(first >= 0 && count >= 0, "host_randomize: negative range");
        host_randomize(kind, seed, first, count, out);
    });
}
