// Host GF(2)[x] / P arithmetic (see gf2poly.hpp). Carry-less multiply
// (PCLMULQDQ) schoolbook products + Barrett reduction: ~0.1 ms per mulmod.
#include "gf2poly.hpp"

#include <algorithm>
#include <cstring>
#include <stdexcept>

#if defined(__x86_64__)
#include <cpuid.h>
#include <immintrin.h>
#endif

namespace vmt_b200 {

namespace {

constexpr std::uint32_t kUpper = 0x80000000u;
constexpr std::uint32_t kLower = 0x7FFFFFFFu;
constexpr std::uint32_t kMatrixA = 0x9908B0DFu;

inline std::uint32_t mul_a(std::uint32_t u) { return (u >> 1) ^ ((0u - (u & 1u)) & kMatrixA); }

inline void clmul_portable(std::uint64_t a, std::uint64_t b, std::uint64_t& lo, std::uint64_t& hi) {
    std::uint64_t l = 0, h = 0;
    for (int i = 0; i < 64; ++i)
        if ((b >> i) & 1u) {
            l ^= a << i;
            if (i)
                h ^= a >> (64 - i);
        }
    lo = l;
    hi = h;
}

#if defined(__x86_64__)
__attribute__((target("pclmul,sse4.1"))) void mul_clmul(const std::uint64_t* a, int aw,
                                                          const std::uint64_t* b, int bw,
                                                          std::uint64_t* out) {
    std::memset(out, 0, sizeof(std::uint64_t) * (aw + bw));
    for (int i = 0; i < aw; ++i) {
        const std::uint64_t ai = a[i];
        if (!ai)
            continue;
        const __m128i va = _mm_set_epi64x(0, (long long)ai);
        __m128i carry = _mm_setzero_si128(); // [hi of the previous odd product, 0]
        int j = 0;
        for (; j + 1 < bw; j += 2) {
            const __m128i vb = _mm_loadu_si128(reinterpret_cast<const __m128i*>(b + j));
            const __m128i p0 = _mm_clmulepi64_si128(va, vb, 0x00); // ai * b[j]
            const __m128i p1 = _mm_clmulepi64_si128(va, vb, 0x10); // ai * b[j+1]
            __m128i t = _mm_xor_si128(p0, _mm_slli_si128(p1, 8));  // [lo0, hi0^lo1]
            t = _mm_xor_si128(t, carry);
            __m128i* o = reinterpret_cast<__m128i*>(out + i + j);
            _mm_storeu_si128(o, _mm_xor_si128(_mm_loadu_si128(o), t));
            carry = _mm_srli_si128(p1, 8); // [hi1, 0]
        }
        out[i + j] ^= (std::uint64_t)_mm_cvtsi128_si64(carry);
        if (j < bw) {
            const __m128i p = _mm_clmulepi64_si128(va, _mm_set_epi64x(0, (long long)b[j]), 0x00);
            out[i + j] ^= (std::uint64_t)_mm_cvtsi128_si64(p);
            out[i + j + 1] ^= (std::uint64_t)_mm_extract_epi64(p, 1);
        }
    }
}
#endif

void mul_portable(const std::uint64_t* a, int aw, const std::uint64_t* b, int bw, std::uint64_t* out) {
    std::memset(out, 0, sizeof(std::uint64_t) * (aw + bw));
    for (int i = 0; i < aw; ++i) {
        if (!a[i])
            continue;
        for (int j = 0; j < bw; ++j) {
            std::uint64_t lo, hi;
            clmul_portable(a[i], b[j], lo, hi);
            out[i + j] ^= lo;
            out[i + j + 1] ^= hi;
        }
    }
}

bool detect_clmul() {
#if defined(__x86_64__)
    unsigned eax, ebx, ecx, edx;
    if (!__get_cpuid(1, &eax, &ebx, &ecx, &edx))
        return false;
    return (ecx & bit_PCLMUL) && (ecx & bit_SSE4_1);
#else
    return false;
#endif
}

const bool g_has_clmul = detect_clmul();

inline bool getbit(const std::uint64_t* a, int i) { return (a[i >> 6] >> (i & 63)) & 1u; }

int degree(const std::uint64_t* a, int words) {
    for (int w = words - 1; w >= 0; --w)
        if (a[w])
            return w * 64 + 63 - __builtin_clzll(a[w]);
    return -1;
}

// out = a >> s (bits), out has ow words
void shr_bits(const std::uint64_t* a, int aw, int s, std::uint64_t* out, int ow) {
    const int ws = s >> 6, bs = s & 63;
    for (int w = 0; w < ow; ++w) {
        const int src = w + ws;
        std::uint64_t v = src < aw ? a[src] >> bs : 0;
        if (bs && src + 1 < aw)
            v |= a[src + 1] << (64 - bs);
        out[w] = v;
    }
}

// a ^= b << s (bits); b has bw words, a has aw words (excess dropped)
void xor_shl(std::uint64_t* a, int aw, const std::uint64_t* b, int bw, int s) {
    const int ws = s >> 6, bs = s & 63;
    for (int w = 0; w < bw; ++w) {
        const std::uint64_t v = b[w];
        if (!v)
            continue;
        if (w + ws < aw)
            a[w + ws] ^= v << bs;
        if (bs && w + ws + 1 < aw)
            a[w + ws + 1] ^= v >> (64 - bs);
    }
}

// Characteristic polynomial of the MT19937 transition by Berlekamp-Massey
// over s_n = bit 0 of x_{n+1} (x = untempered word sequence of seed 5489).
std::vector<std::uint64_t> berlekamp_massey() {
    const int nbits = 2 * kDeg + 64;
    std::vector<std::uint32_t> x(624 + nbits + 2);
    x[0] = 5489u;
    for (std::uint32_t i = 1; i < 624; ++i)
        x[i] = 1812433253u * (x[i - 1] ^ (x[i - 1] >> 30)) + i;
    for (std::size_t n = 0; n + 624 < x.size(); ++n)
        x[n + 624] = x[n + 397] ^ mul_a((x[n] & kUpper) | (x[n + 1] & kLower));
    const int rwords = nbits / 64 + 2;
    std::vector<std::uint64_t> r(rwords, 0); // s reversed
    for (int n = 0; n < nbits; ++n)
        if (x[n + 1] & 1u) {
            const int j = nbits - 1 - n;
            r[j >> 6] |= 1ull << (j & 63);
        }
    const int cw = kFullWords + 1;
    std::vector<std::uint64_t> C(cw, 0), B(cw, 0), T(cw, 0);
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    for (int n = 0; n < nbits; ++n) {
        const int o = nbits - 1 - n;
        std::uint64_t acc = 0;
        const int words = L / 64 + 1;
        for (int w = 0; w < words; ++w) {
            const int bit = o + 64 * w, q = bit >> 6, sh = bit & 63;
            std::uint64_t seg = q < rwords ? r[q] >> sh : 0;
            if (sh && q + 1 < rwords)
                seg |= r[q + 1] << (64 - sh);
            std::uint64_t c = C[w];
            if (w == words - 1 && ((L + 1) & 63))
                c &= (1ull << ((L + 1) & 63)) - 1;
            acc ^= seg & c;
        }
        if (!__builtin_parityll(acc)) {
            ++m;
            continue;
        }
        T = C;
        xor_shl(C.data(), cw, B.data(), cw, m);
        if (2 * L <= n) {
            L = n + 1 - L;
            B = T;
            m = 1;
        } else {
            ++m;
        }
    }
    if (L != kDeg)
        throw std::runtime_error("Berlekamp-Massey: unexpected linear complexity");
    std::vector<std::uint64_t> p(kFullWords, 0);
    for (int j = 0; j <= L; ++j) {
        const int i = L - j;
        if (getbit(C.data(), i))
            p[j >> 6] |= 1ull << (j & 63);
    }
    return p;
}

// floor(x^(2n) / P) by schoolbook long division.
std::vector<std::uint64_t> barrett_mu(const std::vector<std::uint64_t>& p) {
    const int qbits = kDeg + 1;          // quotient degree n
    const int aw = (2 * kDeg) / 64 + 2;  // holds x^(2n)
    std::vector<std::uint64_t> a(aw, 0), q((qbits + 63) / 64 + 1, 0);
    a[(2 * kDeg) >> 6] |= 1ull << ((2 * kDeg) & 63);
    for (int i = 2 * kDeg; i >= kDeg; --i) {
        if (!getbit(a.data(), i))
            continue;
        const int s = i - kDeg;
        q[s >> 6] |= 1ull << (s & 63);
        xor_shl(a.data(), aw, p.data(), kFullWords, s);
    }
    q.resize(kFullWords, 0);
    return q;
}

// Inverse of a mod p (binary extended Euclid, Hankerson et al. alg. 2.48).
Poly invmod(const Poly& a, const std::vector<std::uint64_t>& p) {
    const int W = kFullWords + 2;
    std::vector<std::uint64_t> u(W, 0), v(W, 0), g1(W, 0), g2(W, 0);
    std::copy(a.begin(), a.end(), u.begin());
    std::copy(p.begin(), p.end(), v.begin());
    g1[0] = 1;
    int du = degree(u.data(), W), dv = degree(v.data(), W);
    if (du < 0)
        throw std::invalid_argument("invmod of zero");
    while (du != 0) {
        int j = du - dv;
        if (j < 0) {
            std::swap(u, v);
            std::swap(g1, g2);
            std::swap(du, dv);
            j = -j;
        }
        xor_shl(u.data(), W, v.data(), W, j);
        xor_shl(g1.data(), W, g2.data(), W, j);
        du = degree(u.data(), W);
    }
    Poly out(kPolyWords);
    std::copy(g1.begin(), g1.begin() + kPolyWords, out.begin());
    if (degree(g1.data(), W) >= kDeg)
        throw std::runtime_error("invmod: result not reduced");
    return out;
}

} // namespace

void clmul_mul(const std::uint64_t* a, int aw, const std::uint64_t* b, int bw, std::uint64_t* out) {
#if defined(__x86_64__)
    if (g_has_clmul) {
        mul_clmul(a, aw, b, bw, out);
        return;
    }
#endif
    mul_portable(a, aw, b, bw, out);
}

bool Gf2Field::has_clmul() { return g_has_clmul; }

Gf2Field& Gf2Field::instance() {
    static Gf2Field f;
    return f;
}

Gf2Field::Gf2Field() {
    p_ = berlekamp_massey();
    mu_ = barrett_mu(p_);
    // sqrt(x) = x^(2^(n-1)): with P = Pe(x^2) + x Po(x^2) and P(sqrt x) = 0,
    // sqrt(x) = Pe(x) / Po(x) mod P.
    Poly pe(kPolyWords, 0), po(kPolyWords, 0);
    for (int i = 0; i <= kDeg; ++i)
        if (getbit(p_.data(), i)) {
            const int h = i >> 1;
            if (i & 1)
                po[h >> 6] |= 1ull << (h & 63);
            else
                pe[h >> 6] |= 1ull << (h & 63);
        }
    sqrt_x_ = mulmod(pe, invmod(po, p_));
    // self-check: sqrt(x)^2 == x
    Poly chk = sqrmod(sqrt_x_);
    Poly xx(kPolyWords, 0);
    xx[0] = 2;
    if (chk != xx)
        throw std::runtime_error("sqrt(x) self-check failed");
}

void Gf2Field::barrett_reduce(const std::uint64_t* a, std::uint64_t* out) const {
    // a: product of two residues, 2*kPolyWords words, degree <= 2n-2.
    constexpr int AW = 2 * kPolyWords;
    std::uint64_t q1[kFullWords], q2[2 * kFullWords], q3[kFullWords], t[2 * kFullWords];
    shr_bits(a, AW, kDeg, q1, kFullWords);
    clmul_mul(q1, kFullWords, mu_.data(), kFullWords, q2);
    shr_bits(q2, 2 * kFullWords, kDeg, q3, kFullWords);
    clmul_mul(q3, kFullWords, p_.data(), kFullWords, t);
    for (int w = 0; w < kPolyWords; ++w)
        out[w] = a[w] ^ t[w];
    out[kPolyWords - 1] &= (1ull << (kDeg & 63)) - 1; // keep degree < n
}

Poly Gf2Field::one() const {
    Poly r(kPolyWords, 0);
    r[0] = 1;
    return r;
}

Poly Gf2Field::mulmod(const Poly& a, const Poly& b) const {
    std::uint64_t prod[2 * kPolyWords];
    clmul_mul(a.data(), kPolyWords, b.data(), kPolyWords, prod);
    Poly r(kPolyWords);
    barrett_reduce(prod, r.data());
    return r;
}

Poly Gf2Field::sqrmod(const Poly& a) const {
    std::uint64_t prod[2 * kPolyWords];
    // squaring spreads the bits (no cross terms over GF(2))
    for (int w = 0; w < kPolyWords; ++w) {
        std::uint64_t lo, hi;
        const std::uint64_t v = a[w];
        std::uint64_t l = 0, h = 0;
        for (int i = 0; i < 32; ++i) {
            l |= ((v >> i) & 1ull) << (2 * i);
            h |= ((v >> (i + 32)) & 1ull) << (2 * i);
        }
        lo = l;
        hi = h;
        prod[2 * w] = lo;
        prod[2 * w + 1] = hi;
    }
    Poly r(kPolyWords);
    barrett_reduce(prod, r.data());
    return r;
}

Poly Gf2Field::powmod(const Poly& a, std::uint64_t e) const {
    Poly r = one();
    Poly b = a;
    while (e) {
        if (e & 1u)
            r = mulmod(r, b);
        e >>= 1;
        if (e)
            b = sqrmod(b);
    }
    return r;
}

Poly Gf2Field::x_pow(std::uint64_t d) const { return x_pow128(d, 0); }

Poly Gf2Field::x_pow128(std::uint64_t lo, std::uint64_t hi) const {
    // left-to-right: r = r^2, then r *= x (a shift plus one conditional
    // subtraction of P) for set bits.
    Poly r = one();
    bool started = false;
    for (int b = 127; b >= 0; --b) {
        const bool bit = b >= 64 ? (hi >> (b - 64)) & 1u : (lo >> b) & 1u;
        if (started)
            r = sqrmod(r);
        if (bit) {
            started = true;
            std::uint64_t carry = 0;
            for (int w = 0; w < kPolyWords; ++w) {
                const std::uint64_t v = r[w];
                r[w] = (v << 1) | carry;
                carry = v >> 63;
            }
            if (getbit(r.data(), kDeg))
                for (int w = 0; w < kPolyWords; ++w)
                    r[w] ^= p_[w];
        }
    }
    return r;
}

Poly Gf2Field::sqrtmod(const Poly& a) const {
    // a = Ae(x^2) + x Ao(x^2)  =>  sqrt(a) = Ae(x) + sqrt(x) Ao(x)
    Poly ae(kPolyWords, 0), ao(kPolyWords, 0);
    for (int i = 0; i < kDeg; ++i)
        if (getbit(a.data(), i)) {
            const int h = i >> 1;
            if (i & 1)
                ao[h >> 6] |= 1ull << (h & 63);
            else
                ae[h >> 6] |= 1ull << (h & 63);
        }
    Poly t = mulmod(sqrt_x_, ao);
    for (int w = 0; w < kPolyWords; ++w)
        t[w] ^= ae[w];
    return t;
}

Poly Gf2Field::x_pow2(unsigned q) const {
    {
        std::lock_guard<std::mutex> lk(cache_mu_);
        if (q < pow2_cache_.size() && !pow2_cache_[q].empty())
            return pow2_cache_[q];
    }
    Poly r;
    // x^(2^kDeg) == x (the period is 2^kDeg - 1), so reduce q mod kDeg and
    // walk whichever way is shorter: squarings up from x, or square roots
    // down from x^(2^kDeg) = x.
    const unsigned qq = q % unsigned(kDeg);
    Poly xx(kPolyWords, 0);
    xx[0] = 2;
    if (unsigned(kDeg) - qq > 4096) {
        r = xx;
        for (unsigned i = 0; i < qq; ++i)
            r = sqrmod(r);
    } else {
        r = xx;
        for (unsigned i = 0; i < unsigned(kDeg) - qq; ++i)
            r = sqrtmod(r);
    }
    std::lock_guard<std::mutex> lk(cache_mu_);
    if (pow2_cache_.size() <= q)
        pow2_cache_.resize(q + 1);
    pow2_cache_[q] = r;
    return r;
}

} // namespace vmt_b200
