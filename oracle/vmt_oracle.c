/*
 * vmt_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference's VMT19937 algorithms, written so
 * that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg can
 * check the CUDA product against it. The product (paper_2309_16682_b200/)
 * never links, loads or calls this file.
 *
 * Pinned against: the reference's own KATs (proj/tests/test_mt19937.cpp:35-101),
 * the golden vectors produced by the unmodified reference library in
 * oracle/_ref (tests/golden/make_golden.py), and SURVEY.md Appendix A.
 *
 * Section map (reference file:line each function follows):
 *   A. MT19937 scalar core ............ proj/include/vmt19937/mt19937.hpp:61-72,
 *                                       proj/src/mt19937.cpp:22-55
 *   B. VMT interleaved engine ......... proj/include/vmt19937/engine.hpp:54-63,110-142
 *                                       (lane count generalised to any power of two,
 *                                       SURVEY.md G1)
 *   C. Effective-state layout ......... proj/src/mt19937.cpp:57-101
 *   D. GF(2) matrix jump .............. proj/src/f2_matrix.cpp:119-228,
 *                                       proj/src/jump.cpp:27-53
 *   E. Polynomial jump (new, G3) ...... characteristic polynomial by
 *      Berlekamp-Massey, x^d mod P by square-and-multiply, and the state
 *      jump p(F)s as a word convolution over the generated sequence. Pinned
 *      to section D at small exponents by tests/test_oracle.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NN 624
#define MM 397
#define UPPER 0x80000000u
#define LOWER 0x7FFFFFFFu
#define MATRIX_A 0x9908B0DFu
#define DIM 19937
#define RW 312 /* u64 words per 19937-bit row, F2Vector::word_count */

/* ---------------------------------------------------------------- A ---- */

/* mt19937.hpp:61-66 */
uint32_t or_temper(uint32_t x) {
    uint32_t y = x ^ (x >> 11);
    y ^= (y << 7) & 0x9D2C5680u;
    y ^= (y << 15) & 0xEFC60000u;
    return y ^ (y >> 18);
}

/* mt19937.hpp:70-72 */
uint32_t or_mul_a(uint32_t u) { return (u >> 1) ^ ((0u - (u & 1u)) & MATRIX_A); }

/* mt19937.cpp:22-27 (init_genrand); the state is left at the boundary. */
void or_seed(uint32_t seed, uint32_t *w) {
    w[0] = seed;
    for (uint32_t i = 1; i < NN; ++i)
        w[i] = 1812433253u * (w[i - 1] ^ (w[i - 1] >> 30)) + i;
}

/* mt19937.cpp:36-49: the 227 / 396 / 1 loops. */
void or_regenerate(uint32_t *x) {
    int k;
    for (k = 0; k < NN - MM; ++k)
        x[k] = x[k + MM] ^ or_mul_a((x[k] & UPPER) | (x[k + 1] & LOWER));
    for (; k < NN - 1; ++k)
        x[k] = x[k + MM - NN] ^ or_mul_a((x[k] & UPPER) | (x[k + 1] & LOWER));
    x[NN - 1] = x[MM - 1] ^ or_mul_a((x[NN - 1] & UPPER) | (x[0] & LOWER));
}

/* Outputs [skip, skip+count) of the scalar generator whose boundary state is
 * `words` (Mt19937::from_words + next_u32, mt19937.cpp:29-55). */
void or_mt_stream_from_words(const uint32_t *words, uint64_t skip, uint64_t count, uint32_t *out) {
    uint32_t x[NN];
    memcpy(x, words, sizeof x);
    uint64_t blocks = skip / NN;
    for (uint64_t b = 0; b < blocks; ++b)
        or_regenerate(x);
    uint64_t cur = NN; /* cursor at the boundary */
    uint64_t lead = skip % NN;
    for (uint64_t i = 0; i < lead + count; ++i) {
        if (cur == NN) {
            or_regenerate(x);
            cur = 0;
        }
        uint32_t v = or_temper(x[cur++]);
        if (i >= lead)
            out[i - lead] = v;
    }
}

void or_mt_stream(uint32_t seed, uint64_t skip, uint64_t count, uint32_t *out) {
    uint32_t w[NN];
    or_seed(seed, w);
    or_mt_stream_from_words(w, skip, count, out);
}

/* ---------------------------------------------------------------- B ---- */

/* VmtEngine::regenerate (engine.hpp:110-133) on an interleaved 624*L state,
 * any L: the same three loops, each op widened to an L-lane group. */
void or_vmt_regenerate(uint32_t *s, unsigned L) {
    for (unsigned t = 0; t < L; ++t) {
        int k;
        for (k = 0; k < NN - MM; ++k)
            s[k * L + t] = s[(k + MM) * L + t] ^
                           or_mul_a((s[k * L + t] & UPPER) | (s[(k + 1) * L + t] & LOWER));
        for (; k < NN - 1; ++k)
            s[k * L + t] = s[(k + MM - NN) * L + t] ^
                           or_mul_a((s[k * L + t] & UPPER) | (s[(k + 1) * L + t] & LOWER));
        s[(NN - 1) * L + t] =
            s[(MM - 1) * L + t] ^ or_mul_a((s[(NN - 1) * L + t] & UPPER) | (s[t] & LOWER));
    }
}

/* Interleave L boundary lane states (engine.hpp:58-60). */
void or_vmt_interleave(const uint32_t *lane_states, unsigned L, uint32_t *s) {
    for (unsigned k = 0; k < NN; ++k)
        for (unsigned t = 0; t < L; ++t)
            s[k * L + t] = lane_states[(size_t)t * NN + k];
}

/* Combined-stream words [start, start+count) of a VMT generator whose lanes
 * start from `lane_states` (boundary states, lane-major 624 words each):
 * block-by-block regenerate + temper (engine.hpp:92-98,137-142). Blocks before
 * `start` are regenerated and discarded. */
int or_vmt_stream(const uint32_t *lane_states, unsigned L, uint64_t start, uint64_t count,
                  uint32_t *out) {
    const uint64_t bw = (uint64_t)NN * L;
    uint32_t *s = (uint32_t *)malloc(bw * sizeof(uint32_t));
    if (!s)
        return -1;
    or_vmt_interleave(lane_states, L, s);
    uint64_t b0 = start / bw;
    for (uint64_t b = 0; b < b0; ++b)
        or_vmt_regenerate(s, L);
    uint64_t pos = b0 * bw, done = 0;
    while (done < count) {
        or_vmt_regenerate(s, L);
        for (uint64_t i = 0; i < bw && done < count; ++i, ++pos)
            if (pos >= start)
                out[done++] = or_temper(s[i]);
    }
    free(s);
    return 0;
}

/* XOR fold of combined-stream words [start, start+count) (bench.cpp:13-18). */
uint32_t or_vmt_checksum(const uint32_t *lane_states, unsigned L, uint64_t start, uint64_t count) {
    const uint64_t bw = (uint64_t)NN * L;
    uint32_t *s = (uint32_t *)malloc(bw * sizeof(uint32_t));
    or_vmt_interleave(lane_states, L, s);
    uint64_t b0 = start / bw;
    for (uint64_t b = 0; b < b0; ++b)
        or_vmt_regenerate(s, L);
    uint64_t pos = b0 * bw, done = 0;
    uint32_t acc = 0;
    while (done < count) {
        or_vmt_regenerate(s, L);
        for (uint64_t i = 0; i < bw && done < count; ++i, ++pos)
            if (pos >= start) {
                acc ^= or_temper(s[i]);
                ++done;
            }
    }
    free(s);
    return acc;
}

/* ---------------------------------------------------------------- C ---- */

/* words_to_effective (mt19937.cpp:57-69) for the canonical parameters. */
void or_words_to_effective(const uint32_t *w, uint64_t *v) {
    memset(v, 0, RW * sizeof(uint64_t));
    size_t pos = 0;
    for (unsigned j = 31; j < 32; ++j, ++pos)
        if ((w[0] >> j) & 1u)
            v[pos >> 6] |= 1ull << (pos & 63);
    for (unsigned i = 1; i < NN; ++i)
        for (unsigned j = 0; j < 32; ++j, ++pos)
            if ((w[i] >> j) & 1u)
                v[pos >> 6] |= 1ull << (pos & 63);
}

/* effective_to_words (mt19937.cpp:71-88): the dead bits of word 0 are 0. */
void or_effective_to_words(const uint64_t *v, uint32_t *w) {
    size_t pos = 0;
    w[0] = (uint32_t)((v[0] & 1ull) << 31);
    pos = 1;
    for (unsigned i = 1; i < NN; ++i) {
        uint32_t x = 0;
        for (unsigned j = 0; j < 32; ++j, ++pos)
            x |= (uint32_t)((v[pos >> 6] >> (pos & 63)) & 1ull) << j;
        w[i] = x;
    }
}

/* ---------------------------------------------------------------- D ---- */

static inline void mset(uint64_t *m, size_t r, size_t c) { m[r * RW + (c >> 6)] ^= 1ull << (c & 63); }

/* build_transition_matrix (f2_matrix.cpp:179-228) for the canonical
 * parameters: row convention v(step(s)) = v(s) * F. `f` is DIM*RW u64, zeroed
 * here. Restated from the recurrence, not from the reference's code: step()
 * shifts words 1..623 down one place and appends
 * x_new = x_397 ^ mulA((x_0 & UPPER) | (x_1 & LOWER)). */
void or_build_transition(uint64_t *f) {
    memset(f, 0, (size_t)DIM * RW * sizeof(uint64_t));
    /* effective position of bit j of window word i */
#define POS(i, j) ((i) == 0 ? (size_t)((j)-31) : (size_t)(1 + 32 * ((i)-1) + (j)))
    /* basis bit (i,j) of the old state maps to: (i-1, j) when i >= 1 (shift),
     * plus its contribution to x_new (new word 623). */
    for (unsigned i = 0; i < NN; ++i)
        for (unsigned j = (i == 0 ? 31u : 0u); j < 32; ++j) {
            size_t row = POS(i, j);
            if (i >= 1 && !(i == 1 && j < 31))
                mset(f, row, POS(i - 1, j));
            /* contribution to x_new */
            uint32_t contrib = 0;
            if (i == MM)
                contrib ^= 1u << j;
            if ((i == 0 && j == 31) || (i == 1 && j < 31))
                contrib ^= or_mul_a(1u << j);
            for (unsigned b = 0; b < 32; ++b)
                if ((contrib >> b) & 1u)
                    mset(f, row, POS(NN - 1, b));
        }
#undef POS
}

/* vec_mat_mul (f2_matrix.cpp:119-136): XOR of the rows at the set bits. */
void or_vec_mat_mul(const uint64_t *v, const uint64_t *m, uint64_t *out) {
    uint64_t acc[RW];
    memset(acc, 0, sizeof acc);
    for (size_t w = 0; w < RW; ++w) {
        uint64_t bits = v[w];
        while (bits) {
            size_t i = w * 64 + (size_t)__builtin_ctzll(bits);
            bits &= bits - 1;
            const uint64_t *r = m + i * RW;
            for (size_t k = 0; k < RW; ++k)
                acc[k] ^= r[k];
        }
    }
    memcpy(out, acc, sizeof acc);
}

/* mat_mul (f2_matrix.cpp:138-168), single-threaded row by row. */
void or_mat_mul(const uint64_t *a, const uint64_t *b, uint64_t *c) {
    for (size_t r = 0; r < DIM; ++r)
        or_vec_mat_mul(a + r * RW, b, c + r * RW);
}

/* jump_state (jump.cpp:27-33) for a boundary state and a jump matrix. */
void or_jump_state_matrix(const uint32_t *in, const uint64_t *m, uint32_t *out) {
    uint64_t v[RW], r[RW];
    or_words_to_effective(in, v);
    or_vec_mat_mul(v, m, r);
    or_effective_to_words(r, out);
}

/* ---------------------------------------------------------------- E ---- */
/* Polynomials over GF(2): bit i of a u64 array is the coefficient of x^i. */

#define PW 313 /* words holding a degree-19937 polynomial */

/* Characteristic polynomial of F (degree 19937) by Berlekamp-Massey over the
 * bit sequence s_n = bit 0 of x_{n+1}, where x is the untempered word sequence
 * of seed 5489 (any non-zero linear functional has minimal polynomial P because
 * P is irreducible). Returns the degree (19937 on success); P in p[0..PW). */
int or_charpoly(uint64_t *p) {
    const size_t nbits = 2 * DIM + 64;
    const size_t nw = NN + nbits + 2;
    uint32_t *x = (uint32_t *)malloc(nw * sizeof(uint32_t));
    or_seed(5489u, x);
    for (size_t n = 0; n + NN < nw; ++n)
        x[n + NN] = x[n + MM] ^ or_mul_a((x[n] & UPPER) | (x[n + 1] & LOWER));
    /* r holds s reversed: r[j] = s[nbits-1-j] */
    const size_t rwords = nbits / 64 + 2;
    uint64_t *r = (uint64_t *)calloc(rwords, sizeof(uint64_t));
    for (size_t n = 0; n < nbits; ++n)
        if (x[n + 1] & 1u) {
            size_t j = nbits - 1 - n;
            r[j >> 6] |= 1ull << (j & 63);
        }
    uint64_t *C = (uint64_t *)calloc(PW + 1, sizeof(uint64_t));
    uint64_t *B = (uint64_t *)calloc(PW + 1, sizeof(uint64_t));
    uint64_t *T = (uint64_t *)calloc(PW + 1, sizeof(uint64_t));
    C[0] = B[0] = 1;
    size_t L = 0, m = 1;
    for (size_t n = 0; n < nbits; ++n) {
        /* d = sum_{i=0..L} c_i s_{n-i}; s_{n-i} = r[nbits-1-n+i] */
        size_t o = nbits - 1 - n;
        uint64_t acc = 0;
        size_t words = L / 64 + 1;
        for (size_t w = 0; w < words; ++w) {
            size_t bit = o + 64 * w, q = bit >> 6, sh = bit & 63;
            uint64_t seg = r[q] >> sh;
            if (sh && q + 1 < rwords)
                seg |= r[q + 1] << (64 - sh);
            uint64_t cw = C[w];
            if (w == words - 1 && ((L + 1) & 63))
                cw &= (1ull << ((L + 1) & 63)) - 1;
            acc ^= seg & cw;
        }
        int d = __builtin_parityll(acc);
        if (!d) {
            ++m;
            continue;
        }
        memcpy(T, C, (PW + 1) * sizeof(uint64_t));
        /* C ^= B << m */
        size_t ws = m >> 6, bs = m & 63;
        for (long w = PW; w >= (long)ws; --w) {
            size_t src = (size_t)w - ws;
            uint64_t v = B[src] << bs;
            if (bs && src > 0)
                v |= B[src - 1] >> (64 - bs);
            C[w] ^= v;
        }
        if (2 * L <= n) {
            L = n + 1 - L;
            memcpy(B, T, (PW + 1) * sizeof(uint64_t));
            m = 1;
        } else {
            ++m;
        }
    }
    /* P(x) = x^L C(1/x): p_j = c_{L-j} */
    memset(p, 0, PW * sizeof(uint64_t));
    for (size_t j = 0; j <= L && j < (size_t)PW * 64; ++j) {
        size_t i = L - j;
        if ((C[i >> 6] >> (i & 63)) & 1ull)
            p[j >> 6] |= 1ull << (j & 63);
    }
    free(x);
    free(r);
    free(C);
    free(B);
    free(T);
    return (int)L;
}

/* a (up to 2*PW words, degree < 2*DIM) reduced mod p (degree DIM) in place;
 * naive top-down bit elimination. */
static void poly_reduce(uint64_t *a, size_t aw, const uint64_t *p) {
    for (size_t i = aw * 64; i-- > DIM;) {
        if (!((a[i >> 6] >> (i & 63)) & 1ull))
            continue;
        size_t s = i - DIM; /* xor p << s */
        size_t ws = s >> 6, bs = s & 63;
        for (size_t w = 0; w < PW; ++w) {
            uint64_t v = p[w];
            if (!v)
                continue;
            a[w + ws] ^= v << bs;
            if (bs && w + ws + 1 < aw)
                a[w + ws + 1] ^= v >> (64 - bs);
        }
    }
}

/* out = a * b mod p; residues have RW words (degree < DIM). */
void or_poly_mulmod(const uint64_t *a, const uint64_t *b, const uint64_t *p, uint64_t *out) {
    uint64_t prod[2 * PW];
    memset(prod, 0, sizeof prod);
    for (size_t i = 0; i < (size_t)RW * 64; ++i) {
        if (!((a[i >> 6] >> (i & 63)) & 1ull))
            continue;
        size_t ws = i >> 6, bs = i & 63;
        for (size_t w = 0; w < RW; ++w) {
            uint64_t v = b[w];
            prod[w + ws] ^= v << bs;
            if (bs)
                prod[w + ws + 1] ^= v >> (64 - bs);
        }
    }
    poly_reduce(prod, 2 * PW, p);
    memcpy(out, prod, RW * sizeof(uint64_t));
}

void or_poly_sqrmod(const uint64_t *a, const uint64_t *p, uint64_t *out) {
    uint64_t prod[2 * PW];
    memset(prod, 0, sizeof prod);
    for (size_t i = 0; i < (size_t)RW * 64; ++i)
        if ((a[i >> 6] >> (i & 63)) & 1ull)
            prod[(2 * i) >> 6] |= 1ull << ((2 * i) & 63);
    poly_reduce(prod, 2 * PW, p);
    memcpy(out, prod, RW * sizeof(uint64_t));
}

/* out = x * a mod p */
static void poly_mulx(uint64_t *a, const uint64_t *p) {
    uint64_t t[PW];
    memset(t, 0, sizeof t);
    for (size_t w = 0; w < RW; ++w) {
        t[w] |= a[w] << 1;
        t[w + 1] |= a[w] >> 63;
    }
    if ((t[DIM >> 6] >> (DIM & 63)) & 1ull)
        for (size_t w = 0; w < PW; ++w)
            t[w] ^= p[w];
    memcpy(a, t, RW * sizeof(uint64_t));
}

/* x^d mod p for a 64-bit d (left-to-right square and multiply-by-x). */
void or_x_pow_mod(uint64_t d, const uint64_t *p, uint64_t *out) {
    uint64_t r[RW];
    memset(r, 0, sizeof r);
    r[0] = 1;
    for (int b = 63; b >= 0; --b) {
        or_poly_sqrmod(r, p, r);
        if ((d >> b) & 1ull)
            poly_mulx(r, p);
    }
    memcpy(out, r, sizeof r);
}

/* x^(2^q) mod p by q squarings (slow for large q; golden generation only). */
void or_x_pow2_mod(unsigned q, const uint64_t *p, uint64_t *out) {
    uint64_t r[RW];
    memset(r, 0, sizeof r);
    r[0] = 2; /* x */
    for (unsigned i = 0; i < q; ++i)
        or_poly_sqrmod(r, p, r);
    memcpy(out, r, sizeof r);
}

/* p(F) s for a boundary state s: with x_0..x_623 = s and
 * x_{n+624} = x_{n+397} ^ mulA((x_n & UPPER) | (x_{n+1} & LOWER)),
 * F^i s is the window x_i..x_{i+623}, so word j of p(F)s is
 * XOR_{i : p_i = 1} x_{i+j}; word 0 keeps only its live bit (mt19937.cpp:79). */
void or_poly_jump(const uint32_t *in, const uint64_t *poly, uint32_t *out) {
    const size_t n = DIM + NN;
    uint32_t *x = (uint32_t *)malloc(n * sizeof(uint32_t));
    memcpy(x, in, NN * sizeof(uint32_t));
    for (size_t i = 0; i + NN < n; ++i)
        x[i + NN] = x[i + MM] ^ or_mul_a((x[i] & UPPER) | (x[i + 1] & LOWER));
    uint32_t y[NN];
    memset(y, 0, sizeof y);
    for (size_t i = 0; i < DIM; ++i)
        if ((poly[i >> 6] >> (i & 63)) & 1ull)
            for (size_t j = 0; j < NN; ++j)
                y[j] ^= x[i + j];
    y[0] &= UPPER;
    memcpy(out, y, sizeof y);
    free(x);
}

/* ---------------------------------------------------------------- F ---- */
/* MT19937-64 (the std::mt19937_64 parameter set), used only to draw the
 * config-5 jump distances "from seed 7" (BASELINE.json configs[4]). */
void or_mt64(uint64_t seed, uint64_t count, uint64_t *out) {
    uint64_t mt[312];
    mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    int idx = 312;
    for (uint64_t c = 0; c < count; ++c) {
        if (idx >= 312) {
            for (int i = 0; i < 312; ++i) {
                uint64_t x = (mt[i] & 0xFFFFFFFF80000000ull) | (mt[(i + 1) % 312] & 0x7FFFFFFFull);
                uint64_t xa = x >> 1;
                if (x & 1ull)
                    xa ^= 0xB5026F5AA96619E9ull;
                mt[i] = mt[(i + 156) % 312] ^ xa;
            }
            idx = 0;
        }
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        y ^= y >> 43;
        out[c] = y;
    }
}
