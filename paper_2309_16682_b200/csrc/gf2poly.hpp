// Host-side jump-polynomial arithmetic for VMT19937 on B200.
//
// The reference de-phases lanes with a dense GF(2) jump MATRIX (19937^2 bits,
// proj/src/jump.cpp:27-53, proj/src/f2_matrix.cpp:119-177) that takes ~50 h to
// build at full period. This build uses the equivalent jump
// POLYNOMIAL instead: with P the characteristic polynomial of
// the one-step transition F, F^d = (x^d mod P)(F), so a d-step jump of a state
// s is p(F)s with p = x^d mod P -- computed here on the host, applied on the
// GPU by the convolution kernel in vmt_kernels.cuh.
//
// Representation: bit i of a little-endian u64 array is the coefficient of
// x^i. Residues mod P have degree < 19937 and fit kPolyWords = 312 words.
#pragma once

#include <cstdint>
#include <mutex>
#include <vector>

namespace vmt_b200 {

constexpr int kDeg = 19937;        // deg P = effective state bits (mt19937.hpp:57)
constexpr int kPolyWords = 312;    // words of a residue (F2Vector::word_count)
constexpr int kFullWords = 313;    // words of P itself (bit 19937 set)

using Poly = std::vector<std::uint64_t>; // kPolyWords words (residue) unless noted

class Gf2Field {
public:
    // The process-wide instance; first use runs Berlekamp-Massey (~40 ms).
    static Gf2Field& instance();

    const std::vector<std::uint64_t>& charpoly() const { return p_; } // kFullWords

    Poly one() const;
    Poly x_pow(std::uint64_t d) const;                          // x^d mod P
    Poly x_pow128(std::uint64_t lo, std::uint64_t hi) const;     // x^(hi*2^64+lo) mod P
    Poly x_pow2(unsigned q) const;                               // x^(2^q) mod P
    Poly mulmod(const Poly& a, const Poly& b) const;
    Poly sqrmod(const Poly& a) const;
    Poly powmod(const Poly& a, std::uint64_t e) const;
    Poly sqrtmod(const Poly& a) const;                           // a^(2^(kDeg-1))
    // True when the product uses the carry-less-multiply instruction.
    static bool has_clmul();

private:
    Gf2Field();
    void barrett_reduce(const std::uint64_t* a /*2*kFullWords*/, std::uint64_t* out) const;

    std::vector<std::uint64_t> p_;   // P, kFullWords
    std::vector<std::uint64_t> mu_;  // floor(x^(2*kDeg) / P), kFullWords
    Poly sqrt_x_;                    // x^(2^(kDeg-1)) mod P
    mutable std::mutex cache_mu_;
    mutable std::vector<Poly> pow2_cache_; // index q -> x^(2^q) (lazily filled)
};

// Raw helpers (exposed for tests through the C ABI).
void clmul_mul(const std::uint64_t* a, int aw, const std::uint64_t* b, int bw, std::uint64_t* out);

} // namespace vmt_b200
