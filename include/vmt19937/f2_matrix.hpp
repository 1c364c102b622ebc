// vmt19937/f2_matrix.hpp -- dense GF(2) matrices, source-compatible with the
// reference's proj/include/vmt19937/f2_matrix.hpp:13-87.
//
// F2Matrix is the same host container (row-major, rows packed like
// F2Vector, the .vmtj payload layout). The products run on the GPU through
// the C ABI (vmt_vec_mat_mul: each output row is the XOR of the rows of b
// selected by a row of a / by v), and build_transition_matrix is F^1 from
// vmt_jump_matrix. The GPU implements the MT19937 dimension (19937); other
// dimensions are rejected with std::invalid_argument.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <vector>

#include "vmt19937/detail/abi.hpp"
#include "vmt19937/f2_vector.hpp"
#include "vmt19937/mt19937.hpp"

namespace vmt19937 {

class F2Matrix {
public:
    F2Matrix() = default;
    explicit F2Matrix(std::size_t dim)
        : dim_(dim), row_words_(F2Vector::word_count(dim)), words_(dim * row_words_, 0) {}

    static F2Matrix identity(std::size_t dim) {
        F2Matrix m(dim);
        for (std::size_t i = 0; i < dim; ++i)
            m.set(i, i);
        return m;
    }

    std::size_t dim() const { return dim_; }
    std::size_t row_words() const { return row_words_; }

    std::span<std::uint64_t> row(std::size_t i) { return {words_.data() + i * row_words_, row_words_}; }
    std::span<const std::uint64_t> row(std::size_t i) const { return {words_.data() + i * row_words_, row_words_}; }

    bool get(std::size_t r, std::size_t c) const { return (words_[r * row_words_ + c / 64] >> (c % 64)) & 1u; }
    void set(std::size_t r, std::size_t c, bool v = true) {
        std::uint64_t& w = words_[r * row_words_ + c / 64];
        const std::uint64_t m = std::uint64_t(1) << (c % 64);
        w = v ? (w | m) : (w & ~m);
    }

    F2Vector row_vector(std::size_t i) const {
        F2Vector v(dim_);
        std::copy(row(i).begin(), row(i).end(), v.words().begin());
        return v;
    }
    void set_row(std::size_t i, const F2Vector& v) {
        if (v.size() != dim_)
            throw std::invalid_argument("row length does not match matrix dimension");
        std::copy(v.words().begin(), v.words().end(), row(i).begin());
    }

    std::span<const std::uint64_t> data() const { return words_; }
    std::span<std::uint64_t> data() { return words_; }

    bool padding_clear() const {
        const std::size_t tail = dim_ % 64;
        if (tail == 0)
            return true;
        for (std::size_t i = 0; i < dim_; ++i)
            if (row(i).back() >> tail)
                return false;
        return true;
    }

    friend bool operator==(const F2Matrix&, const F2Matrix&) = default;

private:
    std::size_t dim_ = 0;
    std::size_t row_words_ = 0;
    std::vector<std::uint64_t> words_;
};

namespace detail {
inline void require_mt_dim(std::size_t dim) {
    if (dim != kEffectiveBits)
        throw std::invalid_argument("the B200 build multiplies 19937-dimension (MT19937) matrices only");
}
} // namespace detail

// v * M (f2_matrix.cpp:119-136) on the GPU.
inline F2Vector vec_mat_mul(const F2Vector& v, const F2Matrix& m) {
    if (v.size() != m.dim())
        throw std::invalid_argument("vector length does not match matrix dimension");
    detail::require_mt_dim(m.dim());
    F2Vector out(m.dim());
    detail::check(vmt_vec_mat_mul(v.words().data(), 1, m.data().data(), out.words().data(), default_device(),
                                  nullptr));
    return out;
}

// a * b (f2_matrix.cpp:138-168): every row of a is one vector of a single
// batched GPU product. `workers` is accepted for source compatibility.
inline F2Matrix mat_mul(const F2Matrix& a, const F2Matrix& b, unsigned workers = 0) {
    (void)workers;
    if (a.dim() != b.dim())
        throw std::invalid_argument("matrix dimensions do not match");
    detail::require_mt_dim(a.dim());
    F2Matrix c(a.dim());
    detail::check(vmt_vec_mat_mul(a.data().data(), a.dim(), b.data().data(), c.data().data(), default_device(),
                                  nullptr));
    return c;
}

// m^(2^q) by q squarings (f2_matrix.cpp:170-177), the sink seeing every rung.
using SquaringSink = std::function<void(const F2Matrix&, unsigned completed)>;
inline F2Matrix mat_pow2(F2Matrix m, unsigned q, const SquaringSink& sink = {}, unsigned workers = 0) {
    for (unsigned i = 0; i < q; ++i) {
        m = mat_mul(m, m, workers);
        if (sink)
            sink(m, i + 1);
    }
    return m;
}

// One-step transition matrix F (f2_matrix.cpp:179-228) for the canonical
// parameters: row i is basis state e_i advanced one step, computed on the GPU
// (byte-identical to the reference's structural construction).
inline F2Matrix build_transition_matrix(const Mt19937Params& p) {
    p.validate();
    if (!(p == mt19937_params()))
        throw std::invalid_argument("the B200 build implements the canonical MT19937 parameters only");
    F2Matrix f(kEffectiveBits);
    detail::check(vmt_jump_matrix(1, 0, f.data().data(), default_device(), nullptr));
    return f;
}

// Extensions (no reference counterpart): F^(2^q) and F^d for any 64-bit d,
// built directly on the GPU as 19937 basis-state polynomial jumps --
// jump_matrix_pow2(q) == mat_pow2(build_transition_matrix(mt19937_params()), q)
// byte for byte, including the full-period exponents the reference cannot
// reach (~50 h of squarings).
inline F2Matrix jump_matrix_pow2(unsigned q, int device = default_device()) {
    F2Matrix m(kEffectiveBits);
    detail::check(vmt_jump_matrix_pow2(q, m.data().data(), device, nullptr));
    return m;
}
inline F2Matrix jump_matrix(std::uint64_t d, int device = default_device()) {
    F2Matrix m(kEffectiveBits);
    detail::check(vmt_jump_matrix(d, 0, m.data().data(), device, nullptr));
    return m;
}

} // namespace vmt19937
