// vmt19937/mt19937.hpp -- MT19937 parameters, scalar helpers and the scalar
// generator, source-compatible with the reference's
// proj/include/vmt19937/mt19937.hpp:16-125.
//
// Mt19937 keeps the reference's value semantics (copyable; seeding and
// from_words leave it at the pre-regeneration boundary, cursor == 624) but
// generates on the GPU: the object records its boundary start words plus
// how many blocks it has regenerated and how far into the current block it
// is; next_u32 pulls words from a lazily created single-lane vmt_handle
// (VmtEngine<1> on the device), and words() of an advanced generator is
// the start state jumped by 624 * blocks on the GPU. Copies share nothing:
// a copy creates its own handle and seeks to the same position.
#pragma once

#include <algorithm>
#include <array>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>

#include "vmt19937/detail/abi.hpp"
#include "vmt19937/f2_vector.hpp"

namespace vmt19937 {

// (w, n, m, r, a, d, b, c, u, s, t, l) of the recurrence and tempering
// (mt19937.hpp:16-48). Generic tuples are accepted by the layout helpers
// below; the GPU paths implement the canonical instance only.
struct Mt19937Params {
    unsigned word_bits;
    unsigned state_len;
    unsigned shift;
    unsigned split;
    std::uint32_t matrix_a;
    std::uint32_t temper_d;
    std::uint32_t temper_b;
    std::uint32_t temper_c;
    unsigned temper_u;
    unsigned temper_s;
    unsigned temper_t;
    unsigned temper_l;

    std::uint32_t word_mask() const {
        return word_bits >= 32 ? 0xFFFFFFFFu : ((std::uint32_t(1) << word_bits) - 1u);
    }
    std::uint32_t upper_mask() const { return word_mask() & ~lower_mask(); }
    std::uint32_t lower_mask() const {
        return split >= 32 ? 0xFFFFFFFFu : ((std::uint32_t(1) << split) - 1u) & word_mask();
    }
    std::size_t effective_bits() const { return std::size_t(state_len) * word_bits - split; }

    // mt19937.cpp:7-20: same checks, same exception class and messages.
    void validate() const {
        if (word_bits < 1 || word_bits > 32)
            throw std::invalid_argument("word_bits must be in [1,32]");
        if (state_len < 2)
            throw std::invalid_argument("state_len must be at least 2");
        if (split + 1 > word_bits)
            throw std::invalid_argument("split must be in [0, word_bits-1]");
        if (shift == 0 || shift >= state_len)
            throw std::invalid_argument("shift must be in [1, state_len-1]");
        if ((matrix_a | word_mask()) != word_mask())
            throw std::invalid_argument("matrix_a exceeds the word width");
        if ((upper_mask() | lower_mask()) != word_mask() || (upper_mask() & lower_mask()) != 0)
            throw std::invalid_argument("split masks do not partition the word");
    }

    friend constexpr bool operator==(const Mt19937Params&, const Mt19937Params&) = default;
};

constexpr Mt19937Params mt19937_params() {
    Mt19937Params p{};
    p.word_bits = 32;
    p.state_len = 624;
    p.shift = 397;
    p.split = 31;
    p.matrix_a = 0x9908B0DFu;
    p.temper_d = 0xFFFFFFFFu;
    p.temper_b = 0x9D2C5680u;
    p.temper_c = 0xEFC60000u;
    p.temper_u = 11;
    p.temper_s = 7;
    p.temper_t = 15;
    p.temper_l = 18;
    return p;
}

inline constexpr std::size_t kStateLen = 624;
inline constexpr std::size_t kShift = 397;
inline constexpr std::size_t kEffectiveBits = 19937;

// Scalar output transform and companion-matrix product (mt19937.hpp:61-72),
// kept for callers' known-answer checks; the generators temper on the GPU.
inline std::uint32_t temper(std::uint32_t x) {
    x ^= x >> 11;
    x ^= (x << 7) & 0x9D2C5680u;
    x ^= (x << 15) & 0xEFC60000u;
    return x ^ (x >> 18);
}
inline std::uint32_t mul_a(std::uint32_t u) { return (u >> 1) ^ (0x9908B0DFu & (0u - (u & 1u))); }

class Mt19937 {
public:
    static constexpr std::size_t state_len = kStateLen;

    // init_genrand (mt19937.cpp:22-27), run by vmt_seed_states on the GPU.
    explicit Mt19937(std::uint32_t seed) {
        detail::check(vmt_seed_states(&seed, 1, start_.data(), default_device(), nullptr));
        words_ = start_;
    }

    // mt19937.cpp:29-34: the words become the pre-regeneration boundary.
    static Mt19937 from_words(std::span<const std::uint32_t, state_len> words) {
        Mt19937 s;
        std::copy(words.begin(), words.end(), s.start_.begin());
        s.words_ = s.start_;
        return s;
    }

    Mt19937(const Mt19937& o)
        : start_(o.start_), words_(o.words_), words_block_(o.words_block_), blocks_(o.blocks_),
          cursor_(o.cursor_) {}
    Mt19937& operator=(const Mt19937& o) {
        if (this != &o) {
            start_ = o.start_;
            words_ = o.words_;
            words_block_ = o.words_block_;
            blocks_ = o.blocks_;
            cursor_ = o.cursor_;
            gen_.reset();
        }
        return *this;
    }
    Mt19937(Mt19937&&) noexcept = default;
    Mt19937& operator=(Mt19937&&) noexcept = default;

    std::uint32_t next_u32() {
        if (cursor_ == state_len) {
            ++blocks_;
            cursor_ = 0;
        }
        sync_handle();
        std::uint32_t v;
        detail::check(vmt_next_u32(gen_->get(), &v));
        ++cursor_;
        ++gen_pos_;
        return v;
    }

    // mt19937.cpp:36-55: the next block replaces the state and the cursor
    // rewinds (the rest of a partly consumed block is dropped).
    void regenerate() {
        ++blocks_;
        cursor_ = 0;
    }

    // The current block's untempered words (the start state after blocks_
    // regenerations), materialised on the GPU on demand.
    std::span<const std::uint32_t, state_len> words() const {
        if (words_block_ != blocks_) {
            const std::uint64_t d = std::uint64_t(state_len) * blocks_;
            detail::check(vmt_jump_states(start_.data(), 1, &d, words_.data(), default_device(), nullptr));
            words_block_ = blocks_;
        }
        return std::span<const std::uint32_t, state_len>(words_);
    }
    std::size_t cursor() const { return cursor_; }

private:
    Mt19937() = default;

    // stream position of the next output
    std::uint64_t position() const { return std::uint64_t(state_len) * blocks_ + cursor_ - state_len; }

    void sync_handle() {
        const std::uint64_t pos = position();
        if (!gen_ || !*gen_ || gen_pos_ > pos) {
            vmt_handle h = nullptr;
            detail::check(vmt_create_from_states(start_.data(), 1, default_device(), &h));
            gen_ = std::make_unique<detail::Handle>(h);
            gen_pos_ = 0;
        }
        if (gen_pos_ < pos) {
            detail::check(vmt_skip(gen_->get(), pos - gen_pos_));
            gen_pos_ = pos;
        }
    }

    std::array<std::uint32_t, state_len> start_{};
    mutable std::array<std::uint32_t, state_len> words_{};
    mutable std::uint64_t words_block_ = 0;
    std::uint64_t blocks_ = 0;
    std::size_t cursor_ = state_len;
    std::unique_ptr<detail::Handle> gen_; // copies start without one
    std::uint64_t gen_pos_ = 0;
};

// --- effective-state layout (mt19937.hpp:106-125, mt19937.cpp:57-101) ------
// Bit 0 = bit r of word 0, then the remaining high bits of word 0, then all
// bits of words 1..n-1, LSB first. Host-side format conversion.

inline F2Vector words_to_effective(std::span<const std::uint32_t> words, const Mt19937Params& p) {
    p.validate();
    if (words.size() != p.state_len)
        throw std::invalid_argument("state has the wrong number of words");
    F2Vector v(p.effective_bits());
    std::size_t pos = 0;
    for (unsigned j = p.split; j < p.word_bits; ++j, ++pos)
        if ((words[0] >> j) & 1u)
            v.set(pos);
    for (std::size_t i = 1; i < p.state_len; ++i)
        for (unsigned j = 0; j < p.word_bits; ++j, ++pos)
            if ((words[i] >> j) & 1u)
                v.set(pos);
    return v;
}

inline void effective_to_words(const F2Vector& v, const Mt19937Params& p, std::span<std::uint32_t> words_out) {
    p.validate();
    if (v.size() != p.effective_bits())
        throw std::invalid_argument("effective vector has the wrong length");
    if (words_out.size() != p.state_len)
        throw std::invalid_argument("state has the wrong number of words");
    std::size_t pos = 0;
    std::uint32_t w0 = 0; // the dead low r bits of word 0 come out zero
    for (unsigned j = p.split; j < p.word_bits; ++j, ++pos)
        w0 |= std::uint32_t(v.get(pos)) << j;
    words_out[0] = w0;
    for (std::size_t i = 1; i < p.state_len; ++i) {
        std::uint32_t w = 0;
        for (unsigned j = 0; j < p.word_bits; ++j, ++pos)
            w |= std::uint32_t(v.get(pos)) << j;
        words_out[i] = w;
    }
}

inline F2Vector state_to_effective(const Mt19937& s) {
    if (s.cursor() != Mt19937::state_len)
        throw std::logic_error("effective-state extraction requires the pre-regeneration boundary");
    return words_to_effective(s.words(), mt19937_params());
}

inline Mt19937 effective_to_state(const F2Vector& v) {
    std::array<std::uint32_t, Mt19937::state_len> w{};
    effective_to_words(v, mt19937_params(), w);
    return Mt19937::from_words(w);
}

} // namespace vmt19937
