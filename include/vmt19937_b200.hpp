// vmt19937_b200.hpp -- C++ mirror of the reference's generator interface
// (proj/include/vmt19937/engine.hpp, jump.hpp) over the C ABI in
// vmt19937_b200.h. Reference code written against VmtEngine / VmtGenerator /
// JumpSpec / F2Matrix / the .vmtj functions compiles against this header:
// the matrix constructors de-phase with the caller's matrix on the GPU
// (make_dephased_states), the matrix-free ones with the jump polynomial.
//
// Errors are rethrown as the reference's exception classes:
//   VMT_EINVAL -> std::invalid_argument, VMT_ESTATE -> std::logic_error,
//   VMT_EIO / VMT_ECUDA / VMT_ENOMEM -> std::runtime_error.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "vmt19937_b200.h"

namespace vmt19937_b200 {

inline void check(int rc) {
    if (rc == VMT_OK)
        return;
    const std::string msg = vmt_last_error();
    if (rc == VMT_EINVAL)
        throw std::invalid_argument(msg);
    if (rc == VMT_ESTATE)
        throw std::logic_error(msg);
    throw std::runtime_error(std::string(vmt_status_string(rc)) + ": " + msg);
}

inline constexpr std::size_t kStateLen = 624;        // mt19937.hpp:55
inline constexpr std::size_t kEffectiveBits = 19937; // mt19937.hpp:57

enum class QueryMode { kSingle = VMT_QUERY_SINGLE, kBlock16 = VMT_QUERY_BLOCK16, kStateBlock = VMT_QUERY_STATE_BLOCK };

// jump.hpp:13-21
struct JumpSpec {
    unsigned exponent;
    unsigned lanes;
    void validate() const {
        if (lanes < 1 || (lanes & (lanes - 1)))
            throw std::invalid_argument("lanes must be a power of two");
    }
    bool is_full_period_split() const { return exponent == full_period_exponent(lanes); }
    static JumpSpec full_period_split(unsigned lanes) {
        JumpSpec s{full_period_exponent(lanes), lanes};
        s.validate();
        return s;
    }
    static unsigned full_period_exponent(unsigned lanes) { return vmt_full_period_exponent(lanes); }
};

// engine.hpp:18-33 (lanes up to 32)
struct VmtConfig {
    unsigned lanes = 1;
    QueryMode mode = QueryMode::kSingle;
    unsigned jump_exponent;
    explicit VmtConfig(unsigned lanes_, QueryMode mode_ = QueryMode::kSingle)
        : lanes(lanes_), mode(mode_), jump_exponent(JumpSpec::full_period_exponent(lanes_)) {}
    VmtConfig(unsigned lanes_, QueryMode mode_, unsigned q) : lanes(lanes_), mode(mode_), jump_exponent(q) {}
    void validate() const {
        if (lanes != 1 && lanes != 2 && lanes != 4 && lanes != 8 && lanes != 16 && lanes != 32)
            throw std::invalid_argument("lanes must be one of 1, 2, 4, 8, 16, 32");
    }
};

// Dense 19937 x 19937 GF(2) matrix (f2_matrix.hpp:13-61), row-major payload
// of 312 u64 per row -- the .vmtj layout. Only the MT19937 dimension.
class F2Matrix {
public:
    F2Matrix() = default;
    static F2Matrix zeros() {
        F2Matrix m;
        m.words_.assign(VMT_MATRIX_WORDS, 0);
        return m;
    }
    std::size_t dim() const { return words_.empty() ? 0 : VMT_MATRIX_DIM; }
    std::size_t row_words() const { return VMT_MATRIX_ROW_WORDS; }
    const std::uint64_t* row(std::size_t i) const { return words_.data() + i * VMT_MATRIX_ROW_WORDS; }
    bool get(std::size_t r, std::size_t c) const { return (row(r)[c >> 6] >> (c & 63)) & 1u; }
    const std::vector<std::uint64_t>& data() const { return words_; }
    std::vector<std::uint64_t>& data() { return words_; }
    friend bool operator==(const F2Matrix& a, const F2Matrix& b) { return a.words_ == b.words_; }

private:
    std::vector<std::uint64_t> words_;
};

// F^(2^q) == mat_pow2(build_transition_matrix(), q) (f2_matrix.cpp:138-228),
// computed on the GPU.
inline F2Matrix jump_matrix_pow2(unsigned q, int device = 0) {
    F2Matrix m = F2Matrix::zeros();
    check(vmt_jump_matrix_pow2(q, m.data().data(), device, nullptr));
    return m;
}
// F^d for any 64-bit d.
inline F2Matrix jump_matrix(std::uint64_t d, int device = 0) {
    F2Matrix m = F2Matrix::zeros();
    check(vmt_jump_matrix(d, 0, m.data().data(), device, nullptr));
    return m;
}

// jump_file.hpp:26-45
struct LoadedJumpMatrix {
    F2Matrix matrix;
    unsigned exponent;
};
inline void write_jump_matrix_file(const std::string& path, const F2Matrix& m, unsigned exponent) {
    check(vmt_write_jump_matrix_file(path.c_str(), m.data().data(), exponent));
}
inline LoadedJumpMatrix read_jump_matrix_file(const std::string& path) {
    LoadedJumpMatrix out{F2Matrix::zeros(), 0};
    check(vmt_read_jump_matrix_file(path.c_str(), out.matrix.data().data(), &out.exponent));
    return out;
}
inline std::string jump_matrix_file_name(unsigned exponent) { return "F_2p" + std::to_string(exponent) + ".vmtj"; }
// compute_jump_matrix (jump_file.cpp:171-209) without checkpoints: the GPU
// needs milliseconds, not hours.
inline void compute_jump_matrix(unsigned exponent, const std::string& out, int device = 0) {
    check(vmt_compute_jump_matrix_file(out.c_str(), exponent, device));
}

// Runtime-lane-count generator (engine.hpp:160-207). One owner per
// instance; movable, not copyable.
class VmtGenerator {
public:
    VmtGenerator(std::uint32_t seed, const VmtConfig& cfg, int device = 0) {
        cfg.validate();
        check(vmt_create(seed, cfg.lanes, cfg.jump_exponent, device, &h_));
    }
    // VmtGenerator(seed, cfg, jump_matrix) (engine.hpp:162-163): matrix de-phasing
    VmtGenerator(std::uint32_t seed, const VmtConfig& cfg, const F2Matrix& jump_matrix, int device = 0) {
        cfg.validate();
        check(vmt_create_from_matrix(seed, cfg.lanes, jump_matrix.dim() ? jump_matrix.data().data() : nullptr,
                                     cfg.jump_exponent, device, &h_));
    }
    // lane count 1 needs no jump (engine.hpp:164-167)
    explicit VmtGenerator(std::uint32_t seed) : VmtGenerator(seed, VmtConfig(1, QueryMode::kSingle, 0)) {}
    VmtGenerator(const VmtGenerator&) = delete;
    VmtGenerator& operator=(const VmtGenerator&) = delete;
    VmtGenerator(VmtGenerator&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    VmtGenerator& operator=(VmtGenerator&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    ~VmtGenerator() {
        if (h_)
            vmt_destroy(h_);
    }

    std::uint32_t next_u32() {
        std::uint32_t v;
        check(vmt_next_u32(h_, &v));
        return v;
    }
    void next_block16(std::uint32_t* out) { check(vmt_next_block16(h_, out)); }
    void next_block_state(std::uint32_t* out) { check(vmt_next_block_state(h_, out)); }
    unsigned lanes() const { return vmt_lanes(h_); }
    std::size_t state_words() const { return static_cast<std::size_t>(vmt_state_words(h_)); }
    unsigned jump_exponent() const { return vmt_jump_exponent(h_); }
    std::vector<std::uint32_t> interleaved_state() const {
        std::vector<std::uint32_t> s(state_words());
        check(vmt_export_state(h_, s.data()));
        return s;
    }

    // Bulk output (device or host destination, any length).
    void fill_u32(std::uint32_t* dst, std::uint64_t n, void* stream = nullptr) {
        check(vmt_fill_u32(h_, dst, n, stream));
    }
    void fill_f32(float* dst, std::uint64_t n, void* stream = nullptr) {
        check(vmt_fill_f32(h_, dst, n, VMT_F32_24, stream));
    }
    void fill_f64(double* dst, std::uint64_t n, int rule = VMT_F64_32, void* stream = nullptr) {
        check(vmt_fill_f64(h_, dst, n, rule, stream));
    }
    std::uint32_t checksum_xor(std::uint64_t n, void* stream = nullptr) {
        std::uint32_t x;
        check(vmt_checksum_xor(h_, n, &x, stream));
        return x;
    }
    void skip(std::uint64_t d) { check(vmt_skip(h_, d)); }
    void seek(std::uint64_t pos) { check(vmt_seek(h_, pos)); }
    void synchronize() { check(vmt_synchronize(h_)); }
    vmt_handle handle() const { return h_; }

private:
    vmt_handle h_ = nullptr;
};

// Fixed-lane spelling (engine.hpp:41-68).
template <int M>
class VmtEngine : public VmtGenerator {
    static_assert(M == 1 || M == 2 || M == 4 || M == 8 || M == 16 || M == 32, "lanes must be 1..32");

public:
    static constexpr int lanes_v = M;
    static constexpr std::size_t state_words_v = kStateLen * M;
    static constexpr std::size_t buffer_words = 16;
    VmtEngine(std::uint32_t seed, unsigned jump_exponent, int device = 0)
        : VmtGenerator(seed, VmtConfig(M, QueryMode::kSingle, jump_exponent), device) {}
    // the reference's constructor (engine.hpp:54): de-phase with B = jump_matrix
    VmtEngine(std::uint32_t seed, const F2Matrix& jump_matrix, unsigned jump_exponent, int device = 0)
        : VmtGenerator(seed, VmtConfig(M, QueryMode::kSingle, jump_exponent), jump_matrix, device) {}
    // library-default (full-period) de-phasing on device 0; VmtEngine<1>(seed)
    // is engine.hpp:66-68
    explicit VmtEngine(std::uint32_t seed)
        : VmtGenerator(seed, VmtConfig(M, QueryMode::kSingle, M == 1 ? 0u : JumpSpec::full_period_exponent(M))) {}
};

} // namespace vmt19937_b200
