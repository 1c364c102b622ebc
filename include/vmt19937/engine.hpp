// vmt19937/engine.hpp -- the VMT19937 generator, source-compatible with the
// reference's proj/include/vmt19937/engine.hpp:13-209: QueryMode, VmtConfig,
// VmtEngine<M, Ops> (static constexpr lanes / state_words / buffer_words,
// the (seed, jump_matrix, jump_exponent) constructor, next_u32 /
// next_block16 / next_block_state, jump_exponent(), interleaved_state() as a
// std::span<const std::uint32_t, state_words>, state_data()) and the
// runtime-lane VmtGenerator.
//
// The engine is a handle to a GPU generator (vmt19937_b200.h): de-phasing,
// regeneration and tempering run as sm_100a kernels; queries are served from
// a pinned staging buffer the GPU refills. The interleaved state is mirrored
// into the object on request, so interleaved_state() / state_data() return
// host memory that stays valid until the next call on the engine.
//
// Differences from the reference, all extensions: lanes may also be 32;
// every constructor takes an optional CUDA device; a matrix-free
// (seed, jump_exponent) constructor de-phases with the jump polynomial on the
// GPU (any exponent, VMT_FULL_PERIOD for the library default); bulk
// fill_u32 / fill_f32 / fill_f64 / checksum_xor / skip / seek.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

#include "vmt19937/detail/abi.hpp"
#include "vmt19937/f2_matrix.hpp"
#include "vmt19937/jump.hpp"
#include "vmt19937/lane_ops.hpp"
#include "vmt19937/mt19937.hpp"

namespace vmt19937 {

enum class QueryMode { kSingle, kBlock16, kStateBlock };

// engine.hpp:18-33 (lanes up to 32)
struct VmtConfig {
    unsigned lanes = 1;
    QueryMode mode = QueryMode::kSingle;
    unsigned jump_exponent;

    VmtConfig(unsigned lanes_, QueryMode mode_ = QueryMode::kSingle)
        : lanes(lanes_), mode(mode_), jump_exponent(JumpSpec::full_period_exponent(lanes_)) {}
    VmtConfig(unsigned lanes_, QueryMode mode_, unsigned jump_exponent_)
        : lanes(lanes_), mode(mode_), jump_exponent(jump_exponent_) {}

    void validate() const {
        if (lanes != 1 && lanes != 2 && lanes != 4 && lanes != 8 && lanes != 16 && lanes != 32)
            throw std::invalid_argument("lanes must be one of 1, 2, 4, 8, 16, 32");
    }
};

namespace detail {

// The GPU generator behind VmtEngine and VmtGenerator.
class GpuGenerator {
public:
    GpuGenerator() = default;
    explicit GpuGenerator(vmt_handle h) : h_(h) {}
    GpuGenerator(const GpuGenerator& o) {
        if (o.h_) {
            vmt_handle c = nullptr;
            check(vmt_clone(o.h_.get(), &c));
            h_ = Handle(c);
        }
    }
    GpuGenerator& operator=(const GpuGenerator& o) {
        if (this != &o)
            *this = GpuGenerator(o);
        return *this;
    }
    GpuGenerator(GpuGenerator&&) noexcept = default;
    GpuGenerator& operator=(GpuGenerator&&) noexcept = default;

    static vmt_handle from_matrix(std::uint32_t seed, unsigned lanes, const F2Matrix& m, unsigned q, int device) {
        if (lanes > 1 && m.dim() != kEffectiveBits)
            throw std::invalid_argument("jump matrix dimension mismatch");
        vmt_handle h = nullptr;
        check(vmt_create_from_matrix(seed, lanes, lanes > 1 ? m.data().data() : nullptr, q, device, &h));
        return h;
    }
    static vmt_handle from_poly(std::uint32_t seed, unsigned lanes, unsigned q, int device) {
        vmt_handle h = nullptr;
        check(vmt_create(seed, lanes, q, device, &h));
        return h;
    }

    std::uint32_t next_u32() {
        std::uint32_t v;
        check(vmt_next_u32(h_.get(), &v));
        return v;
    }
    void next_block16(std::uint32_t* out) { check(vmt_next_block16(h_.get(), out)); }
    void next_block_state(std::uint32_t* out) { check(vmt_next_block_state(h_.get(), out)); }
    unsigned jump_exponent() const { return vmt_jump_exponent(h_.get()); }
    void export_state(std::uint32_t* out) const { check(vmt_export_state(h_.get(), out)); }

    void fill_u32(std::uint32_t* dst, std::uint64_t n, void* stream = nullptr) {
        check(vmt_fill_u32(h_.get(), dst, n, stream));
    }
    void fill_f32(float* dst, std::uint64_t n, void* stream = nullptr) {
        check(vmt_fill_f32(h_.get(), dst, n, VMT_F32_24, stream));
    }
    void fill_f64(double* dst, std::uint64_t n, int rule = VMT_F64_32, void* stream = nullptr) {
        check(vmt_fill_f64(h_.get(), dst, n, rule, stream));
    }
    std::uint32_t checksum_xor(std::uint64_t n, void* stream = nullptr) {
        std::uint32_t x;
        check(vmt_checksum_xor(h_.get(), n, &x, stream));
        return x;
    }
    void skip(std::uint64_t d) { check(vmt_skip(h_.get(), d)); }
    void seek(std::uint64_t pos) { check(vmt_seek(h_.get(), pos)); }
    std::uint64_t position() const { return vmt_position(h_.get()); }
    void synchronize() { check(vmt_synchronize(h_.get())); }
    vmt_handle handle() const { return h_.get(); }

private:
    Handle h_;
};

} // namespace detail

template <int M, class Ops = DefaultLanesT<M>>
class alignas(64) VmtEngine : public detail::GpuGenerator {
    static_assert(M == 1 || M == 2 || M == 4 || M == 8 || M == 16 || M == 32, "lanes must be 1, 2, 4, 8, 16 or 32");
    static_assert(Ops::lanes == M, "backend lane count mismatch");

public:
    static constexpr int lanes = M;
    static constexpr std::size_t state_words = kStateLen * M;
    static constexpr std::size_t buffer_words = 16;

    // engine.hpp:54-63: de-phase M copies of Mt19937(seed) with the caller's
    // matrix B = F^(2^q) (make_dephased_states, on the GPU).
    VmtEngine(std::uint32_t seed, const F2Matrix& jump_matrix, unsigned jump_exponent,
              int device = default_device())
        : GpuGenerator(from_matrix(seed, M, jump_matrix, jump_exponent, device)) {}

    // engine.hpp:66-68
    explicit VmtEngine(std::uint32_t seed)
        requires(M == 1)
        : GpuGenerator(from_poly(seed, 1, 0, default_device())) {}

    // Extension: de-phasing by the jump polynomial x^(2^q) mod P on the GPU
    // (no matrix; any q, VMT_FULL_PERIOD = JumpSpec::full_period_exponent(M)).
    VmtEngine(std::uint32_t seed, unsigned jump_exponent, int device = default_device())
        : GpuGenerator(from_poly(seed, M, jump_exponent, device)) {}

    // interleaved_state (engine.hpp:100): the state after ceil(position /
    // state_words) regenerations, copied into this object.
    std::span<const std::uint32_t, state_words> interleaved_state() const {
        export_state(mirror_->data());
        return std::span<const std::uint32_t, state_words>(*mirror_);
    }
    const std::uint32_t* state_data() const { return interleaved_state().data(); }

private:
    struct Mirror : std::array<std::uint32_t, state_words> {};
    std::unique_ptr<Mirror> mirror_ = std::make_unique<Mirror>();

public:
    VmtEngine(const VmtEngine& o) : GpuGenerator(o) {}
    VmtEngine& operator=(const VmtEngine& o) {
        GpuGenerator::operator=(o);
        return *this;
    }
    VmtEngine(VmtEngine&&) noexcept = default;
    VmtEngine& operator=(VmtEngine&&) noexcept = default;
};

// engine.hpp:160-207, any of 1, 2, 4, 8, 16, 32 lanes at run time.
class VmtGenerator : public detail::GpuGenerator {
public:
    VmtGenerator(std::uint32_t seed, const VmtConfig& cfg, const F2Matrix& jump_matrix,
                 int device = default_device())
        : GpuGenerator((cfg.validate(), from_matrix(seed, cfg.lanes, jump_matrix, cfg.jump_exponent, device))) {}

    explicit VmtGenerator(std::uint32_t seed) : GpuGenerator(from_poly(seed, 1, 0, default_device())) {}

    // Extension: polynomial de-phasing with cfg.jump_exponent.
    VmtGenerator(std::uint32_t seed, const VmtConfig& cfg, int device = default_device())
        : GpuGenerator((cfg.validate(), from_poly(seed, cfg.lanes, cfg.jump_exponent, device))) {}

    unsigned lanes() const { return vmt_lanes(handle()); }
    std::size_t state_words() const { return std::size_t(vmt_state_words(handle())); }
    std::vector<std::uint32_t> interleaved_state() const {
        std::vector<std::uint32_t> s(state_words());
        export_state(s.data());
        return s;
    }
};

} // namespace vmt19937
