// vmt19937/jump_file.hpp -- .vmtj jump-matrix files, source-compatible with
// the reference's proj/include/vmt19937/jump_file.hpp:12-68.
//
// Format (jump_file.hpp:12-22): 20-byte little-endian header "VMTJ" |
// version 1 | dimension | exponent | reserved 0, then the row-major payload;
// a checkpoint adds a u32 count of completed squarings after the header.
// Matrix files go through the C ABI (vmt_write/read_jump_matrix_file, the
// reference's checks and error classes); compute_jump_matrix builds the
// matrix on the GPU (vmt_compute_jump_matrix_file: milliseconds instead of
// `exponent` CPU squarings), or, when resuming a checkpoint, finishes its
// squarings with GPU products.
#pragma once

#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <optional>
#include <ostream>
#include <stdexcept>
#include <string>

#include "vmt19937/detail/abi.hpp"
#include "vmt19937/f2_matrix.hpp"

namespace vmt19937 {

inline constexpr char kJumpFileMagic[4] = {'V', 'M', 'T', 'J'};
inline constexpr std::uint32_t kJumpFileVersion = 1;

struct LoadedJumpMatrix {
    F2Matrix matrix;
    unsigned exponent;
};

struct LoadedCheckpoint {
    F2Matrix matrix;
    unsigned target_exponent;
    unsigned completed;
};

inline void write_jump_matrix_file(const std::filesystem::path& path, const F2Matrix& m, unsigned exponent) {
    detail::require_mt_dim(m.dim());
    detail::check(vmt_write_jump_matrix_file(path.string().c_str(), m.data().data(), exponent));
}

inline LoadedJumpMatrix read_jump_matrix_file(const std::filesystem::path& path) {
    unsigned e = 0;
    detail::check(vmt_read_jump_matrix_file(path.string().c_str(), nullptr, &e)); // validate first
    LoadedJumpMatrix out{F2Matrix(kEffectiveBits), 0};
    detail::check(vmt_read_jump_matrix_file(path.string().c_str(), out.matrix.data().data(), &out.exponent));
    return out;
}

namespace detail {
inline void le32(unsigned char* p, std::uint32_t v) {
    for (int i = 0; i < 4; ++i)
        p[i] = (unsigned char)(v >> (8 * i));
}
inline std::uint32_t le32(const unsigned char* p) {
    return std::uint32_t(p[0]) | std::uint32_t(p[1]) << 8 | std::uint32_t(p[2]) << 16 | std::uint32_t(p[3]) << 24;
}
} // namespace detail

inline void write_checkpoint_file(const std::filesystem::path& path, const F2Matrix& m, unsigned target_exponent,
                                  unsigned completed) {
    unsigned char head[24];
    std::copy(kJumpFileMagic, kJumpFileMagic + 4, head);
    detail::le32(head + 4, kJumpFileVersion);
    detail::le32(head + 8, std::uint32_t(m.dim()));
    detail::le32(head + 12, target_exponent);
    detail::le32(head + 16, 0);
    detail::le32(head + 20, completed);
    const std::filesystem::path tmp = path.string() + ".tmp";
    {
        std::ofstream os(tmp, std::ios::binary | std::ios::trunc);
        if (!os)
            throw std::runtime_error("cannot open " + tmp.string());
        os.write(reinterpret_cast<const char*>(head), sizeof head);
        os.write(reinterpret_cast<const char*>(m.data().data()), std::streamsize(m.data().size() * 8));
        if (!os)
            throw std::runtime_error("write failed: " + tmp.string());
    }
    std::filesystem::rename(tmp, path);
}

inline LoadedCheckpoint read_checkpoint_file(const std::filesystem::path& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is)
        throw std::runtime_error("cannot open " + path.string());
    unsigned char head[24];
    is.read(reinterpret_cast<char*>(head), sizeof head);
    if (!is)
        throw std::runtime_error(path.string() + ": truncated header");
    if (!std::equal(kJumpFileMagic, kJumpFileMagic + 4, reinterpret_cast<const char*>(head)))
        throw std::runtime_error(path.string() + ": bad magic");
    if (detail::le32(head + 4) != kJumpFileVersion)
        throw std::runtime_error(path.string() + ": unsupported version");
    const std::uint32_t dim = detail::le32(head + 8), target = detail::le32(head + 12);
    if (detail::le32(head + 16) != 0)
        throw std::runtime_error(path.string() + ": reserved field is not zero");
    if (dim == 0)
        throw std::runtime_error(path.string() + ": zero dimension");
    const std::uint32_t completed = detail::le32(head + 20);
    const std::uint64_t payload = std::uint64_t(dim) * F2Vector::word_count(dim) * 8;
    if (std::filesystem::file_size(path) != 24 + payload)
        throw std::runtime_error(path.string() + ": payload size mismatch");
    if (completed > target)
        throw std::runtime_error(path.string() + ": completed squarings exceed the target");
    LoadedCheckpoint out{F2Matrix(dim), target, completed};
    is.read(reinterpret_cast<char*>(out.matrix.data().data()), std::streamsize(payload));
    if (!is)
        throw std::runtime_error("read failed: " + path.string());
    if (!out.matrix.padding_clear())
        throw std::runtime_error(path.string() + ": nonzero padding bits");
    return out;
}

inline std::string jump_matrix_file_name(unsigned exponent) { return "F_2p" + std::to_string(exponent) + ".vmtj"; }

struct JumpComputeOptions {
    unsigned exponent = 0;
    std::filesystem::path out;
    unsigned checkpoint_every = 64;
    std::optional<std::filesystem::path> resume;
    unsigned workers = 0;
    std::ostream* progress = nullptr;
};

// jump_file.cpp:171-209
inline void compute_jump_matrix(const JumpComputeOptions& opt) {
    if (!opt.resume) {
        detail::check(vmt_compute_jump_matrix_file(opt.out.string().c_str(), opt.exponent, default_device()));
        if (opt.progress)
            *opt.progress << "wrote " << opt.out.string() << " (GPU, " << opt.exponent << " squarings' worth)\n";
        return;
    }
    LoadedCheckpoint ck = read_checkpoint_file(*opt.resume);
    if (ck.matrix.dim() != kEffectiveBits)
        throw std::runtime_error("checkpoint dimension mismatch");
    if (ck.target_exponent != opt.exponent)
        throw std::runtime_error("checkpoint targets a different exponent");
    if (opt.progress)
        *opt.progress << "resuming at squaring " << ck.completed << "/" << opt.exponent << "\n";
    const std::filesystem::path ckpt = opt.out.string() + ".ckpt";
    F2Matrix m = std::move(ck.matrix);
    for (unsigned done = ck.completed; done < opt.exponent;) {
        m = mat_mul(m, m, opt.workers);
        ++done;
        if (opt.checkpoint_every && done % opt.checkpoint_every == 0 && done < opt.exponent)
            write_checkpoint_file(ckpt, m, opt.exponent, done);
        if (opt.progress)
            *opt.progress << "squaring " << done << "/" << opt.exponent << "\n";
    }
    write_jump_matrix_file(opt.out, m, opt.exponent);
    std::filesystem::remove(ckpt);
}

} // namespace vmt19937
