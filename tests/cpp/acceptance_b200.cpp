// Acceptance checks of the GPU-only extensions of the reference-compatible
// C++ headers (include/vmt19937/*.hpp), in the style of
// proj/tests/acceptance.cpp: one
// PASS/FAIL line per criterion, exit code = number of failures. Built and run
// by tests/test_cpp_abi.py (GPU) and compiled (not run) on CPU.
#include <cstdint>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "vmt19937/engine.hpp"
#include "vmt19937/jump_file.hpp"

using namespace vmt19937;

namespace {

int failures = 0;

void criterion(const char* label, const std::function<std::string()>& body) {
    std::string detail;
    bool ok = false;
    try {
        detail = body();
        ok = true;
    } catch (const std::exception& e) {
        detail = e.what();
    }
    std::printf("[%s] %s: %s\n", ok ? "PASS" : "FAIL", label, detail.c_str());
    if (!ok)
        ++failures;
}

void require(bool c, const std::string& what) {
    if (!c)
        throw std::runtime_error(what);
}

// Independent modular-index MT19937 (the recurrence of PAPER.md:137-151),
// test-only, in the spirit of proj/tests/support/mt_oracle.hpp.
struct Scalar {
    std::vector<std::uint32_t> x;
    std::size_t k = 0;
    explicit Scalar(std::uint32_t seed) : x(624) {
        x[0] = seed;
        for (std::uint32_t i = 1; i < 624; ++i)
            x[i] = 1812433253u * (x[i - 1] ^ (x[i - 1] >> 30)) + i;
    }
    std::uint32_t next() {
        const std::uint32_t u = (x[k % 624] & 0x80000000u) | (x[(k + 1) % 624] & 0x7FFFFFFFu);
        std::uint32_t y = x[(k + 397) % 624] ^ (u >> 1) ^ ((u & 1u) ? 0x9908B0DFu : 0u);
        x[k % 624] = y;
        ++k;
        y ^= y >> 11;
        y ^= (y << 7) & 0x9D2C5680u;
        y ^= (y << 15) & 0xEFC60000u;
        return y ^ (y >> 18);
    }
};

} // namespace

int main() {
    criterion("first outputs for the default seed (test_mt19937.cpp:78-83)", [] {
        VmtEngine<1> g(5489);
        require(g.next_u32() == 3499211612u && g.next_u32() == 581869302u && g.next_u32() == 3890346734u,
                "mismatch");
        return std::string("3499211612 581869302 3890346734");
    });
    criterion("interleave identity L=4 q=8 (test_engine.cpp:37-49)", [] {
        const unsigned q = 8, L = 4;
        const std::size_t w = std::size_t(1) << q;
        Scalar s(5489);
        std::vector<std::uint32_t> scalar(w * L);
        for (auto& v : scalar)
            v = s.next();
        VmtEngine<4> g(5489, q);
        for (std::size_t i = 0; i < w; ++i)
            for (std::size_t t = 0; t < L; ++t)
                require(g.next_u32() == scalar[t * w + i], "mismatch at i=" + std::to_string(i));
        return std::string("1024 words");
    });
    criterion("query modes emit identical streams (acceptance.cpp:109-135)", [] {
        const std::size_t n = 100000;
        VmtEngine<8> a(99, 10), b(99, 10), c(99, 10);
        std::vector<std::uint32_t> va(n), vb(n), vc(n + 4992);
        for (auto& v : va)
            v = a.next_u32();
        for (std::size_t i = 0; i < n; i += 16) {
            std::uint32_t buf[16];
            b.next_block16(buf);
            for (std::size_t k = 0; k < 16 && i + k < n; ++k)
                vb[i + k] = buf[k];
        }
        for (std::size_t i = 0; i < n; i += 4992)
            c.next_block_state(vc.data() + i);
        for (std::size_t i = 0; i < n; ++i)
            require(va[i] == vb[i] && va[i] == vc[i], "mismatch at " + std::to_string(i));
        return std::string("100000 words, 3 modes");
    });
    criterion("state-block cadence is enforced (engine.hpp:93-94)", [] {
        VmtEngine<4> g(7, 6);
        std::vector<std::uint32_t> blk(2496);
        g.next_block_state(blk.data());
        g.next_u32();
        try {
            g.next_block_state(blk.data());
        } catch (const std::logic_error&) {
            return std::string("std::logic_error");
        }
        throw std::runtime_error("no exception");
    });
    criterion("copies continue identically (VmtEngine value semantics)", [] {
        VmtEngine<16> a(77, 12);
        for (int i = 0; i < 12345; ++i)
            a.next_u32();
        VmtEngine<16> b = a;
        for (int i = 0; i < 30000; ++i)
            require(a.next_u32() == b.next_u32(), "copy diverges at " + std::to_string(i));
        Mt19937 s(5489);
        for (int i = 0; i < 700; ++i)
            s.next_u32();
        Mt19937 t = s;
        require(s.cursor() == 76 && t.cursor() == 76, "cursor");
        for (int i = 0; i < 2000; ++i)
            require(s.next_u32() == t.next_u32(), "scalar copy diverges at " + std::to_string(i));
        return std::string("engine and scalar copies");
    });
    criterion("interleaved_state() span and state_data() (engine.hpp:100-102)", [] {
        VmtEngine<8> g(5489, 10);
        std::span<const std::uint32_t, VmtEngine<8>::state_words> s0 = g.interleaved_state();
        require(s0[0] == 5489u, "lane 0 word 0 keeps the raw seed before the first query");
        std::vector<std::uint32_t> blk(VmtEngine<8>::state_words);
        g.next_block_state(blk.data());
        const std::uint32_t* p = g.state_data();
        for (std::size_t i = 0; i < blk.size(); ++i)
            require(temper(p[i]) == blk[i], "state words temper to the block at " + std::to_string(i));
        return std::string("state words == untempered block");
    });
    criterion("bad lane count is invalid_argument (engine.hpp:29-32)", [] {
        try {
            VmtGenerator g(1, VmtConfig(3, QueryMode::kSingle, 4));
        } catch (const std::invalid_argument&) {
            return std::string("std::invalid_argument");
        }
        throw std::runtime_error("no exception");
    });
    criterion("Appendix A checksum L=16 q=16 2^26 words (bulk host fill + fused XOR)", [] {
        const std::uint64_t n = std::uint64_t(1) << 26;
        VmtEngine<16> g(5489, 16);
        std::vector<std::uint32_t> out(n);
        g.fill_u32(out.data(), n);
        std::uint32_t x = 0;
        for (auto v : out)
            x ^= v;
        require(x == 0x5E141D5Bu, "stored checksum");
        VmtEngine<16> h(5489, 16);
        require(h.checksum_xor(n) == 0x5E141D5Bu, "fused checksum");
        return std::string("0x5E141D5B");
    });
    criterion("full-period default de-phasing starts at the scalar first output", [] {
        VmtEngine<32> g(5489, VMT_FULL_PERIOD);
        require(g.jump_exponent() == 19932, "exponent");
        require(g.next_u32() == 3499211612u, "first output");
        return std::string("q=19932");
    });
    criterion("reference constructor VmtEngine<M>(seed, F2Matrix, q) + .vmtj round trip", [] {
        const unsigned q = 10;
        const F2Matrix B = jump_matrix_pow2(q);
        const std::string path = "/tmp/acceptance_b200_" + jump_matrix_file_name(q);
        JumpComputeOptions opt;
        opt.exponent = q;
        opt.out = path;
        compute_jump_matrix(opt);
        const LoadedJumpMatrix m = read_jump_matrix_file(path);
        std::remove(path.c_str());
        require(m.exponent == q && m.matrix == B, "file round trip");
        VmtEngine<8> a(4242, m.matrix, m.exponent), b(4242, q);
        for (int i = 0; i < 20000; ++i)
            require(a.next_u32() == b.next_u32(), "matrix vs polynomial de-phasing at " + std::to_string(i));
        return std::string("q=10, 20000 words");
    });
    std::printf("%d failure(s)\n", failures);
    return failures;
}
