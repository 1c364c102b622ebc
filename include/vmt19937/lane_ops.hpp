// vmt19937/lane_ops.hpp -- the lane-register vocabulary of the reference's
// proj/include/vmt19937/lane_ops.hpp (Ops::Reg, load/store/broadcast/bxor,
// DefaultLanesT<M>, has_simd_lanes<N>) for host code written against it,
// e.g. the running XOR fold of proj/src/bench.cpp:37-58.
//
// The B200 build generates on the GPU, so it carries no CPU SIMD generation
// backend: DefaultLanesT<M> is a plain M-word array type (the compiler may
// vectorise it) offering the bitwise operations host callers use, and
// has_simd_lanes<N>() is false (criteria that assume CPU SIMD backends, e.g.
// acceptance.cpp's throughput ratios, report instead of asserting).
#pragma once

#include <array>
#include <cstdint>
#include <cstring>

namespace vmt19937 {

template <int M>
struct HostLanes {
    static constexpr int lanes = M;
    using Reg = std::array<std::uint32_t, M>;

    static Reg load(const std::uint32_t* p) {
        Reg r;
        std::memcpy(r.data(), p, sizeof(Reg));
        return r;
    }
    static Reg loadu(const std::uint32_t* p) { return load(p); }
    static void store(std::uint32_t* p, const Reg& v) { std::memcpy(p, v.data(), sizeof(Reg)); }
    static void storeu(std::uint32_t* p, const Reg& v) { store(p, v); }
    static Reg broadcast(std::uint32_t x) {
        Reg r;
        r.fill(x);
        return r;
    }
    template <class F>
    static Reg zip(const Reg& a, const Reg& b, F f) {
        Reg r;
        for (int i = 0; i < M; ++i)
            r[i] = f(a[i], b[i]);
        return r;
    }
    static Reg bxor(const Reg& a, const Reg& b) { return zip(a, b, [](std::uint32_t x, std::uint32_t y) { return x ^ y; }); }
    static Reg band(const Reg& a, const Reg& b) { return zip(a, b, [](std::uint32_t x, std::uint32_t y) { return x & y; }); }
    static Reg bor(const Reg& a, const Reg& b) { return zip(a, b, [](std::uint32_t x, std::uint32_t y) { return x | y; }); }
    template <int S>
    static Reg shr(const Reg& a) {
        Reg r;
        for (int i = 0; i < M; ++i)
            r[i] = a[i] >> S;
        return r;
    }
    template <int S>
    static Reg shl(const Reg& a) {
        Reg r;
        for (int i = 0; i < M; ++i)
            r[i] = a[i] << S;
        return r;
    }
};

template <int M>
using DefaultLanesT = HostLanes<M>;

template <int N>
constexpr bool has_simd_lanes() {
    return false;
}

} // namespace vmt19937
