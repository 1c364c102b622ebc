// sm_100a kernels for VMT19937 (arXiv 2309.16682) on B200.
//
//   vmt_gen_kernel   twist + temper + emit, the hot path. Replaces
//                    VmtEngine::regenerate + temper_words (engine.hpp:110-142)
//                    and the lane backends' twist/temper (lane_ops.hpp:81-93,
//                    184-195).
//   vmt_jump_kernel  p(F)s for a jump polynomial p = x^d mod P: replaces
//                    jump_state / make_dephased_states (jump.cpp:27-53), which
//                    use a dense 19937^2 GF(2) matrix (f2_matrix.cpp:119-136).
//   vmt_seed_kernel  init_genrand (mt19937.cpp:22-27), one thread per seed.
//
// Generation layout. A CTA owns one chunk of the
// combined stream for a group of G lanes. Each lane's MT19937 word sequence
// x_0, x_1, ... (x_{n+624} = x_{n+397} ^ mulA((x_n & h) | (x_{n+1} & l)),
// PAPER.md:137-151) lives in a shared-memory ring of 832 = 624 + 208 slots
// (plus R mirror slots), interleaved [slot][lane] like the reference's
// interleaved state (engine.hpp:58-60). A "window" computes 208 new words of
// every lane: they only read slots written >= 1 window earlier and write the
// 208 slots freed by the previous window, so one __syncthreads per window is
// the only synchronisation (the reference's 227/396/1 loop split is the
// sequential special case, engine.hpp:119-131). Three windows are one
// 624*L-word block; blocks are emitted tempered, in the combined-stream order
// word[b*624L + k*L + t], with 128-bit stores.
#pragma once

#include <cstdint>

namespace vmt_b200 {

constexpr int kN = 624;
constexpr int kM = 397;
constexpr int kWin = 208;  // new words per lane per window
constexpr int kRing = 832; // kN + kWin
constexpr std::uint32_t kUpperMask = 0x80000000u;
constexpr std::uint32_t kLowerMask = 0x7FFFFFFFu;
constexpr std::uint32_t kMatA = 0x9908B0DFu;

enum GenMode : int {
    MODE_U32 = 0,       // uint32 words (vmt_fill_u32)
    MODE_XOR = 1,       // fused XOR checksum, nothing stored (vmt_checksum_xor)
    MODE_F32 = 2,       // (x >> 8) * 2^-24 in [0,1)
    MODE_F64 = 3,       // x * 2^-32 in [0,1)              (genrand_real2)
    MODE_F64_REAL3 = 4, // (x + 0.5) * 2^-32 in (0,1)      (stats.cpp:118)
    MODE_F64_RES53 = 5, // ((a>>5)*2^26 + (b>>6)) * 2^-53  (two words per value)
    MODE_BENCH_TEMPER_XOR = 6, // scratch/ microbenchmarks only (not reachable from the C ABI)
    MODE_STATS = 7,     // fused statistics consumer, nothing stored: one-bit count (monobit,
                        // stats.cpp:65-81) + byte-value histogram (chi2_bytes, stats.cpp:83-107)
};
constexpr int kModes = 8;
constexpr int kStatWords = 257; // MODE_STATS partial per CTA: ones, count[256]

struct GenParams {
    const std::uint32_t* chunk_states; // [C][624][L] interleaved boundary states
    void* out;                         // element of stream word pos_begin (per-chunk offset in batch mode)
    std::uint32_t* xor_partials;       // [gridDim.x] (MODE_XOR)
    unsigned long long* stats_partials; // [gridDim.x][257] (MODE_STATS)
    std::uint32_t* save_state;         // [624][L] boundary state at save_block (nullable); batch
                                       // mode: [chunk][624][L], one per generator
    unsigned long long first_block;    // absolute block of chunk 0
    unsigned long long end_block;      // exclusive
    unsigned long long pos_begin;      // absolute word range emitted
    unsigned long long pos_end;
    unsigned long long save_block;     // ~0ull: none
    unsigned long long out_chunk_stride; // batch mode: elements between chunks' outputs (0 = single stream)
    unsigned int blocks_per_chunk;
    unsigned int lanes;
#ifdef VMT_TIMELINE
    unsigned long long* tl; // experiments: per-CTA {start ns, end ns, SM id} (profiles/scripts/timeline.py)
#endif
};

#ifdef VMT_TIMELINE
__device__ __forceinline__ unsigned long long tl_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned tl_smid() {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}
#endif

// ---- per-word arithmetic (hand-scheduled LOP3 forms; SASS: 3 ALU + 2 FMA-pipe
// ops for the twist, 6 ALU + 2 FMA-pipe ops for the temper) -----------------

__device__ __forceinline__ std::uint32_t lop3_sel_hi(std::uint32_t hi_src, std::uint32_t lo_src) {
    // (hi_src & 0x80000000) | (lo_src & 0x7FFFFFFF)
    std::uint32_t r;
    asm("lop3.b32 %0, %1, 0x80000000, %2, 0xE2;" : "=r"(r) : "r"(hi_src), "r"(lo_src));
    return r;
}
__device__ __forceinline__ std::uint32_t xor3(std::uint32_t a, std::uint32_t b, std::uint32_t c) {
    std::uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
template <std::uint32_t MASK>
__device__ __forceinline__ std::uint32_t xor_and(std::uint32_t y, std::uint32_t t) {
    // y ^ (t & MASK)
    std::uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x6A;" : "=r"(r) : "r"(t), "n"(MASK), "r"(y));
    return r;
}
__device__ __forceinline__ std::uint32_t mul_lo(std::uint32_t a, std::uint32_t b) {
    std::uint32_t r;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// x_k <- x_{k+m} ^ mulA((x_k & h) | (x_{k+1} & l))   (mt19937.cpp:44, mt19937.hpp:70-72;
// lane form: lane_ops.hpp:81-85)
#ifndef VMT_TWIST_FMA_MAG
#define VMT_TWIST_FMA_MAG 1
#endif
__device__ __forceinline__ std::uint32_t mad_lo(std::uint32_t a, std::uint32_t b, std::uint32_t c) {
    std::uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
// Right shifts by s as the high word of a multiply by 2^(32-s) (IMAD.HI, FMA
// pipe) instead of SHF (ALU pipe): the twist + temper is ALU-pipe bound, so
// moving some of the three right shifts per word to the FMA pipe balances the
// two pipes. Bit 0: the twist's u >> 1; bit 1: temper's y >> 11; bit 2:
// temper's y >> 18.
#ifndef VMT_SHR_FMA
#define VMT_SHR_FMA 0
#endif
template <int S, bool FMA>
__device__ __forceinline__ std::uint32_t shr(std::uint32_t x) {
    if (FMA) {
        std::uint32_t r;
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "n"(1u << (32 - S)));
        return r;
    }
    return x >> S;
}

__device__ __forceinline__ std::uint32_t twist(std::uint32_t xk, std::uint32_t xk1, std::uint32_t xm) {
    const std::uint32_t u = lop3_sel_hi(xk, xk1);
    const std::uint32_t uh = shr<1, (VMT_SHR_FMA & 1) != 0>(u);
#if VMT_TWIST_FMA_MAG
    // mag = (u & 1) * A = u*A - (u >> 1)*2A: two IMADs on the FMA pipe instead
    // of a LOP3 + IMAD, so the twist costs 3 ALU-pipe ops (LOP3, SHF, LOP3)
    const std::uint32_t mag = mad_lo(u, kMatA, mul_lo(uh, 0u - 2u * kMatA));
#else
    const std::uint32_t mag = mul_lo(xk1 & 1u, kMatA); // odd(u) == odd(x_{k+1}); IMAD on the FMA pipe
#endif
    return xor3(xm, uh, mag);
}

// Tempering (mt19937.hpp:61-66; lane form lane_ops.hpp:88-93). Left shifts
// are multiplies so they issue on the FMA pipe. (Right shifts as the high word
// of IMAD.WIDE were measured 6% slower: the wide multiply is not FMA-pipe only.)
#ifndef VMT_TEMPER_SHL_ALU
#define VMT_TEMPER_SHL_ALU 0 // experiment: bit 0 / bit 1 = the << 7 / << 15 as ALU-pipe shifts
#endif
template <int S, bool ALU>
__device__ __forceinline__ std::uint32_t shl(std::uint32_t x) {
    if (ALU) {
        std::uint32_t r;
        // (ptxas turns a plain shl into IMAD.SHL; the funnel shift stays an SHF)
        asm("shf.l.wrap.b32 %0, 0, %1, %2;" : "=r"(r) : "r"(x), "n"(S));
        return r;
    }
    return mul_lo(x, 1u << S);
}
__device__ __forceinline__ std::uint32_t temper(std::uint32_t y) {
    y ^= shr<11, (VMT_SHR_FMA & 2) != 0>(y);
    y = xor_and<0x9D2C5680u>(y, shl<7, (VMT_TEMPER_SHL_ALU & 1) != 0>(y));
    y = xor_and<0xEFC60000u>(y, shl<15, (VMT_TEMPER_SHL_ALU & 2) != 0>(y));
    return y ^ shr<18, (VMT_SHR_FMA & 4) != 0>(y);
}

template <int V>
struct VecT;
template <>
struct VecT<4> {
    using T = uint4;
    __device__ static void get(const T& v, std::uint32_t* a) { a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w; }
    __device__ static T make(const std::uint32_t* a) { return make_uint4(a[0], a[1], a[2], a[3]); }
};
template <>
struct VecT<2> {
    using T = uint2;
    __device__ static void get(const T& v, std::uint32_t* a) { a[0] = v.x; a[1] = v.y; }
    __device__ static T make(const std::uint32_t* a) { return make_uint2(a[0], a[1]); }
};
template <>
struct VecT<1> {
    using T = std::uint32_t;
    __device__ static void get(const T& v, std::uint32_t* a) { a[0] = v; }
    __device__ static T make(const std::uint32_t* a) { return a[0]; }
};

template <int MODE>
struct ElemT {
    using T = std::uint32_t;
};
template <>
struct ElemT<MODE_F32> {
    using T = float;
};
template <>
struct ElemT<MODE_F64> {
    using T = double;
};
template <>
struct ElemT<MODE_F64_REAL3> {
    using T = double;
};
template <>
struct ElemT<MODE_F64_RES53> {
    using T = double;
};

__device__ __forceinline__ float to_f32(std::uint32_t x) { return __uint2float_rn(x >> 8) * 5.9604644775390625e-08f; }
__device__ __forceinline__ double to_f64(std::uint32_t x) { return __uint2double_rn(x) * 2.3283064365386963e-10; }
__device__ __forceinline__ double to_f64_real3(std::uint32_t x) {
    return (__uint2double_rn(x) + 0.5) * 2.3283064365386963e-10;
}
__device__ __forceinline__ double to_f64_res53(std::uint32_t a, std::uint32_t b) {
    return (__uint2double_rn(a >> 5) * 67108864.0 + __uint2double_rn(b >> 6)) * 1.1102230246251565e-16;
}

// Output stores (streamed once, never re-read by this kernel). Default 3: L2
// evict-first policy, so the output stream does not push the co-resident
// positioning GEMM's operands (the 47 MB FP4 state operand, read once per
// output slice, and the 200 MB matrix) out of L2: in the driver's 20-step
// shape 12.47-12.52 vs 12.72-12.81 ms per 2^34-word step, burst 11.30-11.34
// vs 11.72 (profiles/r02_microbench/README.md). 1: st.global.cs (similar),
// 0: plain.
#ifndef VMT_STORE_HINT
#define VMT_STORE_HINT 3
#endif
template <class VT>
__device__ __forceinline__ void store_out(VT* p, const VT& v) {
    *p = v;
}
template <>
__device__ __forceinline__ void store_out<uint2>(uint2* p, const uint2& v) {
#if VMT_STORE_HINT == 3
    unsigned long long pol; // (not volatile: one createpolicy per thread, hoisted)
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(v.x), "r"(v.y), "l"(pol)
                 : "memory");
#elif VMT_STORE_HINT == 1
    __stcs(p, v);
#else
    *p = v;
#endif
}
template <>
__device__ __forceinline__ void store_out<uint4>(uint4* p, const uint4& v) {
#if VMT_STORE_HINT == 1
    __stcs(p, v);
#elif VMT_STORE_HINT == 2
    asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
#elif VMT_STORE_HINT == 3
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
#else
    *p = v;
#endif
}

} // namespace vmt_b200
