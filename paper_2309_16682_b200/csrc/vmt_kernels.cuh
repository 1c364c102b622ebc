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
};

struct GenParams {
    const std::uint32_t* chunk_states; // [C][624][L] interleaved boundary states
    void* out;                         // element of stream word pos_begin (per-chunk offset in batch mode)
    std::uint32_t* xor_partials;       // [gridDim.x] (MODE_XOR)
    std::uint32_t* save_state;         // [624][L] boundary state at save_block (nullable)
    unsigned long long first_block;    // absolute block of chunk 0
    unsigned long long end_block;      // exclusive
    unsigned long long pos_begin;      // absolute word range emitted
    unsigned long long pos_end;
    unsigned long long save_block;     // ~0ull: none
    unsigned long long out_chunk_stride; // batch mode: elements between chunks' outputs (0 = single stream)
    unsigned int blocks_per_chunk;
    unsigned int lanes;
};

// ---- per-word arithmetic (hand-scheduled LOP3 forms; SASS: 4 ALU + 1 FMA-pipe
// op for the twist, 6 ALU + 2 FMA-pipe ops for the temper) -------------------

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
__device__ __forceinline__ std::uint32_t twist(std::uint32_t xk, std::uint32_t xk1, std::uint32_t xm) {
    const std::uint32_t u = lop3_sel_hi(xk, xk1);
    const std::uint32_t mag = mul_lo(xk1 & 1u, kMatA); // odd(u) == odd(x_{k+1}); IMAD on the FMA pipe
    return xor3(xm, u >> 1, mag);
}

// Tempering (mt19937.hpp:61-66; lane form lane_ops.hpp:88-93). Left shifts
// are multiplies so they issue on the FMA pipe.
__device__ __forceinline__ std::uint32_t temper(std::uint32_t y) {
    y ^= y >> 11;
    y = xor_and<0x9D2C5680u>(y, mul_lo(y, 1u << 7));
    y = xor_and<0xEFC60000u>(y, mul_lo(y, 1u << 15));
    return y ^ (y >> 18);
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

// CTA shape: a CTA owns all L lanes of one chunk; thread (rho, q) computes
// R consecutive sequence words of lanes q*V .. q*V+V-1 in every window.
// VW (1, 2 or 4) is the vector width: smaller VW = more threads per lane
// state (more warps per SM for the same shared memory).
template <int L, int R, int VW = 4>
struct GenShape {
    static constexpr int V = L >= VW ? VW : L;    // lanes per thread (vector width)
    static constexpr int Q = L / V;               // threads across a slot row
    static constexpr int RUNS = kWin / R;         // runs per window
    static constexpr int NT = RUNS * Q;           // threads per CTA
    static constexpr int SLOTS = kRing + R;       // ring + mirror of slots [0, R)
    static constexpr int SMEM = SLOTS * L * 4;
    // CTAs per SM that shared memory allows (227 KB usable, 1 KB reserved per CTA)
    static constexpr int SMEM_CTAS = (227 * 1024) / (SMEM + 1024) > 0 ? (227 * 1024) / (SMEM + 1024) : 1;
    // registers are capped so that they never limit occupancy below that
    static constexpr int MINB = (SMEM_CTAS * NT > 2048) ? (2048 / NT > 0 ? 2048 / NT : 1) : SMEM_CTAS;
    static_assert(kWin % R == 0 && kN % R == 0 && kRing % R == 0, "run length must divide 208");
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

// Stores V tempered words that are consecutive in the stream; `o` points at
// the element of the first one. Edge (!FULL) words outside [pos_begin,
// pos_end) are skipped.
template <int MODE, int V, bool VEC, bool FULL>
__device__ __forceinline__ void emit(const std::uint32_t* w, unsigned long long g, const GenParams& p,
                                     typename ElemT<MODE>::T* o) {
    bool in[V];
    bool all_in = true;
#pragma unroll
    for (int v = 0; v < V; ++v) {
        in[v] = FULL || (g + v >= p.pos_begin && g + v < p.pos_end);
        all_in = all_in && in[v];
    }
    if (MODE == MODE_U32) {
        if (VEC && all_in) {
            using VT = typename VecT<V>::T;
            *reinterpret_cast<VT*>(o) = VecT<V>::make(w);
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v)
                if (in[v])
                    o[v] = w[v];
        }
    } else if (MODE == MODE_F32) {
        float f[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
            f[v] = to_f32(w[v]);
        if (VEC && V == 4 && all_in) {
            *reinterpret_cast<float4*>(o) = make_float4(f[0], f[1], f[2], f[3]);
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v)
                if (in[v])
                    o[v] = f[v];
        }
    } else if (MODE == MODE_F64 || MODE == MODE_F64_REAL3) {
        double d[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
            d[v] = MODE == MODE_F64 ? to_f64(w[v]) : to_f64_real3(w[v]);
        if (VEC && V == 4 && all_in) {
            reinterpret_cast<double2*>(o)[0] = make_double2(d[0], d[1]);
            reinterpret_cast<double2*>(o)[1] = make_double2(d[2], d[3]);
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v)
                if (in[v])
                    o[v] = d[v];
        }
    } else if (MODE == MODE_F64_RES53) {
        // value i consumes stream words (pos_begin + 2i, +2i+1): o indexes
        // values, pos_begin is even and so is g (V even)
#pragma unroll
        for (int v = 0; v + 1 < V; v += 2)
            if (in[v] && in[v + 1])
                o[v >> 1] = to_f64_res53(w[v], w[v + 1]);
    }
}

// One window of one thread: R new words of V lanes. base: slot of x_p for
// the run's first p; a: slot of x_{p+397}; wsl: slot receiving x_{p+624}.
// All ring loads are issued before any ring store (the stores go to slots no
// thread reads in this window), so the compiler is free to overlap them.
template <int L, int R, int VW, int MODE, bool VEC, bool FULL>
__device__ __forceinline__ void gen_window(std::uint32_t* ring, int base, int a, int wsl, int q,
                                           unsigned long long g0, const GenParams& p, void* out,
                                           std::uint32_t* acc) {
    constexpr int V = GenShape<L, R, VW>::V;
    using VT = typename VecT<V>::T;
    using E = typename ElemT<MODE>::T;
    std::uint32_t X[R + 1][V], M[R][V];
#pragma unroll
    for (int i = 0; i <= R; ++i)
        VecT<V>::get(*reinterpret_cast<const VT*>(ring + (base + i) * L + q * V), X[i]);
#pragma unroll
    for (int i = 0; i < R; ++i)
        VecT<V>::get(*reinterpret_cast<const VT*>(ring + (a + i) * L + q * V), M[i]);
    E* o = nullptr;
    if (MODE != MODE_XOR) {
        const unsigned long long rel = g0 - p.pos_begin;
        o = static_cast<E*>(out) + (MODE == MODE_F64_RES53 ? (rel >> 1) : rel);
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        std::uint32_t nw[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
            nw[v] = twist(X[i][v], X[i + 1][v], M[i][v]);
        *reinterpret_cast<VT*>(ring + (wsl + i) * L + q * V) = VecT<V>::make(nw);
        if (MODE == MODE_XOR) {
            // temper is GF(2)-linear: XOR the untempered words, temper once
            // at the end (vmt_xor_reduce_kernel)
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const unsigned long long g = g0 + (unsigned long long)i * L + v;
                if (FULL || (g >= p.pos_begin && g < p.pos_end))
                    acc[v] ^= nw[v];
            }
        } else {
            std::uint32_t tw[V];
#pragma unroll
            for (int v = 0; v < V; ++v)
                tw[v] = temper(nw[v]);
            emit<MODE, V, VEC, FULL>(tw, g0 + (unsigned long long)i * L, p,
                                     o + (MODE == MODE_F64_RES53 ? (i * L) / 2 : i * L));
        }
    }
    if (wsl == 0) {
        // mirror slots [0, R) behind the ring end (this thread wrote them)
#pragma unroll
        for (int i = 0; i < R; ++i)
            *reinterpret_cast<VT*>(ring + (kRing + i) * L + q * V) =
                *reinterpret_cast<const VT*>(ring + i * L + q * V);
    }
}

template <int L>
__device__ __forceinline__ void save_boundary(const std::uint32_t* ring, int blk_base_slot, std::uint32_t* dst,
                                              int tid, int nt) {
    for (int i = tid; i < kN * L; i += nt) {
        const int k = i / L, t = i % L;
        int slot = blk_base_slot + k;
        if (slot >= kRing)
            slot -= kRing;
        dst[i] = ring[slot * L + t];
    }
}

// One CTA = one chunk (all L lanes). Dynamic shared memory GenShape::SMEM
// bytes: ring[slot][L].
template <int L, int R, int VW, int MODE, bool VEC>
__global__ void __launch_bounds__(GenShape<L, R, VW>::NT, GenShape<L, R, VW>::MINB) vmt_gen_kernel(GenParams p) {
    using S = GenShape<L, R, VW>;
    constexpr int V = S::V;
    using VT = typename VecT<V>::T;
    extern __shared__ __align__(16) std::uint32_t ring[];
    __shared__ std::uint32_t red;

    const unsigned chunk = blockIdx.x;
    const int tid = threadIdx.x;
    const int q = tid % S::Q;   // vector column (lanes q*V .. q*V+V-1)
    const int rho = tid / S::Q; // run index within a window

    const bool batch = p.out_chunk_stride != 0;
    const unsigned long long b_lo =
        batch ? p.first_block : p.first_block + (unsigned long long)chunk * p.blocks_per_chunk;
    unsigned long long b_hi = batch ? p.end_block : b_lo + p.blocks_per_chunk;
    if (b_hi > p.end_block)
        b_hi = p.end_block;
    void* out = p.out;
    if (batch)
        out = static_cast<void*>(static_cast<typename ElemT<MODE>::T*>(out) +
                                 (MODE == MODE_F64_RES53 ? p.out_chunk_stride / 2 : p.out_chunk_stride) * chunk);

    // -- the chunk's boundary state (words x_0..x_623 -> slots 0..623)
    const std::uint32_t* src = p.chunk_states + (unsigned long long)chunk * kN * L;
    for (int i = tid; i < kN * S::Q; i += S::NT) {
        const VT v = reinterpret_cast<const VT*>(src)[i];
        reinterpret_cast<VT*>(ring)[i] = v;
        if (i < R * S::Q)
            reinterpret_cast<VT*>(ring)[kRing * S::Q + i] = v;
    }
    if (MODE == MODE_XOR && tid == 0)
        red = 0;
    __syncthreads();

    std::uint32_t acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v)
        acc[v] = 0;
    constexpr unsigned long long bw = (unsigned long long)kN * L;
    const bool save_here = p.save_state != nullptr && (!batch || chunk == 0);
    int blk_base_slot = 0; // slot of x_{624 r} for the current block r (= 624 r mod 832)
    for (unsigned long long blk = b_lo; blk < b_hi; ++blk) {
        if (save_here && blk == p.save_block)
            save_boundary<L>(ring, blk_base_slot, p.save_state, tid, S::NT);
        const bool full = blk * bw >= p.pos_begin && (blk + 1) * bw <= p.pos_end;
#pragma unroll 1
        for (int third = 0; third < 3; ++third) {
            int wstart = blk_base_slot + third * kWin;
            if (wstart >= kRing)
                wstart -= kRing;
            const int base = wstart + rho * R;
            int a = base + kM;
            if (a >= kRing)
                a -= kRing;
            int wsl = base + kN;
            if (wsl >= kRing)
                wsl -= kRing;
            const unsigned long long g0 = blk * bw + (unsigned long long)(third * kWin + rho * R) * L + q * V;
            if (full)
                gen_window<L, R, VW, MODE, VEC, true>(ring, base, a, wsl, q, g0, p, out, acc);
            else
                gen_window<L, R, VW, MODE, VEC, false>(ring, base, a, wsl, q, g0, p, out, acc);
            __syncthreads();
        }
        blk_base_slot += kN;
        if (blk_base_slot >= kRing)
            blk_base_slot -= kRing;
    }
    // end-of-range boundary state (block b_hi) when it is the requested one
    if (save_here && b_hi == p.save_block && b_hi == p.end_block)
        save_boundary<L>(ring, blk_base_slot, p.save_state, tid, S::NT);
    if (MODE == MODE_XOR) {
        std::uint32_t x = 0;
#pragma unroll
        for (int v = 0; v < V; ++v)
            x ^= acc[v];
        atomicXor(&red, x);
        __syncthreads();
        if (tid == 0)
            p.xor_partials[blockIdx.x] = red; // untempered; tempered by the reduce kernel
    }
}

// ---------------------------------------------------------------------------
// Jump kernel: one warp per job. Job j computes dst_j = poly_j(F) src_j with
// the convolution y_k = XOR_{i : p_i = 1} x_{i+k} over the word sequence
// generated from src (x_0..x_623 = src), y_0 keeping only its live bit
// (mt19937.cpp:79). Thread tau owns output words 20*tau .. 20*tau+19 (the top
// 16 of lane 31 are discarded) and keeps the 20 sequence words they need in
// registers; each group of 20 coefficient steps reads the next 20 words with
// five conflict-free 128-bit shared loads from a 1024-word per-warp sequence
// ring that lanes 0..19 extend by 20 words per group.
struct JumpParams {
    const std::uint32_t* src;
    std::uint32_t* dst;
    const std::uint64_t* polys;       // [npoly][312]
    const long long* job_src;         // word offset of state j in src (nullable: affine map below)
    const long long* job_dst;         // word offset of state j in dst
    const int* job_poly;              // poly index of job j
    int src_stride;                   // word k of a state at offset + k*stride
    int dst_stride;
    int njobs;
    // affine job map when job_src == nullptr: a = j / div, b = j % div
    int div;
    long long s_a, s_b, s_c, d_a, d_b, d_c;
    int p_a, p_b, p_c;
};

constexpr int kJumpWarps = 1;
constexpr int kSeqRing = 1024;
constexpr int kGroups = 998; // 998 * 20 = 19960 >= 19937 coefficient steps

template <int S>
__device__ __forceinline__ void jump_pair(std::uint32_t (&Y)[20], const std::uint32_t (&A)[20],
                                          const std::uint32_t (&B)[20], unsigned bits) {
    // steps S and S+1 of a 20-step group: position k sees x at offset S+k / S+1+k
    // of the 40-word window A ++ B.
    if (bits == 3u) {
#pragma unroll
        for (int k = 0; k < 20; ++k) {
            const std::uint32_t v0 = (S + k) < 20 ? A[(S + k) % 20] : B[(S + k) % 20];
            const std::uint32_t v1 = (S + 1 + k) < 20 ? A[(S + 1 + k) % 20] : B[(S + 1 + k) % 20];
            Y[k] ^= v0 ^ v1;
        }
    } else if (bits == 1u) {
#pragma unroll
        for (int k = 0; k < 20; ++k)
            Y[k] ^= (S + k) < 20 ? A[(S + k) % 20] : B[(S + k) % 20];
    } else if (bits == 2u) {
#pragma unroll
        for (int k = 0; k < 20; ++k)
            Y[k] ^= (S + 1 + k) < 20 ? A[(S + 1 + k) % 20] : B[(S + 1 + k) % 20];
    }
}

__device__ __forceinline__ unsigned poly_bits20(const std::uint32_t* p32, int i) {
    // 20 coefficient bits starting at bit i (p32 in shared memory)
    const int w = i >> 5, o = i & 31;
    const unsigned long long two = ((unsigned long long)p32[w + 1] << 32) | p32[w];
    return (unsigned)(two >> o) & 0xFFFFFu;
}

__device__ __forceinline__ void jump_produce(std::uint32_t* seq, int m) {
    // x_m from x_{m-624}, x_{m-623}, x_{m-227}
    seq[m & (kSeqRing - 1)] = twist(seq[(m - kN) & (kSeqRing - 1)], seq[(m - kN + 1) & (kSeqRing - 1)],
                                    seq[(m - kN + kM) & (kSeqRing - 1)]);
}

__device__ __forceinline__ void jump_load20(const std::uint32_t* seq, int start, std::uint32_t (&B)[20]) {
#pragma unroll
    for (int v = 0; v < 5; ++v) {
        const uint4 t = *reinterpret_cast<const uint4*>(seq + ((start + 4 * v) & (kSeqRing - 1)));
        B[4 * v] = t.x;
        B[4 * v + 1] = t.y;
        B[4 * v + 2] = t.z;
        B[4 * v + 3] = t.w;
    }
}

// One warp per CTA, so everything derived from the job index (the polynomial
// coefficients driving the branches) is CTA-uniform.
#ifndef VMT_JUMP_MINB
#define VMT_JUMP_MINB 32
#endif
__global__ void __launch_bounds__(32, VMT_JUMP_MINB) vmt_jump_kernel(JumpParams p) {
    __shared__ __align__(16) std::uint32_t seq[kSeqRing];
    const int lane = threadIdx.x;
    const int job = blockIdx.x;
    if (job >= p.njobs)
        return;
    long long so, dof;
    int pidx;
    if (p.job_src != nullptr) {
        so = p.job_src[job];
        dof = p.job_dst[job];
        pidx = p.job_poly[job];
    } else {
        const long long a = job / p.div, b = job % p.div;
        so = a * p.s_a + b * p.s_b + p.s_c;
        dof = a * p.d_a + b * p.d_b + p.d_c;
        pidx = (int)(a * p.p_a + b * p.p_b + p.p_c);
    }
    const std::uint32_t* src = p.src + so;
    for (int k = lane; k < kN; k += 32)
        seq[k] = src[(long long)k * p.src_stride];
    __syncwarp();
    jump_produce(seq, kN + lane); // x_624 .. x_655
    __syncwarp();
    if (lane < 4)
        jump_produce(seq, kN + 32 + lane); // x_656 .. x_659
    __syncwarp();

    // coefficients to shared memory (+1 zero word for the look-ahead past bit 19967)
    __shared__ std::uint32_t p32[kN + 2];
    {
        const std::uint32_t* pg = reinterpret_cast<const std::uint32_t*>(p.polys + (long long)pidx * 312);
        for (int k = lane; k < kN; k += 32)
            p32[k] = __ldg(pg + k);
        if (lane < 2)
            p32[kN + lane] = 0;
        __syncwarp();
    }
    std::uint32_t Y[20], A[20], B[20];
#pragma unroll
    for (int k = 0; k < 20; ++k)
        Y[k] = 0;
    jump_load20(seq, 20 * lane, A);
    unsigned cm = poly_bits20(p32, 0);

#pragma unroll 1
    for (int g = 0; g < kGroups; g += 2) {
        // ---- group g (window A ++ B)
        {
            const int i = 20 * g;
            jump_load20(seq, i + 20 * lane + 20, B);
            if (lane < 20)
                jump_produce(seq, i + 660 + lane);
            const unsigned cn = poly_bits20(p32, i + 20);
            jump_pair<0>(Y, A, B, cm & 3u);
            jump_pair<2>(Y, A, B, (cm >> 2) & 3u);
            jump_pair<4>(Y, A, B, (cm >> 4) & 3u);
            jump_pair<6>(Y, A, B, (cm >> 6) & 3u);
            jump_pair<8>(Y, A, B, (cm >> 8) & 3u);
            jump_pair<10>(Y, A, B, (cm >> 10) & 3u);
            jump_pair<12>(Y, A, B, (cm >> 12) & 3u);
            jump_pair<14>(Y, A, B, (cm >> 14) & 3u);
            jump_pair<16>(Y, A, B, (cm >> 16) & 3u);
            jump_pair<18>(Y, A, B, (cm >> 18) & 3u);
            cm = cn;
            __syncwarp();
        }
        // ---- group g+1 (window B ++ A)
        {
            const int i = 20 * (g + 1);
            jump_load20(seq, i + 20 * lane + 20, A);
            if (lane < 20)
                jump_produce(seq, i + 660 + lane);
            const unsigned cn = (g + 2 < kGroups) ? poly_bits20(p32, i + 20) : 0u;
            jump_pair<0>(Y, B, A, cm & 3u);
            jump_pair<2>(Y, B, A, (cm >> 2) & 3u);
            jump_pair<4>(Y, B, A, (cm >> 4) & 3u);
            jump_pair<6>(Y, B, A, (cm >> 6) & 3u);
            jump_pair<8>(Y, B, A, (cm >> 8) & 3u);
            jump_pair<10>(Y, B, A, (cm >> 10) & 3u);
            jump_pair<12>(Y, B, A, (cm >> 12) & 3u);
            jump_pair<14>(Y, B, A, (cm >> 14) & 3u);
            jump_pair<16>(Y, B, A, (cm >> 16) & 3u);
            jump_pair<18>(Y, B, A, (cm >> 18) & 3u);
            cm = cn;
            __syncwarp();
        }
    }
    std::uint32_t* dst = p.dst + dof;
#pragma unroll
    for (int k = 0; k < 20; ++k) {
        const int j = 20 * lane + k;
        if (j < kN)
            dst[(long long)j * p.dst_stride] = (j == 0) ? (Y[k] & kUpperMask) : Y[k];
    }
}

// init_genrand (mt19937.cpp:22-27): state n = seeds[n] written at
// dst + n*state_stride + k*word_stride.
__global__ void vmt_seed_kernel(const std::uint32_t* seeds, int n, std::uint32_t* dst, long long state_stride,
                                int word_stride) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    std::uint32_t w = seeds[i];
    std::uint32_t* d = dst + (long long)i * state_stride;
    d[0] = w;
    for (std::uint32_t k = 1; k < (std::uint32_t)kN; ++k) {
        w = 1812433253u * (w ^ (w >> 30)) + k;
        d[(long long)k * word_stride] = w;
    }
}

// XOR-reduce per-CTA (untempered) partials into out[0] and temper the total.
__global__ void vmt_xor_reduce_kernel(const std::uint32_t* partials, int n, std::uint32_t* out) {
    std::uint32_t acc = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        acc ^= partials[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        acc ^= __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    __shared__ std::uint32_t red[32];
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        std::uint32_t x = 0;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w)
            x ^= red[w];
        out[0] = temper(x); // XOR of tempered words == temper(XOR of words)
    }
}

} // namespace vmt_b200
