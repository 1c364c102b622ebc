// sm_100a jump-ahead, seeding and reduction kernels (see vmt_common.cuh).
#pragma once

#include "vmt_common.cuh"

namespace vmt_b200 {

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

// Four coefficient steps S..S+3 with bit pattern PAT: position k XORs the
// window words at offsets S+b+k for the set bits b, two per LOP3.
template <int S, unsigned PAT>
__device__ __forceinline__ void jump_quad_apply(std::uint32_t (&Y)[20], const std::uint32_t (&A)[20],
                                                const std::uint32_t (&B)[20]) {
#pragma unroll
    for (int k = 0; k < 20; ++k) {
        std::uint32_t t[4];
        int n = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if ((PAT >> b) & 1u) {
                const int idx = S + b + k;
                t[n++] = idx < 20 ? A[idx % 20] : B[idx % 20];
            }
        if (n == 1)
            Y[k] ^= t[0];
        else if (n == 2)
            Y[k] ^= t[0] ^ t[1];
        else if (n == 3)
            Y[k] = xor3(xor3(Y[k], t[0], t[1]), t[2], 0u);
        else if (n == 4)
            Y[k] = xor3(xor3(Y[k], t[0], t[1]), t[2], t[3]);
    }
}

template <int S>
__device__ __forceinline__ void jump_quad(std::uint32_t (&Y)[20], const std::uint32_t (&A)[20],
                                          const std::uint32_t (&B)[20], unsigned m) {
    switch (m) {
    case 1: jump_quad_apply<S, 1>(Y, A, B); break;
    case 2: jump_quad_apply<S, 2>(Y, A, B); break;
    case 3: jump_quad_apply<S, 3>(Y, A, B); break;
    case 4: jump_quad_apply<S, 4>(Y, A, B); break;
    case 5: jump_quad_apply<S, 5>(Y, A, B); break;
    case 6: jump_quad_apply<S, 6>(Y, A, B); break;
    case 7: jump_quad_apply<S, 7>(Y, A, B); break;
    case 8: jump_quad_apply<S, 8>(Y, A, B); break;
    case 9: jump_quad_apply<S, 9>(Y, A, B); break;
    case 10: jump_quad_apply<S, 10>(Y, A, B); break;
    case 11: jump_quad_apply<S, 11>(Y, A, B); break;
    case 12: jump_quad_apply<S, 12>(Y, A, B); break;
    case 13: jump_quad_apply<S, 13>(Y, A, B); break;
    case 14: jump_quad_apply<S, 14>(Y, A, B); break;
    case 15: jump_quad_apply<S, 15>(Y, A, B); break;
    default: break;
    }
}

// All 20 steps of a group applied to the window A ++ B.
__device__ __forceinline__ void jump_group(std::uint32_t (&Y)[20], const std::uint32_t (&A)[20],
                                           const std::uint32_t (&B)[20], unsigned cm);

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

#ifndef VMT_JUMP_QUADS
#define VMT_JUMP_QUADS 0 // 16-way quad switch measured 1.7x slower (code size; a 7-way
                         // triple switch, 11% fewer LOP3s, measured 1.3x slower too)
#endif
__device__ __forceinline__ void jump_group(std::uint32_t (&Y)[20], const std::uint32_t (&A)[20],
                                           const std::uint32_t (&B)[20], unsigned cm) {
#if VMT_JUMP_QUADS
    jump_quad<0>(Y, A, B, cm & 15u);
    jump_quad<4>(Y, A, B, (cm >> 4) & 15u);
    jump_quad<8>(Y, A, B, (cm >> 8) & 15u);
    jump_quad<12>(Y, A, B, (cm >> 12) & 15u);
    jump_quad<16>(Y, A, B, (cm >> 16) & 15u);
#else
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
#endif
}

#ifndef VMT_JUMP_UNIFORM
#define VMT_JUMP_UNIFORM 1
#endif
#ifndef VMT_JUMP_SINGLE_BODY
#define VMT_JUMP_SINGLE_BODY 0
#endif
__device__ __forceinline__ unsigned poly_bits20(const std::uint32_t* p32, int i) {
    // 20 coefficient bits starting at bit i (p32 in shared memory)
    const int w = i >> 5, o = i & 31;
    const unsigned long long two = ((unsigned long long)p32[w + 1] << 32) | p32[w];
    const unsigned v = (unsigned)(two >> o) & 0xFFFFFu;
#if VMT_JUMP_UNIFORM
    // every lane holds the same value; REDUX.OR moves it into a uniform
    // register so the per-pair bit tests and branches run on the uniform
    // datapath instead of the vector ALU
    return __reduce_or_sync(0xFFFFFFFFu, v);
#else
    return v;
#endif
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

// One job per CTA, so everything derived from the job index (the polynomial
// coefficients driving the branches) is CTA-uniform. SPLIT warps share a job:
// warp w takes the w-th slice of the coefficient groups (after advancing its
// own copy of the sequence to the slice start) and the partial results are
// XOR-reduced through shared memory -- SPLIT > 1 trades ~10% extra work for a
// SPLIT-fold shorter latency when there are few jobs.
// MINB: one-warp jobs resident per SM (the register cap): 24 = 77 registers,
// no spills; 28 = 72 registers, one wave for up to 28 jobs per SM (config 5's
// 4096 jobs on 148 SMs: 4.99 vs 5.39 ms over three launches); 32 = 64
// registers with spills, 4% slower per job.
#ifndef VMT_JUMP_MINB
#define VMT_JUMP_MINB 24
#endif
template <int SPLIT, int MINB = VMT_JUMP_MINB>
__global__ void __launch_bounds__(32 * SPLIT, (SPLIT == 1 ? MINB : 32 / SPLIT)) vmt_jump_kernel(JumpParams p) {
    __shared__ __align__(16) std::uint32_t seq_all[SPLIT][kSeqRing];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int job = blockIdx.x;
    if (job >= p.njobs)
        return;
    std::uint32_t* seq = seq_all[warp];
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
        // (a job_poly table may still supply the polynomial per job)
        pidx = p.job_poly != nullptr ? p.job_poly[job] : (int)(a * p.p_a + b * p.p_b + p.p_c);
    }
    const std::uint32_t* src = p.src + so;
    for (int k = lane; k < kN; k += 32)
        seq[k] = src[(long long)k * p.src_stride];
    __syncwarp();
    // this warp's coefficient groups [g_lo, g_hi) (even bounds: the loop
    // below handles groups in pairs)
    constexpr int kPer = ((kGroups / 2 + SPLIT - 1) / SPLIT) * 2;
    const int g_lo = warp * kPer;
    const int g_hi = g_lo + kPer < kGroups ? g_lo + kPer : kGroups;
    // extend the sequence to x_{20*g_lo + 659} (32 independent words per batch)
    const int last = 20 * g_lo + 659;
    for (int m0 = kN; m0 <= last; m0 += 32) {
        if (m0 + lane <= last)
            jump_produce(seq, m0 + lane);
        __syncwarp();
    }

    // coefficients to shared memory (+1 zero word for the look-ahead past bit 19967)
    __shared__ std::uint32_t p32[kN + 2];
    {
        const std::uint32_t* pg = reinterpret_cast<const std::uint32_t*>(p.polys + (long long)pidx * 312);
        for (int k = threadIdx.x; k < kN; k += 32 * SPLIT)
            p32[k] = __ldg(pg + k);
        if (threadIdx.x < 2)
            p32[kN + threadIdx.x] = 0;
        if (SPLIT == 1)
            __syncwarp();
        else
            __syncthreads();
    }
    std::uint32_t Y[20], A[20], B[20];
#pragma unroll
    for (int k = 0; k < 20; ++k)
        Y[k] = 0;
    jump_load20(seq, 20 * g_lo + 20 * lane, A);
    unsigned cm = g_lo < g_hi ? poly_bits20(p32, 20 * g_lo) : 0u;

#pragma unroll 1
    for (int g = g_lo; g < g_hi; g += 2) {
        // ---- group g (window A ++ B)
        {
            const int i = 20 * g;
            jump_load20(seq, i + 20 * lane + 20, B);
            if (lane < 20)
                jump_produce(seq, i + 660 + lane);
            const unsigned cn = poly_bits20(p32, i + 20);
            jump_group(Y, A, B, cm);
            cm = cn;
            __syncwarp();
        }
        // ---- group g+1 (window B ++ A)
        {
            const int i = 20 * (g + 1);
            jump_load20(seq, i + 20 * lane + 20, A);
            if (lane < 20)
                jump_produce(seq, i + 660 + lane);
            const unsigned cn = (g + 2 < g_hi) ? poly_bits20(p32, i + 20) : 0u;
            jump_group(Y, B, A, cm);
            cm = cn;
            __syncwarp();
        }
    }
    std::uint32_t* dst = p.dst + dof;
    if (SPLIT == 1) {
#pragma unroll
        for (int k = 0; k < 20; ++k) {
            const int j = 20 * lane + k;
            if (j < kN)
                dst[(long long)j * p.dst_stride] = (j == 0) ? (Y[k] & kUpperMask) : Y[k];
        }
    } else {
        // XOR the warps' partial sums (the sequence rings are free now)
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 20; ++k)
            seq[20 * lane + k] = Y[k];
        __syncthreads();
        for (int j = threadIdx.x; j < kN; j += 32 * SPLIT) {
            std::uint32_t v = 0;
#pragma unroll
            for (int w = 0; w < SPLIT; ++w)
                v ^= seq_all[w][j];
            dst[(long long)j * p.dst_stride] = (j == 0) ? (v & kUpperMask) : v;
        }
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

// MODE_STATS: out[j] = sum over CTAs of partials[cta][j], j < 257.
__global__ void vmt_stats_reduce_kernel(const unsigned long long* partials, int n, unsigned long long* out) {
    const int j = threadIdx.x;
    if (j >= kStatWords)
        return;
    unsigned long long s = 0;
    for (int i = 0; i < n; ++i)
        s += partials[(long long)i * kStatWords + j];
    out[j] = s;
}

} // namespace vmt_b200
