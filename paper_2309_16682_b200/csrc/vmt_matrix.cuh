// sm_100a kernels for the GF(2) jump-matrix path.
//
// The reference de-phases lanes with a dense 19937 x 19937 bit matrix
// B = F^(2^q) (f2_matrix.hpp:13-21, jump.cpp:27-53) that it builds by q
// successive squarings (mat_pow2, f2_matrix.cpp:138-177; ~50 h at the full
// period) and stores as a .vmtj file (jump_file.hpp:12-22). Here:
//
//   * row i of F^d is the effective state of the basis state e_i jumped by d
//     steps, so the whole matrix is 19937 independent polynomial jumps
//     (vmt_jump_kernel on vmt_basis_kernel's states, then
//     vmt_words_to_eff_kernel) -- milliseconds for any d, byte-identical to
//     the reference's squaring ladder;
//   * vec_mat_mul (f2_matrix.cpp:119-136: XOR of the rows at the set bits of
//     v) runs as vmt_vec_mat_kernel, used to de-phase with a caller-supplied
//     matrix exactly like make_dephased_states.
//
// Effective layout (mt19937.cpp:57-101): bit 0 = bit 31 of word 0, bits
// 1..19936 = words 1..623 LSB first, packed into 312 little-endian u64 (624
// u32 halves, the last 31 bits zero). As a 32-bit funnel:
//   e32[h] = (W[h] >> 31) | (W[h+1] << 1)         h = 0..623, W[624] = 0
//   W[0] = (e32[0] & 1) << 31,  W[k] = (e32[k-1] >> 1) | (e32[k] << 31)
#pragma once

#include <cstdint>

#include "vmt_common.cuh"

namespace vmt_b200 {

constexpr int kDim = 19937;    // effective bits
constexpr int kRowWords = 312; // u64 per row / vector
constexpr int kRowHalves = 624;

// Basis states e_{row0 + j}, j < n, as [n][624] words (buffer pre-zeroed).
__global__ void vmt_basis_kernel(std::uint32_t* dst, int row0, int n) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n)
        return;
    const int row = row0 + j;
    std::uint32_t* d = dst + (long long)j * kN;
    if (row == 0)
        d[0] = kUpperMask;
    else
        d[1 + (row - 1) / 32] = 1u << ((row - 1) % 32);
}

// words -> effective: state s word k at src + s*state_stride + k*word_stride,
// effective halves to dst + s*624 (u32 view of the 312 u64).
__global__ void vmt_words_to_eff_kernel(const std::uint32_t* src, long long state_stride, int word_stride,
                                        std::uint32_t* dst, int n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)n * kRowHalves)
        return;
    const long long s = i / kRowHalves;
    const int h = (int)(i % kRowHalves);
    const std::uint32_t* w = src + s * state_stride;
    const std::uint32_t lo = w[(long long)h * word_stride];
    const std::uint32_t hi = h + 1 < kN ? w[(long long)(h + 1) * word_stride] : 0u;
    dst[i] = (lo >> 31) | (hi << 1);
}

// effective -> words (effective_to_words: the dead low bits of word 0 are zero).
__global__ void vmt_eff_to_words_kernel(const std::uint32_t* src, std::uint32_t* dst, long long state_stride,
                                        int word_stride, int n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)n * kN)
        return;
    const long long s = i / kN;
    const int k = (int)(i % kN);
    const std::uint32_t* e = src + s * kRowHalves;
    const std::uint32_t w = k == 0 ? (e[0] & 1u) << 31 : (e[k - 1] >> 1) | (e[k] << 31);
    dst[s * state_stride + (long long)k * word_stride] = w;
}

// out[s] = v[s] * M for S vectors per CTA: CTA (cg, sb) owns the 32-byte
// column group cg (4 u64, one DRAM sector) of vectors sb*S .. sb*S+S-1. Each
// thread XORs the selected rows i = tid (mod 256) into its accumulators and
// the CTA reduces them. Rows are read once per S vectors.
constexpr int kVmS = 4;
constexpr int kVmThreads = 256;
constexpr int kVmGroups = kRowWords / 4; // 78

__global__ void __launch_bounds__(kVmThreads) vmt_vec_mat_kernel(const std::uint64_t* __restrict__ vecs,
                                                                   const std::uint64_t* __restrict__ mat,
                                                                   std::uint64_t* __restrict__ out, int n) {
    __shared__ std::uint64_t vs[kVmS][kRowWords];
    __shared__ ulonglong4 red[kVmThreads / 32][kVmS];
    const int cg = blockIdx.x, s0 = blockIdx.y * kVmS;
    const int ns = n - s0 < kVmS ? n - s0 : kVmS;
    for (int i = threadIdx.x; i < kVmS * kRowWords; i += kVmThreads) {
        const int s = i / kRowWords, w = i % kRowWords;
        vs[s][w] = s < ns ? vecs[(long long)(s0 + s) * kRowWords + w] : 0ull;
    }
    __syncthreads();
    std::uint64_t acc[kVmS][4];
#pragma unroll
    for (int s = 0; s < kVmS; ++s)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            acc[s][c] = 0;
    for (int i = threadIdx.x; i < kDim; i += kVmThreads) {
        unsigned sel = 0;
#pragma unroll
        for (int s = 0; s < kVmS; ++s)
            sel |= (unsigned)((vs[s][i >> 6] >> (i & 63)) & 1ull) << s;
        if (sel == 0)
            continue;
        const ulonglong4 r = *reinterpret_cast<const ulonglong4*>(mat + (long long)i * kRowWords + cg * 4);
#pragma unroll
        for (int s = 0; s < kVmS; ++s)
            if ((sel >> s) & 1u) {
                acc[s][0] ^= r.x;
                acc[s][1] ^= r.y;
                acc[s][2] ^= r.z;
                acc[s][3] ^= r.w;
            }
    }
#pragma unroll
    for (int s = 0; s < kVmS; ++s)
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                acc[s][c] ^= __shfl_xor_sync(0xFFFFFFFFu, acc[s][c], o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int s = 0; s < kVmS; ++s)
            red[warp][s] = make_ulonglong4(acc[s][0], acc[s][1], acc[s][2], acc[s][3]);
    __syncthreads();
    if (threadIdx.x < ns * 4) {
        const int s = threadIdx.x / 4, c = threadIdx.x % 4;
        std::uint64_t v = 0;
#pragma unroll
        for (int w = 0; w < kVmThreads / 32; ++w) {
            const ulonglong4 t = red[w][s];
            v ^= c == 0 ? t.x : c == 1 ? t.y : c == 2 ? t.z : t.w;
        }
        out[(long long)(s0 + s) * kRowWords + cg * 4 + c] = v;
    }
}

} // namespace vmt_b200

// ---------------------------------------------------------------------------
// Chunk positioning as one integer GEMM on the tensor cores (capi_gemmpos.inl).
// Word-bit coordinates: column 32k + b = bit b of state word k (word 0 holds
// only its live bit 31: columns 0..30 are always zero), 624*32 = 19968
// columns. In these coordinates the jump F^d is a 19968 x 19968 0/1 matrix;
// new_states = old_states * F^d over the integers, mod 2.
namespace vmt_b200 {

constexpr int kWB = kN * 32; // 19968 word-bit columns

// effective index e <-> word-bit column: e = 0 <-> 31, e >= 1 <-> e + 31
__device__ __forceinline__ int wb_to_eff(int c) { return c == 31 ? 0 : (c >= 32 ? c - 31 : -1); }

} // namespace vmt_b200

// FP4 (e2m1) GEMM positioning operands (vmt_posmma.cuh): 1.0 = code 0x2, two
// values per byte, low nibble first; unit block scales make the product exact
// (0/1 inputs, fp32 accumulation of at most 19937 ones). The tcgen05 kernel's
// epilogue packs the parities of the accumulators straight back into words.
namespace vmt_b200 {

__global__ void vmt_gemm_matrix_fp4_kernel(const std::uint64_t* __restrict__ rows, std::uint8_t* __restrict__ mwt) {
    const int ip2 = blockIdx.x * blockDim.x + threadIdx.x; // column pair
    const int jc = blockIdx.y;
    if (2 * ip2 >= kWB)
        return;
    const int j = wb_to_eff(jc);
    std::uint8_t v = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int i = wb_to_eff(2 * ip2 + h);
        if (i >= 0 && j >= 0 && ((rows[(long long)i * kRowWords + (j >> 6)] >> (j & 63)) & 1ull))
            v |= (std::uint8_t)(0x2u << (4 * h));
    }
    mwt[(long long)jc * (kWB / 2) + ip2] = v;
}

// a[r][.] for r = c*nl + j: lane lane0+j of state c of an interleaved
// [C][624][L] array (nl = L, lane0 = 0: every lane state), rows [rows,
// rows_pad) zeroed. One thread per row and group of 8 state words: 8 reads
// coalesced across the lanes of a warp, one whole 128-byte line written (one
// word per thread wrote 16-byte pieces of 32 different lines per warp).
__global__ void vmt_states_to_fp4_kernel(const std::uint32_t* __restrict__ st, int L, int lane0, int nl,
                                         long long rows, long long rows_pad, std::uint8_t* __restrict__ a) {
    constexpr int kG = kN / 8; // 78 groups of 8 words per row
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows_pad * kG)
        return;
    // consecutive threads: consecutive lanes j of one (state, word group), then word groups, then states
    long long r;
    int k8;
    const long long live = rows * kG;
    uint4* dst;
    if (idx < live) {
        const int j = (int)(idx % nl);
        const long long cg = idx / nl;
        k8 = (int)(cg % kG);
        const long long c = cg / kG;
        r = c * nl + j;
        dst = reinterpret_cast<uint4*>(a + r * (kWB / 2) + 128 * k8);
        const std::uint32_t* src = st + (c * kN + 8 * k8) * L + lane0 + j;
        std::uint32_t ws[8]; // all eight loads in flight before the first conversion
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
            ws[kk] = __ldg(src + (long long)kk * L);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            std::uint32_t w = ws[kk];
            if (k8 == 0 && kk == 0)
                w &= kUpperMask;
            // byte n holds bits 2n (low nibble) and 2n+1 (high nibble) as code 0x2:
            // bit i of each byte of w moves to bit 4i+1 of a 32-bit word
            std::uint32_t q[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                std::uint32_t x = (w >> (8 * m)) & 0xFFu;
                x = (x | (x << 12)) & 0x000F000Fu;
                x = (x | (x << 6)) & 0x03030303u;
                x = (x | (x << 3)) & 0x11111111u;
                q[m] = x << 1;
            }
            dst[kk] = make_uint4(q[0], q[1], q[2], q[3]);
        }
    } else {
        const long long p = idx - live;
        r = rows + p / kG;
        k8 = (int)(p % kG);
        dst = reinterpret_cast<uint4*>(a + r * (kWB / 2) + 128 * k8);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
            dst[kk] = make_uint4(0u, 0u, 0u, 0u);
    }
}

} // namespace vmt_b200

// Advances k whole blocks: every state of an interleaved [C][624][L] array
// regenerated k times in place (the reference's regenerate,
// mt19937.cpp:36-49). One CTA per chunk: the chunk's 624 x L words are one
// contiguous block, loaded and stored with coalesced 128-byte rows (word i of
// lane t at [i][t]; a warp per lane state read them at a stride of L words, one
// sector per word: 40 us for the bench's 4736 states, now ~6). The block
// splits into the recurrence's dependency phases [0,227), [227,454),
// [454,623), {623}: inside a phase every new word depends only on words the
// phase does not write, so each phase is computed into registers and written
// after a barrier. Used to reuse the positioning matrix of a block delta D
// for deltas D+1..D+4.
namespace vmt_b200 {

constexpr int kAdvThreads = 256;
constexpr int kAdvMaxItems = (227 * 32 + kAdvThreads - 1) / kAdvThreads; // phase words per thread at L = 32
__host__ __device__ constexpr int adv_smem(int L) { return kN * L * 4; }

__global__ void __launch_bounds__(kAdvThreads) vmt_advance_blocks_kernel(std::uint32_t* st, int lgL, int k) {
    extern __shared__ __align__(16) std::uint32_t adv_x[]; // [624][L], L = 2^lgL
    const int L = 1 << lgL;
    std::uint32_t* g = st + (long long)blockIdx.x * kN * L;
    const int total = kN * L;
    if (lgL >= 2) { // (624 L words: a multiple of 4)
#pragma unroll 4
        for (int i = threadIdx.x; i < total / 4; i += kAdvThreads)
            reinterpret_cast<uint4*>(adv_x)[i] = reinterpret_cast<const uint4*>(g)[i];
    } else {
        for (int i = threadIdx.x; i < total; i += kAdvThreads)
            adv_x[i] = g[i];
    }
    __syncthreads();
    for (int r = 0; r < k; ++r) {
#pragma unroll 1
        for (int ph = 0; ph < 3; ++ph) {
            const int lo = ph * 227, cnt = (ph == 2 ? kN - 1 - lo : 227) * L; // (word, lane) items of the phase
            std::uint32_t y[kAdvMaxItems];
#pragma unroll
            for (int j = 0; j < kAdvMaxItems; ++j) {
                const int idx = threadIdx.x + kAdvThreads * j;
                if (idx < cnt) {
                    const int i = lo + (idx >> lgL), t = idx & (L - 1);
                    const int im = i + kM < kN ? i + kM : i + kM - kN;
                    y[j] = twist(adv_x[i * L + t], adv_x[(i + 1) * L + t], adv_x[im * L + t]);
                }
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kAdvMaxItems; ++j) {
                const int idx = threadIdx.x + kAdvThreads * j;
                if (idx < cnt)
                    adv_x[lo * L + idx] = y[j];
            }
            __syncthreads();
        }
        if ((int)threadIdx.x < L) {
            const int t = threadIdx.x;
            adv_x[(kN - 1) * L + t] = twist(adv_x[(kN - 1) * L + t], adv_x[t], adv_x[(kM - 1) * L + t]);
        }
        __syncthreads();
    }
    if (lgL >= 2) {
#pragma unroll 4
        for (int i = threadIdx.x; i < total / 4; i += kAdvThreads)
            reinterpret_cast<uint4*>(g)[i] = reinterpret_cast<const uint4*>(adv_x)[i];
    } else {
        for (int i = threadIdx.x; i < total; i += kAdvThreads)
            g[i] = adv_x[i];
    }
}

// Advances every state of a [n][624] array by its own small step count
// (steps[i] >> shift & mask, < 2^16): the window x_r .. x_{r+623} of the MT
// sequence the state starts, generated in a 1024-word ring in phases of 227
// new words (x_k needs x_{k-227}, x_{k-624}, x_{k-623}: all at least one phase
// old). Word 0 of the result keeps only its live bit, as the polynomial jump's
// output does (mt19937.cpp:79), also for r = 0. ~13x cheaper than a polynomial jump for
// r < 2^16; vmt_jump_states uses it for the low 16 bits of each distance.
constexpr int kStepThreads = 256;
constexpr int kStepPhases = 8;                    // phases generated linearly before the window moves back
constexpr int kStepBuf = kN + 227 * kStepPhases;  // words per state
__global__ void __launch_bounds__(kStepThreads) vmt_advance_steps_kernel(std::uint32_t* st, long long nstates,
                                                                        const unsigned long long* steps,
                                                                        unsigned mask) {
    // One CTA per state: the window x_0..x_623 followed by up to 8 phases of
    // new words, x_{624+k} = twist(x_k, x_{k+1}, x_{k+397}), thread t computing
    // word t of each 227-word phase (one barrier per phase); after 8 phases
    // the last 624 words move back to the front. A warp per state (8 rounds
    // per phase, ring masks) was latency-bound at ~16% occupancy with a long
    // tail behind the largest step counts: 4096 states with 16-bit step
    // counts 0.25 ms.
    __shared__ std::uint32_t x[kStepBuf];
    const int t = threadIdx.x;
    const long long s = blockIdx.x;
    if (s >= nstates)
        return;
    const int r = (int)(steps[s] & mask);
    std::uint32_t* g = st + s * kN;
    if (r == 0) { // the effective state: dead bits of word 0 cleared (mt19937.cpp:79)
        if (t == 0)
            g[0] &= kUpperMask;
        return;
    }
    for (int i = t; i < kN; i += kStepThreads)
        x[i] = g[i];
    __syncthreads();
    int produced = 0, batch = 0;
    for (;;) {
        batch = min(r - produced, 227 * kStepPhases);
        for (int base = 0; base < batch; base += 227) {
            if (t < min(227, batch - base))
                x[kN + base + t] = twist(x[base + t], x[base + t + 1], x[base + t + kM]);
            __syncthreads();
        }
        produced += batch;
        if (produced >= r)
            break;
        // a whole batch (1816 >= 624 new words): the last 624 words become the window
        for (int i = t; i < kN; i += kStepThreads)
            x[i] = x[batch + i];
        __syncthreads();
    }
    for (int i = t; i < kN; i += kStepThreads) {
        const std::uint32_t v = x[batch + i];
        g[i] = i == 0 ? (v & kUpperMask) : v;
    }
}

} // namespace vmt_b200
