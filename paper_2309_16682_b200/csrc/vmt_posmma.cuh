// Chunk positioning on the tensor cores, co-resident with the generation
// kernel (hand-written tcgen05, sm_100a).
//
// Steady-state fills of the same shape move every chunk start by the same
// block delta D, so the next fill's chunk lane states are this fill's times
// ONE GF(2) matrix F^(624 D) (capi_gemmpos.inl): in word-bit coordinates
//   new[r][j] = sum_i bits(old[r])[i] * M[j][i]  (mod 2),  i, j < 19968.
// This kernel computes that product while the store-bound generation kernel
// runs: the generation CTA (one per SM, 108 KB of shared memory, 168
// registers x 256 threads) leaves ~120 KB of shared memory, 22.5k registers
// and the whole tensor core of every SM idle, and one CTA of this kernel
// (192 threads, 80 KB) fits beside it. The positioning then costs the
// generation kernel only the issue slots of the operand expansion instead of
// a serial 0.8 ms GEMM between fills.
//
// Tile: 128 lane states (M) x 512 output bit columns (N, two N=256
// accumulators = all 512 TMEM columns), K staged 64 bytes at a time through a
// 2-deep ring. kind::i8 with 0/1 operands and s32 accumulation is exact
// (sums <= 19937); bit j of the new state is the low bit of column j.
//   warp 0     TMA producer: B = M[j][i] int8, K-major, 64B-swizzled boxes
//   warp 1     TMEM allocator; one elected lane issues tcgen05.mma
//   warps 2-5  A producers: expand the compact state words of their 32 rows
//              into 0/1 bytes in the 64B-swizzled K-major layout (no operand
//              buffer in HBM); then the epilogue of the same rows: tcgen05.ld
//              32 columns = one state word per load, packed to bits, stored
//              into the interleaved [C][624][L] chunk-state array.
// Tiles are ordered N-slice-major so the CTAs running at the same time share
// B slices through L2; the 12 MB of compact states stay L2-resident.
#pragma once

#include <cuda.h>

#include "vmt_common.cuh"
#include "vmt_gen.cuh"

namespace vmt_b200 {

constexpr int kPmM = 128;                  // lane states per tile
constexpr int kPmN = 512;                  // output bit columns per tile
constexpr int kPmK = 64;                   // K bytes per stage (= one 64B swizzle atom row)
constexpr int kPmStages = 2;
constexpr int kPmABytes = kPmM * kPmK;     // 8 KB
constexpr int kPmBBytes = kPmN * kPmK;     // 32 KB (two 256-row TMA boxes)
constexpr int kPmStageBytes = kPmABytes + kPmBBytes;
constexpr int kPmKSteps = (kN * 32) / kPmK; // 312
constexpr int kPmNTiles = (kN * 32) / kPmN; // 39
constexpr int kPmThreads = 192;
constexpr int kPmSmem = kPmStages * kPmStageBytes + 1024 /* align */ + 128 /* barriers */;

struct PosMmaParams {
    const std::uint32_t* src; // [C][624][L] chunk lane states (this fill's)
    std::uint32_t* dst;       // [C][624][L] jumped by the matrix (the next fill's)
    int L;
    int rows;                 // C * L
    int m_tiles;              // ceil(rows / 128)
    unsigned flags;           // experiment knobs (VMT_PM_FLAGS): bit0 polite waits, bit1 no A expansion,
                              // bit2 no MMA, bits 8..23 MMA pacing in 64 ns units per stage
};

// Waits without competing for issue slots with the co-resident generation
// warps: a suspending try_wait, then exponential __nanosleep backoff.
__device__ __forceinline__ void mbar_wait_polite(unsigned long long* bar, unsigned parity) {
    unsigned ns = 32;
    for (;;) {
        unsigned done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 100000;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done)
            return;
        __nanosleep(ns);
        ns = ns < 2048 ? ns * 2 : ns;
    }
}
__device__ __forceinline__ void pm_wait(unsigned long long* bar, unsigned parity, unsigned flags) {
    if (flags & 1u)
        mbar_wait_polite(bar, parity);
    else
        mbar_wait_parity(bar, parity);
}

// ---- tcgen05 / TMA primitives -------------------------------------------------
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// TMA tile load with an L2 eviction-priority policy (the B slices are shared
// by the CTAs working on the same N slice; keep them against the generation
// kernel's store stream)
__device__ __forceinline__ void tma_load_2d(void* sdst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar, unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
        "{%2, %3}], [%4], %5;" ::"r"(smem_u32(sdst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(unsigned long long* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_i8(unsigned tmem_d, unsigned long long adesc, unsigned long long bdesc,
                                          unsigned idesc, unsigned accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// K-major operand in the 64-byte swizzle layout: 8-row groups of 8 x 64 B
// (stride 512 B), 16-byte chunk c of row r at chunk c ^ ((r >> 1) & 3).
__device__ __forceinline__ unsigned long long sw64_desc(unsigned saddr) {
    unsigned long long d = 0;
    d |= (unsigned long long)((saddr & 0x3FFFFu) >> 4);  // start address
    d |= (unsigned long long)1 << 16;                     // leading byte offset (unused when swizzled)
    d |= (unsigned long long)(512 >> 4) << 32;            // stride byte offset: next 8-row group
    d |= (unsigned long long)1 << 46;                     // descriptor version (sm_100)
    d |= (unsigned long long)4 << 61;                     // SWIZZLE_64B
    return d;
}
// kind::i8 instruction descriptor: s32 accumulator, u8 x u8, both K-major,
// N = 256, M = 128
constexpr unsigned kPmIdesc = (2u << 4) | ((256u >> 3) << 17) | ((128u >> 4) << 24);

// 32 bits -> 32 bytes of 0/1, as 8 u32 (byte b = bit b)
__device__ __forceinline__ void expand_bits(std::uint32_t w, std::uint32_t q[8]) {
#pragma unroll
    for (int n = 0; n < 8; ++n)
        q[n] = (((w >> (4 * n)) & 15u) * 0x00204081u) & 0x01010101u;
}

__global__ void __launch_bounds__(kPmThreads, 1)
    vmt_posmma_kernel(const __grid_constant__ CUtensorMap tmap_b, const PosMmaParams p) {
    extern __shared__ unsigned char pm_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(pm_raw) + 1023) &
                                                           ~static_cast<std::uintptr_t>(1023));
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + kPmStages * kPmStageBytes);
    unsigned long long* empty = full + kPmStages;
    unsigned long long* accf = empty + kPmStages;
    unsigned* tmem_slot = reinterpret_cast<unsigned*>(accf + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kPmStages; ++s) {
            mbar_init(&full[s], 5); // 4 A-producer warps + the TMA producer's expect_tx
            mbar_init(&empty[s], 1);
        }
        mbar_init(accf, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tmap_b)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned tmem = *tmem_slot;

    const int ntiles = p.m_tiles * kPmNTiles;
    if (warp == 0) {
        if (lane == 0) {
            const unsigned long long pol = l2_policy_evict_last();
            unsigned it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int n = tile / p.m_tiles;
                for (int ks = 0; ks < kPmKSteps; ++ks, ++it) {
                    const int s = it % kPmStages;
                    const unsigned u = it / kPmStages;
                    if (u > 0)
                        pm_wait(&empty[s], (u - 1) & 1, p.flags);
                    unsigned char* b = smem + s * kPmStageBytes + kPmABytes;
                    mbar_arrive_expect_tx(&full[s], kPmBBytes);
                    tma_load_2d(b, &tmap_b, ks * kPmK, n * kPmN, &full[s], pol);
                    tma_load_2d(b + kPmBBytes / 2, &tmap_b, ks * kPmK, n * kPmN + 256, &full[s], pol);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            unsigned it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int ks = 0; ks < kPmKSteps; ++ks, ++it) {
                    const int s = it % kPmStages;
                    pm_wait(&full[s], (it / kPmStages) & 1, p.flags);
                    tc_fence_after();
                    const unsigned a = smem_u32(smem + s * kPmStageBytes);
                    const unsigned b = a + kPmABytes;
                    if (p.flags >> 8)
                        __nanosleep(64u * ((p.flags >> 8) & 0xFFFFu));
                    if (!(p.flags & 4u))
#pragma unroll
                    for (int kk = 0; kk < kPmK / 32; ++kk) {
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            tc_mma_i8(tmem + 256 * h, sw64_desc(a + 32 * kk),
                                      sw64_desc(b + h * (kPmBBytes / 2) + 32 * kk), kPmIdesc,
                                      (ks | kk) != 0);
                    }
                    tc_commit(&empty[s]); // frees the stage when these MMAs are done
                }
                tc_commit(accf); // the tile's accumulators are complete
            }
        }
    } else {
        // A producers + epilogue: TMEM lane quarter (warp % 4) = rows 32*(warp%4) + lane
        const int rq = (warp & 3) * 32;
        const int r = rq + lane; // row within the tile
        unsigned it = 0, tcount = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
            const int n = tile / p.m_tiles, m = tile % p.m_tiles;
            const int row = m * kPmM + r;
            const bool valid = row < p.rows;
            const int c = valid ? row / p.L : 0, t = valid ? row % p.L : 0;
            const std::uint32_t* src = p.src + (long long)c * kN * p.L + t;
            unsigned char* arow = smem + (r >> 3) * 512 + (r & 7) * 64;
            const int sw = (r >> 1) & 3;
            for (int ks = 0; ks < kPmKSteps; ++ks, ++it) {
                const int s = it % kPmStages;
                const unsigned u = it / kPmStages;
                std::uint32_t w0 = 0, w1 = 0;
                if (valid) {
                    w0 = __ldg(src + (long long)(2 * ks) * p.L);
                    w1 = __ldg(src + (long long)(2 * ks + 1) * p.L);
                    if (ks == 0)
                        w0 &= kUpperMask;
                }
                if (u > 0)
                    pm_wait(&empty[s], (u - 1) & 1, p.flags);
                unsigned char* a = arow + s * kPmStageBytes;
                std::uint32_t q[8];
                if (!(p.flags & 2u)) {
                expand_bits(w0, q);
                *reinterpret_cast<uint4*>(a + 16 * (0 ^ sw)) = make_uint4(q[0], q[1], q[2], q[3]);
                *reinterpret_cast<uint4*>(a + 16 * (1 ^ sw)) = make_uint4(q[4], q[5], q[6], q[7]);
                expand_bits(w1, q);
                *reinterpret_cast<uint4*>(a + 16 * (2 ^ sw)) = make_uint4(q[0], q[1], q[2], q[3]);
                *reinterpret_cast<uint4*>(a + 16 * (3 ^ sw)) = make_uint4(q[4], q[5], q[6], q[7]);
                }
                fence_proxy_async_smem(); // generic-proxy writes -> visible to the tensor core
                __syncwarp();
                if (lane == 0)
                    mbar_arrive(&full[s]);
            }
            // epilogue: 16 state words (512 columns) of this row
            pm_wait(accf, tcount & 1, p.flags);
            tc_fence_after();
            std::uint32_t* dst = p.dst + (long long)c * kN * p.L + t;
#pragma unroll 1
            for (int j = 0; j < kPmN / 32; ++j) {
                std::uint32_t v[32];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
                      "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
                      "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(tmem + ((unsigned)rq << 16) + 32u * j));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                std::uint32_t w = 0;
#pragma unroll
                for (int b = 0; b < 32; ++b)
                    w |= (v[b] & 1u) << b;
                const int k = n * (kPmN / 32) + j;
                if (valid)
                    dst[(long long)k * p.L] = k == 0 ? (w & kUpperMask) : w;
            }
            tc_fence_before(); // TMEM reads ordered before the next tile's MMAs
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

} // namespace vmt_b200
