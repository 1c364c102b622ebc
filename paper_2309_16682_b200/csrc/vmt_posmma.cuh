// Chunk positioning on the tensor cores, co-resident with the generation
// kernel (hand-written tcgen05, sm_100a).
//
// Steady-state fills of the same shape move every chunk start by the same
// block delta D, so the next fill's chunk lane states are this fill's times
// ONE GF(2) matrix F^(624 D) (capi_gemmpos.inl): in word-bit coordinates
//   new[r][j] = sum_i bits(old[r])[i] * M[j][i]  (mod 2),  i, j < 19968.
// This kernel computes that product while the store-bound generation kernel
// runs: the generation CTA (one per SM at L=32: 86 KB of shared memory, 162
// registers x 256 threads) leaves ~140 KB of shared memory, 24k registers
// and the whole tensor core of every SM idle, and one CTA of this kernel
// (192 threads, a 3-stage operand ring of 130 KB) fits beside it.
//
// What it costs the generation kernel is mostly shared-memory bandwidth: the
// tensor core reads its operands from shared memory, (1/M + 1/N) bytes per
// MAC per byte-wide element, and the generation kernel's ring traffic runs
// through the same ports (measured with an int8 version: ~0.8 ms added to an
// 11.2 ms generation kernel, all of it the MMA operand reads). So the
// operands are FP4 (kind::mxf4: e2m1 0/1 values, unit ue8m0 block scales held
// in TMEM, fp32 accumulation -- exact, sums <= 19937), half the bytes of int8.
//
// Tile: 128 lane states (M) x 416 output bit columns (two N=208 MMAs side by
// side in TMEM = 13 whole state words), K staged 256 elements (128 bytes per
// operand row = one L2 line) at a time through a ring, both operands by TMA
// (128-byte swizzle, L2 evict_last so the CTAs on the same N slice share B
// through L2):
//   warp 0     TMA producer: A = the states' FP4 operand [rows][9984 B]
//              (vmt_states_to_fp4_kernel), B = F^(624D) FP4 [19968][9984 B]
//   warp 1     TMEM allocator; one elected lane issues tcgen05.mma
//   warps 2-5  unit scale factors into TMEM; epilogue: tcgen05.ld 32 columns
//              = one state word per load, parity of each sum -> bit, stored
//              into the interleaved [C][624][L] chunk-state array.
#pragma once

#include <cuda.h>

#include "vmt_common.cuh"
#include "vmt_gen.cuh"

namespace vmt_b200 {

constexpr int kPmM = 128;                  // lane states per tile
#ifndef VMT_POSMMA_NH
#define VMT_POSMMA_NH 208
#endif
constexpr int kPmNH = VMT_POSMMA_NH;       // output bit columns per MMA (N); 2 x kPmNH must be whole state words
static_assert((2 * VMT_POSMMA_NH) % 32 == 0 && (kN * 32) % (2 * VMT_POSMMA_NH) == 0 && VMT_POSMMA_NH % 16 == 0,
              "tile = whole state words, tiling 19968 columns");
constexpr int kPmN = 2 * kPmNH;            // per tile: two MMAs side by side in TMEM = 13 state words
// K elements (input bits) per stage: 256 = 128 bytes of FP4 per operand row, one
// whole L2 line per row and TMA box (128-byte swizzle); 128 = 64 bytes (64-byte
// swizzle, half lines: the round-1/2 shape, kept for A/B builds)
#ifndef VMT_POSMMA_KE
#define VMT_POSMMA_KE 256
#endif
constexpr int kPmKE = VMT_POSMMA_KE;
static_assert(kPmKE == 128 || kPmKE == 256, "one swizzle span per operand row and stage");
constexpr int kPmStages = 3;              // single-CTA kernel (the pair kernel's depth is a template argument)
constexpr int kPmABytes = kPmM * kPmKE / 2;        // 8 KB
constexpr int kPmBHBytes = kPmNH * kPmKE / 2;      // 13 KB per N half
constexpr int kPmStageBytes = kPmABytes + 2 * kPmBHBytes;
constexpr int kPmKSteps = (kN * 32) / kPmKE; // 156
constexpr int kPmNTiles = (kN * 32) / kPmN;  // 48
constexpr int kPmThreads = 192;
constexpr int kPmSmem = kPmStages * kPmStageBytes + 1024 /* align */ + 128 /* barriers */;
constexpr int kPmSfCol = 448;              // TMEM columns [448, 512): unit scale factors

// Parity of an fp32 accumulator holding an exact integer sum v < 2^23: the
// lowest mantissa bit of v + 2^23 (one FADD on the FMA pipe instead of an
// F2I conversion on the slow pipe; 416 per epilogue thread and tile)
__device__ __forceinline__ std::uint32_t parity_bit(std::uint32_t acc) {
    return __float_as_uint(__uint_as_float(acc) + 8388608.0f) & 1u;
}
// The 32 parities of v[0..31] as one word, bit b from v[b]: each step shifts
// the word right by one and takes the lowest mantissa bit of v[b] + 2^23 in at
// bit 31 (one FADD + one funnel shift per bit instead of FADD, AND, SHL, OR)
__device__ __forceinline__ std::uint32_t parity_word(const std::uint32_t (&v)[32]) {
    std::uint32_t w = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b)
        w = __funnelshift_r(w, __float_as_uint(__uint_as_float(v[b]) + 8388608.0f), 1);
    return w;
}

struct PosMmaParams {
    std::uint32_t* dst;       // [C][624][L] jumped by the matrix (the next fill's)
    int L;
    int rows;                 // C * nl
    int m_tiles;              // ceil(rows / 128) (pair kernel: ceil(rows / 256))
    int nl, lane0;            // row r -> state r / nl, lane lane0 + r % nl (all lanes: nl = L, lane0 = 0)
    unsigned* tile_ctr;       // pair kernel: the launch's tile counter (zero before and after every launch)
#ifdef VMT_TIMELINE
    unsigned long long* tl;   // experiments: per-CTA {start ns, end ns, SM id}
#endif
};

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
// D[tmem] (+)= A[smem] x B[smem]^T, FP4 e2m1 operands with per-32-element
// ue8m0 scale factors read from TMEM (all 1.0 here), fp32 accumulation
__device__ __forceinline__ void tc_mma_mxf4(unsigned tmem_d, unsigned long long adesc, unsigned long long bdesc,
                                            unsigned idesc, unsigned tmem_sfa, unsigned tmem_sfb,
                                            unsigned accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(
            tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(tmem_sfa), "r"(tmem_sfb), "r"(accumulate)
        : "memory");
}
// K-major operand in the swizzled layout of one stage: rows of kPmKE / 2 bytes
// in 8-row groups (stride 8 rows). 64-byte rows: 16-byte chunk c of row r at
// chunk c ^ ((r >> 1) & 3) (SWIZZLE_64B); 128-byte rows: at chunk c ^ (r & 7)
// (SWIZZLE_128B). The K = 64 slices of a stage are 32 bytes apart.
__device__ __forceinline__ unsigned long long sw64_desc(unsigned saddr) {
    unsigned long long d = 0;
    d |= (unsigned long long)((saddr & 0x3FFFFu) >> 4);  // start address
    d |= (unsigned long long)1 << 16;                     // leading byte offset (unused when swizzled)
    d |= (unsigned long long)((8 * kPmKE / 2) >> 4) << 32; // stride byte offset: next 8-row group
    d |= (unsigned long long)1 << 46;                     // descriptor version (sm_100)
    d |= (unsigned long long)(kPmKE == 256 ? 2 : 4) << 61; // SWIZZLE_128B / SWIZZLE_64B
    return d;
}
// kind::mxf4 instruction descriptor: A and B e2m1 (MXF4 format 1), both
// K-major, N = 208, ue8m0 scales, M = 128, K = 64, scale-factor ids 0
constexpr unsigned kPmIdesc = (1u << 7) | (1u << 10) | ((unsigned)(kPmNH >> 3) << 17) | (1u << 23) |
                              ((128u >> 4) << 24);

__global__ void __launch_bounds__(kPmThreads, 1)
    vmt_posmma_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                      const PosMmaParams p) {
    extern __shared__ unsigned char pm_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(pm_raw) + 1023) &
                                                           ~static_cast<std::uintptr_t>(1023));
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + kPmStages * kPmStageBytes);
    unsigned long long* empty = full + kPmStages;
    unsigned long long* accf = empty + kPmStages; // MMA -> epilogue: accumulators complete
    unsigned long long* accd = accf + 1;           // epilogue -> MMA: accumulators drained
    unsigned* tmem_slot = reinterpret_cast<unsigned*>(accd + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kPmStages; ++s) {
            mbar_init(&full[s], 1); // the TMA producer's expect_tx (A + B bytes)
            mbar_init(&empty[s], 1);
        }
        mbar_init(accf, 1);
        mbar_init(accd, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tmap_a)) : "memory");
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
    if (warp >= 2) {
        // unit scale factors (ue8m0 0x7F = 1.0) in every byte of TMEM columns
        // [448, 512) of this warp's lane quarter: whatever the scale-factor
        // layout inside that range, every factor reads as 1.0
        const unsigned one4 = 0x7F7F7F7Fu;
#pragma unroll
        for (int c0 = kPmSfCol; c0 < 512; c0 += 16)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                    tmem + ((unsigned)((warp & 3) * 32) << 16) + (unsigned)c0),
                "r"(one4)
                : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const int ntiles = p.m_tiles * kPmNTiles;
    if (warp == 0) {
        if (lane == 0) {
            const unsigned long long pol = l2_policy_evict_last();
            unsigned it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int n = tile / p.m_tiles, m = tile % p.m_tiles;
                for (int ks = 0; ks < kPmKSteps; ++ks, ++it) {
                    const int s = it % kPmStages;
                    const unsigned u = it / kPmStages;
                    if (u > 0)
                        mbar_wait_parity(&empty[s], (u - 1) & 1);
                    unsigned char* a = smem + s * kPmStageBytes;
                    unsigned char* b = a + kPmABytes;
                    mbar_arrive_expect_tx(&full[s], kPmStageBytes);
                    tma_load_2d(a, &tmap_a, ks * (kPmKE / 2), m * kPmM, &full[s], pol);
                    tma_load_2d(b, &tmap_b, ks * (kPmKE / 2), n * kPmN, &full[s], pol);
                    tma_load_2d(b + kPmBHBytes, &tmap_b, ks * (kPmKE / 2), n * kPmN + kPmNH, &full[s], pol);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            unsigned it = 0, tcount = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
                if (tcount > 0) { // the previous tile's epilogue has read the accumulators
                    mbar_wait_parity(accd, (tcount - 1) & 1);
                    tc_fence_after();
                }
                for (int ks = 0; ks < kPmKSteps; ++ks, ++it) {
                    const int s = it % kPmStages;
                    mbar_wait_parity(&full[s], (it / kPmStages) & 1);
                    tc_fence_after();
                    const unsigned a = smem_u32(smem + s * kPmStageBytes);
                    const unsigned b = a + kPmABytes;
#pragma unroll
                    for (int kk = 0; kk < kPmKE / 64; ++kk) { // K=64 MMAs (32 bytes each) per stage
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            tc_mma_mxf4(tmem + kPmNH * h, sw64_desc(a + 32 * kk),
                                        sw64_desc(b + h * kPmBHBytes + 32 * kk), kPmIdesc, tmem + kPmSfCol,
                                        tmem + kPmSfCol + 32, (ks | kk) != 0);
                    }
                    tc_commit(&empty[s]); // frees the stage when these MMAs are done
                }
                tc_commit(accf); // the tile's accumulators are complete
            }
        }
    } else {
        // epilogue: TMEM lane quarter (warp % 4) = rows 32*(warp%4) + lane
        const int rq = (warp & 3) * 32;
        const int r = rq + lane; // row within the tile
        unsigned tcount = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
            const int n = tile / p.m_tiles, m = tile % p.m_tiles;
            const int row = m * kPmM + r;
            const bool valid = row < p.rows;
            const int c = valid ? row / p.nl : 0, t = valid ? p.lane0 + row % p.nl : 0;
            // 13 state words (416 columns) of this row
            mbar_wait_parity(accf, tcount & 1);
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
                const std::uint32_t w = parity_word(v); // exact fp32 sums of 0/1 products: bit = parity
                const int k = n * (kPmN / 32) + j;
                if (valid)
                    dst[(long long)k * p.L] = k == 0 ? (w & kUpperMask) : w;
            }
            tc_fence_before(); // TMEM reads ordered before the next tile's MMAs
            __syncwarp();
            if (lane == 0)
                mbar_arrive(accd); // this warp's rows are drained
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// ---- CTA-pair form (cta_group::2) -------------------------------------------
// The same product with M = 256 lane states per MMA across a cluster of two
// CTAs on one TPC: each CTA holds its own 128 rows of A and HALF of every B
// tile (104 of the 208 rows per MMA), the leader CTA issues
// tcgen05.mma.cta_group::2 and each CTA's TMEM receives its 128 rows of the
// accumulators. Per SM the tensor core reads (1/208 + 1/256) instead of
// (1/208 + 1/128) operand bytes per MAC from shared memory, and the B tiles
// cross L2 -> SM half as often: less of what the co-resident GEMM takes from
// the generation kernel (§4.6).
constexpr int kP2BQ = kPmNH / 2;                    // 104 B rows per CTA per MMA
constexpr int kP2BQBytes = kP2BQ * kPmKE / 2;       // 6656
constexpr int kP2StageBytes = kPmABytes + 2 * kP2BQBytes; // 21504
// Operand-ring depth (stages of 43 KB with the 256-element K stage): 3 fit
// beside the 86 KB L=32 generation CTA on one SM (the co-resident prefetch), 4
// beside the L=16 one, 5 when the kernel runs alone (serial positioning, batch
// de-phasing); the B operand (200 MB) streams from HBM, it does not fit in L2.
constexpr int kP2Stages = 4;
__host__ __device__ constexpr int p2_smem(int stages) { return stages * kP2StageBytes + 1024 + 256; }
constexpr int kP2Smem = p2_smem(kP2Stages);
// kind::mxf4, M = 256 (pair), N = 208
constexpr unsigned kP2Idesc = (1u << 7) | (1u << 10) | ((unsigned)(kPmNH >> 3) << 17) | (1u << 23) |
                              ((256u >> 4) << 24);

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (a shared::cta variable) in CTA `rank`
__device__ __forceinline__ unsigned map_to_rank(const void* p, unsigned rank) {
    unsigned out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
    return out;
}
__device__ __forceinline__ void tma_load_2d_pair(void* sdst, const CUtensorMap* map, int x, int y,
                                                 unsigned bar_cluster, unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(sdst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(bar_cluster), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tc_commit_pair(unsigned long long* bar) {
    // arrives on the barrier at the same offset in both CTAs of the pair
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((unsigned short)3)
        : "memory");
}
__device__ __forceinline__ void tc_mma_mxf4_pair(unsigned tmem_d, unsigned long long adesc,
                                                 unsigned long long bdesc, unsigned idesc, unsigned tmem_sfa,
                                                 unsigned tmem_sfb, unsigned accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(
            tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(tmem_sfa), "r"(tmem_sfb), "r"(accumulate)
        : "memory");
}

// Tile scheduler of the pair kernel: the leader CTA's producer thread takes the
// next tile from a global counter and publishes it to both CTAs of the pair
// (a 4-slot ring per CTA, one mbarrier per slot), so a pair slowed by the
// generation CTAs it shares its SMs with takes fewer tiles than a pair on free
// SMs (config 1: 60-75 generation CTAs on 148 SMs). Consecutive tiles share
// their N slice, so the pairs running together still share B through L2.
// Every role reads the same sequence; a slot is rewritten four fetches later,
// by which time the producer has loaded three more whole tiles, i.e. the MMA
// thread is in tile i+3 and both epilogues are done with tile i+2.
constexpr int kP2TileSlots = 4;
__device__ __forceinline__ void mbar_wait_parity_cluster(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "VMT_WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra VMT_WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(unsigned bar_cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
// the seq-th tile of this pair (every thread of every role calls it with the same seq order)
__device__ __forceinline__ int p2_next_tile(unsigned long long* tfull, const volatile unsigned* tslot, unsigned seq) {
    mbar_wait_parity_cluster(&tfull[seq % kP2TileSlots], (seq / kP2TileSlots) & 1);
    return (int)tslot[seq % kP2TileSlots];
}

// p.m_tiles = ceil(rows / 256) pair tiles; tmap_b boxes are 104 rows
template <int kStages>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPmThreads, 1)
    vmt_posmma2_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                       const PosMmaParams p) {
    extern __shared__ unsigned char pm_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(pm_raw) + 1023) &
                                                           ~static_cast<std::uintptr_t>(1023));
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + kStages * kP2StageBytes);
    unsigned long long* empty = full + kStages;
    unsigned long long* accf = empty + kStages; // MMA -> epilogues (both CTAs)
    unsigned long long* accd = accf + 1;           // epilogues (both CTAs) -> leader's MMA thread
    unsigned long long* tfull = accd + 1;          // leader's producer -> every role of both CTAs: tile published
    unsigned* tslot = reinterpret_cast<unsigned*>(tfull + kP2TileSlots);
    unsigned* tmem_slot = tslot + kP2TileSlots;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned rank = cluster_rank();
    const bool leader = rank == 0;
#ifdef VMT_TIMELINE
    if (p.tl && threadIdx.x == 0 && blockIdx.x < 1024) {
        p.tl[blockIdx.x * 3] = tl_now();
        p.tl[blockIdx.x * 3 + 2] = tl_smid();
    }
#endif
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);  // leader: its producer's expect_tx for both CTAs' bytes
            mbar_init(&empty[s], 1); // MMA commit, multicast to both CTAs
        }
        mbar_init(accf, 1);
        mbar_init(accd, 8); // 4 epilogue warps x 2 CTAs
        for (int i = 0; i < kP2TileSlots; ++i)
            mbar_init(&tfull[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tmap_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&tmap_b)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const unsigned tmem = *tmem_slot;
    if (warp >= 2) { // unit scale factors in this CTA's TMEM columns [448, 512)
        const unsigned one4 = 0x7F7F7F7Fu;
#pragma unroll
        for (int c0 = kPmSfCol; c0 < 512; c0 += 16)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                    tmem + ((unsigned)((warp & 3) * 32) << 16) + (unsigned)c0),
                "r"(one4)
                : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();

    const int npairs = gridDim.x >> 1;
    const int ntiles = p.m_tiles * kPmNTiles;
    if (warp == 0) {
        if (lane == 0) {
            const unsigned long long pol = l2_policy_evict_last();
            unsigned it = 0;
            for (unsigned seq = 0;; ++seq) {
                int tile;
                if (leader) {
                    // no counter: the static round-robin (every pair equally loaded)
                    const unsigned t = p.tile_ctr ? atomicAdd(p.tile_ctr, 1u)
                                                  : (unsigned)(blockIdx.x >> 1) + seq * (unsigned)npairs;
                    const unsigned sl = seq % kP2TileSlots;
                    tslot[sl] = t;
                    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(map_to_rank(&tslot[sl], 1)), "r"(t)
                                 : "memory");
                    mbar_arrive_cluster(map_to_rank(&tfull[sl], 0));
                    mbar_arrive_cluster(map_to_rank(&tfull[sl], 1));
                    // every pair draws exactly one tile >= ntiles: the last of them re-zeroes the counter
                    if (p.tile_ctr && t == (unsigned)(ntiles + npairs - 1))
                        atomicExch(p.tile_ctr, 0u);
                    tile = (int)t;
                } else
                    tile = p2_next_tile(tfull, tslot, seq);
                if (tile >= ntiles)
                    break;
                const int n = tile / p.m_tiles, m = tile % p.m_tiles;
                for (int ks = 0; ks < kPmKSteps; ++ks, ++it) {
                    const int s = it % kStages;
                    const unsigned u = it / kStages;
                    if (u > 0)
                        mbar_wait_parity(&empty[s], (u - 1) & 1);
                    unsigned char* a = smem + s * kP2StageBytes;
                    unsigned char* b = a + kPmABytes;
                    if (leader)
                        mbar_arrive_expect_tx(&full[s], 2 * kP2StageBytes);
                    const unsigned fb = map_to_rank(&full[s], 0);
                    const int kx = ks * (kPmKE / 2);
                    tma_load_2d_pair(a, &tmap_a, kx, m * 2 * kPmM + (int)rank * kPmM, fb, pol);
                    tma_load_2d_pair(b, &tmap_b, kx, n * kPmN + (int)rank * kP2BQ, fb, pol);
                    tma_load_2d_pair(b + kP2BQBytes, &tmap_b, kx, n * kPmN + kPmNH + (int)rank * kP2BQ, fb, pol);
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            unsigned it = 0, tcount = 0;
            for (;; ++tcount) {
                if (p2_next_tile(tfull, tslot, tcount) >= ntiles)
                    break;
                if (tcount > 0) { // both CTAs' epilogues have read the previous accumulators
                    mbar_wait_parity(accd, (tcount - 1) & 1);
                    tc_fence_after();
                }
                for (int ks = 0; ks < kPmKSteps; ++ks, ++it) {
                    const int s = it % kStages;
                    mbar_wait_parity(&full[s], (it / kStages) & 1);
                    tc_fence_after();
                    const unsigned a = smem_u32(smem + s * kP2StageBytes);
                    const unsigned b = a + kPmABytes;
#pragma unroll
                    for (int kk = 0; kk < kPmKE / 64; ++kk)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            tc_mma_mxf4_pair(tmem + kPmNH * h, sw64_desc(a + 32 * kk),
                                             sw64_desc(b + h * kP2BQBytes + 32 * kk), kP2Idesc, tmem + kPmSfCol,
                                             tmem + kPmSfCol + 32, (ks | kk) != 0);
                    tc_commit_pair(&empty[s]);
                }
                tc_commit_pair(accf);
            }
        }
    } else {
        const int rq = (warp & 3) * 32;
        const int r = (int)rank * kPmM + rq + lane; // row within the 256-row pair tile
        const unsigned accd_leader = map_to_rank(accd, 0);
        unsigned tcount = 0;
        for (;; ++tcount) {
            const int tile = p2_next_tile(tfull, tslot, tcount);
            if (tile >= ntiles)
                break;
            const int n = tile / p.m_tiles, m = tile % p.m_tiles;
            const int row = m * 2 * kPmM + r;
            const bool valid = row < p.rows;
            const int c = valid ? row / p.nl : 0, t = valid ? p.lane0 + row % p.nl : 0;
            mbar_wait_parity(accf, tcount & 1);
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
                const std::uint32_t w = parity_word(v);
                const int k = n * (kPmN / 32) + j;
                if (valid)
                    dst[(long long)k * p.L] = k == 0 ? (w & kUpperMask) : w;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(accd_leader)
                             : "memory");
        }
    }
#ifdef VMT_TIMELINE
    if (p.tl && threadIdx.x == 64 && blockIdx.x < 1024) // an epilogue warp: after its last tile
        p.tl[blockIdx.x * 3 + 1] = tl_now();
#endif
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

} // namespace vmt_b200
