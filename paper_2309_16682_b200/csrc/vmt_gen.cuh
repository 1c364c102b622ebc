// sm_100a generation kernel for VMT19937: twist + temper + emit (the hot path).
//
// Replaces VmtEngine::regenerate + temper_words (engine.hpp:110-142) and the
// lane backends' twist/temper (lane_ops.hpp:81-93, 184-195).
//
// A CTA owns one chunk of the combined stream (all L lanes). Each lane's
// MT19937 word sequence x_0, x_1, ... (x_{n+624} = x_{n+397} ^
// mulA((x_n & h) | (x_{n+1} & l))) lives in a shared-memory
// ring of RING = 624 + W slots (+R mirror slots), interleaved [slot][lane]
// like the reference's interleaved state (engine.hpp:58-60). A window computes
// W new words of every lane (W <= 227, the recurrence's parallel width): it
// reads only slots written >= 1 window earlier and writes the W slots freed by
// the previous window, so one __syncthreads per window is the only
// synchronisation (the reference's 227/396/1 loop split is the sequential
// special case, engine.hpp:119-131). 624/W windows make one 624*L-word block,
// emitted tempered in combined-stream order word[b*624L + k*L + t] (SURVEY.md
// A13).
//
// Output path: one window's output is ONE contiguous W*L-element range of the
// stream, so store-mode windows are staged in shared memory and written by a
// single TMA bulk copy (cp.async.bulk.global.shared::cta) issued by one
// thread after the window barrier -- the per-thread store traffic never goes
// through the LSU/L1 path that the ring loads use. An mbarrier tells the
// writers of the next window when the bulk copy has finished reading the
// staging buffer. Edge windows (range start/end) use direct predicated stores.
#pragma once

#include "vmt_common.cuh"

namespace vmt_b200 {

// ---- TMA bulk-store / mbarrier helpers --------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* ptr) {
    return static_cast<unsigned>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "VMT_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra VMT_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

#ifndef VMT_GEN_HIST
#define VMT_GEN_HIST 1
#endif

template <int MODE>
__host__ __device__ constexpr int elem_bytes() {
    return (MODE == MODE_F64 || MODE == MODE_F64_REAL3 || MODE == MODE_F64_RES53) ? 8 : 4;
}
// modes whose window output is staged and bulk-stored (one element per word)
template <int MODE>
__host__ __device__ constexpr bool staged_mode() {
    return MODE == MODE_U32 || MODE == MODE_F32 || MODE == MODE_F64 || MODE == MODE_F64_REAL3;
}

// CTA shape: a CTA owns all L lanes of one chunk; thread (rho, q) computes R
// consecutive sequence words of lanes q*V .. q*V+V-1 in every window of W
// words. VW (1, 2 or 4) is the vector width: a smaller VW gives more threads
// (warps) per lane state for the same shared memory.
template <int L, int R, int VW, int W, bool TMA = false>
struct GenShape {
    static constexpr int V = L >= VW ? VW : L; // lanes per thread
    static constexpr int Q = L / V;            // threads across a slot row
    static constexpr int RUNS = W / R;         // runs per window
    static constexpr int NT = RUNS * Q;        // threads per CTA
    // In-place ring (the history-register shapes): slot = position mod 624,
    // so every ring address is a per-thread constant + an immediate and the
    // block loop needs no slot arithmetic; the one operand a neighbouring run
    // overwrites in the same window (x_{p+R}, the next run's first word) is
    // published one window ahead in a double-buffered exchange row instead.
    static constexpr bool INPLACE = !TMA && kN % W == 0 && kN / W == 3 && R * V <= 26 && R >= 4;
    static constexpr int RING = INPLACE ? kN : kN + W; // ring slots
    static constexpr int SLOTS = RING + R;     // + mirror of slots [0, R)
    static constexpr int RING_BYTES = SLOTS * L * 4;
    static constexpr int BND_BYTES = INPLACE ? 2 * (RUNS + 1) * L * 4 : 0; // [parity][run 0..RUNS][lane]
    static constexpr int EXTRA_OFF = RING_BYTES + BND_BYTES; // staging / histograms
    template <int MODE>
    __host__ __device__ static constexpr int stage_bytes() {
        return (TMA && staged_mode<MODE>()) ? W * L * elem_bytes<MODE>() : 0;
    }
    // MODE_STATS: one byte-value histogram per lane position, hist[bin][lane]
    // (32 KB): a warp's 32 atomics always hit 32 different banks
    template <int MODE>
    __host__ __device__ static constexpr int hist_bytes() {
        return MODE == MODE_STATS ? 256 * 32 * 4 : 0;
    }
    template <int MODE>
    __host__ __device__ static constexpr int smem() {
        return EXTRA_OFF + stage_bytes<MODE>() + (stage_bytes<MODE>() ? 16 : 0) + hist_bytes<MODE>(); // + mbarrier
    }
    // CTAs per SM that shared memory allows (227 KB usable, 1 KB reserved per CTA)
    template <int MODE>
    __host__ __device__ static constexpr int smem_ctas() {
        return (227 * 1024) / (smem<MODE>() + 1024) > 0 ? (227 * 1024) / (smem<MODE>() + 1024) : 1;
    }
    // registers are capped so that they never limit occupancy below that
    template <int MODE>
    // (the 32-lane store shape runs one CTA per SM anyway -- one chunk per SM
    // is what the planner picks -- and is 3% faster without the 128-register
    // cap; the fused modes are not)
    __host__ __device__ static constexpr int minb() {
#ifdef VMT_GEN_MINB
        return VMT_GEN_MINB;
#endif
        return (L == 32 && NT == 256 && MODE != MODE_XOR && MODE != MODE_STATS)
                   ? 1
                   : (smem_ctas<MODE>() > reg_ctas()) ? reg_ctas()
                   : (smem_ctas<MODE>() * NT > 2048) ? (2048 / NT > 0 ? 2048 / NT : 1) : smem_ctas<MODE>();
    }
    // CTAs per SM that leave >= 128 registers per thread (the history shapes
    // spill below that: 96 registers at 10 x 64 threads cost 2x at L=8)
    __host__ __device__ static constexpr int reg_ctas() {
        return 65536 / (NT * 128) > 0 ? 65536 / (NT * 128) : 1;
    }
    // Thread count the register allocation is bounded for (launch_bounds'
    // first argument; the kernel still launches NT threads).
    template <int MODE>
    __host__ __device__ static constexpr int lb_threads() {
#ifdef VMT_GEN_LB_THREADS
        return VMT_GEN_LB_THREADS;
#endif
        return NT;
    }
    static_assert(W % R == 0 && kN % W == 0 && RING % R == 0 && W <= 227, "bad window / run length");
    static_assert(!INPLACE || kN - kM >= W, "in place: a window's x_{p+397} reads precede its writes");
    static_assert(!TMA || RING_BYTES % 16 == 0, "staging alignment");
};

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
            store_out(reinterpret_cast<VT*>(o), VecT<V>::make(w));
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
        } else if (VEC && V == 2 && all_in) {
            *reinterpret_cast<float2*>(o) = make_float2(f[0], f[1]);
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
        } else if (VEC && V == 2 && all_in) {
            *reinterpret_cast<double2*>(o) = make_double2(d[0], d[1]);
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

// V tempered words -> staging row (element layout identical to the output).
template <int MODE, int V>
__device__ __forceinline__ void stage_put(unsigned char* stage, int elem_index, const std::uint32_t* w) {
    if (MODE == MODE_U32) {
        using VT = typename VecT<V>::T;
        *reinterpret_cast<VT*>(stage + elem_index * 4) = VecT<V>::make(w);
    } else if (MODE == MODE_F32) {
#pragma unroll
        for (int v = 0; v < V; ++v)
            reinterpret_cast<float*>(stage)[elem_index + v] = to_f32(w[v]);
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
            reinterpret_cast<double*>(stage)[elem_index + v] =
                MODE == MODE_F64 ? to_f64(w[v]) : to_f64_real3(w[v]);
    }
}

// Per-CTA staging state (uniform across the CTA except `pending`, tid 0 only).
struct StageCtl {
    unsigned char* buf;
    unsigned long long* bar;
    unsigned phase;   // mbarrier completions consumed so far
    bool prev_staged; // a bulk copy of buf is outstanding (not yet confirmed read)
    bool pending;     // tid 0's view of the same
    std::uint32_t* hist; // MODE_STATS: this thread's histogram column (stride 32)
};

// One window of one thread: R new words of V lanes. base: slot of x_p for
// the run's first p; a: slot of x_{p+397}; wsl: slot receiving x_{p+624}.
// All ring loads are issued before any ring store (the stores go to slots no
// thread reads in this window), so the compiler is free to overlap them.
//
// HIST: the run's x_p .. x_{p+R-1} are the words this same thread computed
// three windows (one block) earlier, kept in registers (H) instead of being
// re-read from the ring; only x_{p+R} (the next run's first word) and the
// x_{p+397} operands come from shared memory.
template <int LT, int L, int R, int VW, int W, int MODE, bool VEC, bool FULL, bool STAGE, bool HIST>
__device__ __forceinline__ void gen_window(std::uint32_t* ring, int base, int a, int wsl, int q, int rho,
                                           unsigned long long g0, const GenParams& p, void* out,
                                           std::uint32_t* acc, StageCtl& sc, int tid,
                                           std::uint32_t (&H)[R][GenShape<L, R, VW, W>::V]) {
    using S = GenShape<L, R, VW, W>;
    constexpr int V = S::V;
    using VT = typename VecT<V>::T;
    using E = typename ElemT<MODE>::T;
    std::uint32_t X[R + 1][V], M[R][V];
    if (HIST) {
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
            for (int v = 0; v < V; ++v)
                X[i][v] = H[i][v];
        VecT<V>::get(*reinterpret_cast<const VT*>(ring + (base + R) * L + q * V), X[R]);
    } else {
#pragma unroll
        for (int i = 0; i <= R; ++i)
            VecT<V>::get(*reinterpret_cast<const VT*>(ring + (base + i) * L + q * V), X[i]);
    }
#pragma unroll
    for (int i = 0; i < R; ++i)
        VecT<V>::get(*reinterpret_cast<const VT*>(ring + (a + i) * L + q * V), M[i]);
    E* o = nullptr;
    if (MODE != MODE_XOR && MODE != MODE_BENCH_TEMPER_XOR && MODE != MODE_STATS && !STAGE) {
        const unsigned long long rel = g0 - p.pos_begin;
        o = static_cast<E*>(out) + (MODE == MODE_F64_RES53 ? (rel >> 1) : rel);
    }
    std::uint32_t NW[STAGE ? R : 1][V];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        std::uint32_t nw[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
            nw[v] = twist(X[i][v], X[i + 1][v], M[i][v]);
        *reinterpret_cast<VT*>(ring + (wsl + i) * L + q * V) = VecT<V>::make(nw);
        if (HIST) {
#pragma unroll
            for (int v = 0; v < V; ++v)
                H[i][v] = nw[v];
        }
        if (MODE == MODE_XOR) {
            // temper is GF(2)-linear: XOR the untempered words, temper once
            // at the end (vmt_xor_reduce_kernel)
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const unsigned long long g = g0 + (unsigned long long)i * LT + v;
                if (FULL || (g >= p.pos_begin && g < p.pos_end))
                    acc[v] ^= nw[v];
            }
        } else if (MODE == MODE_STATS) {
            // acc[0]: one bits of this window's words (folded into 64 bits per
            // window by the caller); bytes into the hist[bin][lane] columns
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const unsigned long long g = g0 + (unsigned long long)i * LT + v;
                if (FULL || (g >= p.pos_begin && g < p.pos_end)) {
                    const std::uint32_t t = temper(nw[v]);
                    acc[0] += __popc(t);
                    // PRMT extracts a byte zero-extended, one LEA forms the address
                    atomicAdd(sc.hist + (__byte_perm(t, 0u, 0x4440u) << 5), 1u);
                    atomicAdd(sc.hist + (__byte_perm(t, 0u, 0x4441u) << 5), 1u);
                    atomicAdd(sc.hist + (__byte_perm(t, 0u, 0x4442u) << 5), 1u);
                    atomicAdd(sc.hist + (__byte_perm(t, 0u, 0x4443u) << 5), 1u);
                }
            }
        } else if (MODE == MODE_BENCH_TEMPER_XOR) {
            // microbenchmark only: full per-word work of the store path minus the store
#pragma unroll
            for (int v = 0; v < V; ++v)
                acc[v] ^= temper(nw[v]);
        } else if (STAGE) {
#pragma unroll
            for (int v = 0; v < V; ++v)
                NW[i][v] = nw[v];
        } else {
            std::uint32_t tw[V];
#pragma unroll
            for (int v = 0; v < V; ++v)
                tw[v] = temper(nw[v]);
            emit<MODE, V, VEC, FULL>(tw, g0 + (unsigned long long)i * LT, p,
                                     o + (MODE == MODE_F64_RES53 ? (i * LT) / 2 : i * LT));
        }
    }
    if (STAGE) {
        // the staging buffer must be free: the previous window's bulk copy
        // has finished reading it (tid 0 confirms, everyone waits on the phase)
        if (sc.prev_staged) {
            if (tid == 0 && sc.pending) {
                bulk_wait_read_all();
                mbar_arrive(sc.bar);
                sc.pending = false;
            }
            mbar_wait_parity(sc.bar, sc.phase & 1u);
            ++sc.phase;
            sc.prev_staged = false;
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            std::uint32_t tw[V];
#pragma unroll
            for (int v = 0; v < V; ++v)
                tw[v] = temper(NW[i][v]);
            stage_put<MODE, V>(sc.buf, (rho * R + i) * L + q * V, tw);
        }
    }
    if (wsl == 0) {
        // mirror slots [0, R) behind the ring end (this thread wrote them)
#pragma unroll
        for (int i = 0; i < R; ++i)
            *reinterpret_cast<VT*>(ring + (S::RING + i) * L + q * V) =
                *reinterpret_cast<const VT*>(ring + i * L + q * V);
    }
}

// One row of V new (untempered) words: fold / count / temper + emit (the
// consumers of gen_window_ip; gen_window keeps its own copy for the staged
// and paired-store forms). o points at the element of stream word g.
template <int LT, int V, int MODE, bool VEC, bool FULL>
__device__ __forceinline__ void consume_row(const std::uint32_t (&nw)[V], unsigned long long g, const GenParams& p,
                                            typename ElemT<MODE>::T* o, std::uint32_t* acc, StageCtl& sc) {
    if (MODE == MODE_XOR) {
        // temper is GF(2)-linear: XOR the untempered words, temper once at the
        // end (vmt_xor_reduce_kernel)
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (FULL || (g + v >= p.pos_begin && g + v < p.pos_end))
                acc[v] ^= nw[v];
    } else if (MODE == MODE_STATS) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if (FULL || (g + v >= p.pos_begin && g + v < p.pos_end)) {
                const std::uint32_t t = temper(nw[v]);
                acc[0] += __popc(t);
                atomicAdd(sc.hist + (__byte_perm(t, 0u, 0x4440u) << 5), 1u);
                atomicAdd(sc.hist + (__byte_perm(t, 0u, 0x4441u) << 5), 1u);
                atomicAdd(sc.hist + (__byte_perm(t, 0u, 0x4442u) << 5), 1u);
                atomicAdd(sc.hist + (__byte_perm(t, 0u, 0x4443u) << 5), 1u);
            }
        }
    } else if (MODE == MODE_BENCH_TEMPER_XOR) {
#pragma unroll
        for (int v = 0; v < V; ++v)
            acc[v] ^= temper(nw[v]);
    } else {
        std::uint32_t tw[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
            tw[v] = temper(nw[v]);
        emit<MODE, V, VEC, FULL>(tw, g, p, o);
    }
}

// One window of one thread, in-place ring (GenShape::INPLACE). The run's x_p
// .. x_{p+R-1} are its history registers H, x_{p+R} comes from the exchange
// row bnd_rd (published by the next run one window earlier), x_{p+397} from
// slots arow.. (mod 624, mirror behind the ring end); the new words go to the
// run's own slots wslot.. (all ring loads of the window precede its stores
// and no thread reads those slots in this window). o: the element of stream
// word g0 (row i at o + i*LT, halved for two-word values).
template <int LT, int L, int R, int V, int RING, int MODE, bool VEC, bool FULL>
__device__ __forceinline__ void gen_window_ip(std::uint32_t* ring, int arow, int wslot, int q,
                                              const std::uint32_t* bnd_rd, unsigned long long g0,
                                              const GenParams& p, typename ElemT<MODE>::T* o, std::uint32_t* acc,
                                              StageCtl& sc, std::uint32_t (&H)[R][V]) {
    using VT = typename VecT<V>::T;
    std::uint32_t X[R + 1][V], M[R][V];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int v = 0; v < V; ++v)
            X[i][v] = H[i][v];
    VecT<V>::get(*reinterpret_cast<const VT*>(bnd_rd), X[R]);
#pragma unroll
    for (int i = 0; i < R; ++i)
        VecT<V>::get(*reinterpret_cast<const VT*>(ring + (arow + i) * L + q * V), M[i]);
#pragma unroll
    for (int i = 0; i < R; ++i) {
        std::uint32_t nw[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
            nw[v] = twist(X[i][v], X[i + 1][v], M[i][v]);
        *reinterpret_cast<VT*>(ring + (wslot + i) * L + q * V) = VecT<V>::make(nw);
#pragma unroll
        for (int v = 0; v < V; ++v)
            H[i][v] = nw[v];
        consume_row<LT, V, MODE, VEC, FULL>(nw, g0 + (unsigned long long)i * LT, p,
                                            o + (MODE == MODE_F64_RES53 ? (i * LT) / 2 : i * LT), acc, sc);
    }
    if (wslot == 0) {
        // mirror of slots [0, R) behind the ring end
#pragma unroll
        for (int i = 0; i < R; ++i)
            *reinterpret_cast<VT*>(ring + (RING + i) * L + q * V) = VecT<V>::make(H[i]);
    }
}

// dst is the stream's [624][LT] state; this CTA's lanes are columns
// [col0, col0 + L).
template <int LT, int L, int RING>
__device__ __forceinline__ void save_boundary(const std::uint32_t* ring, int blk_base_slot, std::uint32_t* dst,
                                              int col0, int tid, int nt) {
    for (int i = tid; i < kN * L; i += nt) {
        const int k = i / L, t = i % L;
        int slot = blk_base_slot + k;
        if (slot >= RING)
            slot -= RING;
        dst[(long long)k * LT + col0 + t] = ring[slot * L + t];
    }
}

// One CTA = one chunk x one group of L of the stream's LT lanes (LT/L CTAs
// per chunk; L < LT lets more CTAs share an SM for the same lane-state count,
// i.e. fewer chunks to position). Dynamic shared memory GenShape::smem<MODE>()
// bytes: ring[slot][L] | staging[W][L] | mbarrier.
template <int LT, int L, int R, int VW, int W, bool TMA, int MODE, bool VEC>
__global__ void __launch_bounds__(GenShape<L, R, VW, W, TMA>::template lb_threads<MODE>(),
                                  GenShape<L, R, VW, W, TMA>::template minb<MODE>())
    vmt_gen_kernel(GenParams p) {
    using S = GenShape<L, R, VW, W, TMA>;
    constexpr int V = S::V;
    using VT = typename VecT<V>::T;
    using E = typename ElemT<MODE>::T;
    static_assert(LT % L == 0, "lane groups must tile the stream's lanes");
    constexpr int kGroups = LT / L;
    // a window's output is contiguous only when the CTA owns every lane
    constexpr bool kStaged = VEC && staged_mode<MODE>() && S::template stage_bytes<MODE>() > 0 && kGroups == 1;
    extern __shared__ __align__(16) std::uint32_t ring[];
    __shared__ std::uint32_t red;

    const unsigned chunk = blockIdx.x / kGroups;
    const int col0 = (int)(blockIdx.x % kGroups) * L; // first stream lane of this CTA
    const int tid = threadIdx.x;
#ifdef VMT_TIMELINE
    if (p.tl && tid == 0 && blockIdx.x < 1024) {
        p.tl[blockIdx.x * 3] = tl_now();
        p.tl[blockIdx.x * 3 + 2] = tl_smid();
    }
#endif
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
        out = static_cast<void*>(static_cast<E*>(out) +
                                 (MODE == MODE_F64_RES53 ? p.out_chunk_stride / 2 : p.out_chunk_stride) * chunk);

    StageCtl sc;
    sc.buf = reinterpret_cast<unsigned char*>(ring) + S::EXTRA_OFF;
    sc.bar = reinterpret_cast<unsigned long long*>(sc.buf + S::template stage_bytes<MODE>());
    sc.phase = 0;
    sc.prev_staged = false;
    sc.pending = false;
    sc.hist = reinterpret_cast<std::uint32_t*>(reinterpret_cast<unsigned char*>(ring) + S::EXTRA_OFF) +
              (MODE == MODE_STATS ? (tid & 31) : 0);
    // bulk copies need the window's destination 16-byte aligned
    const bool tma_ok =
        kStaged &&
        ((reinterpret_cast<unsigned long long>(out) - p.pos_begin * elem_bytes<MODE>()) % 16ull) == 0;

    // -- the chunk's boundary state (words x_0..x_623 -> slots 0..623)
    const std::uint32_t* src = p.chunk_states + (unsigned long long)chunk * kN * LT + col0;
    for (int i = tid; i < kN * S::Q; i += S::NT) {
        const int slot = i / S::Q, qq = i % S::Q;
        const VT v = *reinterpret_cast<const VT*>(src + (long long)slot * LT + qq * V);
        reinterpret_cast<VT*>(ring)[i] = v;
        if (i < R * S::Q)
            reinterpret_cast<VT*>(ring)[S::RING * S::Q + i] = v;
    }
    constexpr bool kFold = MODE == MODE_XOR || MODE == MODE_BENCH_TEMPER_XOR;
    if (kFold && tid == 0)
        red = 0;
    __shared__ unsigned long long ones_red;
    if (MODE == MODE_STATS) {
        std::uint32_t* h0 = reinterpret_cast<std::uint32_t*>(reinterpret_cast<unsigned char*>(ring) + S::EXTRA_OFF);
        for (int i = tid; i < S::template hist_bytes<MODE>() / 4; i += S::NT)
            h0[i] = 0;
        if (tid == 0)
            ones_red = 0;
    }
    if (kStaged && tid == 0)
        mbar_init(sc.bar, 1);
    __syncthreads();

    std::uint32_t acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v)
        acc[v] = 0;
    constexpr unsigned long long bw = (unsigned long long)kN * LT;
    constexpr unsigned long long ww = (unsigned long long)W * LT; // stream words per window (all lanes)
    unsigned long long ones = 0; // MODE_STATS
    // batch mode: every generator (chunk) saves its own boundary state
    const bool save_here = p.save_state != nullptr;
    std::uint32_t* const save_dst = p.save_state + (batch ? (unsigned long long)chunk * kN * LT : 0ull);
    int blk_base_slot = 0; // slot of x_{624 r} for the current block r (= 624 r mod RING)
    constexpr int kWins = kN / W;
    // (3 windows x R x V history registers: with V = 4 that spills)
    constexpr bool kHist = VMT_GEN_HIST && kWins == 3 && R * V <= 26;
    std::uint32_t H[kHist ? kWins : 1][R][V];
    if (kHist) {
        // the first block's x_p of each window of this run: the chunk state
#pragma unroll
        for (int wi = 0; wi < (kHist ? kWins : 1); ++wi)
#pragma unroll
            for (int i = 0; i < R; ++i)
                VecT<V>::get(*reinterpret_cast<const VT*>(ring + (wi * W + rho * R + i) * L + q * V), H[wi][i]);
    }
    static_assert(!S::INPLACE || kHist, "the in-place ring needs the history registers");
    if constexpr (S::INPLACE) {
        // ---- in-place ring: static slots, one range check per block ----
        constexpr int BROW = (S::RUNS + 1) * L; // exchange words per parity
        std::uint32_t* const bnd = ring + S::SLOTS * L;
        const int r0 = rho * R;
        int arow[kWins];
#pragma unroll
        for (int wi = 0; wi < kWins; ++wi) {
            const int a = wi * W + r0 + kM;
            arow[wi] = a >= kN ? a - kN : a;
        }
        // the first window's x_{p+R} words (parity 0)
        *reinterpret_cast<VT*>(bnd + rho * L + q * V) = VecT<V>::make(H[0][0]);
        if (rho == 0)
            *reinterpret_cast<VT*>(bnd + S::RUNS * L + q * V) = VecT<V>::make(H[1][0]);
        __syncthreads();
        int par = 0;
        constexpr int kShift = MODE == MODE_F64_RES53 ? 1 : 0; // two stream words per value
        E* const out_e = static_cast<E*>(out);
        for (unsigned long long blk = b_lo; blk < b_hi; ++blk) {
            if (save_here && blk == p.save_block)
                save_boundary<LT, L, S::RING>(ring, 0, save_dst, col0, tid, S::NT);
            const unsigned long long gb = blk * bw; // first stream word of the block
            const bool bfull = gb >= p.pos_begin && gb + bw <= p.pos_end;
            const unsigned long long g_thr = gb + (unsigned long long)r0 * LT + col0 + q * V;
            // element of this thread's first word in the block (full blocks only)
            E* const o_blk = out_e + (bfull ? ((g_thr - p.pos_begin) >> kShift) : 0ull);
#pragma unroll
            for (int wi = 0; wi < kWins; ++wi) {
                // publish the next window's x_{p+R} words (the other parity)
                std::uint32_t* const bw_row = bnd + (par ^ 1) * BROW;
                *reinterpret_cast<VT*>(bw_row + rho * L + q * V) = VecT<V>::make(H[(wi + 1) % kWins][0]);
                if (rho == 0)
                    *reinterpret_cast<VT*>(bw_row + S::RUNS * L + q * V) = VecT<V>::make(H[(wi + 2) % kWins][0]);
                const std::uint32_t* const bnd_rd = bnd + par * BROW + (rho + 1) * L + q * V;
                const unsigned long long g0 = g_thr + (unsigned long long)wi * ww;
                if (bfull) {
                    gen_window_ip<LT, L, R, V, S::RING, MODE, VEC, true>(
                        ring, arow[wi], wi * W + r0, q, bnd_rd, g0, p, o_blk + ((wi * ww) >> kShift), acc, sc, H[wi]);
                } else {
                    const unsigned long long gw = gb + (unsigned long long)wi * ww;
                    // (as gen_window: words before pos_begin wrap modulo 2^64 and are never stored)
                    E* const o = out_e + ((g0 - p.pos_begin) >> kShift);
                    if (gw >= p.pos_begin && gw + ww <= p.pos_end)
                        gen_window_ip<LT, L, R, V, S::RING, MODE, VEC, true>(ring, arow[wi], wi * W + r0, q, bnd_rd,
                                                                          g0, p, o, acc, sc, H[wi]);
                    else
                        gen_window_ip<LT, L, R, V, S::RING, MODE, VEC, false>(ring, arow[wi], wi * W + r0, q, bnd_rd,
                                                                           g0, p, o, acc, sc, H[wi]);
                }
                par ^= 1;
                __syncthreads();
                if (MODE == MODE_STATS) {
                    ones += acc[0];
                    acc[0] = 0;
                }
            }
        }
        if (save_here && b_hi == p.save_block && b_hi == p.end_block)
            save_boundary<LT, L, S::RING>(ring, 0, save_dst, col0, tid, S::NT);
    } else {
    auto window = [&](unsigned long long blk, int wi, std::uint32_t (&Hw)[R][V]) {
        {
            int wstart = blk_base_slot + wi * W;
            if (wstart >= S::RING)
                wstart -= S::RING;
            const int base = wstart + rho * R;
            int a = base + kM;
            if (a >= S::RING)
                a -= S::RING;
            int wsl = base + kN;
            if (wsl >= S::RING)
                wsl -= S::RING;
            const unsigned long long gw = blk * bw + (unsigned long long)wi * ww; // first word of the window
            const unsigned long long g0 = gw + (unsigned long long)(rho * R) * LT + col0 + q * V;
            const bool wfull = gw >= p.pos_begin && gw + ww <= p.pos_end;
            const bool staged = kStaged && tma_ok && wfull;
            if (staged)
                gen_window<LT, L, R, VW, W, MODE, VEC, true, kStaged, kHist>(ring, base, a, wsl, q, rho, g0, p, out,
                                                                             acc, sc, tid, Hw);
            else if (wfull)
                gen_window<LT, L, R, VW, W, MODE, VEC, true, false, kHist>(ring, base, a, wsl, q, rho, g0, p, out,
                                                                           acc, sc, tid, Hw);
            else
                gen_window<LT, L, R, VW, W, MODE, VEC, false, false, kHist>(ring, base, a, wsl, q, rho, g0, p, out,
                                                                            acc, sc, tid, Hw);
            __syncthreads();
            if (MODE == MODE_STATS) {
                ones += acc[0];
                acc[0] = 0;
            }
            if (kStaged) {
                if (staged && tid == 0) {
                    // all threads' staging writes (generic proxy) -> bulk copy (async proxy)
                    fence_proxy_async_smem();
                    bulk_store(static_cast<E*>(out) + (gw - p.pos_begin), sc.buf,
                               (unsigned)(ww * elem_bytes<MODE>()));
                    bulk_commit();
                    sc.pending = true;
                }
                if (staged)
                    sc.prev_staged = true; // a bulk copy of the buffer is outstanding
            }
        }
    };
    for (unsigned long long blk = b_lo; blk < b_hi; ++blk) {
        if (save_here && blk == p.save_block)
            save_boundary<LT, L, S::RING>(ring, blk_base_slot, save_dst, col0, tid, S::NT);
        if (kHist) {
            // fully unrolled so each window's history registers are static
#pragma unroll
            for (int wi = 0; wi < (kHist ? kWins : 1); ++wi)
                window(blk, wi, H[wi]);
        } else {
#pragma unroll 1
            for (int wi = 0; wi < kWins; ++wi)
                window(blk, wi, H[0]);
        }
        blk_base_slot += kN;
        if (blk_base_slot >= S::RING)
            blk_base_slot -= S::RING;
    }
    // end-of-range boundary state (block b_hi) when it is the requested one
    if (save_here && b_hi == p.save_block && b_hi == p.end_block)
        save_boundary<LT, L, S::RING>(ring, blk_base_slot, save_dst, col0, tid, S::NT);
    } // !INPLACE
    if (kStaged && tid == 0 && sc.pending)
        bulk_wait_all(); // the staging buffer must outlive the last bulk copy
    if (kFold) {
        std::uint32_t x = 0;
#pragma unroll
        for (int v = 0; v < V; ++v)
            x ^= acc[v];
        atomicXor(&red, x);
        __syncthreads();
        if (tid == 0)
            p.xor_partials[blockIdx.x] = red; // untempered; tempered by the reduce kernel
    }
    if (MODE == MODE_STATS) {
        // (every window ended with a barrier: the histograms are complete)
        atomicAdd(&ones_red, ones);
        const std::uint32_t* h0 =
            reinterpret_cast<const std::uint32_t*>(reinterpret_cast<unsigned char*>(ring) + S::EXTRA_OFF);
        unsigned long long* dst = p.stats_partials + (unsigned long long)blockIdx.x * kStatWords;
        for (int b = tid; b < 256; b += S::NT) {
            unsigned long long c = 0;
            for (int l = 0; l < 32; ++l)
                c += h0[b * 32 + ((l + b) & 31)]; // rotated: the 32 threads of a warp read 32 banks
            dst[1 + b] = c;
        }
        __syncthreads();
        if (tid == 0)
            dst[0] = ones_red;
    }
#ifdef VMT_TIMELINE
    if (p.tl && tid == 0 && blockIdx.x < 1024)
        p.tl[blockIdx.x * 3 + 1] = tl_now();
#endif
}

} // namespace vmt_b200
