// Steady-state chunk positioning on the tensor cores (included by vmt_capi.cu).
//
// Consecutive fills of the same shape (same chunk count C and blocks per chunk
// B) advance every chunk start by the same block delta D: chunk c of the next
// fill is chunk c of this one jumped by 624*D words -- one and the same GF(2)
// matrix F^(624 D) for all C*L lane states. Instead of C*L polynomial jumps
// (~0.39 us of GPU each), the new states are one GEMM
//   new[C*L][19968] = old[C*L][19968] x F^(624 D)[19968][19968]  (mod 2)
// in word-bit coordinates (vmt_matrix.cuh) with FP4 e2m1 0/1 operands, unit
// block scales and fp32 accumulation (exact: sums <= 19937):
// our own tcgen05 kernels (vmt_posmma.cuh; no cuBLAS) -- serially between
// fills, or co-resident with the generation kernel as the prefetch of the
// next fill (VMT_PREFETCH_TENSOR). Where the kernel cannot be set up (no TMA
// descriptor encoder) the caller falls back to the polynomial jumps.
// The 200 MB FP4 matrix for a delta is built once (19937 basis jumps +
// expansion) when the delta repeats; four are cached, and deltas up to 4 blocks
// above a cached one reuse it (the rest regenerated in place).
#include <cudaTypedefs.h>

#ifndef VMT_GEMM_MIN_ROWS
#define VMT_GEMM_MIN_ROWS 256
#endif

namespace {

// below this many lane states the polynomial jumps win (env VMT_GEMM_MIN_ROWS
// overrides). 256 since round 2: our GEMM positions 592 lane states in ~0.1 ms
// against ~0.25 ms of jumps (config 1 0.22 -> 0.20 ms per fill, 2^24-word
// fills at L=16 0.20 -> 0.12 ms; profiles/r02_plan_sweep.log)
inline std::uint64_t gemm_min_rows() {
    static const std::uint64_t v =
        std::getenv("VMT_GEMM_MIN_ROWS") ? std::strtoull(std::getenv("VMT_GEMM_MIN_ROWS"), nullptr, 10)
                                         : (std::uint64_t)VMT_GEMM_MIN_ROWS;
    return v;
}
constexpr std::size_t kGemmMatBytes = (std::size_t)kWB * kWB;
// positioning matrices cached per generator (200 MB each): a generator that
// alternates between fill shapes (e.g. float and double fills of the same
// count, each with block deltas D and D+1) keeps all of them
constexpr std::size_t kGemmCachedMats = 4;

struct GemmPos {
    std::map<std::uint64_t, std::unique_ptr<DevBuf<std::int8_t>>> mats; // delta -> F^(624 delta), FP4 word-bit
    // TMA descriptors of the FP4 matrices (B operand of vmt_posmma_kernel)
    std::map<std::uint64_t, CUtensorMap> tmaps;
    std::map<std::uint64_t, CUtensorMap> tmaps2; // 104-row boxes for the CTA-pair kernel
    DevBuf<std::int8_t> pm_a; // FP4 state operand
    DevBuf<unsigned> pm_ctr;  // tile counter of the pair kernel's scheduler (vmt_posmma.cuh)
    // pm_a already holds the operand of these states (written at the end of the
    // prefetch that produced them): consumed or dropped by the next posmma_prepare
    const void* fp4_src = nullptr;
    std::uint64_t fp4_rows = 0;
    unsigned fp4_nl = 0;
    CUtensorMap pm_tmap_a;
    const void* pm_tmap_ptr = nullptr;
    std::uint64_t pm_tmap_rows = 0;
    std::map<std::uint64_t, std::uint64_t> last_use;                     // delta -> tick of its last use
    std::map<std::uint64_t, int> seen;                                   // delta -> transitions observed
    std::uint64_t tick = 0;
    bool last_valid = false;
    std::uint64_t last_b0 = 0, last_B = 0, last_C = 0;
};

// TMA descriptor of a K-major FP4 operand [rows][19968 elements = 9984 B]:
// boxes of 64 B (128 elements) x box_rows rows, 64-byte swizzle.
bool make_tmap_fp4(CUtensorMap& m, const void* base, std::uint64_t rows, unsigned box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    if (!enc)
        return false;
    const cuuint64_t dims[2] = {(cuuint64_t)(kWB / 2), (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(kWB / 2)};
    const cuuint32_t box[2] = {(cuuint32_t)(kPmKE / 2), box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    return enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, kPmKE == 256 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// dst = src jumped by 624*delta words with the co-resident tcgen05 kernel
// (vmt_posmma.cuh), launched on `st` (a side stream, after the generation
// kernel): the FP4 state operand, then the GEMM. false: no FP4 matrix cached
// for exactly this delta.
// the CTA-pair kernel (cta_group::2) unless VMT_POSMMA_SINGLE is set
bool posmma_pair() {
    static const bool pair = std::getenv("VMT_POSMMA_SINGLE") == nullptr;
    return pair;
}

// Operand-ring depths the CTA-pair kernel is instantiated for; a launch takes
// the deepest that fits the shared memory it may use (kP2MaxStages when it
// runs alone, fewer beside a generation CTA).
constexpr int kP2MaxStages = 10;
int p2_stages_for(int smem_bytes) {
    for (int s : {10, 8, 7, 6, 5, 4, 3, 2})
        if (p2_smem(s) <= smem_bytes)
            return s;
    return 0;
}

bool posmma_run(GemmPos& gp, const CUtensorMap& tmap_b, const std::uint32_t* src, std::uint32_t* dst, unsigned L,
                std::uint64_t rows, int sms, cudaStream_t st, unsigned nl, unsigned lane0,
                int stages = kP2MaxStages, bool prepared = false, bool dynamic_tiles = true);

// Whether posmma_launch has a matrix (and its TMA descriptor) for this delta
bool posmma_ready(GemmPos& gp, std::uint64_t delta) {
    const bool pair = posmma_pair();
    auto& maps = pair ? gp.tmaps2 : gp.tmaps;
    return maps.find(delta) != maps.end() && gp.mats.count(delta) != 0;
}

// prepared: posmma_prepare has already written the states' FP4 operand
bool posmma_launch(GemmPos& gp, std::uint64_t delta, const std::uint32_t* src, std::uint32_t* dst, unsigned L,
                   std::uint64_t rows, int sms, cudaStream_t st, int stages = kP2MaxStages, bool prepared = false,
                   bool dynamic_tiles = true) {
    const bool pair = posmma_pair();
    auto it = (pair ? gp.tmaps2 : gp.tmaps).find(delta);
    if (it == (pair ? gp.tmaps2 : gp.tmaps).end() || !gp.mats.count(delta))
        return false;
    gp.last_use[delta] = gp.tick;
    return posmma_run(gp, it->second, src, dst, L, rows, sms, st, L, 0, stages, prepared, dynamic_tiles);
}

#ifdef VMT_TIMELINE
// experiments: per-CTA {start ns, end ns, SM id} of the last generation launch
// ([0, 3072)) and the last positioning GEMM ([3072, 6144)); vmt_debug_timeline
unsigned long long* timeline_buf() {
    static unsigned long long* buf = nullptr;
    if (!buf) {
        VMT_CUDA(cudaMalloc(&buf, 6144 * sizeof(unsigned long long)));
        VMT_CUDA(cudaMemset(buf, 0, 6144 * sizeof(unsigned long long)));
    }
    return buf;
}
#endif

// (ring depths whose shared memory no CTA can have are never launched: p2_stages_for)
constexpr int kSmemPerCtaMax = 227 * 1024;
template <int S>
void p2_set_smem() {
    if (p2_smem(S) <= kSmemPerCtaMax)
        VMT_CUDA(cudaFuncSetAttribute(vmt_posmma2_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, p2_smem(S)));
}

template <int S>
void p2_launch(int grid, cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const PosMmaParams& pp) {
    vmt_posmma2_kernel<S><<<grid, kPmThreads, p2_smem(S), st>>>(a, b, pp);
}

// Lanes [lane0, lane0 + nl) of every state of dst (interleaved [.][624][L])
// = lanes [0, nl) of src times the FP4 matrix behind tmap_b (nl = L, lane0 =
// 0: every lane, chunk positioning).
// The A operand of posmma_run: lanes [0, nl) of the `rows` lane states of src as
// FP4 rows (zero-padded to whole tiles) in gp.pm_a, with its TMA descriptor.
// The co-resident prefetch calls it on the fill's own stream BEFORE the
// generation kernel: queued on the side stream, the conversion's many small
// CTAs raced the generation kernel for the SMs and, when they won, the
// generation CTAs were packed 3-4 per SM onto the first SMs that drained
// (config 1: 0.20 ms per fill at 60 chunks but 0.32 ms at 48 / 64 / 80,
// profiles/r02_summary.md).
bool posmma_prepare(GemmPos& gp, const std::uint32_t* src, unsigned L, std::uint64_t rows, cudaStream_t st,
                    unsigned nl) {
    const std::uint64_t tile_rows = posmma_pair() ? 2 * kPmM : kPmM;
    const std::uint64_t rows_pad = (rows + tile_rows - 1) / tile_rows * tile_rows;
    const bool ready = gp.fp4_src == src && gp.fp4_rows == rows && gp.fp4_nl == nl && gp.pm_a.p &&
                       gp.pm_tmap_ptr == gp.pm_a.p && gp.pm_tmap_rows == rows_pad;
    gp.fp4_src = nullptr; // one use: the buffer is rewritten by whatever is prepared next
    if (ready)
        return true;
    gp.pm_a.reserve(rows_pad * kWB / 2);
    if (gp.pm_tmap_ptr != gp.pm_a.p || gp.pm_tmap_rows != rows_pad) {
        if (!make_tmap_fp4(gp.pm_tmap_a, gp.pm_a.p, rows_pad, kPmM))
            return false;
        gp.pm_tmap_ptr = gp.pm_a.p;
        gp.pm_tmap_rows = rows_pad;
    }
    const long long nthreads = (long long)rows_pad * (kN / 8);
    vmt_states_to_fp4_kernel<<<(unsigned)((nthreads + 127) / 128), 128, 0, st>>>(
        src, (int)L, 0, (int)nl, (long long)rows, (long long)rows_pad, reinterpret_cast<std::uint8_t*>(gp.pm_a.p));
    VMT_CUDA(cudaGetLastError());
    return true;
}

bool posmma_run(GemmPos& gp, const CUtensorMap& tmap_b, const std::uint32_t* src, std::uint32_t* dst, unsigned L,
                std::uint64_t rows, int sms, cudaStream_t st, unsigned nl, unsigned lane0, int stages,
                bool prepared, bool dynamic_tiles) {
    const bool pair = posmma_pair();
    {
        // function attributes are per device (vmt_multi_gpu_fill drives several)
        static std::mutex mu;
        static std::set<int> done;
        int dev = 0;
        VMT_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(mu);
        if (!done.count(dev)) {
            VMT_CUDA(cudaFuncSetAttribute(vmt_posmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPmSmem));
            p2_set_smem<2>();
            p2_set_smem<3>();
            p2_set_smem<4>();
            p2_set_smem<5>();
            p2_set_smem<6>();
            p2_set_smem<7>();
            p2_set_smem<8>();
            p2_set_smem<10>();
            done.insert(dev);
        }
    }
    const std::uint64_t tile_rows = pair ? 2 * kPmM : kPmM;
    const std::uint64_t rows_pad = (rows + tile_rows - 1) / tile_rows * tile_rows;
    if (!prepared && !posmma_prepare(gp, src, L, rows, st, nl))
        return false;
    PosMmaParams pp;
#ifdef VMT_TIMELINE
    pp.tl = timeline_buf() + 3072;
#endif
    if (!gp.pm_ctr.p) { // the pair kernel's tile counter: zero here, re-zeroed by every launch
        gp.pm_ctr.reserve(1);
        VMT_CUDA(cudaMemsetAsync(gp.pm_ctr.p, 0, sizeof(unsigned), st));
    }
    static const int tile_mode = std::getenv("VMT_POSMMA_TILES") ? std::atoi(std::getenv("VMT_POSMMA_TILES")) : 0;
    // tiles from the counter unless the caller knows every pair is equally loaded
    pp.tile_ctr = (tile_mode == 1 || (tile_mode == 0 && dynamic_tiles)) ? gp.pm_ctr.p : nullptr;
    pp.dst = dst;
    pp.L = (int)L;
    pp.rows = (int)rows;
    pp.nl = (int)nl;
    pp.lane0 = (int)lane0;
    pp.m_tiles = (int)(rows_pad / tile_rows);
    const int tiles = pp.m_tiles * kPmNTiles;
    if (pair) {
        const int grid = 2 * std::min(tiles, sms / 2);
        // the deepest instantiated ring that is no deeper than asked for and fits a CTA
        int sg = std::min(stages, p2_stages_for(kSmemPerCtaMax));
        sg = sg >= 10 ? 10 : sg == 9 ? 8 : sg < 2 ? 2 : sg;
        switch (sg) {
        case 10: p2_launch<10>(grid, st, gp.pm_tmap_a, tmap_b, pp); break;
        case 8: p2_launch<8>(grid, st, gp.pm_tmap_a, tmap_b, pp); break;
        case 7: p2_launch<7>(grid, st, gp.pm_tmap_a, tmap_b, pp); break;
        case 6: p2_launch<6>(grid, st, gp.pm_tmap_a, tmap_b, pp); break;
        case 5: p2_launch<5>(grid, st, gp.pm_tmap_a, tmap_b, pp); break;
        case 4: p2_launch<4>(grid, st, gp.pm_tmap_a, tmap_b, pp); break;
        case 3: p2_launch<3>(grid, st, gp.pm_tmap_a, tmap_b, pp); break;
        default: p2_launch<2>(grid, st, gp.pm_tmap_a, tmap_b, pp); break;
        }
    } else
        vmt_posmma_kernel<<<std::min(tiles, sms), kPmThreads, kPmSmem, st>>>(gp.pm_tmap_a, tmap_b, pp);
    VMT_CUDA(cudaGetLastError());
    return true;
}

// p(F) in word-bit coordinates as the GEMM's B operand: FP4 [out][in], two
// elements per byte.
void build_gemm_matrix(const Poly& poly, DevBuf<std::int8_t>& m, cudaStream_t st) {
    DevBuf<std::uint64_t> rows;
    rows.reserve(kMatWords);
    Counters cnt;
    matrix_from_poly(poly, rows.p, st, cnt);
    m.reserve(kGemmMatBytes / 2);
    vmt_gemm_matrix_fp4_kernel<<<dim3((kWB / 2 + 255) / 256, kWB), 256, 0, st>>>(
        rows.p, reinterpret_cast<std::uint8_t*>(m.p));
    VMT_CUDA(cudaGetLastError());
    VMT_CUDA(cudaStreamSynchronize(st)); // rows is released on return
}

// The matrix for a delta, building it when there is room: at most
// kGemmCachedMats are cached, and one is only replaced after 32 positionings
// without a use -- so
// sizes that wander cannot turn every fill into a 10 ms matrix build.
// nullptr: no matrix (the caller uses the polynomial jumps).
const std::int8_t* gemm_matrix(vmt_generator* h, GemmPos& gp, std::uint64_t delta, cudaStream_t st) {
    auto it = gp.mats.find(delta);
    if (it != gp.mats.end()) {
        gp.last_use[delta] = gp.tick;
        return it->second->p;
    }
    if (gp.mats.size() >= kGemmCachedMats) {
        std::uint64_t victim = 0;
        bool found = false;
        for (auto& kv : gp.mats)
            if (gp.tick - gp.last_use[kv.first] > 32) {
                victim = kv.first;
                found = true;
                break;
            }
        if (!found)
            return nullptr;
        VMT_CUDA(cudaStreamSynchronize(st));
        gp.mats.erase(victim);
        gp.tmaps.erase(victim);
        gp.tmaps2.erase(victim);
        gp.last_use.erase(victim);
    }
    Gf2Field& F = Gf2Field::instance();
    const unsigned __int128 d = (unsigned __int128)kN * delta;
    std::unique_ptr<DevBuf<std::int8_t>> m(new DevBuf<std::int8_t>());
    build_gemm_matrix(F.x_pow128((std::uint64_t)d, (std::uint64_t)(d >> 64)), *m, st);
    h->cnt.other += 1;
    const std::int8_t* p = m->p;
    CUtensorMap tm;
    if (make_tmap_fp4(tm, p, kWB, kPmNH))
        gp.tmaps[delta] = tm;
    if (make_tmap_fp4(tm, p, kWB, kP2BQ))
        gp.tmaps2[delta] = tm;
    gp.mats[delta] = std::move(m);
    gp.last_use[delta] = gp.tick;
    return p;
}

// dst[C][624][L] = src[C][624][L] jumped by 624*delta words, by one GEMM.
// A cached matrix usable for `delta`: exact, or a base delta at most 4 blocks
// below (the rest is regenerated); 0 when there is none.
std::uint64_t usable_base(const GemmPos& gp, std::uint64_t delta) {
    std::uint64_t best = 0;
    for (auto& kv : gp.mats)
        if (kv.first <= delta && delta - kv.first <= 4 && kv.first > best)
            best = kv.first;
    return best;
}

bool gemm_position_exact(vmt_generator* h, GemmPos& gp, const std::uint32_t* src, std::uint32_t* dst,
                         std::uint64_t rows, std::uint64_t delta, cudaStream_t st);

// every state of the `chunks` chunks of states[chunks][624][L] advanced by k blocks in place
void launch_advance_blocks(std::uint32_t* states, unsigned L, std::uint64_t chunks, int k, cudaStream_t st) {
    {
        static std::mutex mu;
        static std::set<int> done;
        int dev = 0;
        VMT_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(mu);
        if (!done.count(dev)) {
            VMT_CUDA(cudaFuncSetAttribute(vmt_advance_blocks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          adv_smem(32)));
            done.insert(dev);
        }
    }
    int lgL = 0;
    while ((1u << lgL) < L)
        ++lgL;
    vmt_advance_blocks_kernel<<<(unsigned)chunks, kAdvThreads, adv_smem((int)L), st>>>(states, lgL, k);
    VMT_CUDA(cudaGetLastError());
}

// dst = src jumped by 624*delta words: one GEMM with the matrix of a cached
// base delta B in [delta-4, delta] (the largest, so exact when cached)
// followed by delta-B blocks of in-place regeneration (microseconds), or with
// a new matrix built for delta -- a fill size alternating between block
// deltas D and D+1 then needs one matrix when D repeats first.
// floor_delta: floor(words between the starts of consecutive fills / block), when
// the caller knows it (0: unknown) -- the block deltas of such a sequence are
// floor_delta and floor_delta + 1, so a matrix for floor_delta serves both and
// the fills whose delta is the floor need no advance at all.
bool gemm_position(vmt_generator* h, GemmPos& gp, const std::uint32_t* src, std::uint32_t* dst, std::uint64_t rows,
                   std::uint64_t delta, cudaStream_t st, std::uint64_t floor_delta = 0) {
    std::uint64_t base = usable_base(gp, delta);
    if (base == 0 && floor_delta != 0 && (floor_delta == delta || floor_delta + 1 == delta)) {
        base = floor_delta;
    } else if (base == 0) {
        // no matrix yet: build it for the smallest recently seen delta in
        // [delta-4, delta], and at most delta-1: fills of n words alternate
        // between block deltas floor(n/bw) and floor(n/bw)+1 in whichever
        // order the first repeats come, and both must reuse this matrix (a
        // second 200 MB build, ~8 ms, cost 2^26-word fills at L=32 4x their
        // steady-state time: profiles/r02_plan_sweep.log); the block of
        // in-place advance this adds to exact repeats costs microseconds
        base = delta > 1 ? delta - 1 : delta;
        for (std::uint64_t k = 4; k >= 2; --k)
            if (k < delta && gp.seen.count(delta - k)) {
                base = delta - k;
                break;
            }
    }
    if (!gemm_position_exact(h, gp, src, dst, rows, base, st))
        return false;
    if (delta > base) {
        launch_advance_blocks(dst, h->L, rows / h->L, (int)(delta - base), st);
        h->cnt.other += 1;
    }
    return true;
}

bool gemm_position_exact(vmt_generator* h, GemmPos& gp, const std::uint32_t* src, std::uint32_t* dst,
                         std::uint64_t rows, std::uint64_t delta, cudaStream_t st) {
    ++gp.tick;
    if (!gemm_matrix(h, gp, delta, st))
        return false;
    // our tcgen05 kernel at every row count: operand expansion + GEMM with a
    // packing epilogue (config 1's 1200 states: 0.375 ms per fill; the
    // bench's 4736: 0.81 ms)
    if (!posmma_launch(gp, delta, src, dst, h->L, rows, device_info(h->device).sms, st))
        return false;
    h->cnt.other += 2;
    h->cnt.gemm_positionings += 1;
    return true;
}

// ---- de-phasing many generators at once (config 3) -------------------------
// Lanes [s, s+n) of every generator = lanes [0, n) x F^(s 2^q): log2(L) FP4
// GEMMs (s = 1, 2, 4, ...) with a process-wide cache of the matrices per
// (device, q, s), instead of ngen*(L-1) polynomial jumps.
struct DephaseGemm {
    std::mutex mu;
    GemmPos gp; // operand buffer and its TMA descriptor
    std::map<std::pair<unsigned, unsigned>, std::unique_ptr<DevBuf<std::int8_t>>> mats;
    std::map<std::pair<unsigned, unsigned>, CUtensorMap> tmaps; // for vmt_posmma(2)_kernel
};

std::mutex g_dephase_mu;
std::map<int, std::unique_ptr<DephaseGemm>> g_dephase;

DephaseGemm& dephase_gemm(int dev) {
    std::lock_guard<std::mutex> lk(g_dephase_mu);
    auto& slot = g_dephase[dev];
    if (!slot)
        slot.reset(new DephaseGemm());
    return *slot;
}

// states: [ngen][624][L], lane 0 seeded; fills lanes 1..L-1. false: not done
// (no TMA descriptor encoder; the caller uses the polynomial jumps).
bool dephase_by_gemm(int device, cudaStream_t st, unsigned ngen, unsigned L, unsigned q, std::uint32_t* states,
                     Counters& cnt) {
    if (L < 2)
        return false;
    DephaseGemm& D = dephase_gemm(device);
    std::lock_guard<std::mutex> lk(D.mu);
    Gf2Field& F = Gf2Field::instance();
    for (unsigned s = 1; s < L; s *= 2) {
        const unsigned n = std::min(s, L - s);
        auto key = std::make_pair(q, s);
        auto it = D.mats.find(key);
        if (it == D.mats.end()) {
            if (D.mats.size() >= 8) {
                VMT_CUDA(cudaStreamSynchronize(st));
                D.mats.clear();
                D.tmaps.clear();
            }
            std::unique_ptr<DevBuf<std::int8_t>> m(new DevBuf<std::int8_t>());
            build_gemm_matrix(F.powmod(F.x_pow2(q), s), *m, st);
            cnt.other += 1;
            CUtensorMap tm;
            if (!make_tmap_fp4(tm, m->p, kWB, posmma_pair() ? kP2BQ : kPmNH)) {
                if (s == 1)
                    return false; // nothing written yet: the caller jumps instead
                throw VmtError(VMT_ECUDA, "TMA descriptor failed during de-phasing");
            }
            D.tmaps[key] = tm;
            it = D.mats.emplace(key, std::move(m)).first;
        }
        // lanes [s, s+n) of every generator written straight from the accumulators
        const std::uint64_t rows = (std::uint64_t)ngen * n;
        if (!posmma_run(D.gp, D.tmaps.at(key), states, states, L, rows, device_info(device).sms, st, n, s)) {
            if (s == 1)
                return false;
            throw VmtError(VMT_ECUDA, "positioning GEMM failed during de-phasing");
        }
        cnt.other += 2;
    }
    VMT_CUDA(cudaStreamSynchronize(st));
    return true;
}

} // namespace
