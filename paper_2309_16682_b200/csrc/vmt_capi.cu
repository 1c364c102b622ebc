// C ABI of the B200-native VMT19937 generator (include/vmt19937_b200.h).
//
// Host runtime: positions, chunk planning, jump-polynomial caches and
// staging; every word is produced by the sm_100a kernels in vmt_kernels.cuh.
// There is no CPU generation path: without a CUDA device every call that
// produces words fails with VMT_ECUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <cmath>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/vmt19937_b200.h"
#include "gf2poly.hpp"
#include "vmt_kernels.cuh"
#include "vmt_variants.hpp"

using namespace vmt_b200;

namespace {

thread_local std::string g_last_error;

struct VmtError : std::runtime_error {
    int code;
    VmtError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define VMT_CUDA(x)                                                                                   \
    do {                                                                                              \
        cudaError_t e_ = (x);                                                                         \
        if (e_ != cudaSuccess)                                                                        \
            throw VmtError(VMT_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));               \
    } while (0)

void require(bool c, int code, const char* msg) {
    if (!c)
        throw VmtError(code, msg);
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return VMT_OK;
    } catch (const VmtError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return VMT_ENOMEM;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return VMT_EINVAL;
    } catch (const std::logic_error& e) {
        g_last_error = e.what();
        return VMT_ESTATE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return VMT_EIO;
    }
}

// Host-destination fills are staged through device memory in segments of
// this many stream words (two segments in flight).
constexpr std::uint64_t kHostSegmentWords = 1ull << 28;
// Fills at least this large prefetch the positioning of the predicted next fill.
constexpr std::uint64_t kPrefetchMinWords = 1ull << 24;

bool valid_lanes(unsigned L) { return L == 1 || L == 2 || L == 4 || L == 8 || L == 16 || L == 32; }

unsigned log2u(unsigned L) {
    unsigned r = 0;
    while ((1u << r) < L)
        ++r;
    return r;
}

// ---------------------------------------------------------------- kernels --
// Kernel shape variants (vmt_variants.hpp; instantiated in variants_*.cu).
const Variant& pick_variant(unsigned L, int variant) {
    static const std::vector<Variant> table = [] {
        std::vector<Variant> t;
        for (auto part : {variants_l32a, variants_l32b, variants_l16a, variants_l16b, variants_l8, variants_small})
            for (const Variant& v : part())
                t.push_back(v);
        return t;
    }();
    for (const Variant& v : table)
        if (v.L == (int)L && (variant == 0 || v.id == variant))
            return v;
    if (!valid_lanes(L))
        throw VmtError(VMT_EINVAL, "lanes must be one of 1, 2, 4, 8, 16, 32");
    throw VmtError(VMT_EINVAL, "unknown kernel variant for this lane count");
}

struct DeviceInfo {
    int sms = 0;
    std::set<const void*> smem_set;
    std::map<const void*, int> occ;
};
std::mutex g_dev_mu;
std::map<int, DeviceInfo> g_dev;

DeviceInfo& device_info(int dev) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto& d = g_dev[dev];
    if (d.sms == 0) {
        VMT_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return d;
}

// Occupancy (CTAs per SM) of a generation kernel, opting into >48 KB smem.
int prepare_gen(int dev, GenFn fn, int nt, int smem) {
    DeviceInfo& d = device_info(dev);
    std::lock_guard<std::mutex> lk(g_dev_mu);
    const void* key = reinterpret_cast<const void*>(fn);
    if (!d.smem_set.count(key)) {
        VMT_CUDA(cudaFuncSetAttribute(key, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int occ = 0;
        VMT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, key, nt, smem));
        d.occ[key] = std::max(occ, 1);
        d.smem_set.insert(key);
    }
    return d.occ[key];
}

// Whether one vmt_posmma_kernel CTA fits on an SM beside per_sm CTAs of the
// generation kernel `fn` (shared memory incl. the 1 KB per-CTA reservation,
// registers, threads).
int p2_stages_for(int smem_bytes);

// Operand-ring depth of the CTA-pair positioning kernel that fits beside
// per_sm CTAs of the generation kernel `fn` on one SM (shared memory incl. the
// 1 KB per-CTA reservation, registers, threads); 0 when none does.
int posmma_fits(int dev, GenFn fn, int nt, int smem, int per_sm) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int>, int> memo;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(dev, reinterpret_cast<const void*>(fn), per_sm);
    auto it = memo.find(key);
    if (it != memo.end())
        return it->second;
    int sm_smem = 0, sm_regs = 0, sm_threads = 0;
    VMT_CUDA(cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    VMT_CUDA(cudaDeviceGetAttribute(&sm_regs, cudaDevAttrMaxRegistersPerMultiprocessor, dev));
    VMT_CUDA(cudaDeviceGetAttribute(&sm_threads, cudaDevAttrMaxThreadsPerMultiProcessor, dev));
    // the positioning kernel posmma_run launches: the CTA pair unless VMT_POSMMA_SINGLE
    const bool single = std::getenv("VMT_POSMMA_SINGLE") != nullptr;
    const void* pk = single ? reinterpret_cast<const void*>(vmt_posmma_kernel)
                            : reinterpret_cast<const void*>(vmt_posmma2_kernel<4>);
    cudaFuncAttributes ga{}, pa{};
    VMT_CUDA(cudaFuncGetAttributes(&ga, reinterpret_cast<const void*>(fn)));
    VMT_CUDA(cudaFuncGetAttributes(&pa, pk));
    auto regs = [](int per_thread, int threads) { // allocation unit: 256 registers per warp
        return ((per_thread * 32 + 255) / 256 * 256) * ((threads + 31) / 32);
    };
    const int free_smem = sm_smem - per_sm * (smem + 1024) - 1024;
    int stages = single ? (kPmSmem <= free_smem ? kPmStages : 0) : p2_stages_for(free_smem);
    if (const char* cap = std::getenv("VMT_PREF_STAGES")) // experiments: cap the co-resident ring depth
        stages = std::min(stages, std::max(2, std::atoi(cap)));
    const bool ok = stages > 0 && per_sm * regs(ga.numRegs, nt) + regs(pa.numRegs, kPmThreads) <= sm_regs &&
                    per_sm * nt + kPmThreads <= sm_threads && !std::getenv("VMT_NO_TC_PREFETCH");
    if (ok) {
        // both kernels ask for the full shared-memory carveout: an SM whose
        // generation CTA ran with the smallest carveout that fits it (132 KB)
        // would have no room left for the GEMM CTA
        VMT_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                      cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        for (const void* k : {pk, reinterpret_cast<const void*>(vmt_posmma2_kernel<2>),
                              reinterpret_cast<const void*>(vmt_posmma2_kernel<3>),
                              reinterpret_cast<const void*>(vmt_posmma2_kernel<5>),
                              reinterpret_cast<const void*>(vmt_posmma2_kernel<6>),
                              reinterpret_cast<const void*>(vmt_posmma2_kernel<7>),
                              reinterpret_cast<const void*>(vmt_posmma2_kernel<8>),
                              reinterpret_cast<const void*>(vmt_posmma2_kernel<10>)})
            VMT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    memo[key] = ok ? stages : 0;
    return memo[key];
}

// ------------------------------------------------------- device buffers --
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(cap, o.cap);
    }
    void reserve(size_t n) {
        if (n <= cap)
            return;
        if (p)
            cudaFree(p);
        p = nullptr;
        cap = 0;
        VMT_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
        cap = n;
    }
    ~DevBuf() {
        if (p)
            cudaFree(p);
    }
};

// ------------------------------------------------------------ polynomials --
// J^1..J^(n) for J = x^(624*blocks): the chunk-start jump polynomials.
struct PolySet {
    std::vector<Poly> host;
    DevBuf<std::uint64_t> dev;
    size_t dev_count = 0;
};

void powers_parallel(const Poly& J, size_t count, std::vector<Poly>& out, size_t have) {
    // out[c-1] = J^c for c = have+1 .. count
    Gf2Field& F = Gf2Field::instance();
    if (out.size() < count)
        out.resize(count);
    if (have >= count)
        return;
    const size_t todo = count - have;
    unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 16u));
    nt = (unsigned)std::min<size_t>(nt, (todo + 7) / 8);
    std::vector<std::thread> th;
    for (unsigned k = 0; k < nt; ++k) {
        const size_t lo = have + 1 + todo * k / nt, hi = have + todo * (k + 1) / nt; // inclusive range
        th.emplace_back([&, lo, hi] {
            if (lo > hi)
                return;
            Poly cur = (lo - 1 >= 1 && lo - 1 <= have) ? out[lo - 2] : F.powmod(J, lo - 1);
            if (lo - 1 == 0)
                cur = F.one();
            for (size_t c = lo; c <= hi; ++c) {
                cur = F.mulmod(cur, J);
                out[c - 1] = cur;
            }
        });
    }
    for (auto& t : th)
        t.join();
}

std::mutex g_poly_mu;

// 16-bit digit tables T_j[v] = x^(v * 2^(16 + 16 j)), j < 3, v < 65536, for
// bits 16..63 of a 64-bit jump distance (config 5; the low 16 bits are
// stepped directly): three jumps per state (four with 12-bit digits: 7.1 ms
// for config 5's 4096 states). 196608 polynomials (491 MB on the device),
// built once per process by host threads (~1 s).
constexpr int kDigitBits = 16, kDigitBase = 16, kDigits = 3, kDigitVals = 1 << kDigitBits;
struct DigitTables {
    std::vector<Poly> host; // index j*4096 + v (v=0 unused)
    std::map<int, std::unique_ptr<DevBuf<std::uint64_t>>> dev;
};
DigitTables& digit_tables() {
    static DigitTables t;
    std::lock_guard<std::mutex> lk(g_poly_mu);
    if (t.host.empty()) {
        Gf2Field& F = Gf2Field::instance();
        t.host.assign((size_t)kDigits * kDigitVals, Poly(kPolyWords, 0));
        const int kParts = std::max(1u, std::thread::hardware_concurrency()) >= 24 ? 16 : 8; // threads per digit
        std::vector<std::thread> th;
        for (int j = 0; j < kDigits; ++j)
            for (int part = 0; part < kParts; ++part)
                th.emplace_back([&, j, part] {
                    const Poly base = F.x_pow2((unsigned)(kDigitBase + kDigitBits * j));
                    const int v0 = part * (kDigitVals / kParts), v1 = v0 + kDigitVals / kParts;
                    Poly cur = v0 == 0 ? F.one() : F.powmod(base, (std::uint64_t)v0);
                    t.host[(size_t)j * kDigitVals + v0] = cur;
                    for (int v = v0 + 1; v < v1; ++v) {
                        cur = F.mulmod(cur, base);
                        t.host[(size_t)j * kDigitVals + v] = cur;
                    }
                });
        for (auto& x : th)
            x.join();
    }
    return t;
}

const std::uint64_t* digit_tables_device(int dev) {
    DigitTables& t = digit_tables();
    std::lock_guard<std::mutex> lk(g_poly_mu);
    auto& slot = t.dev[dev];
    if (!slot) {
        slot.reset(new DevBuf<std::uint64_t>());
        slot->reserve(t.host.size() * kPolyWords);
        std::vector<std::uint64_t> flat(t.host.size() * kPolyWords);
        for (size_t i = 0; i < t.host.size(); ++i)
            std::memcpy(flat.data() + i * kPolyWords, t.host[i].data(), kPolyWords * 8);
        VMT_CUDA(cudaMemcpy(slot->p, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice));
    }
    return slot->p;
}

// Dephasing polynomials x^(t*2^q) mod P, t = 1..L-1.
// (cached per (q, L): they do not depend on the seed, and the L - 2 products
// were ~3 ms of every 32-lane vmt_create)
std::vector<Poly> dephase_polys(unsigned q, unsigned L) {
    std::vector<Poly> out;
    if (L <= 1)
        return out;
    static std::mutex mu;
    static std::map<std::pair<unsigned, unsigned>, std::shared_ptr<const std::vector<Poly>>> cache;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find({q, L});
        if (it != cache.end())
            return *it->second;
    }
    Gf2Field& F = Gf2Field::instance();
    const Poly base = F.x_pow2(q);
    Poly cur = base;
    out.push_back(cur);
    for (unsigned t = 2; t < L; ++t) {
        cur = F.mulmod(cur, base);
        out.push_back(cur);
    }
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() >= 32)
        cache.clear();
    cache[{q, L}] = std::make_shared<const std::vector<Poly>>(out);
    return out;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a{};
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct Counters {
    std::uint64_t gen = 0, jump = 0, other = 0, lane_jumps = 0, gemm_positionings = 0, tc_prefetches = 0, pref_used = 0;
};

// One CTA per job; with few jobs several warps split each job's coefficient
// range (vmt_jump.cuh) to cut latency. One warp per job fills an SM with 32.
void launch_jump_kernel(const JumpParams& jp, cudaStream_t st) {
    int dev = 0;
    VMT_CUDA(cudaGetDevice(&dev));
    const int sms = device_info(dev).sms;
    const int slots = sms * VMT_JUMP_MINB; // resident one-warp jobs
    const int n = jp.njobs;
    // one wave instead of two: the 28-job-per-SM instantiation when it needs
    // fewer waves than the 24-job one (each job ~2% slower)
    auto waves = [&](int per_sm) { return (n + sms * per_sm - 1) / (sms * per_sm); };
    // measured on B200 (scratch/jump_bench.cu): split 8 wins below ~1/4 of the
    // warp slots, split 1 from 1/2 upwards
    if (n >= slots / 2 && waves(28) < waves(VMT_JUMP_MINB))
        vmt_jump_kernel<1, 28><<<n, 32, 0, st>>>(jp);
    else if (n >= slots / 2)
        vmt_jump_kernel<1><<<n, 32, 0, st>>>(jp);
    else if (n >= slots / 4)
        vmt_jump_kernel<4><<<n, 128, 0, st>>>(jp);
    else
        vmt_jump_kernel<8><<<n, 256, 0, st>>>(jp);
    VMT_CUDA(cudaGetLastError());
}

struct AffineJobs {
    int n = 0, div = 1;
    long long s_a = 0, s_b = 0, s_c = 0, d_a = 0, d_b = 0, d_c = 0;
    int p_a = 0, p_b = 0, p_c = 0;
};

// Launches the jump kernel with jobs given by an affine map of the job index
// (no host tables, fully asynchronous).
void launch_jumps_affine(cudaStream_t st, const std::uint32_t* src, int src_stride, std::uint32_t* dst,
                         int dst_stride, const std::uint64_t* d_polys, const AffineJobs& a, Counters& cnt,
                         const int* d_job_poly = nullptr) {
    if (a.n == 0)
        return;
    JumpParams jp{};
    jp.job_poly = d_job_poly; // per-job polynomial index (else affine p_a, p_b, p_c)
    jp.src = src;
    jp.dst = dst;
    jp.polys = d_polys;
    jp.src_stride = src_stride;
    jp.dst_stride = dst_stride;
    jp.njobs = a.n;
    jp.div = a.div;
    jp.s_a = a.s_a;
    jp.s_b = a.s_b;
    jp.s_c = a.s_c;
    jp.d_a = a.d_a;
    jp.d_b = a.d_b;
    jp.d_c = a.d_c;
    jp.p_a = a.p_a;
    jp.p_b = a.p_b;
    jp.p_c = a.p_c;
    launch_jump_kernel(jp, st);
    cnt.jump += 1;
    cnt.lane_jumps += a.n;
}

} // namespace

namespace {
struct GemmPos; // capi_gemmpos.inl

// Prefetch mode of new generators (vmt_set_prefetch); env VMT_PREFETCH overrides.
int default_prefetch() {
    static const int v = [] {
        const char* e = std::getenv("VMT_PREFETCH");
        const int m = e ? std::atoi(e) : VMT_PREFETCH_TENSOR;
        return (m >= VMT_PREFETCH_OFF && m <= VMT_PREFETCH_TENSOR) ? m : VMT_PREFETCH_TENSOR;
    }();
    return v;
}
}

// ------------------------------------------------------------------ handle --
struct vmt_generator {
    int device = 0;
    unsigned L = 1;
    unsigned q = 0;
    std::uint64_t bw = 624;
    cudaStream_t own = nullptr;
    cudaEvent_t last = nullptr;
    cudaStream_t last_stream = nullptr;

    DevBuf<std::uint32_t> base;   // [624][L] boundary states at block 0
    DevBuf<std::uint32_t> cur;    // [624][L] at cur_block
    DevBuf<std::uint32_t> next;   // save target
    std::uint64_t cur_block = 0;
    std::uint64_t pos = 0;  // words consumed by the caller
    std::uint64_t gpos = 0; // words produced by the GPU (>= pos)

    DevBuf<std::uint32_t> chunks;    // [C][624][L]
    DevBuf<std::uint32_t> chunks_alt; // prefetched chunk states of the predicted next fill
    int prefetch = default_prefetch(); // position the predicted next fill while this one generates
    bool pref_valid = false;
    bool pref_inflight = false;      // ev_pref recorded and not yet waited for by a fill
    std::uint64_t pref_b0 = 0, pref_B = 0, pref_C = 0;
    std::uint64_t last_end = ~0ull;  // end position of the previous GPU fill
    std::uint64_t last_fill_n = 0;   // size of the previous GPU fill
    cudaStream_t side = nullptr;     // prefetch stream
    cudaEvent_t ev_chunks = nullptr, ev_pref = nullptr;
    DevBuf<std::uint32_t> partials;  // per-CTA xor partials
    DevBuf<unsigned long long> stat_partials; // per-CTA MODE_STATS partials [grid][257]
    DevBuf<unsigned long long> stat_out;      // reduced MODE_STATS counts [257]
    DevBuf<std::uint32_t> scratch;   // device staging for host destinations
    DevBuf<std::uint64_t> tmp_poly;
    std::uint32_t* hstage = nullptr; // pinned staging for single / block16 queries
    std::uint64_t hstage_cap = 0, hstage_start = 0;
    std::uint32_t* hsmall = nullptr; // pinned 4-byte readback

    std::map<std::uint64_t, std::unique_ptr<PolySet>> polycache; // blocks-per-chunk -> J^c
    std::map<std::uint64_t, std::unique_ptr<DevBuf<std::uint64_t>>> skipcache; // block delta -> x^(624 delta)
    cudaStream_t copy_stream = nullptr;                                  // D2H of host fills
    cudaEvent_t seg_gen[2] = {nullptr, nullptr}, seg_copy[2] = {nullptr, nullptr};
    unsigned max_chunks = 0;
    int variant = 0;
    int positioning = 0; // 0 auto, 1 polynomial jumps only, 2 GEMM whenever the fill shape repeats
    GemmPos* gemm = nullptr;
    Counters cnt;
    bool profile = false;
    // profiling: one event triplet per fill (before jumps, before gen, after
    // gen), folded into running totals when the pool is full or on request
    std::vector<std::array<cudaEvent_t, 3>> evpool;
    std::size_t ev_used = 0;
    std::uint64_t prof_fills = 0;
    double prof_jump_ms = 0, prof_gen_ms = 0;
    float last_jump_ms = -1.f, last_gen_ms = -1.f;

    cudaStream_t pick(void* s) {
        cudaStream_t st = s ? static_cast<cudaStream_t>(s) : own;
        if (last_stream && st != last_stream)
            VMT_CUDA(cudaStreamWaitEvent(st, last, 0));
        return st;
    }
    void mark(cudaStream_t st) {
        VMT_CUDA(cudaEventRecord(last, st));
        last_stream = st;
    }
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        VMT_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0)
            cudaSetDevice(prev);
    }
};

void check_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw VmtError(VMT_ECUDA, "no CUDA device available (the generator has no CPU path)");
    }
    require(device >= 0 && device < n, VMT_EINVAL, "device ordinal out of range");
}

const std::uint64_t* upload_polys(vmt_generator* h, const std::vector<Poly>& polys, cudaStream_t st) {
    h->tmp_poly.reserve(std::max<size_t>(polys.size(), 1) * kPolyWords);
    std::vector<std::uint64_t> flat(polys.size() * kPolyWords);
    for (size_t i = 0; i < polys.size(); ++i)
        std::memcpy(flat.data() + i * kPolyWords, polys[i].data(), kPolyWords * 8);
    VMT_CUDA(cudaMemcpyAsync(h->tmp_poly.p, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, st));
    VMT_CUDA(cudaStreamSynchronize(st));
    return h->tmp_poly.p;
}

// Chunk-start polynomials J^1..J^(C-1) for B blocks per chunk (cached).
// The chunk polynomials J^c, J = x^(624 B) mod P, depend on the chunk size only:
// a process-wide cache behind the per-generator one, so the first fill of a new
// generator does not repeat the C - 1 host multiplications of an earlier one
// with the same chunk size (296 chunks: ~4 ms of host time, measured with a
// 2^20-word first fill at L = 1; 0.3 ms from the cache).
std::mutex g_chunkpoly_mu;
std::map<std::uint64_t, std::shared_ptr<const std::vector<Poly>>> g_chunkpoly;

const std::uint64_t* chunk_polys(vmt_generator* h, std::uint64_t B, size_t C, cudaStream_t st) {
    auto& slot = h->polycache[B];
    if (!slot)
        slot.reset(new PolySet());
    PolySet& ps = *slot;
    const size_t need = C > 0 ? C - 1 : 0;
    if (ps.host.size() < need) {
        {
            std::lock_guard<std::mutex> lk(g_chunkpoly_mu);
            auto it = g_chunkpoly.find(B);
            if (it != g_chunkpoly.end() && it->second->size() > ps.host.size())
                ps.host = *it->second;
        }
        if (ps.host.size() < need) {
            Gf2Field& F = Gf2Field::instance();
            const Poly J = F.x_pow(624ull * B);
            const size_t have = ps.host.size();
            powers_parallel(J, need, ps.host, have);
            auto pub = std::make_shared<const std::vector<Poly>>(ps.host);
            std::lock_guard<std::mutex> lk(g_chunkpoly_mu);
            if (g_chunkpoly.size() >= 64) // ~0.75 MB per 296-chunk entry
                g_chunkpoly.clear();
            auto& g = g_chunkpoly[B];
            if (!g || g->size() < pub->size())
                g = pub;
        }
    }
    if (ps.dev_count < need) {
        ps.dev.reserve(need * kPolyWords);
        std::vector<std::uint64_t> flat(need * kPolyWords);
        for (size_t i = 0; i < need; ++i)
            std::memcpy(flat.data() + i * kPolyWords, ps.host[i].data(), kPolyWords * 8);
        VMT_CUDA(cudaMemcpyAsync(ps.dev.p, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, st));
        VMT_CUDA(cudaStreamSynchronize(st));
        ps.dev_count = need;
    }
    return ps.dev.p;
}

// x^(624*delta) mod P on the device, cached per block distance (repeated
// strides are common: consecutive fills, ranks skipping the other ranks'
// shares, seeking back to a range).
const std::uint64_t* skip_poly(vmt_generator* h, std::uint64_t delta) {
    auto it = h->skipcache.find(delta);
    if (it == h->skipcache.end()) {
        if (h->skipcache.size() >= 16)
            h->skipcache.clear(); // cudaFree synchronises: no in-flight user
        Gf2Field& F = Gf2Field::instance();
        // 624*delta may exceed 64 bits for huge skips
        const unsigned __int128 d = (unsigned __int128)624u * delta;
        const Poly poly = F.x_pow128((std::uint64_t)d, (std::uint64_t)(d >> 64));
        auto& slot = h->skipcache[delta];
        slot.reset(new DevBuf<std::uint64_t>());
        slot->reserve(kPolyWords);
        VMT_CUDA(cudaMemcpy(slot->p, poly.data(), kPolyWords * 8, cudaMemcpyHostToDevice));
        it = h->skipcache.find(delta);
    }
    return it->second->p;
}

// Moves h->cur (block cur_block) to block `target` by one jump (forward from
// cur, or from the block-0 states when going backwards).
void reposition(vmt_generator* h, std::uint64_t target, cudaStream_t st) {
    if (target == h->cur_block)
        return;
    const std::uint32_t* from = h->cur.p;
    std::uint64_t delta = 0;
    if (target > h->cur_block) {
        delta = target - h->cur_block;
    } else {
        from = h->base.p;
        delta = target;
    }
    const std::uint64_t* dp = skip_poly(h, delta);
    AffineJobs a;
    a.n = (int)h->L;
    a.div = (int)h->L;
    a.s_b = 1;
    a.d_b = 1;
    launch_jumps_affine(st, from, (int)h->L, h->next.p, (int)h->L, dp, a, h->cnt);
    h->cur.swap(h->next);
    h->cur_block = target;
}

void matrix_from_poly(const Poly& p, std::uint64_t* rows_dev, cudaStream_t st, Counters& cnt); // capi_matrix.inl
constexpr std::size_t kMatWords = (std::size_t)kDim * kRowWords;

} // namespace
#include "capi_gemmpos.inl"
namespace {

// Profiling event pool (vmt_set_profiling).
constexpr std::size_t kProfPool = 1024;

void prof_fold(vmt_generator* h) {
    for (std::size_t i = 0; i < h->ev_used; ++i) {
        auto& e = h->evpool[i];
        VMT_CUDA(cudaEventSynchronize(e[2]));
        float a = 0, b = 0;
        VMT_CUDA(cudaEventElapsedTime(&a, e[0], e[1]));
        VMT_CUDA(cudaEventElapsedTime(&b, e[1], e[2]));
        h->prof_jump_ms += a;
        h->prof_gen_ms += b;
        h->last_jump_ms = a;
        h->last_gen_ms = b;
        ++h->prof_fills;
    }
    h->ev_used = 0;
}

cudaEvent_t* prof_next(vmt_generator* h) {
    if (h->ev_used == kProfPool)
        prof_fold(h);
    if (h->ev_used == h->evpool.size()) {
        std::array<cudaEvent_t, 3> e{};
        for (auto& x : e)
            VMT_CUDA(cudaEventCreate(&x));
        h->evpool.push_back(e);
    }
    return h->evpool[h->ev_used++].data();
}

// Chunk count for a fill of n words: every chunk but the first costs L lane
// jumps (positioning), every chunk adds generation parallelism. Minimise a
// cost model t(C) with constants measured on B200 (DESIGN.md section 5,
// profiles/r02_chunk_curve*.log):
//  * generation: (n / C) / min(L r_lane, peak_sm / k), k = ceil(C / sms) chunks
//    sharing the busiest SM; one lane of the R=13, VW=2 shape generates
//    ~5.5e8 words/s (8.8e8 with one lane per thread), an SM's store path
//    saturates at ~1.6e12 / 148 words/s. Past one chunk per SM only whole
//    waves (multiples of sms) are candidates.
//  * positioning by polynomial jumps (a fill shape seen for the first time):
//    0.43 us of whole-GPU throughput per lane jump, latency floor 0.16-0.5 ms.
//  * positioning by the FP4 GEMM (the previous fill had the same size):
//    ~0.03 ms + 40 us per 256-state x 416-column tile and SM pair, in whole
//    rounds of sms/2 tiles when it runs alone (1024 rows 0.15 ms, 4736 rows
//    0.55 ms).
//  * `overlap`: that GEMM will run beside the generation kernel as the
//    tensor-core prefetch of the next fill. One chunk per SM: the two share
//    the SMs' shared-memory bandwidth, measured t = max(t_gen + 0.5 t_pos,
//    t_pos + 0.4 t_gen) with the tiles handed out dynamically (no whole
//    rounds; 15% slower beside the 86 KB L=32 CTA, whose neighbour gets a
//    shallower operand ring). More chunks per SM: t_gen + t_pos.
// Fused XOR fills (no stores) run at ~5.5e8 words/s per lane and saturate at
// ~3.4e12 words/s per GPU.
#ifndef VMT_PLAN_RLANE
#define VMT_PLAN_RLANE 5.5e8
#endif
std::uint64_t plan_chunks(unsigned L, std::uint64_t n, std::uint64_t c_max, int sms, int mode = MODE_U32,
                          bool gemm = false, double lane_speed = 1.0, bool overlap = false) {
    const double per_jump = 0.43e-6 * 148.0 / (double)sms;
    auto t_jump = [&](double jobs) -> double {
        if (jobs <= 0)
            return 0.0;
        const double floor_s = jobs <= sms * 4.0 ? 0.16e-3 : (jobs <= sms * 16.0 ? 0.37e-3 : 0.0);
        return std::max(floor_s, jobs * per_jump);
    };
    const bool fused = mode == MODE_XOR;
    // store modes saturate at ~1.6e12 4-byte elements/s per GPU; doubles (one
    // per word) at ~5.1e11/s (measured at L=8: 4.1 TB/s)
    const bool dbl = mode == MODE_F64 || mode == MODE_F64_REAL3;
    // lane_speed: threads per lane of the kernel shape relative to the R=13,
    // VW=2 shape (VW=1 has twice as many and runs a lane 1.6x as fast)
    // (the one-lane kernel runs 208 threads on its lane: 1.8e9 words/s)
    const double r_lane = fused ? 5.5e8 * lane_speed
                          : lane_speed > 8.0 ? 1.8e9
                                             : VMT_PLAN_RLANE * (1.0 + 0.6 * (std::min(lane_speed, 2.0) - 1.0)),
                 // (1- and 2-lane kernels saturate an SM at ~3e9 words/s: measured 2.3-2.9e9 with 2-4 CTAs per SM)
                 peak_sm = fused ? 3.4e12 / 148.0 : dbl ? 5.1e11 / 148.0 : L <= 2 ? 3.0e9 : 1.6e12 / 148.0;
    const double pairs = std::max(1, sms / 2);
    auto gemm_tiles = [&](std::uint64_t C) { return std::ceil(double(C) * L / 256.0) * 48.0; };
    auto t_pos = [&](std::uint64_t C) -> double { // serial positioning
        const double rows = double(C) * L;
        if (gemm && rows >= (double)gemm_min_rows())
            return std::min(t_jump(double(C - 1) * L), 0.03e-3 + std::ceil(gemm_tiles(C) / pairs) * 40e-6);
        return t_jump(double(C - 1) * L);
    };
    auto t = [&](std::uint64_t C) {
        const double k = (double)((C + sms - 1) / sms);
        const double t_gen = (double(n) / double(C)) / std::min(L * r_lane, peak_sm / k);
        if (overlap && gemm && double(C) * L >= (double)gemm_min_rows()) {
            if (k > 1) // (beside several generation CTAs per SM the GEMM hides nothing: measured at L = 2, 8, 16)
                return t_gen + t_pos(C);
            const double tp = (0.03e-3 + gemm_tiles(C) / pairs * 40e-6) * (L == 32 ? 1.15 : 1.0);
            return std::max(t_gen + 0.5 * tp, tp + 0.4 * t_gen);
        }
        return t_pos(C) + t_gen;
    };
    std::uint64_t best = 1;
    double tb = t(1);
    auto consider = [&](std::uint64_t C) {
        const double tc = t(C);
        if (tc < tb * 0.97) { // a candidate must win clearly: fewer chunks is less positioning risk
            tb = tc;
            best = C;
        }
    };
    const std::uint64_t one_wave = std::min<std::uint64_t>(c_max, (std::uint64_t)sms);
    for (std::uint64_t C = 2; C < one_wave; C = (C * 5 + 3) / 4) // ~25% steps
        consider(C);
    consider(one_wave);
    for (std::uint64_t C = 2 * (std::uint64_t)sms; C <= c_max; C += (std::uint64_t)sms)
        consider(C);
    return best;
}

// Core: GPU-produces stream words [h->gpos, h->gpos + n) into `out` in the
// representation of `mode` (out == nullptr only for MODE_XOR). Advances gpos.
void gpu_generate(vmt_generator* h, int mode, void* out, std::uint64_t n, cudaStream_t st, void* reduce_out_dev) {
    if (n == 0)
        return;
    const std::uint64_t P0 = h->gpos, P1 = h->gpos + n;
    const std::uint64_t b0 = P0 / h->bw, b1 = (P1 + h->bw - 1) / h->bw;
    cudaEvent_t* pe = h->profile ? prof_next(h) : nullptr;
    if (pe)
        VMT_CUDA(cudaEventRecord(pe[0], st));
    // fused XOR at 32 lanes: chunks split over four 8-lane CTAs of 64 threads
    // (variant 7) generate 11% faster than one 256-thread CTA per chunk
    // (measured: 6.41 vs 7.10 ms per 2^34 words incl. positioning; nothing is
    // stored, so the 32-byte row segments of a lane group cost nothing), with
    // one wave of chunks (4 CTAs per SM)
    const bool xor_groups = h->variant == 0 && mode == MODE_XOR && h->L == 32;
    // 8-lane store fills: one lane per thread (variant 4, 128 threads per
    // chunk) instead of two (64 threads: 2 warps per chunk leave the SM
    // latency-bound): 2^28 words per fill u32 0.48 -> 0.33 ms, f32 0.51-0.81
    // -> 0.35, f64 0.62 -> 0.47 (profiles/r02_c2_variants.log). Two-word
    // doubles (RES53) need two lanes per thread.
    const bool l8_vw1 = h->variant == 0 && h->L == 8 &&
                        (mode == MODE_U32 || mode == MODE_F32 || mode == MODE_F64 || mode == MODE_F64_REAL3);
    const Variant& v = pick_variant(h->L, xor_groups ? 7 : l8_vw1 ? 4 : h->variant);
    const double lane_speed = double(v.NT) / double(v.G) / 8.0;
    const int groups = v.L / v.G; // CTAs per chunk (lane groups)
    const std::uint64_t nb = b1 - b0;
    // VEC when the destination is aligned for the vector width: the element
    // of stream word g lives at out + (g - P0).
    const int esz = (mode == MODE_U32 || mode == MODE_F32 || mode == MODE_XOR) ? 4 : 8;
    bool vec = false;
    if (mode != MODE_XOR && mode != MODE_STATS && mode != MODE_F64_RES53) {
        const int V = v.G >= v.VW ? v.VW : v.G;
        const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(out);
        const std::uint64_t e = (std::uint64_t)(a / (std::uintptr_t)esz);
        const int need = (esz == 8) ? 2 : V; // double2 / VecT<V> stores
        vec = (a % (std::uintptr_t)esz == 0) && ((e - P0) % (std::uint64_t)need == 0) && (P0 % V == 0) &&
              (esz == 4 || V >= 2);
    }
    GenFn fn = v.fn[mode][vec ? 1 : 0];
    const int smem = v.smem[mode];
    const int occ = prepare_gen(h->device, fn, v.NT, smem);
    const int sms = device_info(h->device).sms;
    const std::uint64_t max_grid = (std::uint64_t)sms * occ;
    const std::uint64_t c_max = std::min<std::uint64_t>(
        std::max<std::uint64_t>(1, xor_groups ? std::min<std::uint64_t>(max_grid / groups, (std::uint64_t)sms)
                                              : max_grid / groups),
        nb);
    // a fill of the same size as the previous one is planned with the GEMM
    // positioning cost (its block delta's matrix is built once the delta
    // repeats): fused XOR once that matrix exists (7.4 -> 7.1 ms per 2^34
    // words at L=32), the other modes from the first repeat on (config 1,
    // 2^26 words at L=16: 38 jump-positioned chunks 0.57 ms per fill -> 64
    // GEMM-positioned chunks 0.35 ms)
    const bool repeat = h->positioning != 1 && h->last_fill_n == n;
    const bool gemm_plan = repeat && (mode != MODE_XOR || (h->gemm && h->gemm->last_valid && b0 > h->gemm->last_b0 &&
                                                           usable_base(*h->gemm, b0 - h->gemm->last_b0) != 0));
    // the GEMM of the next fill will run beside this fill's generation kernel
    const bool overlap_plan = gemm_plan && h->prefetch == VMT_PREFETCH_TENSOR && mode != MODE_XOR &&
                              n >= kPrefetchMinWords;
    std::uint64_t C = h->max_chunks ? std::min<std::uint64_t>(c_max, h->max_chunks)
                                    : plan_chunks(h->L, n, c_max, sms, mode, gemm_plan, lane_speed, overlap_plan);
    static const bool debug = std::getenv("VMT_DEBUG") != nullptr;
    if (debug)
        std::fprintf(stderr, "[vmt] L=%u R=%d NT=%d smem=%d occ=%d chunks=%llu blocks=%llu mode=%d vec=%d\n", h->L,
                     v.R, v.NT, smem, occ, (unsigned long long)C, (unsigned long long)nb, mode, (int)vec);
    const std::uint64_t B = (nb + C - 1) / C;
    C = (nb + B - 1) / B;

    // -- chunk start states: prefetched during the previous fill, by one GEMM
    // from the previous fill's chunks (same shape, repeating block delta), or
    // by polynomial jumps from cur
    const bool use_pref = h->pref_valid && h->pref_b0 == b0 && h->pref_B == B && h->pref_C == C;
    h->pref_valid = false;
    if (h->pref_inflight) {
        // the side stream still reads h->chunks / writes h->chunks_alt
        VMT_CUDA(cudaStreamWaitEvent(st, h->ev_pref, 0));
        h->pref_inflight = false;
    }
    bool positioned = false;
    if (use_pref) {
        // chunk 0 is the prefetched state at b0, so cur needs no re-positioning
        // (the generation kernel saves the next one)
        h->chunks.swap(h->chunks_alt);
        positioned = true;
        h->cnt.pref_used += 1;
    }
    if (!positioned && h->positioning != 1 && C * h->L >= gemm_min_rows()) {
        if (!h->gemm)
            h->gemm = new GemmPos();
        GemmPos& gp = *h->gemm;
        if (gp.last_valid && gp.last_B == B && gp.last_C == C && b0 > gp.last_b0) {
            const std::uint64_t delta = b0 - gp.last_b0;
            if (gp.seen.size() > 64)
                gp.seen.clear();
            ++gp.seen[delta];
            // build the 200 MB matrix only for a delta that repeats; deltas up
            // to 4 blocks apart count as one (a fill size that is not a
            // multiple of the block alternates between D and D+1, and one
            // matrix for D serves both, capi_gemmpos.inl)
            int seen = 0;
            for (std::uint64_t k = 0; k <= 4 && k < delta; ++k) {
                auto it = gp.seen.find(delta - k);
                if (it != gp.seen.end())
                    seen += it->second;
            }
            if (usable_base(gp, delta) || seen >= 2 || h->positioning == 2) {
                h->chunks_alt.reserve((size_t)C * kN * h->L);
                try {
                    // words between this fill's start and the previous one's (same size: repeat)
                    std::uint64_t floor_delta = 0;
                    if (repeat && h->last_end != ~0ull && h->last_end >= n && P0 + n > h->last_end)
                        floor_delta = (P0 - (h->last_end - n)) / h->bw;
                    if (gemm_position(h, gp, h->chunks.p, h->chunks_alt.p, C * h->L, delta, st, floor_delta)) {
                        h->chunks.swap(h->chunks_alt);
                        positioned = true;
                    }
                } catch (const VmtError&) {
                    // e.g. no memory for the matrix / operands: use the jumps
                    // from now on (the chunk states are rebuilt below)
                    cudaGetLastError();
                    VMT_CUDA(cudaStreamSynchronize(st));
                    gp.mats.clear();
                    gp.tmaps.clear();
                    gp.tmaps2.clear();
                    h->positioning = 1;
                }
            }
        }
    }
    if (!positioned) {
        if (h->gemm)
            h->gemm->fp4_src = nullptr; // the chunk buffers are rewritten by the jumps
        reposition(h, b0, st);
        h->chunks.reserve((size_t)C * kN * h->L);
        VMT_CUDA(cudaMemcpyAsync(h->chunks.p, h->cur.p, (size_t)kN * h->L * 4, cudaMemcpyDeviceToDevice, st));
        if (C > 1) {
            const std::uint64_t* dp = chunk_polys(h, B, C, st);
            AffineJobs a;
            a.n = (int)((C - 1) * h->L);
            a.div = (int)h->L;
            a.s_b = 1;
            a.d_a = (long long)kN * h->L;
            a.d_b = 1;
            a.d_c = (long long)kN * h->L;
            a.p_a = 1;
            launch_jumps_affine(st, h->cur.p, (int)h->L, h->chunks.p, (int)h->L, dp, a, h->cnt);
        }
    }
    if (h->gemm) { // h->chunks now holds this fill's chunk starts
        h->gemm->last_valid = true;
        h->gemm->last_b0 = b0;
        h->gemm->last_B = B;
        h->gemm->last_C = C;
    }
    // -- predict the next fill (same size, same gap) and position its chunks
    // on the side stream while this fill's generation kernel runs: chunk c of
    // the next fill is chunk c of this one advanced by the same block delta
    bool prefetch_now = false, pref_prepared = false, pref_ready = false;
    std::uint64_t next_b0 = 0, pref_base = 0;
    const std::uint64_t grid = C * groups;
    // the tensor-core form runs beside the generation kernel: only when that
    // kernel's CTAs spread evenly over the SMs (one wave) and leave room for
    // one positioning CTA on each. Not for the fused XOR: that kernel is
    // issue-bound rather than store-bound and loses more to the co-resident
    // GEMM than the serial GEMM costs (measured 6.53 vs 6.37 ms per 2^34
    // words).
    const int per_sm = (int)((grid + sms - 1) / (std::uint64_t)sms);
    int pref_stages = 0;
    const bool tc_pref = h->prefetch == VMT_PREFETCH_TENSOR && h->positioning != 1 && h->gemm &&
                         mode != MODE_XOR && C * h->L >= gemm_min_rows() &&
                         (grid <= (std::uint64_t)sms || grid % sms == 0) && per_sm <= occ &&
                         (pref_stages = posmma_fits(h->device, fn, v.NT, smem, per_sm)) > 0;
    if ((h->prefetch == VMT_PREFETCH_JUMPS || tc_pref) && C > 1 && n >= kPrefetchMinWords) {
        const std::uint64_t gap = (h->last_end != ~0ull && P0 >= h->last_end) ? P0 - h->last_end : 0;
        const std::uint64_t P0n = P1 + gap;
        next_b0 = P0n / h->bw;
        const std::uint64_t nbn = (P0n + n + h->bw - 1) / h->bw - next_b0;
        const std::uint64_t c_max_n = std::min<std::uint64_t>(
            std::max<std::uint64_t>(1, xor_groups ? std::min<std::uint64_t>(max_grid / groups, (std::uint64_t)sms)
                                                  : max_grid / groups),
            nbn);
        std::uint64_t Cn = h->max_chunks ? std::min<std::uint64_t>(c_max_n, h->max_chunks)
                                         : plan_chunks(h->L, n, c_max_n, sms, mode, gemm_plan, lane_speed, overlap_plan);
        const std::uint64_t Bn = (nbn + Cn - 1) / Cn;
        Cn = (nbn + Bn - 1) / Bn;
        prefetch_now = Cn == C && Bn == B && next_b0 >= b0;
    }
    if (prefetch_now) {
        if (!h->side) {
            VMT_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
            VMT_CUDA(cudaEventCreateWithFlags(&h->ev_chunks, cudaEventDisableTiming));
            VMT_CUDA(cudaEventCreateWithFlags(&h->ev_pref, cudaEventDisableTiming));
        }
        // the tensor-core prefetch's FP4 state operand is written on this
        // stream, ahead of the generation kernel (posmma_prepare)
        if (tc_pref) {
            try {
                pref_base = usable_base(*h->gemm, next_b0 - b0);
                pref_ready = pref_base && posmma_ready(*h->gemm, pref_base);
                // (a generation kernel with one CTA per SM by occupancy cannot be
                // packed; its operand is written on the side stream, in parallel)
                static const int prep_mode = std::getenv("VMT_PREP_AHEAD") ? std::atoi(std::getenv("VMT_PREP_AHEAD")) : 0;
                if (pref_ready && (prep_mode == 1 || (prep_mode == 0 && occ > 1)))
                    pref_prepared = posmma_prepare(*h->gemm, h->chunks.p, h->L, C * h->L, st, h->L);
            } catch (const VmtError&) { // e.g. no memory for the operand: generate without prefetching
                cudaGetLastError();
                h->prefetch = VMT_PREFETCH_OFF;
                prefetch_now = false;
            }
        }
        if (prefetch_now)
            VMT_CUDA(cudaEventRecord(h->ev_chunks, st));
    }
    if (pe)
        VMT_CUDA(cudaEventRecord(pe[1], st));
    if (mode == MODE_XOR)
        h->partials.reserve(grid);
    if (mode == MODE_STATS)
        h->stat_partials.reserve(grid * kStatWords);
    GenParams p{};
    p.chunk_states = h->chunks.p;
    p.out = out;
    p.xor_partials = h->partials.p;
    p.stats_partials = h->stat_partials.p;
    p.save_state = h->next.p;
    p.first_block = b0;
    p.end_block = b1;
    p.pos_begin = P0;
    p.pos_end = P1;
    p.save_block = P1 / h->bw;
    p.out_chunk_stride = 0;
    p.blocks_per_chunk = (unsigned)B;
    p.lanes = h->L;
#ifdef VMT_TIMELINE
    p.tl = timeline_buf();
#endif
    // Everything of the prefetch that can free device memory (growing the
    // alternate chunk buffer, evicting a cached skip polynomial: cudaFree
    // waits for the whole device) happens before the generation kernel is
    // queued, so it never serialises the prefetch behind the generation.
    const std::uint64_t* pref_dp = nullptr;
    if (prefetch_now) {
        try {
            h->chunks_alt.reserve((size_t)C * kN * h->L);
            if (!tc_pref)
                pref_dp = skip_poly(h, next_b0 - b0);
        } catch (const VmtError&) { // e.g. no memory: generate without prefetching
            cudaGetLastError();
            h->prefetch = VMT_PREFETCH_OFF;
            prefetch_now = false;
        }
    }
    fn<<<(unsigned)grid, v.NT, smem, st>>>(p);
    VMT_CUDA(cudaGetLastError());
    h->cnt.gen += 1;
    if (prefetch_now && tc_pref) {
        // one tcgen05 FP4 GEMM with the cached matrix of the next block delta,
        // launched after the generation kernel so its CTAs take the resources
        // the generation CTAs leave free on every SM
        try {
            VMT_CUDA(cudaStreamWaitEvent(h->side, h->ev_chunks, 0));
            // a cached matrix for the delta or for a base at most 4 blocks below
            // it (the rest regenerated in place, as in gemm_position)
            const std::uint64_t delta = next_b0 - b0, base = pref_base;
            // tiles handed out dynamically when the generation CTAs leave some SMs free
            if (pref_ready && posmma_launch(*h->gemm, base, h->chunks.p, h->chunks_alt.p, h->L, C * h->L, sms,
                                            h->side, pref_stages, pref_prepared, grid < (std::uint64_t)sms)) {
                if (delta > base) {
                    launch_advance_blocks(h->chunks_alt.p, h->L, C, (int)(delta - base), h->side);
                    h->cnt.other += 1;
                }
                // the operand of the NEXT fill's GEMM (these states) right behind them on
                // the side stream instead of ahead of the next generation kernel on the
                // fill's stream: hidden whenever the prefetch ends before the generation
                if (pref_prepared && !std::getenv("VMT_NO_EAGER_FP4")) {
                    GemmPos& gp = *h->gemm;
                    if (posmma_prepare(gp, h->chunks_alt.p, h->L, C * h->L, h->side, h->L)) {
                        gp.fp4_src = h->chunks_alt.p;
                        gp.fp4_rows = C * h->L;
                        gp.fp4_nl = h->L;
                    }
                }
                VMT_CUDA(cudaEventRecord(h->ev_pref, h->side));
                h->pref_valid = true;
                h->pref_inflight = true;
                h->pref_b0 = next_b0;
                h->pref_B = B;
                h->pref_C = C;
                h->cnt.tc_prefetches += 1;
                h->cnt.other += 2; // FP4 state operand + vmt_posmma_kernel
            }
        } catch (const VmtError&) {
            // e.g. no memory for the operand: this fill is unaffected (its
            // generation kernel is already queued); stop prefetching
            cudaGetLastError();
            cudaStreamSynchronize(h->side);
            h->prefetch = VMT_PREFETCH_OFF;
            h->pref_valid = h->pref_inflight = false;
        }
        prefetch_now = false;
    }
    if (prefetch_now) {
        // launched after the generation kernel so its CTAs take the resources
        // the generation wave leaves free on every SM
        const std::uint64_t* dp = pref_dp;
        VMT_CUDA(cudaStreamWaitEvent(h->side, h->ev_chunks, 0));
        AffineJobs a;
        a.n = (int)(C * h->L);
        a.div = (int)h->L;
        a.s_a = (long long)kN * h->L;
        a.s_b = 1;
        a.d_a = (long long)kN * h->L;
        a.d_b = 1;
        launch_jumps_affine(h->side, h->chunks.p, (int)h->L, h->chunks_alt.p, (int)h->L, dp, a, h->cnt);
        VMT_CUDA(cudaEventRecord(h->ev_pref, h->side));
        h->pref_valid = true;
        h->pref_inflight = true;
        h->pref_b0 = next_b0;
        h->pref_B = B;
        h->pref_C = C;
    }
    h->last_end = P1;
    h->last_fill_n = n;
    if (pe)
        VMT_CUDA(cudaEventRecord(pe[2], st));
    if (mode == MODE_XOR) {
        vmt_xor_reduce_kernel<<<1, 256, 0, st>>>(h->partials.p, (int)grid, static_cast<std::uint32_t*>(reduce_out_dev));
        VMT_CUDA(cudaGetLastError());
        h->cnt.other += 1;
    }
    if (mode == MODE_STATS) {
        vmt_stats_reduce_kernel<<<1, 288, 0, st>>>(h->stat_partials.p, (int)grid,
                                                   static_cast<unsigned long long*>(reduce_out_dev));
        VMT_CUDA(cudaGetLastError());
        h->cnt.other += 1;
    }
    h->cur.swap(h->next);
    h->cur_block = P1 / h->bw;
    h->gpos = P1;
}

// Serves words [pos, pos+take) from the host staging buffer into dst.
std::uint64_t drain_stage(vmt_generator* h, void* dst, int mode, std::uint64_t n, bool dst_dev, cudaStream_t st) {
    if (h->pos >= h->gpos || mode != MODE_U32)
        return 0;
    const std::uint64_t take = std::min<std::uint64_t>(n, h->gpos - h->pos);
    const std::uint32_t* src = h->hstage + (h->pos - h->hstage_start);
    if (dst_dev)
        VMT_CUDA(cudaMemcpyAsync(dst, src, take * 4, cudaMemcpyHostToDevice, st));
    else
        std::memcpy(dst, src, take * 4);
    h->pos += take;
    return take;
}

void fill_generic(vmt_generator* h, void* dst, std::uint64_t n, int mode, void* stream) {
    require(dst != nullptr || n == 0, VMT_EINVAL, "null destination");
    if (n == 0)
        return;
    DeviceGuard g(h->device);
    cudaStream_t st = h->pick(stream);
    const bool dev = is_device_ptr(dst);
    std::uint64_t words = (mode == MODE_F64_RES53) ? 2 * n : n;
    if (h->pos < h->gpos) {
        require(mode == MODE_U32 || mode == MODE_XOR, VMT_ESTATE,
                "conversion fills cannot resume inside a partially consumed single-query buffer");
        const std::uint64_t took = drain_stage(h, dst, mode, n, dev, st);
        dst = static_cast<std::uint32_t*>(dst) + took;
        words -= took;
        n -= took;
    }
    if (words == 0) {
        h->mark(st);
        return;
    }
    require(mode != MODE_F64_RES53 || (h->gpos % 2) == 0, VMT_ESTATE, "RES53 needs an even stream position");
    const int esz = (mode == MODE_F64 || mode == MODE_F64_REAL3 || mode == MODE_F64_RES53) ? 8 : 4;
    if (dev) {
        gpu_generate(h, mode, dst, words, st, nullptr);
    } else {
        // host destination: generate in segments into two device staging
        // buffers and copy each one out on a second stream while the next
        // segment is generated (pinned destinations overlap fully)
        const std::uint64_t per_elem_words = (mode == MODE_F64_RES53) ? 2 : 1;
        const std::uint64_t seg_elems = std::min<std::uint64_t>(n, kHostSegmentWords / per_elem_words);
        const std::uint64_t seg_words_cap = seg_elems * (std::uint64_t)esz / 4; // scratch words per half
        h->scratch.reserve(2 * seg_words_cap + 8);
        if (!h->copy_stream) {
            VMT_CUDA(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                VMT_CUDA(cudaEventCreateWithFlags(&h->seg_gen[i], cudaEventDisableTiming));
                VMT_CUDA(cudaEventCreateWithFlags(&h->seg_copy[i], cudaEventDisableTiming));
            }
        }
        std::uint64_t done = 0;
        for (int i = 0; done < n; ++i) {
            const int half = i & 1;
            const std::uint64_t ne = std::min<std::uint64_t>(seg_elems, n - done);
            std::uint32_t* buf = h->scratch.p + half * seg_words_cap;
            if (i >= 2)
                VMT_CUDA(cudaStreamWaitEvent(st, h->seg_copy[half], 0));
            gpu_generate(h, mode, buf, ne * per_elem_words, st, nullptr);
            VMT_CUDA(cudaEventRecord(h->seg_gen[half], st));
            VMT_CUDA(cudaStreamWaitEvent(h->copy_stream, h->seg_gen[half], 0));
            VMT_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + done * esz, buf, ne * esz, cudaMemcpyDeviceToHost,
                                     h->copy_stream));
            VMT_CUDA(cudaEventRecord(h->seg_copy[half], h->copy_stream));
            done += ne;
        }
        VMT_CUDA(cudaStreamSynchronize(h->copy_stream));
    }
    h->pos = h->gpos;
    h->mark(st);
}

void refill_stage(vmt_generator* h) {
    DeviceGuard g(h->device);
    cudaStream_t st = h->pick(nullptr);
    const std::uint64_t S = std::max<std::uint64_t>(h->bw, 1u << 16);
    if (h->hstage_cap < S) {
        if (h->hstage)
            cudaFreeHost(h->hstage);
        h->hstage = nullptr;
        VMT_CUDA(cudaMallocHost(&h->hstage, S * 4));
        h->hstage_cap = S;
    }
    h->scratch.reserve(S);
    h->hstage_start = h->gpos;
    gpu_generate(h, MODE_U32, h->scratch.p, S, st, nullptr);
    VMT_CUDA(cudaMemcpyAsync(h->hstage, h->scratch.p, S * 4, cudaMemcpyDeviceToHost, st));
    VMT_CUDA(cudaStreamSynchronize(st));
    h->mark(st);
}

// Builds interleaved [624][L] de-phased states for `ngen` generators with
// seeds seed0.. into dst (generator stride 624*L words).
// Device buffers kept per host thread and device, reused across calls (no
// cudaMalloc/cudaFree -- a device-wide sync -- per call). Slots: 0 seeds,
// 1 batch states, 2 batch host staging, 3 jumped states (vmt_jump_states),
// 4 its table indices, 5 its distances, 6/7 basis states and polynomial of a
// jump-matrix build (capi_matrix.inl).
template <class T>
DevBuf<T>& thread_scratch(int device, int slot) {
    thread_local std::map<std::pair<int, int>, std::unique_ptr<DevBuf<T>>> bufs;
    auto& b = bufs[std::make_pair(device, slot)];
    if (!b)
        b.reset(new DevBuf<T>());
    return *b;
}
DevBuf<std::uint32_t>& thread_scratch_u32(int device, int slot) { return thread_scratch<std::uint32_t>(device, slot); }

// Scratch larger than this is freed when the call that grew it returns (after
// its final synchronisation), so one large host-destination batch fill does
// not pin gigabytes of device memory outside the caller's allocator for the
// rest of the thread's life; smaller buffers stay cached for reuse.
constexpr size_t kScratchKeepBytes = 64ull << 20;
template <class T>
void trim_scratch(DevBuf<T>& b) {
    if (b.cap * sizeof(T) > kScratchKeepBytes) {
        cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
    }
}

void build_dephased(int device, cudaStream_t st, std::uint32_t seed0, unsigned ngen, unsigned L, unsigned q,
                    std::uint32_t* dst, DevBuf<std::uint64_t>& polybuf, Counters& cnt) {
    std::vector<std::uint32_t> seeds(ngen);
    for (unsigned g = 0; g < ngen; ++g)
        seeds[g] = seed0 + g;
    // per-thread, per-device scratch: no cudaMalloc/cudaFree (a device-wide
    // sync) per call
    DevBuf<std::uint32_t>& dseeds = thread_scratch_u32(device, 0);
    dseeds.reserve(ngen);
    VMT_CUDA(cudaMemcpyAsync(dseeds.p, seeds.data(), ngen * 4, cudaMemcpyHostToDevice, st));
    // one warp per CTA: every store of a warp touches 32 different lines (one per
    // state), so the kernel is bound by the LSUs of the SMs it runs on
    vmt_seed_kernel<<<(ngen + 31) / 32, 32, 0, st>>>(dseeds.p, (int)ngen, dst, (long long)kN * L, (int)L);
    VMT_CUDA(cudaGetLastError());
    cnt.other += 1;
    // many generators: log2(L) tensor-core GEMMs with cached matrices
    static const std::uint64_t gemm_min = std::getenv("VMT_DEPHASE_GEMM_MIN")
                                              ? std::strtoull(std::getenv("VMT_DEPHASE_GEMM_MIN"), nullptr, 10)
                                              : 4096;
    if (L > 1 && (std::uint64_t)ngen * (L - 1) >= gemm_min) {
        bool done = false;
        try {
            done = dephase_by_gemm(device, st, ngen, L, q, dst, cnt);
        } catch (const VmtError&) { // e.g. no memory for the matrices: jump instead
            cudaGetLastError();
            VMT_CUDA(cudaStreamSynchronize(st));
        }
        if (done) {
            VMT_CUDA(cudaStreamSynchronize(st));
            return;
        }
    }
    if (L > 1) {
        const std::vector<Poly> polys = dephase_polys(q, L);
        polybuf.reserve(polys.size() * kPolyWords);
        std::vector<std::uint64_t> flat(polys.size() * kPolyWords);
        for (size_t i = 0; i < polys.size(); ++i)
            std::memcpy(flat.data() + i * kPolyWords, polys[i].data(), kPolyWords * 8);
        VMT_CUDA(cudaMemcpyAsync(polybuf.p, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, st));
        AffineJobs a;
        a.n = (int)(ngen * (L - 1));
        a.div = (int)(L - 1);
        a.s_a = (long long)kN * L;
        a.d_a = (long long)kN * L;
        a.d_b = 1;
        a.d_c = 1;
        a.p_b = 1;
        launch_jumps_affine(st, dst, (int)L, dst, (int)L, polybuf.p, a, cnt);
    }
    VMT_CUDA(cudaStreamSynchronize(st));
}

vmt_generator* new_handle(unsigned L, int device) {
    check_device(device);
    auto* h = new vmt_generator();
    h->device = device;
    h->L = L;
    h->bw = 624ull * L;
    DeviceGuard g(device);
    VMT_CUDA(cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking));
    VMT_CUDA(cudaEventCreateWithFlags(&h->last, cudaEventDisableTiming));
    h->base.reserve((size_t)kN * L);
    h->cur.reserve((size_t)kN * L);
    h->next.reserve((size_t)kN * L);
    VMT_CUDA(cudaMallocHost(&h->hsmall, 64));
    return h;
}

} // namespace

// =================================================================== C ABI ==
extern "C" {

unsigned vmt_full_period_exponent(unsigned lanes) { return unsigned(kDeg) - log2u(lanes ? lanes : 1); }

int vmt_create(uint32_t seed, unsigned lanes, unsigned jump_exponent, int device, vmt_handle* out) {
    return guarded([&] {
        require(out != nullptr, VMT_EINVAL, "null handle pointer");
        require(valid_lanes(lanes), VMT_EINVAL, "lanes must be one of 1, 2, 4, 8, 16, 32");
        const unsigned q = jump_exponent == VMT_FULL_PERIOD ? vmt_full_period_exponent(lanes) : jump_exponent;
        std::unique_ptr<vmt_generator> h(new_handle(lanes, device));
        h->q = q;
        DeviceGuard g(device);
        build_dephased(device, h->own, seed, 1, lanes, q, h->base.p, h->tmp_poly, h->cnt);
        VMT_CUDA(cudaMemcpyAsync(h->cur.p, h->base.p, (size_t)kN * lanes * 4, cudaMemcpyDeviceToDevice, h->own));
        VMT_CUDA(cudaStreamSynchronize(h->own));
        *out = h.release();
    });
}

int vmt_create_from_states(const uint32_t* lane_states, unsigned lanes, int device, vmt_handle* out) {
    return guarded([&] {
        require(out != nullptr && lane_states != nullptr, VMT_EINVAL, "null pointer");
        require(valid_lanes(lanes), VMT_EINVAL, "lanes must be one of 1, 2, 4, 8, 16, 32");
        std::unique_ptr<vmt_generator> h(new_handle(lanes, device));
        h->q = 0;
        std::vector<std::uint32_t> il((size_t)kN * lanes), ls((size_t)kN * lanes);
        if (is_device_ptr(lane_states))
            VMT_CUDA(cudaMemcpy(ls.data(), lane_states, ls.size() * 4, cudaMemcpyDeviceToHost));
        else
            std::memcpy(ls.data(), lane_states, ls.size() * 4);
        for (unsigned k = 0; k < (unsigned)kN; ++k)
            for (unsigned t = 0; t < lanes; ++t)
                il[(size_t)k * lanes + t] = ls[(size_t)t * kN + k];
        DeviceGuard g(device);
        VMT_CUDA(cudaMemcpy(h->base.p, il.data(), il.size() * 4, cudaMemcpyHostToDevice));
        VMT_CUDA(cudaMemcpy(h->cur.p, il.data(), il.size() * 4, cudaMemcpyHostToDevice));
        *out = h.release();
    });
}

int vmt_clone(vmt_handle src, vmt_handle* out) {
    return guarded([&] {
        require(src != nullptr && out != nullptr, VMT_EINVAL, "null argument");
        DeviceGuard g(src->device);
        VMT_CUDA(cudaEventSynchronize(src->last)); // every fill / prefetch of src has finished
        VMT_CUDA(cudaStreamSynchronize(src->own));
        if (src->side)
            VMT_CUDA(cudaStreamSynchronize(src->side));
        std::unique_ptr<vmt_generator> h(new_handle(src->L, src->device));
        h->q = src->q;
        const size_t bytes = (size_t)kN * src->L * 4;
        VMT_CUDA(cudaMemcpy(h->base.p, src->base.p, bytes, cudaMemcpyDeviceToDevice));
        VMT_CUDA(cudaMemcpy(h->cur.p, src->cur.p, bytes, cudaMemcpyDeviceToDevice));
        h->cur_block = src->cur_block;
        h->pos = h->gpos = h->hstage_start = src->pos; // nothing staged: the copy starts at src's position
        h->max_chunks = src->max_chunks;
        h->variant = src->variant;
        h->positioning = src->positioning;
        h->prefetch = src->prefetch;
        *out = h.release();
    });
}

int vmt_destroy(vmt_handle h) {
    return guarded([&] {
        if (!h)
            return;
        {
            DeviceGuard g(h->device);
            cudaStreamSynchronize(h->own);
            if (h->hstage)
                cudaFreeHost(h->hstage);
            if (h->hsmall)
                cudaFreeHost(h->hsmall);
            cudaEventDestroy(h->last);
            for (auto& t : h->evpool)
                for (auto& e : t)
                    cudaEventDestroy(e);
            if (h->side) {
                cudaStreamSynchronize(h->side);
                cudaStreamDestroy(h->side);
                cudaEventDestroy(h->ev_chunks);
                cudaEventDestroy(h->ev_pref);
            }
            delete h->gemm;
            if (h->copy_stream) {
                cudaStreamSynchronize(h->copy_stream);
                cudaStreamDestroy(h->copy_stream);
                for (int i = 0; i < 2; ++i) {
                    cudaEventDestroy(h->seg_gen[i]);
                    cudaEventDestroy(h->seg_copy[i]);
                }
            }
            cudaStreamDestroy(h->own);
            delete h;
        }
    });
}

unsigned vmt_lanes(vmt_handle h) { return h ? h->L : 0; }
uint64_t vmt_state_words(vmt_handle h) { return h ? h->bw : 0; }
unsigned vmt_jump_exponent(vmt_handle h) { return h ? h->q : 0; }
uint64_t vmt_position(vmt_handle h) { return h ? h->pos : 0; }

int vmt_next_u32(vmt_handle h, uint32_t* out) {
    return guarded([&] {
        require(h && out, VMT_EINVAL, "null argument");
        if (h->pos >= h->gpos)
            refill_stage(h);
        *out = h->hstage[h->pos - h->hstage_start];
        ++h->pos;
    });
}

int vmt_next_block16(vmt_handle h, uint32_t* out16) {
    return guarded([&] {
        require(h && out16, VMT_EINVAL, "null argument");
        for (int i = 0; i < 16; ++i) {
            if (h->pos >= h->gpos)
                refill_stage(h);
            out16[i] = h->hstage[h->pos - h->hstage_start];
            ++h->pos;
        }
    });
}

int vmt_next_block_state(vmt_handle h, uint32_t* out) {
    return guarded([&] {
        require(h && out, VMT_EINVAL, "null argument");
        if (h->pos % h->bw != 0)
            throw VmtError(VMT_ESTATE, "state-block query off a state-block boundary");
        fill_generic(h, out, h->bw, MODE_U32, nullptr);
        DeviceGuard g(h->device);
        VMT_CUDA(cudaStreamSynchronize(h->last_stream ? h->last_stream : h->own));
    });
}

int vmt_fill_u32(vmt_handle h, uint32_t* dst, uint64_t n, void* stream) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        fill_generic(h, dst, n, MODE_U32, stream);
    });
}

int vmt_fill_f32(vmt_handle h, float* dst, uint64_t n, int rule, void* stream) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        require(rule == VMT_F32_24, VMT_EINVAL, "unknown float32 rule");
        fill_generic(h, dst, n, MODE_F32, stream);
    });
}

int vmt_fill_f64(vmt_handle h, double* dst, uint64_t n, int rule, void* stream) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        int mode = 0;
        switch (rule) {
        case VMT_F64_32: mode = MODE_F64; break;
        case VMT_F64_REAL3: mode = MODE_F64_REAL3; break;
        case VMT_F64_RES53: mode = MODE_F64_RES53; break;
        default: throw VmtError(VMT_EINVAL, "unknown float64 rule");
        }
        fill_generic(h, dst, n, mode, stream);
    });
}

int vmt_checksum_xor(vmt_handle h, uint64_t n, uint32_t* out, void* stream) {
    return guarded([&] {
        require(h && out, VMT_EINVAL, "null argument");
        DeviceGuard g(h->device);
        cudaStream_t st = h->pick(stream);
        std::uint32_t acc = 0;
        if (h->pos < h->gpos) {
            const std::uint64_t take = std::min<std::uint64_t>(n, h->gpos - h->pos);
            for (std::uint64_t i = 0; i < take; ++i)
                acc ^= h->hstage[h->pos - h->hstage_start + i];
            h->pos += take;
            n -= take;
        }
        if (n) {
            h->scratch.reserve(4);
            gpu_generate(h, MODE_XOR, nullptr, n, st, h->scratch.p);
            VMT_CUDA(cudaMemcpyAsync(h->hsmall, h->scratch.p, 4, cudaMemcpyDeviceToHost, st));
            VMT_CUDA(cudaStreamSynchronize(st));
            acc ^= h->hsmall[0];
            h->pos = h->gpos;
        }
        h->mark(st);
        *out = acc;
    });
}

int vmt_synchronize(vmt_handle h) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        DeviceGuard g(h->device);
        VMT_CUDA(cudaStreamSynchronize(h->own));
        if (h->last_stream)
            VMT_CUDA(cudaEventSynchronize(h->last));
    });
}

int vmt_seek(vmt_handle h, uint64_t pos) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        if (pos >= h->pos && pos <= h->gpos) {
            h->pos = pos; // forward inside the words already staged on the host
            return;
        }
        // drop staging; the GPU state is re-positioned lazily by the next
        // fill (forward from the current block, or from block 0 backwards)
        h->pos = pos;
        h->gpos = pos;
        h->hstage_start = pos;
    });
}

int vmt_skip(vmt_handle h, uint64_t d) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        if (h->pos + d <= h->gpos) {
            h->pos += d;
            return;
        }
        h->pos += d;
        h->gpos = h->pos; // staging dropped; the GPU state is re-positioned lazily
    });
}

int vmt_export_state(vmt_handle h, uint32_t* out) {
    return guarded([&] {
        require(h && out, VMT_EINVAL, "null argument");
        DeviceGuard g(h->device);
        cudaStream_t st = h->pick(nullptr);
        // the reference's state after ceil(pos / bw) regenerations
        const std::uint64_t tb = (h->pos + h->bw - 1) / h->bw;
        const std::uint64_t keep_block = h->cur_block;
        DevBuf<std::uint32_t> tmp;
        tmp.reserve((size_t)kN * h->L);
        if (tb == h->cur_block) {
            VMT_CUDA(cudaMemcpyAsync(out, h->cur.p, (size_t)kN * h->L * 4, cudaMemcpyDeviceToHost, st));
        } else {
            // jump from the block-0 states (no change to the live position)
            Gf2Field& F = Gf2Field::instance();
            const unsigned __int128 d = (unsigned __int128)624u * tb;
            std::vector<Poly> polys{F.x_pow128((std::uint64_t)d, (std::uint64_t)(d >> 64))};
            const std::uint64_t* dp = upload_polys(h, polys, st);
            AffineJobs a;
            a.n = (int)h->L;
            a.div = (int)h->L;
            a.s_b = 1;
            a.d_b = 1;
            launch_jumps_affine(st, h->base.p, (int)h->L, tmp.p, (int)h->L, dp, a, h->cnt);
            VMT_CUDA(cudaMemcpyAsync(out, tmp.p, (size_t)kN * h->L * 4, cudaMemcpyDeviceToHost, st));
        }
        VMT_CUDA(cudaStreamSynchronize(st));
        (void)keep_block;
        h->mark(st);
    });
}

int vmt_batch_fill_u32(uint32_t seed0, unsigned ngen, unsigned lanes, unsigned jump_exponent, uint64_t n_per_gen,
                       uint32_t* dst, int device, void* stream) {
    return guarded([&] {
        require(dst != nullptr || n_per_gen == 0, VMT_EINVAL, "null destination");
        require(valid_lanes(lanes), VMT_EINVAL, "lanes must be one of 1, 2, 4, 8, 16, 32");
        require(ngen > 0, VMT_EINVAL, "ngen must be positive");
        check_device(device);
        DeviceGuard g(device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        const unsigned q = jump_exponent == VMT_FULL_PERIOD ? vmt_full_period_exponent(lanes) : jump_exponent;
        DevBuf<std::uint32_t>& states = thread_scratch_u32(device, 1);
        DevBuf<std::uint64_t> polys;
        Counters cnt;
        states.reserve((size_t)ngen * kN * lanes);
        build_dephased(device, st, seed0, ngen, lanes, q, states.p, polys, cnt);
        if (n_per_gen == 0)
            return;
        const Variant& v = pick_variant(lanes, 0);
        const bool dev = is_device_ptr(dst);
        DevBuf<std::uint32_t>& scratch = thread_scratch_u32(device, 2);
        std::uint32_t* out = dst;
        if (!dev) {
            scratch.reserve((size_t)ngen * n_per_gen);
            out = scratch.p;
        }
        const bool vec = (reinterpret_cast<std::uintptr_t>(out) % 16 == 0) && (n_per_gen % 4 == 0);
        GenFn fn = v.fn[MODE_U32][vec ? 1 : 0];
        prepare_gen(device, fn, v.NT, v.smem[MODE_U32]);
        GenParams p{};
        p.chunk_states = states.p;
        p.out = out;
        p.first_block = 0;
        p.end_block = (n_per_gen + 624ull * lanes - 1) / (624ull * lanes);
        p.pos_begin = 0;
        p.pos_end = n_per_gen;
        p.save_block = ~0ull;
        p.out_chunk_stride = n_per_gen;
        p.blocks_per_chunk = (unsigned)p.end_block;
        p.lanes = lanes;
        fn<<<ngen * (unsigned)(v.L / v.G), v.NT, v.smem[MODE_U32], st>>>(p);
        VMT_CUDA(cudaGetLastError());
        if (!dev)
            VMT_CUDA(cudaMemcpyAsync(dst, scratch.p, (size_t)ngen * n_per_gen * 4, cudaMemcpyDeviceToHost, st));
        VMT_CUDA(cudaStreamSynchronize(st));
        trim_scratch(scratch);
        trim_scratch(states);
    });
}

int vmt_jump_states(const uint32_t* src, uint64_t n, const uint64_t* distances, uint32_t* dst, int device,
                    void* stream) {
    return guarded([&] {
        require(src && distances && dst, VMT_EINVAL, "null argument");
        if (n == 0)
            return;
        check_device(device);
        DeviceGuard g(device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        const std::uint64_t* tables = digit_tables_device(device);
        DevBuf<std::uint32_t>& buf = thread_scratch_u32(device, 3);
        buf.reserve(n * kN);
        if (is_device_ptr(src))
            VMT_CUDA(cudaMemcpyAsync(buf.p, src, n * kN * 4, cudaMemcpyDeviceToDevice, st));
        else
            VMT_CUDA(cudaMemcpyAsync(buf.p, src, n * kN * 4, cudaMemcpyHostToDevice, st));
        std::vector<std::uint64_t> d(n);
        if (is_device_ptr(distances))
            VMT_CUDA(cudaMemcpy(d.data(), distances, n * 8, cudaMemcpyDeviceToHost));
        else
            std::memcpy(d.data(), distances, n * 8);
        // bits 16..63 by four 12-bit table jumps, bits 0..15 by direct
        // advance (vmt_advance_steps_kernel): F^d = F^(d_hi) F^(d_lo). The
        // per-job table indices of all four digits go up in one copy and the
        // launches follow back to back (a zero digit jumps by T_j[0] = 1).
        Counters cnt;
        std::vector<int> pidx((size_t)kDigits * n);
        for (int j = 0; j < kDigits; ++j)
            for (std::uint64_t i = 0; i < n; ++i)
                pidx[(size_t)j * n + i] =
                    j * kDigitVals + (int)((d[i] >> (kDigitBase + kDigitBits * j)) & (kDigitVals - 1));
        DevBuf<int>& dp = thread_scratch<int>(device, 4);
        dp.reserve(pidx.size());
        VMT_CUDA(cudaMemcpyAsync(dp.p, pidx.data(), pidx.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        for (int j = 0; j < kDigits; ++j) {
            AffineJobs a;
            a.n = (int)n;
            a.div = 1;
            a.s_a = kN; // job i: state i, in place (each warp reads its whole state before writing it)
            a.d_a = kN;
            launch_jumps_affine(st, buf.p, 1, buf.p, 1, tables, a, cnt, dp.p + (size_t)j * n);
        }
        DevBuf<unsigned long long>& dd = thread_scratch<unsigned long long>(device, 5);
        dd.reserve(n);
        VMT_CUDA(cudaMemcpyAsync(dd.p, d.data(), n * 8, cudaMemcpyHostToDevice, st));
        vmt_advance_steps_kernel<<<(unsigned)n, kStepThreads, 0, st>>>(
            buf.p, (long long)n, dd.p, 0xFFFFu);
        VMT_CUDA(cudaGetLastError());
        if (is_device_ptr(dst))
            VMT_CUDA(cudaMemcpyAsync(dst, buf.p, n * kN * 4, cudaMemcpyDeviceToDevice, st));
        else
            VMT_CUDA(cudaMemcpyAsync(dst, buf.p, n * kN * 4, cudaMemcpyDeviceToHost, st));
        VMT_CUDA(cudaStreamSynchronize(st));
        trim_scratch(buf);
    });
}

int vmt_seed_states(const uint32_t* seeds, uint64_t n, uint32_t* dst, int device, void* stream) {
    return guarded([&] {
        require(seeds && dst, VMT_EINVAL, "null argument");
        if (n == 0)
            return;
        check_device(device);
        DeviceGuard g(device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        DevBuf<std::uint32_t> ds, out;
        ds.reserve(n);
        if (is_device_ptr(seeds))
            VMT_CUDA(cudaMemcpyAsync(ds.p, seeds, n * 4, cudaMemcpyDeviceToDevice, st));
        else
            VMT_CUDA(cudaMemcpyAsync(ds.p, seeds, n * 4, cudaMemcpyHostToDevice, st));
        const bool dev = is_device_ptr(dst);
        std::uint32_t* o = dst;
        if (!dev) {
            out.reserve(n * kN);
            o = out.p;
        }
        vmt_seed_kernel<<<(unsigned)((n + 31) / 32), 32, 0, st>>>(ds.p, (int)n, o, kN, 1);
        VMT_CUDA(cudaGetLastError());
        if (!dev)
            VMT_CUDA(cudaMemcpyAsync(dst, out.p, n * kN * 4, cudaMemcpyDeviceToHost, st));
        VMT_CUDA(cudaStreamSynchronize(st));
    });
}

int vmt_jump_poly(uint64_t d_lo, uint64_t d_hi, uint64_t* out312) {
    return guarded([&] {
        require(out312 != nullptr, VMT_EINVAL, "null argument");
        const Poly p = Gf2Field::instance().x_pow128(d_lo, d_hi);
        std::memcpy(out312, p.data(), kPolyWords * 8);
    });
}

int vmt_jump_poly_pow2(unsigned q, uint64_t* out312) {
    return guarded([&] {
        require(out312 != nullptr, VMT_EINVAL, "null argument");
        const Poly p = Gf2Field::instance().x_pow2(q);
        std::memcpy(out312, p.data(), kPolyWords * 8);
    });
}

int vmt_charpoly(uint64_t* out313) {
    return guarded([&] {
        require(out313 != nullptr, VMT_EINVAL, "null argument");
        const auto& p = Gf2Field::instance().charpoly();
        std::memcpy(out313, p.data(), kFullWords * 8);
    });
}

int vmt_set_tuning(vmt_handle h, unsigned max_chunks, int variant) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        (void)pick_variant(h->L, variant); // validates
        h->max_chunks = max_chunks;
        h->variant = variant;
        h->pref_valid = false;
    });
}

int vmt_set_prefetch(vmt_handle h, int enable) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        require(enable >= VMT_PREFETCH_OFF && enable <= VMT_PREFETCH_TENSOR, VMT_EINVAL, "unknown prefetch mode");
        h->prefetch = enable;
        h->pref_valid = false;
    });
}

int vmt_release_caches(int device) {
    return guarded([&] {
        check_device(device);
        DeviceGuard g(device);
        VMT_CUDA(cudaDeviceSynchronize());
        std::lock_guard<std::mutex> lk(g_dephase_mu);
        auto it = g_dephase.find(device);
        if (it != g_dephase.end()) {
            std::lock_guard<std::mutex> lk2(it->second->mu);
            it->second->mats.clear();
            it->second->tmaps.clear();
        }
        std::lock_guard<std::mutex> lk3(g_chunkpoly_mu); // host side: the chunk polynomials
        g_chunkpoly.clear();
    });
}

int vmt_set_positioning(vmt_handle h, int mode) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        require(mode >= 0 && mode <= 2, VMT_EINVAL, "positioning mode must be 0 (auto), 1 (jumps) or 2 (gemm)");
        h->positioning = mode;
    });
}

int vmt_positioning_stats(vmt_handle h, uint64_t* gemm_positionings, uint64_t* cached_matrices) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        if (gemm_positionings)
            *gemm_positionings = h->cnt.gemm_positionings;
        if (cached_matrices)
            *cached_matrices = h->gemm ? h->gemm->mats.size() : 0;
    });
}

int vmt_prefetch_stats(vmt_handle h, uint64_t* tensor_prefetches, uint64_t* used) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        if (tensor_prefetches)
            *tensor_prefetches = h->cnt.tc_prefetches;
        if (used)
            *used = h->cnt.pref_used;
    });
}

int vmt_set_profiling(vmt_handle h, int enable) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        DeviceGuard g(h->device);
        prof_fold(h);
        h->profile = enable != 0;
    });
}

int vmt_last_timings(vmt_handle h, float* jump_ms, float* gen_ms) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        DeviceGuard g(h->device);
        prof_fold(h);
        require(h->last_gen_ms >= 0.f, VMT_ESTATE, "profiling disabled or no fill recorded");
        if (jump_ms)
            *jump_ms = h->last_jump_ms;
        if (gen_ms)
            *gen_ms = h->last_gen_ms;
    });
}

int vmt_profile_totals(vmt_handle h, uint64_t* fills, double* jump_ms, double* gen_ms) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        DeviceGuard g(h->device);
        prof_fold(h);
        if (fills)
            *fills = h->prof_fills;
        if (jump_ms)
            *jump_ms = h->prof_jump_ms;
        if (gen_ms)
            *gen_ms = h->prof_gen_ms;
        h->prof_fills = 0;
        h->prof_jump_ms = h->prof_gen_ms = 0;
    });
}

int vmt_stats(vmt_handle h, uint64_t* gen_launches, uint64_t* jump_launches, uint64_t* other_launches,
              uint64_t* lane_jumps) {
    return guarded([&] {
        require(h != nullptr, VMT_EINVAL, "null handle");
        if (gen_launches)
            *gen_launches = h->cnt.gen;
        if (jump_launches)
            *jump_launches = h->cnt.jump;
        if (other_launches)
            *other_launches = h->cnt.other;
        if (lane_jumps)
            *lane_jumps = h->cnt.lane_jumps;
    });
}

int vmt_store_bandwidth(int device, uint64_t bytes, int pattern, int ctas_per_sm, double* gbs) {
    return guarded([&] {
        require(gbs != nullptr && bytes >= 16, VMT_EINVAL, "bad argument");
        require(pattern >= 0 && pattern <= 2, VMT_EINVAL,
                "pattern must be 0 (grid-stride), 1 (chunked) or 2 (chunked, random words)");
        check_device(device);
        DeviceGuard g(device);
        const unsigned long long n4 = bytes / 16;
        DevBuf<uint4> buf;
        buf.reserve(n4);
        const int sms = device_info(device).sms;
        const unsigned grid = (unsigned)(sms * std::max(1, ctas_per_sm));
        cudaStream_t st = cudaStreamPerThread;
        auto launch = [&] {
            if (pattern == 0)
                vmt_store_probe_stride<<<grid, 512, 0, st>>>(buf.p, n4);
            else if (pattern == 1)
                vmt_store_probe_chunked<<<grid, 256, 0, st>>>(buf.p, n4);
            else
                vmt_store_probe_chunked_random<<<grid, 256, 0, st>>>(buf.p, n4);
        };
        launch();
        VMT_CUDA(cudaGetLastError());
        cudaEvent_t e0, e1;
        VMT_CUDA(cudaEventCreate(&e0));
        VMT_CUDA(cudaEventCreate(&e1));
        VMT_CUDA(cudaEventRecord(e0, st));
        for (int r = 0; r < 3; ++r)
            launch();
        VMT_CUDA(cudaEventRecord(e1, st));
        VMT_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        VMT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *gbs = double(n4 * 16) * 3 / (ms * 1e-3) / 1e9;
    });
}

const char* vmt_status_string(int status) {
    switch (status) {
    case VMT_OK: return "ok";
    case VMT_EINVAL: return "invalid argument";
    case VMT_ESTATE: return "invalid state (cadence / boundary)";
    case VMT_EIO: return "I/O or format error";
    case VMT_ECUDA: return "CUDA error";
    case VMT_ENOMEM: return "out of memory";
    default: return "unknown status";
    }
}

const char* vmt_last_error(void) { return g_last_error.c_str(); }

int vmt_version(void) { return 100; }

} // extern "C"

// GF(2) jump-matrix path: .vmtj files, vec_mat_mul, matrix de-phasing.
#include "capi_matrix.inl"
// Fused statistics consumer: monobit / chi2_bytes counts in MODE_STATS.
#include "capi_stats.inl"

// Generator batches (config 3) and the single-process multi-GPU fill (config 4).
#include "capi_batch.inl"

#ifdef VMT_TIMELINE
// experiments (profiles/scripts/timeline.py): copies the 6144-word timeline buffer to the host
extern "C" int vmt_debug_timeline(unsigned long long* host_out) {
    if (cudaDeviceSynchronize() != cudaSuccess)
        return -1;
    return cudaMemcpy(host_out, timeline_buf(), 6144 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) ==
                   cudaSuccess
               ? 0
               : -1;
}
#endif
