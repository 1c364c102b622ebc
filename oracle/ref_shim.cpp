// TEST INFRASTRUCTURE ONLY (oracle/): a C-ABI shim over the UNMODIFIED
// reference library, compiled from the sources where they lie under
// /root/reference/proj (see oracle/Makefile). Nothing in the product links
// this; it is loaded by tests/, by __graft_entry__.smoke() only as a checker,
// and by bench.py's reference / cpu_baseline arms.
//
// Every entry point calls the reference's own public C++ API:
//   Mt19937                 proj/include/vmt19937/mt19937.hpp:79-104
//   VmtEngine<M>            proj/include/vmt19937/engine.hpp:41-158
//   make_dephased_states    proj/src/jump.cpp:35-53
//   jump_state              proj/src/jump.cpp:27-33
//   mat_mul / transition F  proj/src/f2_matrix.cpp:138-228
//   run_benchmark           proj/src/bench.cpp:99-120
//   .vmtj files             proj/src/jump_file.cpp:117-209
//   monobit / chi2_bytes    proj/src/stats.cpp:65-107
// Error mapping: invalid_argument -> -1, logic_error -> -2, other -> -3.

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <stdexcept>
#include <thread>
#include <vector>

#include "vmt19937/bench.hpp"
#include "vmt19937/engine.hpp"
#include "vmt19937/jump.hpp"
#include "vmt19937/jump_file.hpp"
#include "vmt19937/lane_ops.hpp"
#include "vmt19937/stats.hpp"

using namespace vmt19937;

namespace {

std::mutex g_mu;
std::map<unsigned, F2Matrix>& ladder() {
    static std::map<unsigned, F2Matrix> cache;
    return cache;
}

// F^(2^q), extended on demand from the highest cached rung (the same
// idiom as proj/tests/test_jump.cpp:14-28).
const F2Matrix& transition_power(unsigned q) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& cache = ladder();
    if (auto it = cache.find(q); it != cache.end())
        return it->second;
    if (cache.empty())
        cache.emplace(0, build_transition_matrix(mt19937_params()));
    auto best = cache.begin();
    for (auto it = cache.begin(); it != cache.end(); ++it)
        if (it->first <= q)
            best = it;
    F2Matrix m = best->second;
    for (unsigned i = best->first; i < q; ++i)
        m = mat_mul(m, m);
    return cache.emplace(q, std::move(m)).first->second;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (const std::logic_error&) {
        return -2;
    } catch (...) {
        return -3;
    }
}

template <int M>
void engine_stream(std::uint32_t seed, unsigned q, std::uint64_t count, std::uint32_t* out) {
    const F2Matrix none;
    const F2Matrix& jm = (M == 1) ? none : transition_power(q);
    auto gen = std::make_unique<VmtEngine<M>>(seed, jm, q);
    std::vector<std::uint32_t> buf(VmtEngine<M>::state_words);
    std::uint64_t done = 0;
    while (done < count) {
        gen->next_block_state(buf.data());
        const std::uint64_t take = std::min<std::uint64_t>(buf.size(), count - done);
        std::memcpy(out + done, buf.data(), take * 4);
        done += take;
    }
}

template <int M>
void engine_state(std::uint32_t seed, unsigned q, unsigned nblocks, std::uint32_t* out) {
    const F2Matrix none;
    const F2Matrix& jm = (M == 1) ? none : transition_power(q);
    auto gen = std::make_unique<VmtEngine<M>>(seed, jm, q);
    std::vector<std::uint32_t> buf(VmtEngine<M>::state_words);
    for (unsigned b = 0; b < nblocks; ++b)
        gen->next_block_state(buf.data());
    std::memcpy(out, gen->state_data(), VmtEngine<M>::state_words * 4);
}

template <int M>
double bench_threads(std::uint32_t seed, unsigned q, std::uint64_t words_per_thread, int threads,
                     std::uint32_t* buf, std::uint32_t* checksum) {
    // One VmtEngine per thread, each writing next_block_state into its own
    // slice of one large buffer (the all-cores plan of BASELINE.md section 3).
    const F2Matrix none;
    const F2Matrix& jm = (M == 1) ? none : transition_power(q);
    const std::uint64_t bw = VmtEngine<M>::state_words;
    const std::uint64_t blocks = (words_per_thread + bw - 1) / bw;
    std::vector<std::unique_ptr<VmtEngine<M>>> gens;
    for (int t = 0; t < threads; ++t)
        gens.push_back(std::make_unique<VmtEngine<M>>(seed + std::uint32_t(t), jm, q));
    std::atomic<int> ready{0};
    std::atomic<bool> go{false};
    std::vector<double> secs(threads, 0.0);
    std::vector<std::uint32_t> sums(threads, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            std::uint32_t* dst = buf + std::uint64_t(t) * blocks * bw;
            ready.fetch_add(1);
            while (!go.load()) {
            }
            const auto t0 = std::chrono::steady_clock::now();
            for (std::uint64_t b = 0; b < blocks; ++b)
                gens[t]->next_block_state(dst + b * bw);
            secs[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            std::uint32_t x = 0;
            for (std::uint64_t i = 0; i < blocks * bw; ++i)
                x ^= dst[i];
            sums[t] = x;
        });
    while (ready.load() < threads) {
    }
    const auto t0 = std::chrono::steady_clock::now();
    go.store(true);
    for (auto& th : pool)
        th.join();
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::uint32_t x = 0;
    for (auto s : sums)
        x ^= s;
    if (checksum)
        *checksum = x;
    (void)secs;
    return wall;
}

} // namespace

extern "C" {

// Scalar MT19937 (mt19937.cpp:22-55): outputs [skip, skip+count) of seed.
int vref_mt_stream(std::uint32_t seed, std::uint64_t skip, std::uint64_t count, std::uint32_t* out) {
    return guarded([&] {
        Mt19937 s(seed);
        for (std::uint64_t i = 0; i < skip; ++i)
            s.next_u32();
        for (std::uint64_t i = 0; i < count; ++i)
            out[i] = s.next_u32();
    });
}

// Scalar outputs of an arbitrary boundary state (Mt19937::from_words).
int vref_mt_stream_from_words(const std::uint32_t* words, std::uint64_t count, std::uint32_t* out) {
    return guarded([&] {
        std::array<std::uint32_t, 624> w;
        std::memcpy(w.data(), words, sizeof(w));
        Mt19937 s = Mt19937::from_words(w);
        for (std::uint64_t i = 0; i < count; ++i)
            out[i] = s.next_u32();
    });
}

// VmtEngine<M>(seed, F^(2^q), q).next_block_state, first count words.
int vref_engine_stream(std::uint32_t seed, unsigned lanes, unsigned q, std::uint64_t count,
                       std::uint32_t* out) {
    return guarded([&] {
        switch (lanes) {
        case 1: engine_stream<1>(seed, q, count, out); break;
        case 2: engine_stream<2>(seed, q, count, out); break;
        case 4: engine_stream<4>(seed, q, count, out); break;
        case 8: engine_stream<8>(seed, q, count, out); break;
        case 16: engine_stream<16>(seed, q, count, out); break;
        default: throw std::invalid_argument("lanes must be one of 1, 2, 4, 8, 16");
        }
    });
}

// VmtEngine<M>::interleaved_state() after nblocks state-block queries.
int vref_engine_state(std::uint32_t seed, unsigned lanes, unsigned q, unsigned nblocks,
                      std::uint32_t* out) {
    return guarded([&] {
        switch (lanes) {
        case 1: engine_state<1>(seed, q, nblocks, out); break;
        case 2: engine_state<2>(seed, q, nblocks, out); break;
        case 4: engine_state<4>(seed, q, nblocks, out); break;
        case 8: engine_state<8>(seed, q, nblocks, out); break;
        case 16: engine_state<16>(seed, q, nblocks, out); break;
        default: throw std::invalid_argument("lanes must be one of 1, 2, 4, 8, 16");
        }
    });
}

// make_dephased_states(Mt19937(seed), JumpSpec{q, lanes}, F^(2^q)); any
// power-of-two lane count (JumpSpec accepts L=32, jump.cpp:8-11).
int vref_dephased_states(std::uint32_t seed, unsigned lanes, unsigned q, std::uint32_t* out) {
    return guarded([&] {
        const F2Matrix& jm = transition_power(q);
        auto st = make_dephased_states(Mt19937(seed), JumpSpec{q, lanes}, jm);
        for (unsigned t = 0; t < lanes; ++t)
            std::memcpy(out + std::size_t(t) * 624, st[t].words().data(), 624 * 4);
    });
}

// jump_state(from_words(in), F^(2^q)).
int vref_jump_state(const std::uint32_t* in, unsigned q, std::uint32_t* out) {
    return guarded([&] {
        std::array<std::uint32_t, 624> w;
        std::memcpy(w.data(), in, sizeof(w));
        Mt19937 j = jump_state(Mt19937::from_words(w), transition_power(q));
        std::memcpy(out, j.words().data(), 624 * 4);
    });
}

// Seeding only (mt19937.cpp:22-27).
int vref_seed_words(std::uint32_t seed, std::uint32_t* out) {
    return guarded([&] {
        Mt19937 s(seed);
        std::memcpy(out, s.words().data(), 624 * 4);
    });
}

// Builds (and caches) the ladder up to F^(2^q); returns 0 when done.
int vref_prepare_ladder(unsigned q) {
    return guarded([&] { (void)transition_power(q); });
}

// The reference's own single-thread benchmark (bench.cpp:99-120).
// mode: 0 single, 1 block16, 2 state-block.
int vref_run_benchmark(unsigned lanes, int mode, std::uint64_t count, std::uint32_t seed,
                       unsigned q, double* seconds, std::uint32_t* checksum) {
    return guarded([&] {
        BenchConfig cfg;
        cfg.generator = BenchGenerator::kVmt;
        cfg.lanes = lanes;
        cfg.block = mode == 0 ? QueryMode::kSingle
                              : (mode == 1 ? QueryMode::kBlock16 : QueryMode::kStateBlock);
        cfg.count = count;
        cfg.seed = seed;
        cfg.jump_exponent = q;
        cfg.jump_matrix = lanes == 1 ? nullptr : &transition_power(q);
        BenchResult r = run_benchmark(cfg);
        *seconds = r.seconds;
        *checksum = r.checksum;
    });
}

// All-cores DRAM-bound run: `threads` independent engines, each writing
// words_per_thread (rounded up to whole blocks) into its own slice of buf.
// Returns wall seconds of the parallel region (setup excluded) or < 0.
double vref_bench_threads(unsigned lanes, std::uint32_t seed, unsigned q,
                          std::uint64_t words_per_thread, int threads, std::uint32_t* buf,
                          std::uint32_t* checksum) {
    double s = -1.0;
    int rc = guarded([&] {
        switch (lanes) {
        case 4: s = bench_threads<4>(seed, q, words_per_thread, threads, buf, checksum); break;
        case 8: s = bench_threads<8>(seed, q, words_per_thread, threads, buf, checksum); break;
        case 16: s = bench_threads<16>(seed, q, words_per_thread, threads, buf, checksum); break;
        default: throw std::invalid_argument("lanes must be one of 4, 8, 16");
        }
    });
    return rc == 0 ? s : double(rc);
}

std::uint64_t vref_state_words(unsigned lanes) { return 624ull * lanes; }

// 1 when lane count M has a SIMD backend in this build (lane_ops.hpp:227-230).
int vref_simd_backend(unsigned lanes) {
    switch (lanes) {
    case 4: return has_simd_lanes<4>() ? 1 : 0;
    case 8: return has_simd_lanes<8>() ? 1 : 0;
    case 16: return has_simd_lanes<16>() ? 1 : 0;
    default: return 0;
    }
}

// Jump by an arbitrary 64-bit distance by composing the ladder rungs
// F^(2^i) at the set bits of d with jump_state.
int vref_jump_by(const std::uint32_t* in, std::uint64_t d, std::uint32_t* out) {
    return guarded([&] {
        std::array<std::uint32_t, 624> w;
        std::memcpy(w.data(), in, sizeof(w));
        Mt19937 s = Mt19937::from_words(w);
        for (unsigned i = 0; i < 64; ++i)
            if ((d >> i) & 1u)
                s = jump_state(s, transition_power(i));
        std::memcpy(out, s.words().data(), 624 * 4);
    });
}

// write_jump_matrix_file(path, F^(2^q), q) with the cached ladder rung --
// the bytes compute_jump_matrix (jump_file.cpp:171-209) writes for exponent q.
int vref_write_pow2_matrix_file(unsigned q, const char* path) {
    return guarded([&] { write_jump_matrix_file(path, transition_power(q), q); });
}

// read_jump_matrix_file (jump_file.cpp:125-137): rows (nullable) and exponent.
int vref_read_jump_matrix_file(const char* path, std::uint64_t* rows, unsigned* dim, unsigned* exponent) {
    return guarded([&] {
        LoadedJumpMatrix m = read_jump_matrix_file(path);
        if (dim)
            *dim = unsigned(m.matrix.dim());
        if (exponent)
            *exponent = m.exponent;
        if (rows)
            std::memcpy(rows, m.matrix.data().data(), m.matrix.data().size() * 8);
    });
}

// make_dephased_states(Mt19937(seed), JumpSpec{exponent, lanes}, B) with B
// read from a .vmtj file.
int vref_dephased_states_file(std::uint32_t seed, unsigned lanes, const char* path, std::uint32_t* out) {
    return guarded([&] {
        LoadedJumpMatrix m = read_jump_matrix_file(path);
        auto st = make_dephased_states(Mt19937(seed), JumpSpec{m.exponent, lanes}, m.matrix);
        for (unsigned t = 0; t < lanes; ++t)
            std::memcpy(out + std::size_t(t) * 624, st[t].words().data(), 624 * 4);
    });
}

// detail::regularized_gamma_q (stats.cpp:52-60).
int vref_regularized_gamma_q(double a, double x, double* out) {
    return guarded([&] { *out = detail::regularized_gamma_q(a, x); });
}

// monobit (which = 0) / chi2_bytes (which = 1) over the first `count` words
// of VmtGenerator(seed, VmtConfig(lanes, kSingle, q), F^(2^q)).next_u32, the
// CLI `stat` wiring (vmt19937_main.cpp:203-214).
int vref_stat_report(std::uint32_t seed, unsigned lanes, unsigned q, std::uint64_t count, int which,
                     double* statistic, double* p_value, int* pass) {
    return guarded([&] {
        auto gen = lanes == 1 ? std::make_shared<VmtGenerator>(seed)
                              : std::make_shared<VmtGenerator>(seed, VmtConfig(lanes, QueryMode::kSingle, q),
                                                               transition_power(q));
        WordSource src = [gen] { return gen->next_u32(); };
        const StatReport r = which == 0 ? monobit(src, count) : chi2_bytes(src, count);
        *statistic = r.statistic;
        *p_value = r.p_value;
        *pass = r.pass ? 1 : 0;
    });
}

// lane_cross_correlation over the CLI's per-lane sources (make_dephased_states
// + regenerate + next_u32, vmt19937_main.cpp:216-229); which = 2 on a
// constant source pair instead when seed_or_word is used as the word.
int vref_lane_corr(std::uint32_t seed, unsigned lanes, unsigned q, std::uint64_t count, double* statistic,
                   double* p_value, int* pass) {
    return guarded([&] {
        auto states = make_dephased_states(Mt19937(seed), JumpSpec{q, lanes}, transition_power(q));
        std::vector<WordSource> sources;
        for (auto& st : states) {
            auto lane = std::make_shared<Mt19937>(st);
            lane->regenerate();
            sources.push_back([lane] { return lane->next_u32(); });
        }
        const StatReport r = lane_cross_correlation(sources, count);
        *statistic = r.statistic;
        *p_value = r.p_value;
        *pass = r.pass ? 1 : 0;
    });
}

// monobit (0) / chi2_bytes (1) / lane_cross_correlation of two copies (2) of
// a constant source (the CLI's --self-test, vmt19937_main.cpp:174-186).
int vref_stat_constant(std::uint32_t word, std::uint64_t count, int which, double* statistic, double* p_value,
                       int* pass) {
    return guarded([&] {
        WordSource c = [word] { return word; };
        const StatReport r = which == 0 ? monobit(c, count)
                             : which == 1 ? chi2_bytes(c, count)
                                          : lane_cross_correlation({c, c}, count);
        *statistic = r.statistic;
        *p_value = r.p_value;
        *pass = r.pass ? 1 : 0;
    });
}

// libstdc++ std::mt19937_64 (the tests' RNG idiom, test_mt19937.cpp:67).
int vref_mt64(std::uint64_t seed, std::uint64_t count, std::uint64_t* out) {
    std::mt19937_64 g(seed);
    for (std::uint64_t i = 0; i < count; ++i)
        out[i] = g();
    return 0;
}

} // extern "C"
