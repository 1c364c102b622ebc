// Driver for the reference's own benchmark code (proj/src/bench.cpp, compiled
// UNCHANGED against include/vmt19937/*.hpp, so its VmtEngine<M> are the GPU
// engines): runs run_benchmark for M in {1,2,4,8,16} in all three query modes
// with F^(2^q) from the GPU ladder and prints one CSV row per run --
// lanes,mode,count,q,seed,checksum,seconds,words_per_sec -- for
// tests/test_cpp_abi.py to compare with the reference's checksums
// (tests/golden/golden.json bench_checksums; vmt19937_main.cpp:71-125 prints
// the same columns).
#include <cstdio>
#include <cstdlib>

#include "vmt19937/bench.hpp"

using namespace vmt19937;

int main(int argc, char** argv) {
    const std::uint64_t count = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000;
    const unsigned q = argc > 2 ? unsigned(std::atoi(argv[2])) : 6;
    const F2Matrix b = mat_pow2(build_transition_matrix(mt19937_params()), q);
    std::printf("lanes,mode,count,q,seed,checksum,seconds,words_per_sec\n");
    const QueryMode modes[3] = {QueryMode::kSingle, QueryMode::kBlock16, QueryMode::kStateBlock};
    for (unsigned lanes : {1u, 2u, 4u, 8u, 16u})
        for (int m = 0; m < 3; ++m) {
            BenchConfig cfg;
            cfg.lanes = lanes;
            cfg.block = modes[m];
            cfg.count = count;
            cfg.jump_exponent = q;
            cfg.jump_matrix = &b;
            const BenchResult r = run_benchmark(cfg);
            std::printf("%u,%d,%llu,%u,%u,0x%08X,%.6f,%.6g\n", lanes, m, (unsigned long long)count, q, cfg.seed,
                        r.checksum, r.seconds, r.words_per_sec);
        }
    BenchConfig scalar;
    scalar.generator = BenchGenerator::kScalar;
    scalar.count = count;
    const BenchResult r = run_benchmark(scalar);
    std::printf("scalar,0,%llu,0,%u,0x%08X,%.6f,%.6g\n", (unsigned long long)count, scalar.seed, r.checksum,
                r.seconds, r.words_per_sec);
    return 0;
}
