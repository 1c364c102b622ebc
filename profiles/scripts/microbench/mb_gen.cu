// Microbenchmark of the generation kernel's store and compute rates for
// compile-time arithmetic variants (build: scratch/mb_gen.sh). Not product code.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../../paper_2309_16682_b200/csrc/vmt_gen.cuh"
using namespace vmt_b200;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

#ifndef MB_VW
#define MB_VW 2
#endif
#ifndef MB_R
#define MB_R 13
#endif
#ifndef MB_W
#define MB_W 208
#endif
#ifndef MB_L
#define MB_L 32
#endif
#ifndef MB_TMA
#define MB_TMA false
#endif
template <int MODE>
float run(GenParams p, int grid, int reps, cudaStream_t st) {
    using S = GenShape<MB_L, MB_R, MB_VW, MB_W, MB_TMA>;
    auto fn = vmt_gen_kernel<MB_L, MB_L, MB_R, MB_VW, MB_W, MB_TMA, MODE, true>;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, S::smem<MODE>()));
    for (int i = 0; i < 3; ++i) fn<<<grid, S::NT, S::smem<MODE>(), st>>>(p);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, st);
    for (int i = 0; i < reps; ++i) fn<<<grid, S::NT, S::smem<MODE>(), st>>>(p);
    cudaEventRecord(b, st);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20;
    const int C = argc > 2 ? atoi(argv[2]) : 148, L = MB_L;
    const unsigned long long B = argc > 3 ? strtoull(argv[3], nullptr, 10) : 1453ull * 148 / C * 32 / L; // blocks per chunk: 148 * 1453 * 19968 ~ 2^32 words
    const unsigned long long n = (unsigned long long)C * B * kN * L;
    std::vector<unsigned> h((size_t)C * kN * L);
    unsigned s = 12345;
    for (auto& v : h) { s = s * 1664525u + 1013904223u; v = s; }
    unsigned *states, *out, *parts;
    CK(cudaMalloc(&states, h.size() * 4));
    CK(cudaMemcpy(states, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&out, n * 4));
    CK(cudaMalloc(&parts, C * 4 * 4));
    cudaStream_t st; cudaStreamCreate(&st);
    GenParams p{};
    p.chunk_states = states; p.out = out; p.xor_partials = parts; p.save_state = nullptr;
    p.first_block = 0; p.end_block = C * B; p.pos_begin = 0; p.pos_end = n; p.save_block = ~0ull;
    p.blocks_per_chunk = (unsigned)B; p.lanes = L;
    // MB_ONLY=store / MB_ONLY=xor: run one of the two (power sampling)
    const char* only = getenv("MB_ONLY");
    const bool do_store = !only || only[0] == 's', do_xor = !only || only[0] == 'x';
    const float ms_store = do_store ? run<MODE_U32>(p, C, reps, st) : 0.f;
    const float ms_xor = do_xor ? run<MODE_BENCH_TEMPER_XOR>(p, C, reps, st) : 0.f;
    std::vector<unsigned> hp(C);
    CK(cudaMemcpy(hp.data(), parts, C * 4, cudaMemcpyDeviceToHost));
    unsigned x = 0; for (auto v : hp) x ^= v;
    // XOR of a sample of the stored output (first/last MB)
    std::vector<unsigned> ho(std::min<unsigned long long>(1 << 18, n));
    CK(cudaMemcpy(ho.data(), out + n - ho.size(), ho.size() * 4, cudaMemcpyDeviceToHost));
    unsigned y = 0; for (auto v : ho) y ^= v;
    printf("{\"L\": %d, \"tma\": %d, \"R\": %d, \"W\": %d, \"C\": %d, \"vw\": %d, \"shr_fma\": %d, \"store_ms\": %.4f, \"store_tbs\": %.4f, \"words_s_per_chunk\": %.4e, \"temperxor_ms\": %.4f, \"temperxor_words_s\": %.4e, \"chk\": \"%08x-%08x\"}\n",
           MB_L, (int)MB_TMA, MB_R, MB_W, C, MB_VW, VMT_SHR_FMA, ms_store, n * 4.0 / ms_store / 1e9, n / (ms_store * 1e-3) / C, ms_xor, n / (ms_xor * 1e-3), x, y);
    return 0;
}
