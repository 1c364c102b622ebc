// Experiment (not product code): store paths compared by rate AND power under
// sustained load -- 64-bit and 128-bit per-thread stores of random-looking
// words (one IMAD per word, like real generator output rather than a
// counter), and TMA bulk stores (cp.async.bulk.global.shared::cta) of a
// shared-memory staging buffer, one chunk per CTA. Usage: probe_power MODE REPS
//   MODE: stg64 | stg128 | tma  (148 CTAs, 16 GiB per launch)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <class T>
__global__ void __launch_bounds__(256, 1) stg(T* out, unsigned long long n) {
    const unsigned long long per = (n + gridDim.x - 1) / gridDim.x;
    const unsigned long long lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
    for (unsigned long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        T v; unsigned* p = reinterpret_cast<unsigned*>(&v);
#pragma unroll
        for (int k = 0; k < (int)(sizeof(T) / 4); ++k) p[k] = ((unsigned)i + k) * 0x9E3779B9u;
        out[i] = v;
    }
}

constexpr int kStage = 26624; // one 208-row x 32-lane window of 32-bit words
__global__ void __launch_bounds__(256, 1) tma(unsigned char* out, unsigned long long bytes, int inflight) {
    extern __shared__ __align__(128) unsigned char buf[];
    unsigned* w = reinterpret_cast<unsigned*>(buf);
    for (int i = threadIdx.x; i < 2 * kStage / 4; i += blockDim.x) w[i] = (i * 2654435761u) ^ blockIdx.x;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const unsigned long long per = bytes / gridDim.x / kStage * kStage;
    unsigned char* dst = out + blockIdx.x * per;
    const unsigned s0 = static_cast<unsigned>(__cvta_generic_to_shared(buf));
    for (unsigned long long off = 0, k = 0; off < per; off += kStage, ++k) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                     "r"(s0 + (unsigned)(k & 1) * kStage), "r"(kStage) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (inflight == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        else if (inflight == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    const char* mode = argc > 1 ? argv[1] : "stg64";
    const int reps = argc > 2 ? atoi(argv[2]) : 20;
    const int inflight = argc > 3 ? atoi(argv[3]) : 2;
    const unsigned long long bytes = 16ull << 30;
    void* p; CK(cudaMalloc(&p, bytes));
    auto launch = [&]() {
        if (!strcmp(mode, "stg64")) stg<uint2><<<148, 256>>>((uint2*)p, bytes / 8);
        else if (!strcmp(mode, "stg128")) stg<uint4><<<148, 256>>>((uint4*)p, bytes / 16);
        else tma<<<148, 32, 2 * kStage>>>((unsigned char*)p, bytes, inflight);
    };
    CK(cudaFuncSetAttribute(tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kStage));
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
    printf("{\"mode\": \"%s\", \"inflight\": %d, \"reps\": %d, \"ms\": %.4f, \"tbs\": %.4f}\n", mode, inflight, reps, ms,
           bytes / (ms * 1e-3) / 1e12);
    return 0;
}
