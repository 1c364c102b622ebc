// Experiment: pure-store ceilings (chunk per CTA) at burst and sustained length.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
template <class T>
__global__ void chunked(T* out, unsigned long long n) {
    const unsigned long long per = (n + gridDim.x - 1) / gridDim.x;
    const unsigned long long lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
    for (unsigned long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        T v; unsigned* p = reinterpret_cast<unsigned*>(&v);
        for (int k = 0; k < (int)(sizeof(T) / 4); ++k) p[k] = (unsigned)i + k;
        out[i] = v;
    }
}
template <class T>
float run(T* out, unsigned long long bytes, int grid, int nt, int reps) {
    const unsigned long long n = bytes / sizeof(T);
    for (int i = 0; i < 3; ++i) chunked<T><<<grid, nt>>>(out, n);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) chunked<T><<<grid, nt>>>(out, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return bytes / (ms / reps * 1e-3) / 1e12;
}
int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20;
    const unsigned long long bytes = 16ull << 30;
    void* p; cudaMalloc(&p, bytes);
    if (argc > 2) { // one probe only (power sampling): v4 or v2, 148 x 256
        const bool v4 = argv[2][1] == '4';
        const float t = v4 ? run((uint4*)p, bytes, 148, 256, reps) : run((uint2*)p, bytes, 148, 256, reps);
        printf("{\"reps\": %d, \"%s_148x256\": %.3f}\n", reps, argv[2], t);
        return 0;
    }
    printf("{\"reps\": %d, \"v4_148x256\": %.3f, \"v2_148x256\": %.3f, \"v4_296x256\": %.3f, \"v4_148x512\": %.3f}\n", reps,
           run((uint4*)p, bytes, 148, 256, reps), run((uint2*)p, bytes, 148, 256, reps),
           run((uint4*)p, bytes, 296, 256, reps), run((uint4*)p, bytes, 148, 512, reps));
}
