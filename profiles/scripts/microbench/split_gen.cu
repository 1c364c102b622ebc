// Experiment (not product code): generation kernel with runs of 6 and 7
// words (32 runs per 208-word window) instead of 16 runs of 13, so that
// each thread can own V = 4 lanes (LDS.128 / STS.128 / STG.128, 256 threads)
// or V = 2 lanes with twice the warps (512 threads). Store mode, whole
// blocks only; prints TB/s of the store kernel and the output checksum of
// the last MB for comparison with mb_gen (same states, same layout).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../../paper_2309_16682_b200/csrc/vmt_common.cuh"
using namespace vmt_b200;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

#ifndef SV
#define SV 4
#endif
#ifndef MINB
#define MINB 1
#endif
constexpr int L = 32, W = 208, RING = 832, RA = 6, RB = 7, NA = 16, NRUN = 32, MIR = RB, SLOTS = RING + MIR;
constexpr int V = SV, Q = L / V, NT = NRUN * Q;
using VT = typename VecT<V>::T;

template <int R>
__device__ __forceinline__ void window(uint32_t* ring, int base, int a, int wsl, int q, uint32_t (&H)[RB][V],
                                       uint32_t* o) {
    uint32_t X[R + 1][V], M[R][V];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int v = 0; v < V; ++v) X[i][v] = H[i][v];
    VecT<V>::get(*reinterpret_cast<const VT*>(ring + (base + R) * L + q * V), X[R]);
#pragma unroll
    for (int i = 0; i < R; ++i) VecT<V>::get(*reinterpret_cast<const VT*>(ring + (a + i) * L + q * V), M[i]);
#pragma unroll
    for (int i = 0; i < R; ++i) {
        uint32_t nw[V], tw[V];
#pragma unroll
        for (int v = 0; v < V; ++v) nw[v] = twist(X[i][v], X[i + 1][v], M[i][v]);
        *reinterpret_cast<VT*>(ring + (wsl + i) * L + q * V) = VecT<V>::make(nw);
#pragma unroll
        for (int v = 0; v < V; ++v) { H[i][v] = nw[v]; tw[v] = temper(nw[v]); }
        *reinterpret_cast<VT*>(o + i * L) = VecT<V>::make(tw);
    }
    if (wsl < MIR) { // mirror of slots [0, MIR) behind the ring end
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (wsl + i < MIR)
                *reinterpret_cast<VT*>(ring + (RING + wsl + i) * L + q * V) = VecT<V>::make(H[i]);
    }
}

template <int R>
__device__ __forceinline__ void run_chunk(uint32_t* ring, int q, int row0, uint32_t* out, unsigned long long B) {
    uint32_t H[3][RB][V];
#pragma unroll
    for (int wi = 0; wi < 3; ++wi)
#pragma unroll
        for (int i = 0; i < R; ++i)
            VecT<V>::get(*reinterpret_cast<const VT*>(ring + (wi * W + row0 + i) * L + q * V), H[wi][i]);
    int bbs = 0;
    for (unsigned long long blk = 0; blk < B; ++blk) {
#pragma unroll
        for (int wi = 0; wi < 3; ++wi) {
            int wstart = bbs + wi * W; if (wstart >= RING) wstart -= RING;
            const int base = wstart + row0;
            int a = base + kM; if (a >= RING) a -= RING;
            int wsl = base + kN; if (wsl >= RING) wsl -= RING;
            uint32_t* o = out + (blk * kN + wi * W + row0) * L + q * V;
            window<R>(ring, base, a, wsl, q, H[wi], o);
            __syncthreads();
        }
        bbs += kN; if (bbs >= RING) bbs -= RING;
    }
}

__global__ void __launch_bounds__(NT, MINB) split_kernel(const uint32_t* states, uint32_t* out, unsigned long long B) {
    extern __shared__ __align__(16) uint32_t ring[];
    const int tid = threadIdx.x;
    const uint32_t* src = states + (size_t)blockIdx.x * kN * L;
    for (int i = tid; i < kN * Q; i += NT) {
        const int slot = i / Q, qq = i % Q;
        const VT v = *reinterpret_cast<const VT*>(src + slot * L + qq * V);
        reinterpret_cast<VT*>(ring)[i] = v;
        if (i < MIR * Q) reinterpret_cast<VT*>(ring)[RING * Q + i] = v;
    }
    __syncthreads();
    const int q = tid % Q, rho = tid / Q;
    uint32_t* o_chunk = out + (size_t)blockIdx.x * B * kN * L;
    if (rho < NA) run_chunk<RA>(ring, q, rho * RA, o_chunk, B);
    else run_chunk<RB>(ring, q, NA * RA + (rho - NA) * RB, o_chunk, B);
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20;
    const int C = 148;
    const unsigned long long B = 1453ull;
    const unsigned long long n = (unsigned long long)C * B * kN * L;
    std::vector<unsigned> h((size_t)C * kN * L);
    unsigned s = 12345;
    for (auto& v : h) { s = s * 1664525u + 1013904223u; v = s; }
    unsigned *states, *out;
    CK(cudaMalloc(&states, h.size() * 4));
    CK(cudaMemcpy(states, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&out, n * 4));
    const int smem = SLOTS * L * 4;
    CK(cudaFuncSetAttribute(split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int i = 0; i < 3; ++i) split_kernel<<<C, NT, smem>>>(states, out, B);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) split_kernel<<<C, NT, smem>>>(states, out, B);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    std::vector<unsigned> ho(1 << 18);
    CK(cudaMemcpy(ho.data(), out + n - ho.size(), ho.size() * 4, cudaMemcpyDeviceToHost));
    unsigned y = 0; for (auto v : ho) y ^= v;
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, split_kernel);
    printf("{\"split\": \"%d/%d\", \"V\": %d, \"threads\": %d, \"regs\": %d, \"local\": %zu, \"reps\": %d, \"store_ms\": %.4f, \"store_tbs\": %.4f, \"chk\": \"%08x\"}\n",
           RA, RB, V, NT, fa.numRegs, fa.localSizeBytes, reps, ms, n * 4.0 / ms / 1e9, y);
    return 0;
}
