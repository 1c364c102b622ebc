// Experiment (not product code): warp-specialised generation kernel. Warps
// 0-7 twist (ring + history registers), warps 8-15 temper + store the
// previous window's words from the ring. Store mode, whole blocks only.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../../paper_2309_16682_b200/csrc/vmt_common.cuh"
using namespace vmt_b200;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int L = 32, R = 13, V = 2, W = 208, Q = 16, RUNS = 16, RING = 832, SLOTS = RING + R;
constexpr int NP = 256; // producer threads
#ifndef NC
#define NC 256 // consumer threads
#endif
#ifndef CV
#define CV 2 // lanes per consumer thread (4: LDS.128 / STG.128)
#endif
#ifndef LBT
#define LBT (NP + NC)
#endif
constexpr int CQ = L / CV;                 // consumer threads across a row
constexpr int CR = W * CQ / NC;            // rows per consumer thread per window

template <bool STORE>
__global__ void __launch_bounds__(LBT, 1) ws_kernel(const uint32_t* states, uint32_t* out, unsigned long long B,
                                                       uint32_t* xparts) {
    extern __shared__ __align__(16) uint32_t ring[];
    const int tid = threadIdx.x;
    const bool prod = tid < NP;
    const uint32_t* src = states + (size_t)blockIdx.x * kN * L;
    for (int i = tid; i < kN * Q; i += NP + NC) {
        const int slot = i / Q, qq = i % Q;
        const uint2 v = *reinterpret_cast<const uint2*>(src + slot * L + qq * V);
        reinterpret_cast<uint2*>(ring)[i] = v;
        if (i < R * Q) reinterpret_cast<uint2*>(ring)[RING * Q + i] = v;
    }
    __syncthreads();
    uint32_t acc = 0;
    uint32_t* o_chunk = out + (size_t)blockIdx.x * B * kN * L;
    if (prod) {
        const int q = tid % Q, rho = tid / Q;
        uint32_t H[3][R][V];
#pragma unroll
        for (int wi = 0; wi < 3; ++wi)
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const uint2 v = *reinterpret_cast<const uint2*>(ring + (wi * W + rho * R + i) * L + q * V);
                H[wi][i][0] = v.x; H[wi][i][1] = v.y;
            }
        int bbs = 0;
        for (unsigned long long blk = 0; blk < B; ++blk) {
#pragma unroll
            for (int wi = 0; wi < 3; ++wi) {
                int wstart = bbs + wi * W; if (wstart >= RING) wstart -= RING;
                const int base = wstart + rho * R;
                int a = base + kM; if (a >= RING) a -= RING;
                int wsl = base + kN; if (wsl >= RING) wsl -= RING;
                uint32_t X[R + 1][V], M[R][V];
#pragma unroll
                for (int i = 0; i < R; ++i) { X[i][0] = H[wi][i][0]; X[i][1] = H[wi][i][1]; }
                { const uint2 v = *reinterpret_cast<const uint2*>(ring + (base + R) * L + q * V); X[R][0] = v.x; X[R][1] = v.y; }
#pragma unroll
                for (int i = 0; i < R; ++i) { const uint2 v = *reinterpret_cast<const uint2*>(ring + (a + i) * L + q * V); M[i][0] = v.x; M[i][1] = v.y; }
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    uint32_t n0 = twist(X[i][0], X[i + 1][0], M[i][0]);
                    uint32_t n1 = twist(X[i][1], X[i + 1][1], M[i][1]);
                    *reinterpret_cast<uint2*>(ring + (wsl + i) * L + q * V) = make_uint2(n0, n1);
                    H[wi][i][0] = n0; H[wi][i][1] = n1;
                }
                if (wsl == 0) {
#pragma unroll
                    for (int i = 0; i < R; ++i)
                        *reinterpret_cast<uint2*>(ring + (RING + i) * L + q * V) = *reinterpret_cast<const uint2*>(ring + i * L + q * V);
                }
                __syncthreads();
            }
            bbs += kN; if (bbs >= RING) bbs -= RING;
        }
        __syncthreads(); // the consumers' drain window
    } else {
        const int t = tid - NP;
        const int q = t % CQ, rho = t / CQ; // consumer rows: NC/CQ rows of CR words
        __syncthreads(); // producers compute window 0; nothing to store yet
        int bbs = 0;
        unsigned long long wcount = 0;
        for (unsigned long long blk = 0; blk < B; ++blk) {
#pragma unroll
            for (int wi = 0; wi < 3; ++wi) {
                int wstart = bbs + wi * W; if (wstart >= RING) wstart -= RING;
                int wsl = wstart + rho * CR + kN; if (wsl >= RING) wsl -= RING;
                uint32_t* o = o_chunk + (size_t)(wcount * W + rho * CR) * L + q * CV;
#pragma unroll
                for (int i = 0; i < CR; ++i) {
                    int s = wsl + i; if (s >= RING) s -= RING;
                    if (CV == 4) {
                        const uint4 v = *reinterpret_cast<const uint4*>(ring + s * L + q * CV);
                        const uint4 tv = make_uint4(temper(v.x), temper(v.y), temper(v.z), temper(v.w));
                        if (STORE) *reinterpret_cast<uint4*>(o + i * L) = tv;
                        else acc ^= tv.x ^ tv.y ^ tv.z ^ tv.w;
                    } else {
                        const uint2 v = *reinterpret_cast<const uint2*>(ring + s * L + q * CV);
                        const uint32_t t0 = temper(v.x), t1 = temper(v.y);
                        if (STORE) *reinterpret_cast<uint2*>(o + i * L) = make_uint2(t0, t1);
                        else acc ^= t0 ^ t1;
                    }
                }
                ++wcount;
                __syncthreads();
            }
            bbs += kN; if (bbs >= RING) bbs -= RING;
        }
    }
    if (!STORE && !prod) atomicXor(xparts + blockIdx.x, acc);
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20;
    const int C = 148;
    const unsigned long long B = 1453, n = (unsigned long long)C * B * kN * L;
    std::vector<unsigned> h((size_t)C * kN * L);
    unsigned s = 12345;
    for (auto& v : h) { s = s * 1664525u + 1013904223u; v = s; }
    unsigned *states, *out, *parts;
    CK(cudaMalloc(&states, h.size() * 4));
    CK(cudaMemcpy(states, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&out, n * 4));
    CK(cudaMalloc(&parts, C * 4));
    const int smem = SLOTS * L * 4;
    CK(cudaFuncSetAttribute(ws_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(ws_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms[2];
    for (int m = 0; m < 2; ++m) {
        for (int i = 0; i < 3; ++i) { if (m == 0) ws_kernel<true><<<C, NP + NC, smem>>>(states, out, B, parts); else ws_kernel<false><<<C, NP + NC, smem>>>(states, out, B, parts); }
        CK(cudaDeviceSynchronize());
        CK(cudaMemset(parts, 0, C * 4));
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i) { if (m == 0) ws_kernel<true><<<C, NP + NC, smem>>>(states, out, B, parts); else ws_kernel<false><<<C, NP + NC, smem>>>(states, out, B, parts); }
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms[m], a, b);
        ms[m] /= reps;
    }
    std::vector<unsigned> ho(1 << 18);
    CK(cudaMemcpy(ho.data(), out + n - ho.size(), ho.size() * 4, cudaMemcpyDeviceToHost));
    unsigned y = 0; for (auto v : ho) y ^= v;
    printf("{\"ws\": %d, \"cv\": %d, \"lbt\": %d, \"store_ms\": %.4f, \"store_tbs\": %.4f, \"temperxor_ms\": %.4f, \"temperxor_words_s\": %.4e, \"chk\": \"%08x\"}\n",
           NC, CV, LBT, ms[0], n * 4.0 / ms[0] / 1e9, ms[1], n / (ms[1] * 1e-3), y);
}
