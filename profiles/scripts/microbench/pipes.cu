// Experiment (not product code): issue/pipe throughput of the integer
// instructions the generation kernel's twist + temper can be written with
// (LOP3 / SHF on the ALU pipe, IMAD / IMAD.SHL / IMAD.HI / IMAD.WIDE on the
// FMA pipe), alone and in the temper's mix. Each thread iterates K
// independent words; prints thread-ops per SM per clock for each variant.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int K = 12; // independent words per thread

__device__ __forceinline__ unsigned shr(unsigned x, int s) { unsigned r; asm volatile("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s)); return r; }
__device__ __forceinline__ unsigned mulhi(unsigned x, unsigned m) { unsigned r; asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(m)); return r; }
__device__ __forceinline__ unsigned mulwide_hi(unsigned x, unsigned m) {
    unsigned long long r; asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(x), "r"(m)); return (unsigned)(r >> 32); }
__device__ __forceinline__ unsigned shl_imad(unsigned x, unsigned m) { unsigned r; asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(m)); return r; }
__device__ __forceinline__ unsigned lop_xa(unsigned a, unsigned b, unsigned c) { // a ^ (b & c)
    unsigned r; asm volatile("lop3.b32 %0, %1, %2, %3, 0x6a;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r; }
__device__ __forceinline__ unsigned lop_x(unsigned a, unsigned b) { unsigned r; asm volatile("xor.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ unsigned fsh(unsigned a, unsigned b) { unsigned r; asm volatile("shf.r.wrap.b32 %0, %1, %2, 3;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ unsigned imad(unsigned a, unsigned b, unsigned c) { unsigned r; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r; }

template <int V>
__device__ __forceinline__ unsigned step(unsigned y, unsigned B, unsigned C) {
    if (V == 0) { // the temper as shipped: 6 ALU + 2 FMA
        y = lop_x(y, shr(y, 11));
        y = lop_xa(y, shl_imad(y, 1u << 7), B);
        y = lop_xa(y, shl_imad(y, 1u << 15), C);
        y = lop_x(y, shr(y, 18));
    } else if (V == 1) { // first right shift as IMAD.HI
        y = lop_x(y, mulhi(y, 1u << 21));
        y = lop_xa(y, shl_imad(y, 1u << 7), B);
        y = lop_xa(y, shl_imad(y, 1u << 15), C);
        y = lop_x(y, shr(y, 18));
    } else if (V == 2) { // first right shift as IMAD.WIDE (high half)
        y = lop_x(y, mulwide_hi(y, 1u << 21));
        y = lop_xa(y, shl_imad(y, 1u << 7), B);
        y = lop_xa(y, shl_imad(y, 1u << 15), C);
        y = lop_x(y, shr(y, 18));
    } else if (V == 3) { // 8 LOP3
        for (int i = 0; i < 8; ++i) y = lop_xa(y, B, C);
    } else if (V == 4) { // 8 SHF (funnel shifts of two registers: not foldable)
        unsigned z = y ^ B;
        for (int i = 0; i < 4; ++i) { y = fsh(y, z); z = fsh(z, y); }
        y ^= z;
    } else if (V == 5) { // 8 IMAD
        for (int i = 0; i < 8; ++i) y = imad(y, B, C);
    } else if (V == 6) { // 8 IMAD.HI
        for (int i = 0; i < 8; ++i) y = mulhi(y, 0x9908b0dfu);
    } else if (V == 7) { // 4 IMAD.WIDE + 4 IMAD (both halves used)
        for (int i = 0; i < 4; ++i) {
            unsigned long long r; asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(y), "r"(0x9908b0dfu));
            y = imad((unsigned)r, B, (unsigned)(r >> 32));
        }
    } else if (V == 8) { // 8 IMAD.SHL
        for (int i = 0; i < 8; ++i) y = shl_imad(y, 1u << 7);
    } else if (V == 9) { // 4 LOP3 + 4 IMAD.HI interleaved
        for (int i = 0; i < 4; ++i) { y = lop_xa(y, B, C); y = mulhi(y, 0x9908b0dfu); }
    } else if (V == 10) { // 4 LOP3 + 4 IMAD interleaved
        for (int i = 0; i < 4; ++i) { y = lop_xa(y, B, C); y = imad(y, B, C); }
    } else if (V == 11) { // 6 LOP3 + 2 IMAD.WIDE
        for (int i = 0; i < 2; ++i) { y = lop_xa(y, B, C); y = lop_xa(y, B, C); y = lop_xa(y, B, C); y = mulwide_hi(y, 0x9908b0dfu); }
    }
    return y;
}

template <int V>
__global__ void k_pipes(unsigned* out, int iters, unsigned B, unsigned C, long long* clk) {
    unsigned y[K];
#pragma unroll
    for (int j = 0; j < K; ++j) y[j] = threadIdx.x * 7919u + j * 104729u + blockIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < K; ++j) y[j] = step<V>(y[j], B, C);
    }
    long long t1 = clock64();
    unsigned x = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) x ^= y[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, int ops, int threads, unsigned* out, long long* clk, int sms) {
    const int iters = 4096;
    for (int r = 0; r < 2; ++r) k_pipes<V><<<sms, threads>>>(out, iters, 0x9d2c5680u, 0xefc60000u, clk);
    CK(cudaDeviceSynchronize());
    long long h[1024];
    CK(cudaMemcpy(h, clk, sms * sizeof(long long), cudaMemcpyDeviceToHost));
    double c = 0; for (int i = 0; i < sms; ++i) c += h[i]; c /= sms;
    const double thread_ops = (double)threads * iters * K * ops;
    printf("{\"variant\": \"%s\", \"threads_per_sm\": %d, \"thread_ops_per_clk_per_sm\": %.2f}\n", name, threads, thread_ops / c);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* out; long long* clk;
    CK(cudaMalloc(&out, sms * 1024 * 4));
    CK(cudaMalloc(&clk, sms * 8));
    for (int threads : {256, 512, 1024}) {
        run<0>("temper_shipped(8 ops)", 8, threads, out, clk, sms);
        run<1>("temper_imadhi(8 ops)", 8, threads, out, clk, sms);
        run<2>("temper_imadwide(8 ops)", 8, threads, out, clk, sms);
        run<3>("lop3", 8, threads, out, clk, sms);
        run<4>("shf", 8, threads, out, clk, sms);
        run<5>("imad", 8, threads, out, clk, sms);
        run<6>("imad.hi", 8, threads, out, clk, sms);
        run<7>("imad.wide", 8, threads, out, clk, sms);
        run<8>("imad.shl", 8, threads, out, clk, sms);
        run<9>("lop3+imad.hi", 8, threads, out, clk, sms);
        run<10>("lop3+imad", 8, threads, out, clk, sms);
        run<11>("3lop3+imad.wide", 8, threads, out, clk, sms);
    }
    return 0;
}
