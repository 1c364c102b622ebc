// Store-bandwidth probes: the pure-store ceilings the generation kernel is
// measured against ("a trivial st.global.v4 kernel as a second
// denominator"). Not on any generation path.
#pragma once

#include <cstdint>

namespace vmt_b200 {

// pattern 0: grid-stride 16-byte stores (all CTAs write neighbouring lines)
__global__ void vmt_store_probe_stride(uint4* out, unsigned long long n4) {
    unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    const unsigned long long s = (unsigned long long)gridDim.x * blockDim.x;
    for (; i < n4; i += s)
        out[i] = make_uint4((unsigned)i, (unsigned)i + 1, (unsigned)i + 2, (unsigned)i + 3);
}

// pattern 1: every CTA writes its own contiguous chunk (the generation kernel's
// output pattern: one chunk of the stream per CTA)
__global__ void vmt_store_probe_chunked(uint4* out, unsigned long long n4) {
    const unsigned long long per = (n4 + gridDim.x - 1) / gridDim.x;
    const unsigned long long lo = blockIdx.x * per, hi = lo + per < n4 ? lo + per : n4;
    for (unsigned long long i = lo + threadIdx.x; i < hi; i += blockDim.x)
        out[i] = make_uint4((unsigned)i, (unsigned)i + 1, (unsigned)i + 2, (unsigned)i + 3);
}

// pattern 2: as pattern 1 with random-looking words (a multiplicative hash
// per word, like generator output): at the B200's 1000 W board limit the
// bits toggled on the HBM interface decide whether the store stream alone is
// power-capped (counter data ~930 W, random words ~990 W at 6.4 TB/s)
__global__ void vmt_store_probe_chunked_random(uint4* out, unsigned long long n4) {
    const unsigned long long per = (n4 + gridDim.x - 1) / gridDim.x;
    const unsigned long long lo = blockIdx.x * per, hi = lo + per < n4 ? lo + per : n4;
    for (unsigned long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const unsigned x = (unsigned)i * 0x9E3779B9u;
        out[i] = make_uint4(x, x * 0x85EBCA6Bu, x * 0xC2B2AE35u, x * 0x27D4EB2Fu);
    }
}

} // namespace vmt_b200
