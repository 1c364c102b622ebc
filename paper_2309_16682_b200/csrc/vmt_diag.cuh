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

} // namespace vmt_b200
