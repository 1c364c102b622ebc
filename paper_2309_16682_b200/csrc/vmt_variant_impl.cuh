// make_variant: instantiates vmt_gen_kernel for every output mode of one
// shape (included by the variants_*.cu translation units only).
#pragma once

#include "vmt_gen.cuh"
#include "vmt_variants.hpp"

namespace vmt_b200 {

template <int LT, int G, int R, int VW, int W, bool TMA, int MODE>
void fill_mode(Variant& v) {
    v.fn[MODE][0] = vmt_gen_kernel<LT, G, R, VW, W, TMA, MODE, false>;
    v.fn[MODE][1] = vmt_gen_kernel<LT, G, R, VW, W, TMA, MODE, true>;
    v.smem[MODE] = GenShape<G, R, VW, W, TMA>::template smem<MODE>();
}

// LT = lanes of the stream, G = lanes per CTA (LT/G CTAs per chunk)
template <int LT, int G, int R, int VW, int W = 208, bool TMA = false>
Variant make_variant(int id) {
    Variant v;
    v.id = id;
    v.L = LT;
    v.G = G;
    v.R = R;
    v.VW = VW;
    v.W = W;
    v.tma = TMA;
    v.NT = GenShape<G, R, VW, W, TMA>::NT;
    fill_mode<LT, G, R, VW, W, TMA, MODE_U32>(v);
    fill_mode<LT, G, R, VW, W, TMA, MODE_XOR>(v);
    fill_mode<LT, G, R, VW, W, TMA, MODE_F32>(v);
    fill_mode<LT, G, R, VW, W, TMA, MODE_F64>(v);
    fill_mode<LT, G, R, VW, W, TMA, MODE_F64_REAL3>(v);
    fill_mode<LT, G, R, VW, W, TMA, MODE_F64_RES53>(v);
    // no output: one instantiation serves both slots
    v.fn[MODE_STATS][0] = v.fn[MODE_STATS][1] = vmt_gen_kernel<LT, G, R, VW, W, TMA, MODE_STATS, false>;
    v.smem[MODE_STATS] = GenShape<G, R, VW, W, TMA>::template smem<MODE_STATS>();
    return v;
}

} // namespace vmt_b200
