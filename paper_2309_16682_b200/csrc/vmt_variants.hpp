// Generation-kernel shape variants (vmt_set_tuning). The instantiations live
// in variants_*.cu -- one translation unit per lane-count group so the build
// compiles them in parallel; vmt_capi.cu only holds the function pointers.
#pragma once

#include <vector>

#include "vmt_common.cuh"

namespace vmt_b200 {

using GenFn = void (*)(GenParams);

struct Variant {
    int id = 0, L = 0, G = 0, R = 0, VW = 0, W = 0, NT = 0;
    bool tma = false;
    int smem[kModes] = {};
    GenFn fn[kModes][2] = {};
};

// Run length R = consecutive words per thread per window, VW = lanes per
// thread, W = window, G = lanes per CTA, TMA = window output staged in shared
// memory and written by one bulk copy. The first entry per lane count is the
// default.
//   id 3: R=13 VW=2   id 1: R=13 VW=4   id 4: R=13 VW=1   id 5: R=1 VW=4
//   id 6: R=13 VW=2 W=104 TMA bulk stores
//   id 7: R=13 VW=2 G=8 (lane groups of 8)   id 8: R=13 VW=2 G=16
std::vector<Variant> variants_l32a();
std::vector<Variant> variants_l32b();
std::vector<Variant> variants_l16a();
std::vector<Variant> variants_l16b();
std::vector<Variant> variants_l8();
std::vector<Variant> variants_small();

} // namespace vmt_b200
