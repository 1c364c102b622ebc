// Generation-kernel instantiations, group l16b (see vmt_variants.hpp).
#include "vmt_variant_impl.cuh"

namespace vmt_b200 {

std::vector<Variant> variants_l16b() { return {make_variant<16, 16, 1, 4>(5), make_variant<16, 16, 13, 2, 104, true>(6), make_variant<16, 8, 13, 2>(7)}; }

} // namespace vmt_b200
