// Generation-kernel instantiations, group l8 (see vmt_variants.hpp).
#include "vmt_variant_impl.cuh"

namespace vmt_b200 {

std::vector<Variant> variants_l8() { return {make_variant<8, 8, 13, 2>(3), make_variant<8, 8, 13, 4>(1), make_variant<8, 8, 13, 1>(4), make_variant<8, 8, 1, 4>(5)}; }

} // namespace vmt_b200
