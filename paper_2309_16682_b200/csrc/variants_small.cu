// Generation-kernel instantiations, group small (see vmt_variants.hpp).
#include "vmt_variant_impl.cuh"

namespace vmt_b200 {

std::vector<Variant> variants_small() { return {make_variant<4, 4, 13, 1>(4), make_variant<4, 4, 1, 4>(5), make_variant<2, 2, 13, 1>(4), make_variant<2, 2, 1, 2>(5), make_variant<1, 1, 1, 1>(5)}; }

} // namespace vmt_b200
