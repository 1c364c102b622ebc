// Generation-kernel instantiations, group l32b (see vmt_variants.hpp).
#include "vmt_variant_impl.cuh"

namespace vmt_b200 {

std::vector<Variant> variants_l32b() { return {make_variant<32, 32, 13, 2, 104, true>(6), make_variant<32, 8, 13, 2>(7), make_variant<32, 16, 13, 2>(8)}; }

} // namespace vmt_b200
