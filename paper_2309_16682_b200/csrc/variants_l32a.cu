// Generation-kernel instantiations, group l32a (see vmt_variants.hpp).
#include "vmt_variant_impl.cuh"

namespace vmt_b200 {

std::vector<Variant> variants_l32a() { return {make_variant<32, 32, 13, 2>(3), make_variant<32, 32, 13, 4>(1), make_variant<32, 32, 13, 1>(4)}; }

} // namespace vmt_b200
