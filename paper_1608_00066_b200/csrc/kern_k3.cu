// K=3 (7,5) textbook code, 4 states (BASELINE config C1).
#include "kern_common.cuh"
namespace pbvd {
using C3 = Code<3, 2, 07, 05>;
void add_variants_k3(std::vector<Variant>& v) { v.push_back(make_variant<C3, 1>(0)); }
}  // namespace pbvd
