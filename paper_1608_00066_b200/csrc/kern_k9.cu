// K=9 (557,663,711) rate-1/3 code, 256 states (BASELINE config C4).
#include "kern_common.cuh"
namespace pbvd {
using C9 = Code<9, 3, 0557, 0663, 0711>;
void add_variants_k9(std::vector<Variant>& v) {
    v.push_back(make_variant<C9, 8>(0));
    v.push_back(make_variant<C9, 4>(1));
}
}  // namespace pbvd
