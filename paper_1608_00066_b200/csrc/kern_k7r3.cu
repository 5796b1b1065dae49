// K=7 rate-1/3 (133,171,165) code, 64 states (LTE / 3GPP style).
#include "kern_common.cuh"
namespace pbvd {
using C7R3 = Code<7, 3, 0133, 0171, 0165>;
void add_variants_k7r3(std::vector<Variant>& v) { v.push_back(make_variant<C7R3, 2>(0)); }
}  // namespace pbvd
