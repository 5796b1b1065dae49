// K=5 (23,35) code, 16 states (GSM-style).
#include "kern_common.cuh"
namespace pbvd {
using C5 = Code<5, 2, 023, 035>;
void add_variants_k5(std::vector<Variant>& v) { v.push_back(make_variant<C5, 1>(0)); }
}  // namespace pbvd
