// K=7 (171,133) CCSDS / 802.11 code, 64 states (the paper's code, P:376;
// BASELINE configs C2, C3, C5).
#include "kern_common.cuh"
namespace pbvd {
using C7 = Code<7, 2, 0171, 0133>;
void add_variants_k7(std::vector<Variant>& v) {
    v.push_back(make_variant<C7, 2>(0));
    v.push_back(make_variant<C7, 1>(1));
    v.push_back(make_variant<C7, 4>(2));
}
}  // namespace pbvd
