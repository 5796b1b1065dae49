// K=9 (557,663,711) rate-1/3 code, 256 states (BASELINE config C4).
#include "kern_common.cuh"
namespace pbvd {
using C9 = Code<9, 3, 0557, 0663, 0711>;
void add_variants_k9(std::vector<Variant>& v) {
    // W=4 is the faster default with the fused traceback (its 16-block
    // survivor ring fits beside the forward's shared memory); W=8 wins for the
    // two-kernel path (pbvd_set_fused(h, 0)) -- see DESIGN.md section 7
    v.push_back(make_variant<C9, 4>(0));
    v.push_back(make_variant<C9, 8>(1));
}
}  // namespace pbvd
