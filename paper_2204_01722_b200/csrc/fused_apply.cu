// Fused brick Jacobian apply — placeholder until the brick kernel lands.
#include "fused_apply.cuh"
#include "operator.hpp"

namespace hxg {
bool fused_supported(int, int) { return false; }
int fused_launches(int, int) { return 1; }
void fused_jacobian(Operator&, const double*, double*) {
  throw Error(HXG_ERR_UNSUPPORTED, "fused apply not available");
}
}  // namespace hxg
