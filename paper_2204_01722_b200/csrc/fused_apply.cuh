// Fused brick Jacobian apply (declared here, defined in fused_apply.cu).
#pragma once

namespace hxg {
class Operator;
bool fused_supported(int p, int q);
int fused_launches(int p, int q);
void fused_jacobian(Operator& op, const double* du, double* y);
void fused_jacobian_host(Operator& op, const double* xh, double* yh);
void fused_residual(Operator& op, const double* u, double* f);
}  // namespace hxg
