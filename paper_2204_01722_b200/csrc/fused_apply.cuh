// Fused brick Jacobian apply (declared here, defined in fused_apply.cu).
#pragma once

#include <cuda_runtime.h>

#include <functional>

namespace hxg {
class Operator;
bool fused_supported(int p, int q);
int fused_launches(int p, int q);
void fused_jacobian(Operator& op, const double* du, double* y);
void fused_jacobian_host(Operator& op, const double* xh, double* yh);
void fused_residual(Operator& op, const double* u, double* f);
// Partitioned apply with the interface exchange overlapped: the bricks
// touching the interface faces (bits iface) and their interface-node sums
// first; `exchange` is then enqueued on the side stream (after them) while
// the remaining bricks and sums run on the operator's stream; the operator's
// stream finally waits for the side stream.
void fused_jacobian_split(Operator& op, const double* du, double* y, int iface, cudaStream_t side,
                          const std::function<void()>& exchange);
}  // namespace hxg
