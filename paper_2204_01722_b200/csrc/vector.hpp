// Device vector kernels for CG / Chebyshev / V-cycle (cg.hpp:81-184,
// smoother.hpp:41-62, multigrid.hpp:167-194).  Reductions are deterministic:
// a fixed grid and a fixed-order tree, independent of the device.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace hxg {

struct DotWorkspace {
  double* partial = nullptr;  // kDotBlocks partials + 2 results
  double* host = nullptr;     // pinned result slots
  DotWorkspace();
  ~DotWorkspace();
  DotWorkspace(const DotWorkspace&) = delete;
  DotWorkspace& operator=(const DotWorkspace&) = delete;
};

// Launches the dot; result lands in ws.host[slot] after a stream sync.
void dot_async(const double* x, const double* y, long long n, DotWorkspace& ws, int slot,
               cudaStream_t s);
// x . y into the device scalar *out (same fixed-order reduction), no sync.
void dot_to(const double* x, const double* y, long long n, DotWorkspace& ws, double* out,
            cudaStream_t s);
// CG updates with alpha = *num / *den, beta = *num / *den read on the device.
void cg_update_xr_dev(double* x, double* r, const double* p, const double* ap, const double* num,
                      const double* den, long long n, cudaStream_t s);
void cg_update_p_dev(double* p, const double* z, const double* num, const double* den, long long n,
                     cudaStream_t s);
// Synchronous convenience: returns x . y.
double dot(const double* x, const double* y, long long n, DotWorkspace& ws, cudaStream_t s);

// x . y over the entries with mask[i] != 0 (all when mask is null), same
// fixed-order reduction; the result stays on the device (slot < 8).
double* dot_masked_device(const double* x, const double* y, const uint8_t* mask, long long n,
                          DotWorkspace& ws, int slot, cudaStream_t s);

void vcopy(double* y, const double* x, long long n, cudaStream_t s);
void vzero(double* y, long long n, cudaStream_t s);
// y = b - y
void vsub_from(double* y, const double* b, long long n, cudaStream_t s);
// y[i] = 0 where mask[i]
void vmask_zero(double* y, const uint8_t* mask, long long n, cudaStream_t s);
// y[i] = src[i] where mask[i]
void vmask_copy(double* y, const double* src, const uint8_t* mask, long long n, cudaStream_t s);
// y[i] = v where mask[i]
void vmask_fill(double* y, double v, const uint8_t* mask, long long n, cudaStream_t s);
// y += x
void vadd(double* y, const double* x, long long n, cudaStream_t s);
// w = x + a y
void vwaxpy(double* w, const double* x, double a, const double* y, long long n, cudaStream_t s);
// y = -x
void vneg(double* y, const double* x, long long n, cudaStream_t s);
// y = a * x
void vscale_mul(double* y, const double* a, const double* x, long long n, cudaStream_t s);
// y[i] = 1 / d[i]; returns false (after sync) if any d[i] == 0.
bool vreciprocal(double* y, const double* d, long long n, cudaStream_t s);
// CG: x += alpha p; r -= alpha ap  (cg.hpp:110-113)
void cg_update_xr(double* x, double* r, const double* p, const double* ap, double alpha,
                  long long n, cudaStream_t s);
// CG: p = z + beta p  (cg.hpp:128)
void cg_update_p(double* p, const double* z, double beta, long long n, cudaStream_t s);
// Chebyshev first step: r = b - r; d = inv_diag * r / theta; x += d
void cheb_first(double* x, double* r, double* d, const double* b, const double* inv_diag,
                double theta, long long n, cudaStream_t s);
// Chebyshev step: r = b - r; d = c1 d + c2 inv_diag r; x += d  (smoother.hpp:55-59)
void cheb_step(double* x, double* r, double* d, const double* b, const double* inv_diag, double c1,
               double c2, long long n, cudaStream_t s);
// Chebyshev first step with x == 0 on entry (A x = 0 skipped):
// d = inv_diag * b / theta; x = d
void cheb_first_zero(double* x, double* d, const double* b, const double* inv_diag, double theta,
                     long long n, cudaStream_t s);

}  // namespace hxg
