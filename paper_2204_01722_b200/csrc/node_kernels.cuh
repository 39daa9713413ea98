// Node-centric deterministic transpose restriction (scatter_add,
// mesh.hpp:105-116): every L-vector entry sums its element contributions in
// increasing element order — the reference's sequential scatter order — so
// the two-pass path reproduces the reference summation bit for bit given the
// same element values.  No atomics.
#pragma once

#include <cuda_runtime.h>

#include "common.hpp"

namespace hxg {

enum NodeEpilogue {
  kEpiNone = 0,      // out = sum
  kEpiJacobian = 1,  // constrained: out = x (operator.hpp:212-214)
  kEpiResidual = 2,  // out = sum - s * load; constrained: 0 (operator.hpp:175-179)
  kEpiDiagonal = 3,  // constrained: 1 (operator.hpp:280-282)
  kEpiInvMult = 4    // out = sum / multiplicity (Prolongation::apply, multigrid.hpp:47-49)
};

struct NodeParams {
  BoxDev box;
  const double* evec;   // (e, c, a)
  double* out;          // L-vector
  const double* x;      // jacobian pass-through source
  const uint8_t* mask;  // may be null
  const double* load;   // residual load, may be null
  double load_scale;
  int epilogue;
  int accumulate;  // start from out[dof] (scatter_add semantics)
};

template <int P>
__global__ void node_sum_kernel(NodeParams prm) {
  constexpr int N = P + 1, N3 = N * N * N;
  const BoxDev& b = prm.box;
  long long nn = b.num_nodes();
  for (long long node = blockIdx.x * (long long)blockDim.x + threadIdx.x; node < nn;
       node += (long long)gridDim.x * blockDim.x) {
    int g[3] = {(int)(node % b.npd[0]), (int)((node / b.npd[0]) % b.npd[1]),
                (int)(node / ((long long)b.npd[0] * b.npd[1]))};
    int lo[3], hi[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      int e = g[d] / P;
      if (g[d] % P == 0) {
        lo[d] = e > 0 ? e - 1 : 0;
        hi[d] = e < b.cells[d] ? e : b.cells[d] - 1;
      } else {
        lo[d] = hi[d] = e;
      }
    }
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (prm.accumulate) {
      s0 = prm.out[3 * node];
      s1 = prm.out[3 * node + 1];
      s2 = prm.out[3 * node + 2];
    }
    int mult = 0;
    for (int ez = lo[2]; ez <= hi[2]; ++ez)
      for (int ey = lo[1]; ey <= hi[1]; ++ey)
        for (int ex = lo[0]; ex <= hi[0]; ++ex) {
          long long e = ex + b.cells[0] * (ey + (long long)b.cells[1] * ez);
          int a = (g[0] - P * ex) + N * ((g[1] - P * ey) + N * (g[2] - P * ez));
          const double* src = prm.evec + e * 3 * N3 + a;
          s0 += src[0];
          s1 += src[N3];
          s2 += src[2 * N3];
          ++mult;
        }
    double s[3] = {s0, s1, s2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      long long dof = 3 * node + c;
      double v = s[c];
      bool fixed = prm.mask && prm.mask[dof];
      switch (prm.epilogue) {
        case kEpiJacobian:
          if (fixed) v = prm.x[dof];
          break;
        case kEpiResidual:
          if (prm.load) v -= prm.load_scale * prm.load[dof];
          if (fixed) v = 0.0;
          break;
        case kEpiDiagonal:
          if (fixed) v = 1.0;
          break;
        case kEpiInvMult:
          v *= 1.0 / (double)mult;
          break;
        default:
          break;
      }
      prm.out[dof] = v;
    }
  }
}

}  // namespace hxg
