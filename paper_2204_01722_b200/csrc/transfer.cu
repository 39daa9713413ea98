// p-level transfer (Prolongation, multigrid.hpp:25-74): P = diag(1/m_f) E_f^T
// (C x C x C) E_c with C the 1D coarse-on-fine-GLL tabulation; R = P^T.
// Element kernels evaluate each output entry with the reference's
// contraction order; the node-ordered sum (node_kernels.cuh) scatters.
#include "transfer.hpp"

#include <cstdlib>

#include "dispatch.hpp"
#include "node_kernels.cuh"

namespace hxg {

namespace {

struct TransferParams {
  BoxDev fine, coarse;
  const double* ctof;  // Nf x Nc
  const double* in;    // L-vector (coarse for prolong, fine for restrict)
  double* evec;        // output E-vector (fine for prolong, coarse for restrict)
  double C[5 * 4];     // ctof by value (uniform operands)
};

__device__ __forceinline__ long long lattice_node(const BoxDev& b, long long e, int i, int j, int k) {
  long long ex = e % b.cells[0], ey = (e / b.cells[0]) % b.cells[1],
            ez = e / ((long long)b.cells[0] * b.cells[1]);
  return (b.p * ex + i) + b.npd[0] * ((b.p * ey + j) + (long long)b.npd[1] * (b.p * ez + k));
}

// Prolong: out[e][c][k][j][i] = sum_kc C[k][kc] sum_jc C[j][jc] sum_ic C[i][ic] xc[..]
template <int NF, int NC>
__global__ void prolong_element_kernel(TransferParams prm) {
  constexpr int NF3 = NF * NF * NF, NC3 = NC * NC * NC;
  long long total = prm.fine.num_elements() * 3 * NF3;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < total;
       r += (long long)gridDim.x * blockDim.x) {
    long long e = r / (3 * NF3);
    int rem = (int)(r % (3 * NF3));
    int c = rem / NF3, a = rem % NF3;
    int i = a % NF, j = (a / NF) % NF, k = a / (NF * NF);
    double xc[NC3];
#pragma unroll
    for (int kc = 0; kc < NC; ++kc)
#pragma unroll
      for (int jc = 0; jc < NC; ++jc)
#pragma unroll
        for (int ic = 0; ic < NC; ++ic)
          xc[(kc * NC + jc) * NC + ic] = prm.in[3 * lattice_node(prm.coarse, e, ic, jc, kc) + c];
    double out = 0.0;
#pragma unroll
    for (int kc = 0; kc < NC; ++kc) {
      double t2 = 0.0;
#pragma unroll
      for (int jc = 0; jc < NC; ++jc) {
        double t1 = 0.0;
#pragma unroll
        for (int ic = 0; ic < NC; ++ic) t1 += prm.ctof[i * NC + ic] * xc[(kc * NC + jc) * NC + ic];
        t2 += prm.ctof[j * NC + jc] * t1;
      }
      out += prm.ctof[k * NC + kc] * t2;
    }
    prm.evec[(e * 3 + c) * NF3 + a] = out;
  }
}

// Prolong fused with the node-ordered average: one thread per fine node.
// A node shared by k elements sits on their common faces, where the 1D
// coarse-on-fine rows are exact unit vectors (the fine and coarse GLL
// endpoints coincide, lagrange_tabulate), so every element's per-entry
// interpolation (the element kernel above, same operation sequence) is the
// same double: it is evaluated once, in the lowest containing element, and
// the node_sum_kernel(kEpiInvMult) epilogue is replayed on k copies (sum from
// 0 in element order, times 1/k) -- bitwise the element kernel + node sum
// pair (tested), without the E-vector round trip or the k-fold recompute.
template <int NF, int NC>
__global__ void __launch_bounds__(256) prolong_node_kernel(TransferParams prm) {
  constexpr int PF = NF - 1, PC = NC - 1;
  const BoxDev& f = prm.fine;
  const BoxDev& cb = prm.coarse;
  const long long nn = f.num_nodes();
  for (long long node = blockIdx.x * (long long)blockDim.x + threadIdx.x; node < nn;
       node += (long long)gridDim.x * blockDim.x) {
    const int g[3] = {(int)(node % f.npd[0]), (int)((node / f.npd[0]) % f.npd[1]),
                      (int)(node / ((long long)f.npd[0] * f.npd[1]))};
    int lo[3], mult = 1;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int e = g[d] / PF;
      const bool shared = g[d] % PF == 0;
      lo[d] = shared && e > 0 ? e - 1 : (e < f.cells[d] ? e : f.cells[d] - 1);
      if (shared && e > 0 && e < f.cells[d]) mult *= 2;
    }
    const int i = g[0] - PF * lo[0], j = g[1] - PF * lo[1], k = g[2] - PF * lo[2];
    const double* xb = prm.in + 3 * ((PC * lo[0]) + cb.npd[0] * ((long long)(PC * lo[1]) +
                                                               (long long)cb.npd[1] * (PC * lo[2])));
    const long long sy = 3LL * cb.npd[0], sz = 3LL * cb.npd[0] * cb.npd[1];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double out = 0.0;
#pragma unroll
      for (int kc = 0; kc < NC; ++kc) {
        double t2 = 0.0;
#pragma unroll
        for (int jc = 0; jc < NC; ++jc) {
          double t1 = 0.0;
#pragma unroll
          for (int ic = 0; ic < NC; ++ic)
            t1 += prm.ctof[i * NC + ic] * __ldg(xb + 3 * ic + sy * jc + sz * kc + c);
          t2 += prm.ctof[j * NC + jc] * t1;
        }
        out += prm.ctof[k * NC + kc] * t2;
      }
      double s = 0.0;
      for (int r = 0; r < mult; ++r) s += out;
      prm.evec[3 * node + c] = s * (1.0 / (double)mult);
    }
  }
}

// Restrict (exact transpose, contraction order z, y, x as apply_transpose):
// out[e][c][kc][jc][ic] = sum_if C[if][ic] sum_jf C[jf][jc] sum_kf C[kf][kc] s[..]
// with s = x_f / m_f gathered on the fine lattice.  One thread per
// (coarse element, component, kc) evaluates its NC^2 outputs with the
// z-sums t1 and y-sums t2 shared between them: every output is the same
// operation sequence as the per-entry formula (bitwise identical), with the
// NF^3 gathers and the lattice arithmetic done once.  1/m_f is the product
// of per-direction factors 1 or 1/2 (exact).
template <int NF, int NC>
__global__ void __launch_bounds__(128) restrict_element_kernel(TransferParams prm) {
  constexpr int NC3 = NC * NC * NC, PF = NF - 1;
  const BoxDev& f = prm.fine;
  const long long total = prm.coarse.num_elements() * 3 * NC;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < total;
       r += (long long)gridDim.x * blockDim.x) {
    const long long e = r / (3 * NC);
    const int rem = (int)(r - e * 3 * NC), c = rem / NC, kc = rem - c * NC;
    const int ex = (int)(e % f.cells[0]), ey = (int)((e / f.cells[0]) % f.cells[1]),
              ez = (int)(e / ((long long)f.cells[0] * f.cells[1]));
    const double* base =
        prm.in + 3 * ((PF * ex) + f.npd[0] * ((long long)(PF * ey) + (long long)f.npd[1] * (PF * ez))) + c;
    const long long sy = 3LL * f.npd[0], sz = 3LL * f.npd[0] * f.npd[1];
    auto half = [](int i, int ecell, int ncell) {
      return (i == 0 && ecell > 0) || (i == PF && ecell < ncell - 1) ? 0.5 : 1.0;
    };
    double out[NC][NC];
#pragma unroll
    for (int jc = 0; jc < NC; ++jc)
#pragma unroll
      for (int ic = 0; ic < NC; ++ic) out[jc][ic] = 0.0;
#pragma unroll
    for (int iff = 0; iff < NF; ++iff) {
      const double hx = half(iff, ex, f.cells[0]);
      double t2[NC];
#pragma unroll
      for (int jc = 0; jc < NC; ++jc) t2[jc] = 0.0;
#pragma unroll
      for (int jf = 0; jf < NF; ++jf) {
        const double hxy = hx * half(jf, ey, f.cells[1]);
        double t1 = 0.0;
#pragma unroll
        for (int kf = 0; kf < NF; ++kf) {
          const double s = base[3 * iff + sy * jf + sz * kf] * (hxy * half(kf, ez, f.cells[2]));
          t1 += prm.C[kf * NC + kc] * s;
        }
#pragma unroll
        for (int jc = 0; jc < NC; ++jc) t2[jc] += prm.C[jf * NC + jc] * t1;
      }
#pragma unroll
      for (int jc = 0; jc < NC; ++jc)
#pragma unroll
        for (int ic = 0; ic < NC; ++ic) out[jc][ic] += prm.C[iff * NC + ic] * t2[jc];
    }
    double* o = prm.evec + (e * 3 + c) * NC3 + kc * NC * NC;
#pragma unroll
    for (int jc = 0; jc < NC; ++jc)
#pragma unroll
      for (int ic = 0; ic < NC; ++ic) o[jc * NC + ic] = out[jc][ic];
  }
}

template <class F>
void dispatch_transfer(int pf, int pc, F&& f) {
  switch (pf * 10 + pc) {
    case 21: f(IC<3>{}, IC<2>{}); return;
    case 31: f(IC<4>{}, IC<2>{}); return;
    case 32: f(IC<4>{}, IC<3>{}); return;
    case 41: f(IC<5>{}, IC<2>{}); return;
    case 42: f(IC<5>{}, IC<3>{}); return;
    case 43: f(IC<5>{}, IC<4>{}); return;
    default:
      throw Error(HXG_ERR_UNSUPPORTED, "unsupported transfer orders");
  }
}

}  // namespace

Transfer::Transfer(const int cells[3], int fine_order, int coarse_order)
    : pf_(fine_order), pc_(coarse_order) {
  fine_ = make_box(cells, fine_order);
  coarse_ = make_box(cells, coarse_order);
  std::vector<double> ctof;
  lagrange_tabulate(gauss_lobatto(coarse_order), gauss_lobatto(fine_order), &ctof, nullptr);
  ctof_.upload(ctof);
  ctof_h_ = ctof;
  dispatch_transfer(pf_, pc_, [](auto, auto) {});
}

void Transfer::prolong(const double* xc, double* xf, cudaStream_t s) {
  if (!getenv("HXG_PROLONG_TWO_PASS")) {
    TransferParams prm{fine_, coarse_, ctof_.p, xc, xf, {}};
    dispatch_transfer(pf_, pc_, [&](auto NFc, auto NCc) {
      constexpr int NF = decltype(NFc)::value, NC = decltype(NCc)::value;
      prolong_node_kernel<NF, NC><<<grid_for(fine_.num_nodes(), 256), 256, 0, s>>>(prm);
    });
    HXG_CUDA(cudaGetLastError());
    return;
  }
  int nf = pf_ + 1;
  size_t need = (size_t)fine_.num_elements() * 3 * nf * nf * nf;
  if (evf_.n != need) evf_.alloc(need);
  TransferParams prm{fine_, coarse_, ctof_.p, xc, evf_.p, {}};
  dispatch_transfer(pf_, pc_, [&](auto NFc, auto NCc) {
    constexpr int NF = decltype(NFc)::value, NC = decltype(NCc)::value;
    prolong_element_kernel<NF, NC><<<grid_for((long long)need, 128), 128, 0, s>>>(prm);
  });
  HXG_CUDA(cudaGetLastError());
  NodeParams np{};
  np.box = fine_;
  np.evec = evf_.p;
  np.out = xf;
  np.epilogue = kEpiInvMult;
  dispatch_p(pf_, [&](auto Pc) {
    constexpr int P = decltype(Pc)::value;
    node_sum_kernel<P><<<grid_for(fine_.num_nodes(), 256), 256, 0, s>>>(np);
  });
  HXG_CUDA(cudaGetLastError());
}

void Transfer::restrict_to(const double* xf, double* xc, cudaStream_t s) {
  int nc = pc_ + 1;
  size_t need = (size_t)coarse_.num_elements() * 3 * nc * nc * nc;
  if (evc_.n != need) evc_.alloc(need);
  TransferParams prm{fine_, coarse_, ctof_.p, xf, evc_.p, {}};
  for (size_t i = 0; i < ctof_h_.size(); ++i) prm.C[i] = ctof_h_[i];
  dispatch_transfer(pf_, pc_, [&](auto NFc, auto NCc) {
    constexpr int NF = decltype(NFc)::value, NC = decltype(NCc)::value;
    const long long threads = (long long)coarse_.num_elements() * 3 * NC;
    restrict_element_kernel<NF, NC><<<grid_for(threads, 128), 128, 0, s>>>(prm);
  });
  HXG_CUDA(cudaGetLastError());
  NodeParams np{};
  np.box = coarse_;
  np.evec = evc_.p;
  np.out = xc;
  np.epilogue = kEpiNone;
  dispatch_p(pc_, [&](auto Pc) {
    constexpr int P = decltype(Pc)::value;
    node_sum_kernel<P><<<grid_for(coarse_.num_nodes(), 256), 256, 0, s>>>(np);
  });
  HXG_CUDA(cudaGetLastError());
}

}  // namespace hxg
