// Fused brick Jacobian apply: y = E^T B^T D B E x (operator.hpp:184-215) in
// one pass over the quadrature state, deterministic and atomic-free.
//
// One CTA per brick of BX x BY x BZ elements (the QLayout brick), one thread
// per quadrature column (element, qx, qy):
//   1. the brick's node block of x is loaded once (coalesced rows, masked
//      entries zeroed: operator.hpp:189-193) into shared memory;
//   2. per element: sum-factorised gradient (basis.hpp:319-335), Neo-Hookean
//      Jacobian q-function on the streamed 17-scalar state
//      (material.hpp:179-194), transpose (basis.hpp:339-355);
//   3. element outputs are summed per node inside the brick in a fixed
//      element order (scatter_add, mesh.hpp:105-116);
//   4. nodes interior to the brick are final and stored to y (constrained
//      entries pass x through, operator.hpp:212-214); nodes on brick
//      boundary planes store their partial sum to a per-brick buffer;
//   5. a light second kernel sums the boundary partials of the (<= 8)
//      bricks sharing each such node in increasing brick order.
// Both steps use fixed summation orders, so y is bitwise reproducible.
#include "fused_apply.cuh"

#include "apply_kernels.cuh"
#include "dispatch.hpp"
#include "operator.hpp"

namespace hxg {

namespace {

struct FusedParams {
  BoxDev box;
  QLayout lay;
  const double* x;
  double* y;
  const uint8_t* mask;
  const double* tab;
  const double* state;
  double mu, lambda, perturb;
  double* partial;
};

template <int P, int Q>
struct FDims : Dims<P, Q> {
  using D = Dims<P, Q>;
  static constexpr int NBX = P * D::BX + 1, NBY = P * D::BY + 1, NBZ = P * D::BZ + 1;
  static constexpr int NB = NBX * NBY * NBZ;  // nodes per (full) brick block
  static constexpr int EO = 3 * D::N3;        // element outputs [c][k][j][i]
  static constexpr int ELEM = EO + 2 * D::Q3; // per-element shared scratch
  // Separable overlap-add buffers (x pass, y pass).
  static constexpr int AXN = D::BZ * D::BY * 3 * D::N * D::N * NBX;
  static constexpr int AYN = D::BZ * 3 * D::N * NBY * NBX;
  static constexpr int SMEM = D::TAB + NB * 3 + D::NE * ELEM + AXN + AYN;
};

// Minimum resident CTAs per SM requested from ptxas (register budget).
#ifndef HXG_EXPERIMENT
#define HXG_EXPERIMENT 0
#endif
#ifndef HXG_FUSED_MINB
#define HXG_FUSED_MINB 2
#endif
template <int Q>
struct MinBlocks {
  static constexpr int value = HXG_FUSED_MINB;
};

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int P, int Q>
__global__ void __launch_bounds__(Dims<P, Q>::T, MinBlocks<Q>::value)
    fused_jacobian_kernel(FusedParams prm) {
  using D = FDims<P, Q>;
  constexpr int N = D::N, N3 = D::N3, T = D::T;
  constexpr int NBX = D::NBX, NBY = D::NBY, NB = D::NB, ROW3 = 3 * NBX;
  extern __shared__ double smem[];
  double* sB = smem;
  double* sD = smem + Q * N;
  double* Xs = smem + D::TAB;  // node block [iz][iy][ix][c]
  const int tid = threadIdx.x;
  const int brick = blockIdx.x;
  const QLayout& lay = prm.lay;
  const BoxDev& box = prm.box;
  const int bx = brick % lay.nb[0], by = (brick / lay.nb[0]) % lay.nb[1],
            bz = brick / (lay.nb[0] * lay.nb[1]);
  // The brick's quadrature state is one contiguous run: start pulling it
  // into L2 now so the q-function loads below hit L2.
  const double* st_brick = prm.state + (size_t)lay.brick_points() * brick * kStateStride;
  if (tid == 0) {
    constexpr unsigned bytes = (unsigned)(sizeof(double) * Q * kStateStride * T);
    constexpr unsigned chunk = 32768;
#pragma unroll
    for (unsigned off = 0; off < bytes; off += chunk)
      prefetch_l2(reinterpret_cast<const char*>(st_brick) + off, off + chunk <= bytes ? chunk : bytes - off);
  }
  // Elements of this brick (clipped at the domain) and its node block.
  const int ecx = min(D::BX, box.cells[0] - bx * D::BX);
  const int ecy = min(D::BY, box.cells[1] - by * D::BY);
  const int ecz = min(D::BZ, box.cells[2] - bz * D::BZ);
  const int nbx = P * ecx + 1, nby = P * ecy + 1, nbz = P * ecz + 1;
  const int npx = box.npd[0], npy = box.npd[1];
  const int node0 = P * bx * D::BX + npx * (P * by * D::BY + npy * (P * bz * D::BZ));

  load_tables<P, Q>(prm.tab, smem);
  // 1. node block of x: rows of 3 * nbx contiguous doubles.
  for (int r = tid; r < NB * 3; r += T) {
    const int c3 = r % ROW3, row = r / ROW3;
    const int iy = row % NBY, iz = row / NBY;
    if (c3 < 3 * nbx && iy < nby && iz < nbz) {
      const int dof = 3 * (node0 + npx * (iy + npy * iz)) + c3;
      double v = prm.x[dof];
      if (prm.mask && prm.mask[dof]) v = 0.0;
      Xs[r] = v;
    }
  }
  __syncthreads();

  const int le = tid / D::Q2, qx = tid % Q, qy = (tid / Q) % Q;
  const int lx = le % D::BX, ly = (le / D::BX) % D::BY, lz = le / (D::BX * D::BY);
  const bool valid = lx < ecx && ly < ecy && lz < ecz;
  double* EOe = smem + D::TAB + D::NB * 3 + le * D::ELEM;
  double* S1 = EOe + D::EO;
  double* S2 = S1 + D::Q3;
  // 2. gradient straight from the node block (no per-element copy).
  const double* Xe = Xs + ((P * lz * NBY + P * ly) * NBX + P * lx) * 3;
  double g[3][3][Q];
#pragma unroll
  for (int c = 0; c < 3; ++c)
    grad_column<P, Q, NBY * NBX * 3, NBX * 3, 3>(sB, sD, Xe + c, S1, S2, qx, qy, g[c]);
  __syncthreads();

  // 3. q-function on the streamed state.
  const double* sp0 = st_brick + tid;
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double H[9];
    if (valid) {
      double st[kStateStride];
      const double* sp = sp0 + qz * T * kStateStride;
#pragma unroll
      for (int s = 0; s < kStateStride; ++s) {
#if HXG_EXPERIMENT == 1
        st[s] = 1.0 + 0.01 * s + 1e-3 * tid;  // compute-only timing experiment
#else
        st[s] = __ldcs(sp + s * T);
#endif
      }
      double G[9];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) G[3 * c + d] = g[c][d][qz];
      jacobian_qf(prm.mu, prm.lambda, G, st, H);
      if (prm.perturb != 0.0) {
#pragma unroll
        for (int k = 0; k < 9; ++k) H[k] += prm.perturb * st[0] * G[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < 9; ++k) H[k] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d) g[c][d][qz] = H[3 * c + d];
  }

  // 4. transpose into per-element outputs [c][k][j][i].
  // Padding elements of a clipped brick contribute exact zeros.
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double* Oc = EOe + c * N3;
    grad_transpose_column<P, Q>(sB, sD, S1, S2, qx, qy, g[c], [&](int k, int j, int i, double v) {
      Oc[(k * N + j) * N + i] = valid ? v : 0.0;
    });
  }

  // 5. Overlap-add of the element patches onto the brick's node block,
  // separably x, then y, then z.  A shared node takes (lower element +
  // upper element) in each direction: a fixed order, so the sums are
  // bitwise reproducible.
  constexpr int BX = D::BX, BY = D::BY, BZ = D::BZ;
  double* AX = smem + D::TAB + D::NB * 3 + D::NE * D::ELEM;  // [lz][ly][c][k][j][ix]
  double* AY = AX + D::AXN;                                   // [lz][c][k][iy][ix]
  const double* Ebase = smem + D::TAB + D::NB * 3;
  constexpr int NAX = BZ * BY * 3 * N * N * NBX;
#pragma unroll 1
  for (int r = tid; r < NAX; r += T) {
    const int ix = r % NBX, rest = r / NBX;  // rest = ((lz*BY + ly)*3 + c)*N*N + k*N + j
    const int kj = rest % (N * N), lzlyc = rest / (N * N);
    const int c = lzlyc % 3, lzly = lzlyc / 3;
    const int lxh = ix / P < BX ? ix / P : BX - 1;
    const int i = ix - P * lxh;
    const double* e = Ebase + (lzly * BX + lxh) * D::ELEM + c * N3 + kj * N;
    double v = e[i];
    if (i == 0 && lxh > 0) v = e[P - D::ELEM] + v;
    AX[r] = v;
  }
  __syncthreads();
  constexpr int NAY = BZ * 3 * N * NBY * NBX;
#pragma unroll 1
  for (int r = tid; r < NAY; r += T) {
    const int ix = r % NBX, rest = r / NBX;  // rest = ((lz*3 + c)*N + k)*NBY + iy
    const int iy = rest % NBY, lzck = rest / NBY;
    const int k = lzck % N, lzc = lzck / N;
    const int c = lzc % 3, lz = lzc / 3;
    const int lyh = iy / P < BY ? iy / P : BY - 1;
    const int j = iy - P * lyh;
    // AX index: ((((lz*BY + ly)*3 + c)*N + k)*N + j)*NBX + ix
    const double* a = AX + ((((lz * BY + lyh) * 3 + c) * N + k) * N + j) * NBX + ix;
    double v = a[0];
    if (j == 0 && lyh > 0) v = a[(P - 3 * N * N) * NBX] + v;  // ly - 1, j = P
    AY[r] = v;
  }
  __syncthreads();
  // z, fused with the stores: node block in [iz][iy][ix][c] order.
  double* part = prm.partial + (size_t)brick * (D::NB * 3);
#pragma unroll 1
  for (int r = tid; r < NB * 3; r += T) {
    const int c3 = r % ROW3, row = r / ROW3;
    const int iy = row % NBY, iz = row / NBY;
    const int ix = c3 / 3, c = c3 - 3 * ix;
    if (!(ix < nbx && iy < nby && iz < nbz)) continue;
    const int lzh = iz / P < BZ ? iz / P : BZ - 1;
    const int k = iz - P * lzh;
    // AY index: (((lz*3 + c)*N + k)*NBY + iy)*NBX + ix
    const double* a = AY + (((lzh * 3 + c) * N + k) * NBY + iy) * NBX + ix;
    double s = a[0];
    if (k == 0 && lzh > 0) s = a[(P - 3 * N) * NBY * NBX] + s;  // lz - 1, k = P
    const bool boundary = ix == 0 || iy == 0 || iz == 0 || ix == nbx - 1 || iy == nby - 1 || iz == nbz - 1;
    if (boundary) {
      __stcg(part + r, s);
    } else {
      const int dof = 3 * (node0 + npx * (iy + npy * iz)) + c3;
      if (prm.mask && prm.mask[dof]) s = prm.x[dof];
      prm.y[dof] = s;
    }
  }
}

// Sums brick-boundary partials: nodes on planes g_d = k P B_d (or the domain's
// far face) in increasing brick order.
template <int P, int Q>
__global__ void fused_fixup_kernel(FusedParams prm) {
  using D = FDims<P, Q>;
  constexpr int PB[3] = {P * D::BX, P * D::BY, P * D::BZ};
  const BoxDev& box = prm.box;
  const QLayout& lay = prm.lay;
  long long nn = box.num_nodes();
  for (long long node = blockIdx.x * (long long)blockDim.x + threadIdx.x; node < nn;
       node += (long long)gridDim.x * blockDim.x) {
    int g[3] = {(int)(node % box.npd[0]), (int)((node / box.npd[0]) % box.npd[1]),
                (int)(node / ((long long)box.npd[0] * box.npd[1]))};
    bool on = false;
#pragma unroll
    for (int d = 0; d < 3; ++d) on = on || g[d] % PB[d] == 0 || g[d] == box.npd[d] - 1;
    if (!on) continue;
    int lo[3], hi[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      int b = g[d] / PB[d];
      if (g[d] % PB[d] == 0) {
        lo[d] = b > 0 ? b - 1 : 0;
        hi[d] = b < lay.nb[d] ? b : lay.nb[d] - 1;
      } else {
        lo[d] = hi[d] = b;
      }
    }
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int b2 = lo[2]; b2 <= hi[2]; ++b2)
      for (int b1 = lo[1]; b1 <= hi[1]; ++b1)
        for (int b0 = lo[0]; b0 <= hi[0]; ++b0) {
          long long brick = b0 + lay.nb[0] * (b1 + (long long)lay.nb[1] * b2);
          int ix = g[0] - PB[0] * b0, iy = g[1] - PB[1] * b1, iz = g[2] - PB[2] * b2;
          const double* p = prm.partial + brick * (long long)(D::NB * 3) +
                            ((iz * D::NBY + iy) * D::NBX + ix) * 3;
          s0 += __ldcg(p);
          s1 += __ldcg(p + 1);
          s2 += __ldcg(p + 2);
        }
    double s[3] = {s0, s1, s2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      long long dof = 3 * node + c;
      double v = s[c];
      if (prm.mask && prm.mask[dof]) v = prm.x[dof];
      prm.y[dof] = v;
    }
  }
}

}  // namespace

bool fused_supported(int p, int q) {
  bool ok = false;
  try {
    dispatch_pq(p, q, [&](auto, auto) { ok = true; });
  } catch (...) {
    ok = false;
  }
  return ok;
}

int fused_launches(int, int) { return 2; }

void fused_jacobian(Operator& op, const double* du, double* y) {
  FusedParams prm{};
  prm.box = op.box_;
  prm.lay = op.lay_;
  prm.x = du;
  prm.y = y;
  prm.mask = op.mask();
  prm.tab = op.tab_.p;
  prm.state = op.state_->data.p;
  prm.mu = op.mu_;
  prm.lambda = op.lambda_;
  prm.perturb = op.perturb_;
  dispatch_pq(op.p_, op.q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    using D = FDims<P, Q>;
    size_t need = (size_t)op.lay_.num_bricks() * D::NB * 3;
    if (op.partial_.n != need) op.partial_.alloc(need);
    prm.partial = op.partial_.p;
    size_t smem = sizeof(double) * D::SMEM;
    auto k = fused_jacobian_kernel<P, Q>;
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)op.lay_.num_bricks(), D::T, smem, op.stream_>>>(prm);
    HXG_CUDA(cudaGetLastError());
    fused_fixup_kernel<P, Q><<<grid_for(op.box_.num_nodes(), 256), 256, 0, op.stream_>>>(prm);
    HXG_CUDA(cudaGetLastError());
  });
}

}  // namespace hxg
