// Fused brick Jacobian apply: y = E^T B^T D B E x (operator.hpp:184-215) in
// one pass over the quadrature state, deterministic and atomic-free.
//
// One CTA per brick of BX x BY x BZ elements (the QLayout brick), one thread
// per quadrature column (element, qx, qy):
//   1. the brick's node block of x is loaded once (coalesced rows; masked
//      entries zeroed, operator.hpp:189-193) into shared memory, one plane
//      per component;
//   2. per element, all three components per phase: sum-factorised gradient
//      (basis.hpp:319-335) with every contraction reading its operand rows
//      from registers, Neo-Hookean Jacobian q-function on the streamed
//      17-scalar state (material.hpp:179-194), exact transpose
//      (basis.hpp:339-355);
//   3. the element patches are overlap-added onto the brick's node block,
//      separably in x, y, z, in a fixed order (scatter_add, mesh.hpp:105-116);
//   4. nodes interior to the brick are final and stored to y (constrained
//      entries pass x through, operator.hpp:212-214); nodes on brick
//      boundary planes store their partial sum to a per-brick buffer;
//   5. a light second kernel sums the boundary partials of the (<= 8)
//      bricks sharing each such node in increasing brick order.
// Every sum has a fixed order, so y is bitwise reproducible run to run.
#include "fused_apply.cuh"

#include "apply_kernels.cuh"
#include "dispatch.hpp"
#include "operator.hpp"

#ifndef HXG_EXPERIMENT
#define HXG_EXPERIMENT 0
#endif
#ifndef HXG_FUSED_MINB
#define HXG_FUSED_MINB 2
#endif

namespace hxg {

namespace {

struct FusedParams {
  BoxDev box;
  QLayout lay;
  const double* x;
  double* y;
  const uint8_t* mask;
  const double* tab;  // B (Q x N) then Dc (Q x Q)
  const double* state;
  double mu, lambda, perturb;
  double* partial;
  int brick0;  // first brick of this launch (pipelined host path)
  int gz0;     // first node plane of this fix-up launch
  // Uniform copies of the 1D tables for the z-direction contractions
  // (constant-bank operands).
  double B[kMaxQ * (kMaxP + 1)];
  double Dc[kMaxQ * kMaxQ];
};

template <int P, int Q>
struct FDims : Dims<P, Q> {
  using D = Dims<P, Q>;
  static constexpr int N = P + 1;
  static constexpr int NBX = P * D::BX + 1, NBY = P * D::BY + 1, NBZ = P * D::BZ + 1;
  static constexpr int NB = NBX * NBY * NBZ;  // nodes per (full) brick block
  static constexpr int A = 3 * D::Q3;         // per-element slab A / B (3 components)
  static constexpr int EO = 3 * D::N3;        // element outputs [c][k][j][i]
  // Element stride == Q^2 (mod 16 doubles): a thread's slab address is then
  // == its thread index (mod 16) for the column-contiguous accesses, so every
  // half-warp hits 16 distinct bank pairs (conflict-free 64-bit accesses).
  static constexpr int ELEM0 = 2 * A + EO;
  static constexpr int ELEM = ELEM0 + (((D::Q2 - ELEM0) % 16) + 16) % 16;
  // Overlap-add rows (NBX doubles each) packed into the elements' A/B
  // slabs, which are free by then: RPS rows per slab.
  static constexpr int RX = D::BZ * D::BY * 3 * N * N;  // x-pass rows [lz][ly][c][k][j]
  static constexpr int RY = D::BZ * 3 * N * NBY;        // y-pass rows [lz][c][k][iy]
  static constexpr int RPS = 2 * A / NBX;
  static_assert(RX + RY <= D::NE * RPS, "overlap-add rows must fit the element slabs");
  static constexpr int SMEM = D::TAB + 3 * NB + D::NE * ELEM;
  // Register cap for two resident CTAs per SM.
  static constexpr int REGS0 = 65536 / (HXG_FUSED_MINB * ((D::T + 31) / 32 * 32)) / 8 * 8 - 8;
  static constexpr int REGS = REGS0 > 255 ? 255 : REGS0;
};

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// L2 eviction policies: the quadrature state is streamed once per apply
// (evict first, no L1 allocation); the brick-boundary partials are re-read
// by the fix-up kernel right after (keep them in L2).
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_stream(const double* a, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_keep(double* a, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_once(const double* a, unsigned long long pol) {
  double v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v)
               : "l"(a), "l"(pol));
  return v;
}

template <int P, int Q>
__global__ void __launch_bounds__(Dims<P, Q>::T, HXG_FUSED_MINB)
    fused_jacobian_kernel(const __grid_constant__ FusedParams prm) {
  using D = FDims<P, Q>;
  constexpr int N = D::N, N3 = D::N3, Q3 = D::Q3, T = D::T;
  constexpr int NBX = D::NBX, NBY = D::NBY, NB = D::NB;
  constexpr int BX = D::BX, BY = D::BY, BZ = D::BZ;
  extern __shared__ double smem[];
  const double* sB = smem;          // Q x N
  const double* sD = smem + Q * N;  // Q x Q
  double* Xs = smem + D::TAB;       // node block [c][iz][iy][ix]
  double* Ebase = Xs + 3 * NB;      // per-element slabs
  const int tid = threadIdx.x;
  const int brick = blockIdx.x + prm.brick0;
  const QLayout& lay = prm.lay;
  const BoxDev& box = prm.box;
  const int bx = brick % lay.nb[0], by = (brick / lay.nb[0]) % lay.nb[1],
            bz = brick / (lay.nb[0] * lay.nb[1]);
  // The brick's quadrature state is one contiguous run: start pulling it
  // into L2 now so the q-function loads below hit L2.
  const double* st_brick = prm.state + (size_t)lay.brick_points() * brick * kStateStride;
#if HXG_EXPERIMENT != 1
  if (tid == 0) {
    constexpr unsigned bytes = (unsigned)(sizeof(double) * Q * kStateStride * T);
    constexpr unsigned chunk = 32768;
#pragma unroll
    for (unsigned off = 0; off < bytes; off += chunk)
      prefetch_l2(reinterpret_cast<const char*>(st_brick) + off,
                  off + chunk <= bytes ? chunk : bytes - off);
  }
#endif
  const int ecx = min(BX, box.cells[0] - bx * BX);
  const int ecy = min(BY, box.cells[1] - by * BY);
  const int ecz = min(BZ, box.cells[2] - bz * BZ);
  const int nbx = P * ecx + 1, nby = P * ecy + 1, nbz = P * ecz + 1;
  const int npx = box.npd[0], npy = box.npd[1];
  const int node0 = P * bx * BX + npx * (P * by * BY + npy * (P * bz * BZ));

  load_tables<P, Q>(prm.tab, smem);
  // 1. node block of x: global rows of 3 nbx contiguous doubles, stored one
  // plane per component.
  constexpr int ROW3 = 3 * NBX;
  for (int r = tid; r < NB * 3; r += T) {
    const int c3 = r % ROW3, row = r / ROW3;
    const int iy = row % NBY, iz = row / NBY;
    const int ix = c3 / 3, c = c3 - 3 * ix;
    if (ix < nbx && iy < nby && iz < nbz) {
      const int dof = 3 * (node0 + npx * (iy + npy * iz)) + c3;
      double v = prm.x[dof];
      if (prm.mask && prm.mask[dof]) v = 0.0;
      Xs[c * NB + (iz * NBY + iy) * NBX + ix] = v;
    }
  }
  const int le = tid / D::Q2, qx = tid % Q, qy = (tid / Q) % Q;
  const int lx = le % BX, ly = (le / BX) % BY, lz = le / (BX * BY);
  const bool valid = lx < ecx && ly < ecy && lz < ecz;
  double* SA = Ebase + le * D::ELEM;  // 3 Q^3
  double* SB = SA + D::A;             // 3 Q^3
  double* EOe = SB + D::A;            // 3 N^3
  __syncthreads();

  // ---- forward: G = (D (x) B (x) B, ...) U, all components per phase ----
  // F1: x-contraction T1[c][k][j][a] = sum_i B[a][i] U[c][k][j][i] (slab A).
  if (qy < N) {
    double bx_[N];
#pragma unroll
    for (int i = 0; i < N; ++i) bx_[i] = sB[qx * N + i];
    const double* Xe = Xs + ((P * lz * NBY + P * ly + qy) * NBX + P * lx);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) s += bx_[i] * Xe[c * NB + k * NBY * NBX + i];
        SA[((c * N + k) * N + qy) * Q + qx] = s;
      }
  }
  __syncthreads();
  // F2: y then z in registers; values V[c][qz][b][a] -> slab B; z-derivative.
  double g[3][3][Q];
  {
    double by_[N];
#pragma unroll
    for (int j = 0; j < N; ++j) by_[j] = sB[qy * N + j];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double t2[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) s += by_[j] * SA[((c * N + k) * N + j) * Q + qx];
        t2[k] = s;
      }
      double v[Q];
#pragma unroll
      for (int z = 0; z < Q; ++z) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) s += prm.B[z * N + k] * t2[k];
        v[z] = s;
        SB[((c * Q + z) * Q + qy) * Q + qx] = s;
      }
#pragma unroll
      for (int z = 0; z < Q; ++z) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < Q; ++r) s += prm.Dc[z * Q + r] * v[r];
        g[c][2][z] = s;
      }
    }
  }
  __syncthreads();
  // F3: x and y collocated derivatives from slab B.
  {
    double dx_[Q], dy_[Q];
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      dx_[r] = sD[qx * Q + r];
      dy_[r] = sD[qy * Q + r];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int z = 0; z < Q; ++z) {
        double sx = 0.0, sy = 0.0;
#pragma unroll
        for (int r = 0; r < Q; ++r) {
          sx += dx_[r] * SB[((c * Q + z) * Q + qy) * Q + r];
          sy += dy_[r] * SB[((c * Q + z) * Q + r) * Q + qx];
        }
        g[c][0][z] = sx;
        g[c][1][z] = sy;
      }
  }

  // ---- q-function on the streamed state --------------------------------
  const double* sp0 = st_brick + tid;
  const unsigned long long pol_stream = policy_evict_first();
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double H[9];
    if (valid) {
      double st[kStateStride];
      const double* sp = sp0 + qz * T * kStateStride;
#pragma unroll
      for (int s = 0; s < kStateStride; ++s) {
#if HXG_EXPERIMENT == 1
        st[s] = 1.0 + 0.01 * s + 1e-3 * tid + 0.0 * sp[0];
#else
        st[s] = ld_stream(sp + s * T, pol_stream);
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
  __syncthreads();  // slabs A/B free

  // ---- backward: exact adjoint ------------------------------------------
  // B1: Hx -> A, Hy -> B.
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int z = 0; z < Q; ++z) {
      SA[((c * Q + z) * Q + qy) * Q + qx] = g[c][0][z];
      SB[((c * Q + z) * Q + qy) * Q + qx] = g[c][1][z];
    }
  __syncthreads();
  // B2: acc = Dx^T Hx + Dy^T Hy + Dz^T Hz (reference order), then z interp^T.
  double w[3][N];
  {
    double dxt[Q], dyt[Q];
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      dxt[r] = sD[r * Q + qx];
      dyt[r] = sD[r * Q + qy];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double acc[Q];
#pragma unroll
      for (int z = 0; z < Q; ++z) {
        double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
        for (int r = 0; r < Q; ++r) {
          sx += dxt[r] * SA[((c * Q + z) * Q + qy) * Q + r];
          sy += dyt[r] * SB[((c * Q + z) * Q + r) * Q + qx];
          sz += prm.Dc[r * Q + z] * g[c][2][r];
        }
        acc[z] = (sx + sy) + sz;
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
#pragma unroll
        for (int z = 0; z < Q; ++z) s += prm.B[z * N + k] * acc[z];
        w[c][k] = s;
      }
    }
  }
  __syncthreads();
  // B3: W[c][k][b][a] -> A.
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int k = 0; k < N; ++k) SA[((c * N + k) * Q + qy) * Q + qx] = w[c][k];
  __syncthreads();
  // B4: y interp^T: T[c][k][j][a] = sum_b B[b][j] W[c][k][b][a] -> B.
  if (qy < N) {
    double bcy[Q];
#pragma unroll
    for (int b = 0; b < Q; ++b) bcy[b] = sB[b * N + qy];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < Q; ++b) s += bcy[b] * SA[((c * N + k) * Q + b) * Q + qx];
        SB[((c * N + k) * N + qy) * Q + qx] = s;
      }
  }
  __syncthreads();
  // B5: x interp^T: EO[c][k][j][i] = sum_a B[a][i] T[c][k][j][a].
  if (qx < N && qy < N) {
    double bcx[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) bcx[a] = sB[a * N + qx];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < Q; ++a) s += bcx[a] * SB[((c * N + k) * N + qy) * Q + a];
        EOe[(c * N + k) * N * N + qy * N + qx] = valid ? s : 0.0;  // padding elements add 0
      }
  }
  __syncthreads();

  // ---- overlap-add onto the node block: x, then y, then z ---------------
  // A shared node takes (lower element + upper element) in each direction.
  // AX [lz][ly][c][k][j][ix] and AY [lz][c][k][iy][ix] live in the elements'
  // A/B slabs (free now; the EO regions they read from stay untouched):
  // slab index r -> element r / 2A, offset r % 2A.
  auto rowp = [&](int r) { return Ebase + (r / D::RPS) * D::ELEM + (r % D::RPS) * NBX; };
  // x pass: one thread per (lz, ly, c, k, j) row of NBX nodes.
  constexpr int RX = D::RX;
  for (int row = tid; row < RX; row += T) {
    const int kj = row % (N * N), lzlyc = row / (N * N);
    const int c = lzlyc % 3, lzly = lzlyc / 3;
    const double* e = Ebase + lzly * BX * D::ELEM + 2 * D::A + c * N3 + kj * N;
    double* out = rowp(row);
#pragma unroll
    for (int ix = 0; ix < NBX; ++ix) {
      const int lxh = ix / P < BX ? ix / P : BX - 1;
      const int i = ix - P * lxh;
      double v = e[lxh * D::ELEM + i];
      if (i == 0 && lxh > 0) v = e[(lxh - 1) * D::ELEM + P] + v;
      out[ix] = v;
    }
  }
  __syncthreads();
  // y pass: one thread per (lz, c, k, iy) row.
  constexpr int RY = D::RY;
  for (int row = tid; row < RY; row += T) {
    const int iy = row % NBY, lzck = row / NBY;
    const int k = lzck % N, lzc = lzck / N;
    const int c = lzc % 3, lz = lzc / 3;
    const int lyh = iy / P < BY ? iy / P : BY - 1;
    const int j = iy - P * lyh;
    const int ra = (((lz * BY + lyh) * 3 + c) * N + k) * N + j;
    const double* a = rowp(ra);
    const bool two = j == 0 && lyh > 0;
    const double* b = rowp(ra + P - 3 * N * N);  // ly - 1, j = P
    double* out = rowp(RX + row);
#pragma unroll
    for (int ix = 0; ix < NBX; ++ix) out[ix] = two ? b[ix] + a[ix] : a[ix];
  }
  __syncthreads();
  // z pass fused with the stores: consecutive threads walk the global node
  // rows (3 nbx interleaved doubles, contiguous) for coalesced stores.
  double* part = prm.partial + (size_t)brick * (D::NB * 3);
  const unsigned long long pol_keep = policy_evict_last();
  for (int w = tid; w < NB * 3; w += T) {
    const int c3 = w % ROW3, row = w / ROW3;
    const int iy = row % NBY, iz = row / NBY;
    const int ix = c3 / 3, c = c3 - 3 * ix;
    if (ix >= nbx || iy >= nby || iz >= nbz) continue;
    const int lzh = iz / P < BZ ? iz / P : BZ - 1;
    const int k = iz - P * lzh;
    const int ra = RX + ((lzh * 3 + c) * N + k) * NBY + iy;
    double s = rowp(ra)[ix];
    if (k == 0 && lzh > 0) s = rowp(ra + (P - 3 * N) * NBY)[ix] + s;  // lz - 1, k = P
    if (ix == 0 || iy == 0 || iz == 0 || ix == nbx - 1 || iy == nby - 1 || iz == nbz - 1) {
      st_keep(part + w, s, pol_keep);
    } else {
      const int dof = 3 * (node0 + npx * (iy + npy * iz)) + c3;
      prm.y[dof] = (prm.mask && prm.mask[dof]) ? prm.x[dof] : s;
    }
  }
}

// Sums brick-boundary partials: nodes on planes g_d = k P B_d (or the domain's
// far face) in increasing brick order.
// One warp per (gy, gz) node row (blockDim = 32 x 4, grid = (ceil(npy/4), npz)).
// Rows on a y or z brick plane are boundary along their whole length; other
// rows only at the x brick planes.
template <int P, int Q>
__global__ void fused_fixup_kernel(const __grid_constant__ FusedParams prm) {
  using D = FDims<P, Q>;
  constexpr int PB0 = P * D::BX, PB1 = P * D::BY, PB2 = P * D::BZ;
  const BoxDev& box = prm.box;
  const QLayout& lay = prm.lay;
  const int gy = blockIdx.x * blockDim.y + threadIdx.y, gz = blockIdx.y + prm.gz0;
  const int npx = box.npd[0], npy = box.npd[1];
  if (gy >= npy) return;
  const bool yb = gy % PB1 == 0 || gy == npy - 1;
  const bool zb = gz % PB2 == 0 || gz == box.npd[2] - 1;
  const bool full = yb || zb;
  // y / z brick ranges of this row.
  const int b1 = gy / PB1, b2 = gz / PB2;
  const int lo1 = (gy % PB1 == 0 && b1 > 0) ? b1 - 1 : b1, hi1 = min(b1, lay.nb[1] - 1);
  const int lo2 = (gz % PB2 == 0 && b2 > 0) ? b2 - 1 : b2, hi2 = min(b2, lay.nb[2] - 1);
  const unsigned long long pol = policy_evict_first();
  const int nx_planes = (npx - 1 + PB0 - 1) / PB0 + 1;  // x brick planes incl. far face
  const int count = full ? npx : nx_planes;
  for (int t = threadIdx.x; t < count; t += 32) {
    const int gx = full ? t : min(t * PB0, npx - 1);
    const int b0 = gx / PB0;
    const int lo0 = (gx % PB0 == 0 && b0 > 0) ? b0 - 1 : b0, hi0 = min(b0, lay.nb[0] - 1);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int c2 = lo2; c2 <= hi2; ++c2)
      for (int c1 = lo1; c1 <= hi1; ++c1)
        for (int c0 = lo0; c0 <= hi0; ++c0) {
          const size_t brick = c0 + (size_t)lay.nb[0] * (c1 + (size_t)lay.nb[1] * c2);
          const int ix = gx - PB0 * c0, iy = gy - PB1 * c1, iz = gz - PB2 * c2;
          const double* p =
              prm.partial + brick * (D::NB * 3) + ((iz * D::NBY + iy) * D::NBX + ix) * 3;
          s0 += ld_once(p, pol);
          s1 += ld_once(p + 1, pol);
          s2 += ld_once(p + 2, pol);
        }
    const size_t dof0 = 3 * ((size_t)gx + (size_t)npx * (gy + (size_t)npy * gz));
    const double s[3] = {s0, s1, s2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double v = s[c];
      if (prm.mask && prm.mask[dof0 + c]) v = prm.x[dof0 + c];
      prm.y[dof0 + c] = v;
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
  for (size_t i = 0; i < op.interp_.size(); ++i) prm.B[i] = op.interp_[i];
  for (size_t i = 0; i < op.colloc_.size(); ++i) prm.Dc[i] = op.colloc_[i];
  dispatch_pq(op.p_, op.q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    using D = FDims<P, Q>;
    size_t need = (size_t)op.lay_.num_bricks() * D::NB * 3;
    if (op.partial_.n != need) op.partial_.alloc(need);
    prm.partial = op.partial_.p;
    size_t smem = sizeof(double) * D::SMEM;
    auto k = fused_jacobian_kernel<P, Q>;
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
    k<<<(unsigned)op.lay_.num_bricks(), D::T, smem, op.stream_>>>(prm);
    HXG_CUDA(cudaGetLastError());
    dim3 fb(32, 4), fg((op.box_.npd[1] + 3) / 4, op.box_.npd[2]);
    fused_fixup_kernel<P, Q><<<fg, fb, 0, op.stream_>>>(prm);
    HXG_CUDA(cudaGetLastError());
  });
}

// Host buffers: the box is cut into C chunks of brick layers along z.  Chunk
// i's x planes go up on the H2D stream; its bricks and the fix-up of the node
// planes it finalises run on the compute stream once those planes have
// landed; its finished y planes go down on the D2H stream.  The three
// engines overlap, so the copies hide the apply (and vice versa).
void fused_jacobian_host(Operator& op, const double* xh, double* yh) {
  if (!op.pipe_) op.pipe_ = std::make_unique<HostPipe>();
  HostPipe& pp = *op.pipe_;
  const size_t n = (size_t)op.size();
  if (pp.x.n != n) {
    pp.x.alloc(n);
    pp.y.alloc(n);
  }
  FusedParams prm{};
  prm.box = op.box_;
  prm.lay = op.lay_;
  prm.x = pp.x.p;
  prm.y = pp.y.p;
  prm.mask = op.mask();
  prm.tab = op.tab_.p;
  prm.state = op.state_->data.p;
  prm.mu = op.mu_;
  prm.lambda = op.lambda_;
  prm.perturb = op.perturb_;
  for (size_t i = 0; i < op.interp_.size(); ++i) prm.B[i] = op.interp_[i];
  for (size_t i = 0; i < op.colloc_.size(); ++i) prm.Dc[i] = op.colloc_[i];
  dispatch_pq(op.p_, op.q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    using D = FDims<P, Q>;
    size_t need = (size_t)op.lay_.num_bricks() * D::NB * 3;
    if (op.partial_.n != need) op.partial_.alloc(need);
    prm.partial = op.partial_.p;
    size_t smem = sizeof(double) * D::SMEM;
    auto k = fused_jacobian_kernel<P, Q>;
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
    const int nbz = op.lay_.nb[2], layer = op.lay_.nb[0] * op.lay_.nb[1];
    const int pb2 = P * D::BZ, npz = op.box_.npd[2];
    const size_t plane = (size_t)op.box_.npd[0] * op.box_.npd[1] * 3;
    const int C = nbz < HostPipe::kMaxChunks / 2 ? nbz : HostPipe::kMaxChunks / 2;
    // Order after earlier work on the operator's stream.
    HXG_CUDA(cudaEventRecord(pp.done_evt, op.stream_));
    HXG_CUDA(cudaStreamWaitEvent(pp.h2d, pp.done_evt, 0));
    HXG_CUDA(cudaStreamWaitEvent(pp.comp, pp.done_evt, 0));
    int sent = 0;  // planes [0, sent) uploaded
    for (int i = 0; i < C; ++i) {
      const int le = (int)((long long)(i + 1) * nbz / C);
      const int upto = (pb2 * le < npz - 1 ? pb2 * le : npz - 1) + 1;
      HXG_CUDA(cudaMemcpyAsync(pp.x.p + sent * plane, xh + sent * plane,
                               (size_t)(upto - sent) * plane * sizeof(double),
                               cudaMemcpyHostToDevice, pp.h2d));
      sent = upto;
      HXG_CUDA(cudaEventRecord(pp.in_ready[i], pp.h2d));
    }
    for (int i = 0; i < C; ++i) {
      const int lb = (int)((long long)i * nbz / C), le = (int)((long long)(i + 1) * nbz / C);
      HXG_CUDA(cudaStreamWaitEvent(pp.comp, pp.in_ready[i], 0));
      FusedParams pc = prm;
      pc.brick0 = lb * layer;
      k<<<(unsigned)((le - lb) * layer), D::T, smem, pp.comp>>>(pc);
      HXG_CUDA(cudaGetLastError());
      const int zs = i == 0 ? 0 : pb2 * lb;
      const int ze = i == C - 1 ? npz : pb2 * le;
      pc.gz0 = zs;
      dim3 fb(32, 4), fg((op.box_.npd[1] + 3) / 4, ze - zs);
      fused_fixup_kernel<P, Q><<<fg, fb, 0, pp.comp>>>(pc);
      HXG_CUDA(cudaGetLastError());
      HXG_CUDA(cudaEventRecord(pp.out_ready[i], pp.comp));
      HXG_CUDA(cudaStreamWaitEvent(pp.d2h, pp.out_ready[i], 0));
      HXG_CUDA(cudaMemcpyAsync(yh + zs * plane, pp.y.p + zs * plane,
                               (size_t)(ze - zs) * plane * sizeof(double), cudaMemcpyDeviceToHost,
                               pp.d2h));
    }
    HXG_CUDA(cudaEventRecord(pp.done_evt, pp.d2h));
    HXG_CUDA(cudaStreamWaitEvent(op.stream_, pp.done_evt, 0));
    HXG_CUDA(cudaStreamSynchronize(pp.d2h));
  });
}

}  // namespace hxg
