// Fused brick Jacobian apply: y = E^T B^T D B E x (operator.hpp:184-215) in
// one pass over the quadrature state, deterministic and atomic-free.
//
// One CTA per brick of BX x BY x BZ elements (the QLayout brick), one thread
// per quadrature column (element, qx, qy):
//   1. the brick's node block of x is copied once (coalesced rows, cp.async
//      one brick ahead) into shared memory, one plane per component; masked
//      entries read as zero (operator.hpp:189-193);
//   2. per element, all three components per phase: sum-factorised gradient
//      (basis.hpp:319-335) with every contraction reading its operand rows
//      from registers, Neo-Hookean Jacobian q-function on the streamed
//      17-scalar state (material.hpp:179-194), exact transpose
//      (basis.hpp:339-355);
//   3. each node of the block sums the element patches sharing it in a
//      fixed order (scatter_add, mesh.hpp:105-116);
//   4. nodes interior to the brick are final and stored to y (constrained
//      entries pass x through, operator.hpp:212-214); nodes on brick
//      boundary planes store their partial sum to a per-brick buffer;
//   5. a light second kernel, one CTA per brick, sums the boundary partials
//      of the (<= 8) bricks sharing each node the brick owns in increasing
//      brick order.
// The residual (MODE = kResidual, operator.hpp:146-180) runs the same pass
// with the residual q-function on the streamed geometry, writing the state.
// Every sum has a fixed order, so y is bitwise reproducible run to run.
#include "fused_apply.cuh"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "apply_kernels.cuh"
#include "dispatch.hpp"
#include "operator.hpp"

#ifndef HXG_EXPERIMENT
#define HXG_EXPERIMENT 0  // 4: per-phase clock64 accounting (scripts/phase_times.py)
#endif
#ifndef HXG_MINB_HIGHP
#define HXG_MINB_HIGHP 3
#endif
#ifndef HXG_MINB_Q2
#define HXG_MINB_Q2 2
#endif
#ifndef HXG_SLOTS_Q2
#define HXG_SLOTS_Q2 1
#endif
#ifndef HXG_MINB_Q4
#define HXG_MINB_Q4 3
#endif
#ifndef HXG_SLOTS_Q4
#define HXG_SLOTS_Q4 1
#endif
// Q2 (2, 3): planes of the gradients / q-function outputs kept in the
// column-private shared slots (the rest in registers).
#ifndef HXG_NSG_Q2
#define HXG_NSG_Q2 3
#endif
#ifndef HXG_NSH_Q2
#define HXG_NSH_Q2 3
#endif
#ifndef HXG_RES_BOX_GEO
#define HXG_RES_BOX_GEO 1  // residual on box meshes: geometry in registers
#endif
#ifndef HXG_HOST_CHUNKS_DEFAULT
#define HXG_HOST_CHUNKS_DEFAULT 8
#endif
constexpr int kHostChunks = HXG_HOST_CHUNKS_DEFAULT;
#ifndef HXG_PIPE_GRID_PCT_DEFAULT
#define HXG_PIPE_GRID_PCT_DEFAULT 100
#endif
constexpr int kPipeGridPct = HXG_PIPE_GRID_PCT_DEFAULT;
#ifndef HXG_SKIP_FIXUP
#define HXG_SKIP_FIXUP 0  // timing experiment only: results are wrong
#endif
#ifndef HXG_SLOTS_HIGHP
#define HXG_SLOTS_HIGHP 0
#endif

namespace hxg {

namespace {

#ifndef HXG_PIPE_Q2
#define HXG_PIPE_Q2 0
#endif
#ifndef HXG_PIPE_ALL_Q5
#define HXG_PIPE_ALL_Q5 0
#endif
#ifndef HXG_BRICK_PDL
#define HXG_BRICK_PDL 0
#endif
#ifndef HXG_FIXUP_PDL
#define HXG_FIXUP_PDL 0
#endif
// Where the bulk L2 prefetch of a brick's quadrature state is issued:
// 0 = the next brick, at the start of the current one; 1 = the current
// brick, at its start (its state is first read after the node-block wait,
// P1 and P2); 2 = the next brick, after the current P1 pass; 3 = the next
// brick, after the current q-function phase.  Measured (ab_time, B200, us
// per apply, modes 0/1/2/3): Q2 64^3 318.1/307.0/308.5/306.5, Q3 43^3
// 335.9/324.2/332.6/327.4, Q4 32^3 364.3/371.3/379.4/388.1 (no prefetch:
// 345.7/354.8/397.5).  A whole brick ahead keeps ~2 x 32 MB of state in
// flight through L2, more than one die's half holds for Q2/Q3.
#ifndef HXG_PF_MODE
#define HXG_PF_MODE -1  // -1: per (P, Q) as measured
#endif
__host__ __device__ constexpr int pf_mode(int q) {
  return HXG_PF_MODE >= 0 ? HXG_PF_MODE : (q == 5 ? 0 : 1);
}
#ifndef HXG_FIXUP_THREADS
#define HXG_FIXUP_THREADS 128
#endif
constexpr int kFixupThreads = HXG_FIXUP_THREADS;
#ifndef HXG_FIXUP_LD
#define HXG_FIXUP_LD 0  // partial loads: 0 L1 no-allocate + L2 evict-first, 1 read-only path, 2 plain
#endif
#ifndef HXG_FIXUP_MINB
#define HXG_FIXUP_MINB 8  // 64 registers: 8 CTAs per SM (Q2 64^3 apply 316.9 -> 310.4 us)
#endif
#ifndef HXG_FIXUP_MAXGRID
#define HXG_FIXUP_MAXGRID (148 * 64)
#endif
constexpr int kFixupMaxGrid = HXG_FIXUP_MAXGRID;

struct FusedParams {
  BoxDev box;
  QLayout lay;
  const double* x;
  double* y;
  const uint8_t* mask;
  const double* tab;  // B (Q x N) then Dc (Q x Q)
  const double* state;
  const double* geo;  // geometric factors (w detJ for the perturbation hook)
  double mu, lambda, perturb;
  double* partial;
  // residual mode: state written, external load, first inverted point
  double* state_out;
  const double* load;
  double load_scale;
  unsigned long long* fail;
  // residual on a box mesh: the geometric factors formed in registers (the
  // stored ones are the same products, Operator::make_box_geometry)
  int geo_box;
  double geo_g[3], geo_jac, geo_qw[kMaxQ];
  // optional brick list: launch brick i is blist[brick0 + i] (the
  // partitioned apply's interface layer / interior split)
  const int* blist;
  // fix-up node filter over the partition-interface faces iface (bits
  // -x,+x,-y,+y,-z,+z of this block): 0 all nodes, 1 only nodes on an
  // interface face, 2 all but those
  int iface, ifilter;
  int brick0;   // first brick of this launch (pipelined host path)
  int nbricks;  // bricks in this launch
  int face_bits;  // >= 0: constraints are these whole faces (analytic), -1: mask array
  // Uniform copies of the 1D tables for the z-direction contractions
  // (constant-bank operands).
  double B[kMaxQ * (kMaxP + 1)];   // interp (Q x N)
  double Bd[kMaxQ * (kMaxP + 1)];  // deriv  (Q x N)
};

// Padding tables (P * 10 + Q) from the bank-conflict search.
__host__ __device__ constexpr int elem_pad(int p, int q) {
  return p * 10 + q == 34 || p * 10 + q == 14 || p * 10 + q == 15 ? 2
         : p * 10 + q == 45 || p * 10 + q == 25 || p * 10 + q == 35 ? 0
                                                                     : 1;
}
// Element-output component padding: spreads the node-centric overlap-add
// reads (lanes over (ix, c)) across banks.
__host__ __device__ constexpr int eo_pad(int p, int q) {
  switch (p * 10 + q) {
    case 12: return 3; case 34: case 35: return 4; case 45: return 8;
    case 24: case 25: return 0;
  }
  return 1;
}
__host__ __device__ constexpr int pad_nbx(int p, int q) {
  switch (p * 10 + q) {
    case 12: return 12; case 23: return 10; case 34: return 7; case 45: return 10;
    case 13: return 12; case 14: return 6; case 24: return 6; case 15: return 4;
    case 25: return 12; case 35: return 10;
  }
  return 0;
}
__host__ __device__ constexpr int pad_nby(int p, int q) {
  switch (p * 10 + q) {
    case 12: return 5; case 23: return 9; case 34: return 7; case 45: return 9;
    case 13: return 5; case 14: return 3; case 24: return 6; case 15: return 6;
    case 25: return 5; case 35: return 10;
  }
  return 0;
}
__host__ __device__ constexpr int pad_plane(int p, int q) {
  switch (p * 10 + q) {
    case 12: return 300; case 23: return 450; case 34: return 343; case 45: return 451;
    case 13: return 180; case 14: return 54; case 24: return 181; case 15: return 50;
    case 25: return 181; case 35: return 400;
  }
  return 0;
}

// Resident CTAs per SM the register allocation targets: two for the 9-warp
// bricks; three for the 4-warp (3, 4) brick (shared memory allows it).
__host__ __device__ constexpr int fused_min_blocks(int p, int q) {
  return p * 10 + q == 34 ? HXG_MINB_HIGHP : p * 10 + q == 23 ? HXG_MINB_Q2 : p * 10 + q == 45 ? HXG_MINB_Q4 : 2;
}
// Fused residual: the residual q-function needs more registers than the
// Jacobian's.  Q2 (2, 3) fits two CTAs per SM without spills (Q2 64^3
// residual 0.667 -> 0.536 ms); the larger bricks keep one.
#ifndef HXG_RES_MINB
#define HXG_RES_MINB 0  // 0: per (P, Q) as measured
#endif
__host__ __device__ constexpr int fused_residual_min_blocks(int p, int q) {
  return HXG_RES_MINB > 0 ? HXG_RES_MINB : (p == 2 && q == 3) ? 2 : 1;
}
// Initial-storage variants (measured, Q2 64^3): Native and AD run 2 CTAs/SM
// in 113 registers (0.525 / 0.667 ms vs 0.547 / 0.770 at 1 CTA); Tuned keeps
// 1 CTA/SM (0.510 vs 0.695 ms).
__host__ __device__ constexpr int variant_min_blocks(int storage) {
  return storage == kStorageInitialTuned ? 1 : 2;
}
// Column-private shared slots for the gradients (see P2).
__host__ __device__ constexpr bool fused_slots(int p, int q) {
  return p * 10 + q == 12 || p * 10 + q == 13 || (HXG_SLOTS_Q2 && p * 10 + q == 23) ||
         (HXG_SLOTS_HIGHP && p * 10 + q == 34) || (HXG_SLOTS_Q4 && p * 10 + q == 45);
}

template <int P, int Q>
struct FDims : Dims<P, Q> {
  using D = Dims<P, Q>;
  static constexpr int N = P + 1;
  static constexpr int NBX = P * D::BX + 1, NBY = P * D::BY + 1, NBZ = P * D::BZ + 1;
  static constexpr int NB = NBX * NBY * NBZ;  // nodes per (full) brick block
  static constexpr int S = 9 * N * D::Q2;     // per-element exchange slab [c][arr][k][b][a]
  // Element outputs [c][k][j][i], component stride EOC >= N^3.
  static constexpr int EOC = D::N3 + eo_pad(P, Q);
  // Element stride and node-block strides padded (exhaustive search over the
  // half-warp access patterns of every phase) so 64-bit shared accesses are
  // (nearly) bank-conflict free; lanes are (column or plane task, element)
  // with elements fastest.  Only ELEM mod 16 matters to the slab phases.
  static constexpr int ELEM0 = S + 3 * EOC;
  static constexpr int ELEM =
      ELEM0 + ((S + 3 * D::N3 + elem_pad(P, Q) - ELEM0) % 16 + 16) % 16;
  static constexpr int NBXP = pad_nbx(P, Q), NBYP = pad_nby(P, Q), NBP = pad_plane(P, Q);
  static_assert(NBXP >= NBX && NBYP >= NBY && NBP >= NBXP * NBYP * NBZ, "node block padding");
  static constexpr int SMEM = 2 * 3 * NBP + D::NE * ELEM;  // two node blocks + slabs
};

#if HXG_EXPERIMENT == 4
__device__ unsigned long long g_phase_cycles[10];
#endif

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
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void ld_stream2(const double* a, unsigned long long pol, double& x,
                                           double& y) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
      : "=d"(x), "=d"(y)
      : "l"(a), "l"(pol));
}
__device__ __forceinline__ void st_keep(double* a, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_stream(double* a, double v, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_stream2(double* a, double x, double y, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(x),
               "d"(y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ double ld_once(const double* a, unsigned long long pol) {
  double v;
  asm("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v)
               : "l"(a), "l"(pol));
  return v;
}


// ST = JacobianStorage: Current streams the 16-scalar state through
// jacobian_qf; the initial-configuration variants (material.hpp:196-239)
// stream their 19 / 26 / 25-scalar reference layout through
// jacobian_qf_initial (one CTA per SM: their q-functions need the registers).
// MODE = kJacobian (y = J x on the streamed state) or kResidual (the
// residual q-function on the streamed geometry, writing the state: the
// residual of operator.hpp:146-180 in one pass, Current storage).
template <int P, int Q, int ST = kStorageCurrent, int MODE = kJacobian>
__global__ void __launch_bounds__(Dims<P, Q>::T,
                                  MODE != kJacobian         ? fused_residual_min_blocks(P, Q)
                                  : ST == kStorageCurrent ? fused_min_blocks(P, Q)
                                                          : variant_min_blocks(ST))
    fused_jacobian_kernel(const __grid_constant__ FusedParams prm) {
  static_assert(MODE != kResidual || ST == kStorageCurrent, "fused residual: Current storage");
  // kResidualBox: the residual on a box mesh, geometric factors formed in
  // registers (diagonal dxi/dX)
  constexpr bool kRes = MODE == kResidual || MODE == kResidualBox;
  constexpr bool kBoxGeo = MODE == kResidualBox;
  constexpr int SS = device_state_stride(ST), SP = state_row(SS, Q);
  constexpr bool kStateV2 = state_paired(Q);  // 16-byte loads of the paired layout
  using D = FDims<P, Q>;
  constexpr int N = D::N, T = D::T;
  constexpr int NBX = D::NBX, NBY = D::NBY;
  constexpr int BX = D::BX, BY = D::BY, BZ = D::BZ;
  extern __shared__ double smem[];
  double* Xs = smem;                // node block [c][iz][iy][ix] (padded strides)
  double* Ebase = Xs + 2 * 3 * D::NBP;  // per-element slabs
  const int tid = threadIdx.x;
  const QLayout& lay = prm.lay;
  const BoxDev& box = prm.box;
  // Persistent CTAs walk bricks brick0 + blockIdx.x, + gridDim.x, ...; each
  // brick's quadrature state is one contiguous run, pulled into L2 one brick
  // ahead so the q-function loads hit L2.
  auto prefetch_state = [&](int b) {
    // residual: the brick's geometry (the state is written, not read)
    constexpr int RS = kRes ? kGeoStride : SP;
    constexpr unsigned bytes = (unsigned)(sizeof(double) * Q * RS * T);
    constexpr unsigned chunk = 32768;
    const char* base = reinterpret_cast<const char*>(
        (kRes ? prm.geo : prm.state) + (size_t)lay.brick_points() * b * RS);
#pragma unroll
    for (unsigned off = 0; off < bytes; off += chunk)
      prefetch_l2(base + off, off + chunk <= bytes ? chunk : bytes - off);
  };
#if HXG_BRICK_PDL
  // launched as a programmatic dependent of whatever precedes it on the
  // stream: nothing global is touched before the predecessor has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  if (pf_mode(Q) != 1 && !kBoxGeo && tid == 0 && (int)blockIdx.x < prm.nbricks)
    prefetch_state(prm.blist ? prm.blist[prm.brick0 + blockIdx.x] : prm.brick0 + blockIdx.x);
#if HXG_EXPERIMENT == 4
  long long t_last = clock64();
  long long ph[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define HXG_PHASE(i)                    \
  if (tid == 0) {                       \
    long long now_ = clock64();         \
    ph[i] += now_ - t_last;             \
    t_last = now_;                      \
  }
#else
#define HXG_PHASE(i)
#endif
  // 1. node blocks of x: global rows of 3 nbx contiguous doubles, one warp per
  // row (lane = interleaved (node, component) offset), copied asynchronously
  // (cp.async) into one of two buffers one brick ahead, so the loads overlap
  // the previous brick's compute.
  constexpr int ROW3 = 3 * NBX;
  static_assert(ROW3 <= 32, "a node row must fit one warp");
  constexpr int WARPS = T / 32;
  const int lane = tid & 31, warp = tid >> 5;
  const int lix = lane / 3, lc = lane - 3 * (lane / 3);
  const int npx = box.npd[0], npy = box.npd[1];
  // Node rows (iy, iz) of a block, strided over the warps, without divisions.
  auto for_rows = [&](int nby_, int nbz_, auto&& f) {
    int iy = warp, iz = 0;
    while (iy >= nby_) iy -= nby_, ++iz;
    while (iz < nbz_) {
      f(iy, iz);
      iy += WARPS;
      while (iy >= nby_) iy -= nby_, ++iz;
    }
  };
  // Brick coordinates, advanced by the grid stride with carries.
  struct BrickXYZ {
    int x, y, z;
  };
  auto decompose = [&](int b) {
    BrickXYZ c;
    c.x = b % lay.nb[0];
    c.y = (b / lay.nb[0]) % lay.nb[1];
    c.z = b / (lay.nb[0] * lay.nb[1]);
    return c;
  };
  const BrickXYZ step = decompose(gridDim.x);
  auto advance = [&](BrickXYZ c) {
    c.x += step.x;
    c.y += step.y;
    c.z += step.z;
    if (c.x >= lay.nb[0]) c.x -= lay.nb[0], ++c.y;
    if (c.y >= lay.nb[1]) c.y -= lay.nb[1], ++c.z;
    return c;
  };
  auto issue_block = [&](BrickXYZ c, double* dst) {
    const int nbx = P * min(BX, box.cells[0] - c.x * BX) + 1;
    const int nby = P * min(BY, box.cells[1] - c.y * BY) + 1;
    const int nbz = P * min(BZ, box.cells[2] - c.z * BZ) + 1;
    const int node0 = P * c.x * BX + npx * (P * c.y * BY + npy * (P * c.z * BZ));
    if (warp < WARPS && lane < 3 * nbx) {
      const double* src0 = prm.x + 3 * node0 + lane;
      const unsigned d0 = (unsigned)__cvta_generic_to_shared(dst + lc * D::NBP + lix);
      auto row = [&](int iy, int iz) {
        const double* src = src0 + 3 * npx * (iy + npy * iz);
        const unsigned d = d0 + (unsigned)sizeof(double) * ((iz * D::NBYP + iy) * D::NBXP);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
      };
      if (nbx == NBX && nby == NBY && nbz == D::NBZ) {
        constexpr int RPW = (NBY * D::NBZ + WARPS - 1) / WARPS;
#pragma unroll(RPW <= 6 ? RPW : 1)
        for (int t = 0; t < RPW; ++t) {
          const int r = warp + t * WARPS;
          if (r < NBY * D::NBZ) row(r % NBY, r / NBY);
        }
      } else {
        for_rows(nby, nbz, row);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto brick_at = [&](int i) { return prm.blist ? prm.blist[prm.brick0 + i] : prm.brick0 + i; };
  BrickXYZ bc = decompose(brick_at(blockIdx.x));
  if ((int)blockIdx.x < prm.nbricks) issue_block(bc, Xs);
  int cur = 0;
#pragma unroll 1
  for (int bi = blockIdx.x; bi < prm.nbricks; bi += gridDim.x, cur ^= 1) {
  const int brick = brick_at(bi);
  const bool pf_next = tid == 0 && bi + (int)gridDim.x < prm.nbricks;
  if (pf_mode(Q) == 0 && pf_next && !kBoxGeo) prefetch_state(brick_at(bi + gridDim.x));
  if (pf_mode(Q) == 1 && tid == 0 && !kBoxGeo) prefetch_state(brick);
  const int bx = bc.x, by = bc.y, bz = bc.z;
  const BrickXYZ bnext = prm.blist ? decompose(brick_at(min(bi + (int)gridDim.x, prm.nbricks - 1)))
                                    : advance(bc);
  const double* st_brick = prm.state + (size_t)lay.brick_points() * brick * SP;
  const int ecx = min(BX, box.cells[0] - bx * BX);
  const int ecy = min(BY, box.cells[1] - by * BY);
  const int ecz = min(BZ, box.cells[2] - bz * BZ);
  const int nbx = P * ecx + 1, nby = P * ecy + 1, nbz = P * ecz + 1;
  const bool full = ecx == BX && ecy == BY && ecz == BZ;
  const int node0 = P * bx * BX + npx * (P * by * BY + npy * (P * bz * BZ));
  const int gx0 = P * bx * BX, gy0 = P * by * BY, gz0 = P * bz * BZ;
  double* Xc = Xs + cur * (3 * D::NBP);
  // Does the brick touch a constrained face (or is the mask general)?
  const int fb = prm.face_bits;
  const bool bmask =
      fb < 0 || (fb > 0 && (((fb & 1) && gx0 == 0) || ((fb & 2) && gx0 + nbx == npx) ||
                            ((fb & 4) && gy0 == 0) || ((fb & 8) && gy0 + nby == npy) ||
                            ((fb & 16) && gz0 == 0) || ((fb & 32) && gz0 + nbz == box.npd[2])));
  // Constrained test: analytic whole-face sets (build_constraints,
  // operator.hpp:36-55) or the general mask array.
  auto fixed = [&](int dof, int gx, int gy, int gz) -> bool {
    if (prm.face_bits >= 0) {
      const int b = prm.face_bits;
      return ((b & 1) && gx == 0) || ((b & 2) && gx == npx - 1) || ((b & 4) && gy == 0) ||
             ((b & 8) && gy == npy - 1) || ((b & 16) && gz == 0) ||
             ((b & 32) && gz == box.npd[2] - 1);
    }
    return prm.mask && prm.mask[dof];
  };
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // General masks: zero constrained inputs (operator.hpp:189-193) in the
  // landed block.  Whole-face masks are applied analytically as P1 reads the
  // block, which keeps x intact for the constrained pass-through.
  if (!kRes && fb < 0 && warp < WARPS && lane < 3 * nbx) {
    for_rows(nby, nbz, [&](int iy, int iz) {
      const int dof = 3 * (node0 + npx * (iy + npy * iz)) + lane;
      if (fixed(dof, gx0 + lix, gy0 + iy, gz0 + iz))
        Xc[lc * D::NBP + (iz * D::NBYP + iy) * D::NBXP + lix] = 0.0;
    });
  }
  // Next brick's block into the other buffer (free: its last readers, the
  // previous brick's P1 pass, are behind the barrier above).
  if (bi + (int)gridDim.x < prm.nbricks) issue_block(bnext, Xs + (cur ^ 1) * (3 * D::NBP));
  bc = bnext;
  // Lanes are (column te = qy Q + qx, element le) with elements fastest, so
  // tid is also the state-layout index t (coalesced state loads).
  const int le = tid % D::NE, te = tid / D::NE;
  const int lx = le % BX, ly = (le / BX) % BY, lz = le / (BX * BY);
  const bool valid = lx < ecx && ly < ecy && lz < ecz;
  // S[c][arr][k][b][a], arr 0 = interpolated, 1 = d/dx, 2 = d/dy (forward)
  // or the z-adjoints (backward); EO[c][k][j][i] element outputs.
  double* S = Ebase + le * D::ELEM;
  double* EOe = S + D::S;
  constexpr int Q2 = D::Q2;
  // Only the general-mask zeroing above writes the landed block; the slab
  // hazards with the previous brick are ordered by the barrier after the
  // cp.async wait (P1 writes S, the overlap-add read EO).
  if (fb < 0) __syncthreads();
  HXG_PHASE(0);

  // ---- forward: G = (Bd (x) B (x) B, B (x) Bd (x) B, B (x) B (x) Bd) U -----
  // The direct tensor-product gradient (deriv tabulated at the points,
  // basis.hpp:144, = colloc_deriv * interp in exact arithmetic).  x and y
  // passes run on (component, z-plane) owners in registers; the z pass on
  // (qx, qy) column owners, so each value crosses shared memory once.
  // P1: plane tasks (c, k), te < 3N.
  // (3N plane tasks per element; Q^2 < 3N only for p = 1, q = 2.)
#pragma unroll 1
  for (int task = te; task < 3 * N; task += Q2) {
    const int c = task / N, k = task - c * N;
    const double* Xp = Xc + c * D::NBP + ((P * lz + k) * D::NBYP + P * ly) * D::NBXP + P * lx;
    double u[N][N];
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) u[j][i] = Xp[j * D::NBXP + i];
    if (!kRes && fb > 0 && bmask) {
      const int gx = gx0 + P * lx, gy = gy0 + P * ly, gz = gz0 + P * lz + k;
      const bool mz = ((fb & 16) && gz == 0) || ((fb & 32) && gz == box.npd[2] - 1);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const bool my = mz || ((fb & 4) && gy + j == 0) || ((fb & 8) && gy + j == npy - 1);
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const bool m = my || ((fb & 1) && gx + i == 0) || ((fb & 2) && gx + i == npx - 1);
          u[j][i] = m ? 0.0 : u[j][i];
        }
      }
    }
    double ab[N][Q], ad[N][Q];
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        double sb = 0.0, sd = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          sb += prm.B[a * N + i] * u[j][i];
          sd += prm.Bd[a * N + i] * u[j][i];
        }
        ab[j][a] = sb;
        ad[j][a] = sd;
      }
    double* S0 = S + ((c * 3 + 0) * N + k) * Q2;
    double* S1 = S + ((c * 3 + 1) * N + k) * Q2;
    double* S2 = S + ((c * 3 + 2) * N + k) * Q2;
#pragma unroll
    for (int b = 0; b < Q; ++b)
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        double tb = 0.0, tdy = 0.0, tdx = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          tb += prm.B[b * N + j] * ab[j][a];
          tdy += prm.Bd[b * N + j] * ab[j][a];
          tdx += prm.B[b * N + j] * ad[j][a];
        }
        S0[b * Q + a] = tb;
        S1[b * Q + a] = tdx;
        S2[b * Q + a] = tdy;
      }
  }
  __syncthreads(); HXG_PHASE(1);
  if (pf_mode(Q) == 2 && pf_next) prefetch_state(brick + gridDim.x);
  // P2: column owners (qx, qy): z pass for the three arrays.
  // Between the P1 and Q2 barriers the slab entries S[idx Q^2 + te] (idx <
  // 9N) belong to this thread alone (its column).  For (p, q) = (1, 2),
  // (1, 3), (2, 3) they hold the gradients and q-function outputs of the
  // column's first N points (shared memory instead of registers: no spills at
  // the two-CTA register cap), registers the remaining Q - N; elsewhere all Q
  // stay in registers (no spills there, and fewer shared accesses).  The slots are volatile so the compiler
  // does not forward them back into registers.
  // NSG / NSH planes of the gradients / q-function outputs live in the
  // slots, the rest in registers.
  constexpr int NSG = !fused_slots(P, Q) ? 0 : (P == 2 && Q == 3) ? HXG_NSG_Q2 : N;
  constexpr int NSH = !fused_slots(P, Q) ? 0 : (P == 2 && Q == 3) ? HXG_NSH_Q2 : N;
  constexpr int QR = Q - NSG, QH = Q - NSH;
  volatile double* slot = S + te;
  double g[3][3][QR > 0 ? QR : 1];
  double hr[3][3][QH > 0 ? QH : 1];
  const double* sp0 = st_brick + state_lane(tid, Q);
  const unsigned long long pol_stream = policy_evict_first();
  auto gslot = [&](int c, int d, int z) { return ((c * 3 + d) * N + z) * Q2; };
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double tb[N], tdx[N], tdy[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      tb[k] = S[((c * 3 + 0) * N + k) * Q2 + te];
      tdx[k] = S[((c * 3 + 1) * N + k) * Q2 + te];
      tdy[k] = S[((c * 3 + 2) * N + k) * Q2 + te];
    }
#pragma unroll
    for (int z = 0; z < Q; ++z) {
      double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        gx += prm.B[z * N + k] * tdx[k];
        gy += prm.B[z * N + k] * tdy[k];
        gz += prm.Bd[z * N + k] * tb[k];
      }
      if (z < NSG) {
        slot[gslot(c, 0, z)] = gx;
        slot[gslot(c, 1, z)] = gy;
        slot[gslot(c, 2, z)] = gz;
      } else {
        g[c][0][z - NSG] = gx;
        g[c][1][z - NSG] = gy;
        g[c][2][z - NSG] = gz;
      }
    }
  }

  // ---- q-function on the streamed state --------------------------------
  // Loads scalars [s0, s1) of plane qz (s0, s1 even on the paired layout).
  auto load_range = [&](int qz, double* st, int s0, int s1) {
    const double* sp = sp0 + qz * T * SP;
    if constexpr (kStateV2) {
#pragma unroll
      for (int s = 0; s < SS; s += 2)
        if (s >= s0 && s < s1) ld_stream2(sp + s * T, pol_stream, st[s], st[s + 1]);
    } else {
#pragma unroll
      for (int s = 0; s < SS; ++s)
        if (s >= s0 && s < s1) st[s] = ld_stream(sp + s * T, pol_stream);
    }
  };
  // Software pipeline of the state planes: the first kPipe scalars of plane
  // qz + 1 are loaded while plane qz is consumed.  Measured: all of them for
  // Q4 (394.5 -> 364.4 us); Q2 / Q3 have no register room for the full plane
  // (+1 % / +8 %).
  constexpr int kPipe = kRes ? 0
                        : (Q == 5 && ST == kStorageCurrent && (P == 4 || HXG_PIPE_ALL_Q5)) ? SP
                        : (P == 2 && Q == 3 && ST == kStorageCurrent)                   ? HXG_PIPE_Q2
                                                                                        : 0;
  double stn[kPipe > 0 ? kPipe : 1];
  if constexpr (kPipe > 0) {
    if (valid) load_range(0, stn, 0, kPipe);
  }
  (void)load_range;
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double H[9];
    if constexpr (kRes) {
      if (valid) {
        const size_t pt = (size_t)lay.brick_points() * brick + (size_t)qz * T;
        double G[9];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d)
            G[3 * c + d] = qz < NSG ? slot[gslot(c, d, qz)] : g[c][d][qz - NSG];
        // the q-function, state stores and failure report for one set of
        // geometric factors (inlined twice: the box branch's zero
        // off-diagonal dxi/dX entries fold away)
        auto qf_store = [&](const double* geo, auto diag) {
          double st[kRefStateScalars];
          const double J = residual_qf<decltype(diag)::value>(prm.mu, prm.lambda, G, geo, geo[9], H, st);
          double* so = prm.state_out + pt * SP + state_lane(tid, Q);
          if (!(J > 0.0)) {  // first inverted (e, q) in reference order (operator.hpp:166-168)
            const int qx = te % Q, qy = te / Q;
            const long long e = (bx * BX + lx) + (long long)box.cells[0] * ((by * BY + ly) +
                                                                       (long long)box.cells[1] * (bz * BZ + lz));
            atomicMin(prm.fail, (unsigned long long)e * (Q * Q * Q) + (unsigned long long)(qx + Q * (qy + Q * qz)));
            so[0] = J;  // read back by the host for the error report
#pragma unroll
            for (int k = 0; k < 9; ++k) H[k] = 0.0;
          } else {
            double sp[kStateStride];
            pack_state(prm.mu, st, sp);
            if constexpr (kStateV2) {
#pragma unroll
              for (int s = 0; s < kStateStride; s += 2) st_stream2(so + s * T, sp[s], sp[s + 1], pol_stream);
            } else {
#pragma unroll
              for (int s = 0; s < kStateStride; ++s) st_stream(so + s * T, sp[s], pol_stream);
            }
          }
        };
        if constexpr (kBoxGeo) {
          const int qx = te % Q, qy = te / Q;
          const double geo[kGeoStride] = {prm.geo_g[0], 0.0, 0.0, 0.0, prm.geo_g[1], 0.0, 0.0, 0.0, prm.geo_g[2],
                                          prm.geo_qw[qx] * prm.geo_qw[qy] * prm.geo_qw[qz] * prm.geo_jac};
          qf_store(geo, std::true_type{});
        } else {
          double geo[kGeoStride];
          const double* gp = prm.geo + pt * kGeoStride + tid;
#pragma unroll
          for (int s = 0; s < kGeoStride; ++s) geo[s] = ld_stream(gp + s * T, pol_stream);
          qf_store(geo, std::false_type{});
        }
      } else {
#pragma unroll
        for (int k = 0; k < 9; ++k) H[k] = 0.0;
      }
    } else if (valid) {
      double st[SP];
      if constexpr (kPipe > 0) {
#pragma unroll
        for (int s = 0; s < kPipe; ++s) st[s] = stn[s];
        load_range(qz, st, kPipe, SP);
        if (qz + 1 < Q) load_range(qz + 1, stn, 0, kPipe);
      } else {
        load_range(qz, st, 0, SP);
      }
      double G[9];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d)
          G[3 * c + d] = qz < NSG ? slot[gslot(c, d, qz)] : g[c][d][qz - NSG];
      if constexpr (ST == kStorageCurrent)
        jacobian_qf(prm.mu, prm.lambda, G, st, H);
      else
        jacobian_qf_initial<ST>(prm.mu, prm.lambda, G, st, H);
      if (!kRes && prm.perturb != 0.0) {  // fault-injection hook: + eps w detJ G
        const double wdet =
            prm.geo[((size_t)lay.brick_points() * brick + (size_t)qz * T) * kGeoStride + 9 * T + tid];
#pragma unroll
        for (int k = 0; k < 9; ++k) H[k] += prm.perturb * wdet * G[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < 9; ++k) H[k] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        if (qz < NSH)
          slot[gslot(c, d, qz)] = H[3 * c + d];
        else
          hr[c][d][qz - NSH] = H[3 * c + d];
      }
  }
  HXG_PHASE(2);
  if (pf_mode(Q) == 3 && pf_next) prefetch_state(brick + gridDim.x);

  // ---- backward: exact adjoint of the forward passes ---------------------
  // Q1: column owners: z adjoints R0 = Bd_z^T Hz, R1 = B_z^T Hx, R2 = B_z^T Hy
  // (into this column's own slab entries: no barrier needed before it).
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double h[3][Q];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int z = 0; z < Q; ++z) h[d][z] = z < NSH ? slot[gslot(c, d, z)] : hr[c][d][z - NSH];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double r0 = 0.0, r1 = 0.0, r2 = 0.0;
#pragma unroll
      for (int z = 0; z < Q; ++z) {
        r0 += prm.Bd[z * N + k] * h[2][z];
        r1 += prm.B[z * N + k] * h[0][z];
        r2 += prm.B[z * N + k] * h[1][z];
      }
      slot[((c * 3 + 0) * N + k) * Q2] = r0;
      slot[((c * 3 + 1) * N + k) * Q2] = r1;
      slot[((c * 3 + 2) * N + k) * Q2] = r2;
    }
  }
  __syncthreads(); HXG_PHASE(3);
  // Q2: plane tasks (c, k): y adjoints then x adjoints, in registers.
#pragma unroll 1
  for (int task = te; task < 3 * N; task += Q2) {
    const int c = task / N, k = task - c * N;
    const double* S0 = S + ((c * 3 + 0) * N + k) * Q2;
    const double* S1 = S + ((c * 3 + 1) * N + k) * Q2;
    const double* S2 = S + ((c * 3 + 2) * N + k) * Q2;
    double ab[N][Q], ad[N][Q];
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        ab[j][a] = 0.0;
        ad[j][a] = 0.0;
      }
#pragma unroll
    for (int b = 0; b < Q; ++b)
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        const double r0 = S0[b * Q + a], r1 = S1[b * Q + a], r2 = S2[b * Q + a];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          ab[j][a] += prm.B[b * N + j] * r0 + prm.Bd[b * N + j] * r2;
          ad[j][a] += prm.B[b * N + j] * r1;
        }
      }
    double* Oc = EOe + c * D::EOC + k * N * N;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < Q; ++a) s += prm.B[a * N + i] * ab[j][a] + prm.Bd[a * N + i] * ad[j][a];
        Oc[j * N + i] = valid ? s : 0.0;  // padding elements add exact zeros
      }
  }
  __syncthreads(); HXG_PHASE(4);

  // ---- overlap-add fused with the stores: node-centric ------------------
  // Node (ix, iy, iz) of the block sums the outputs of the elements sharing
  // it, lower element first in x, then y, then z: a fixed order (the
  // scatter_add of mesh.hpp:105-116, made deterministic).  One warp per node
  // row, lanes over the row's 3 nbx interleaved (node, component) doubles,
  // which are contiguous in y (coalesced stores).
  double* part = prm.partial + (size_t)brick * (D::NB * 3);
  const unsigned long long pol_keep = policy_evict_last();
  if (warp < WARPS && lane < 3 * nbx) {
    const int ix = lix, c = lc;
    const int lxh = ix / P < BX ? ix / P : BX - 1;
    const int i = ix - P * lxh;
    const bool twox = i == 0 && lxh > 0;
    const double* ex = Ebase + lxh * D::ELEM + D::S + c * D::EOC + i;
    constexpr int DX = P - D::ELEM;                 // (lx - 1, i = P)
    constexpr int DY = P * N - BX * D::ELEM;        // (ly - 1, j = P)
    constexpr int DZ = P * N * N - BY * BX * D::ELEM;  // (lz - 1, k = P)
    auto xsum = [&](const double* e) {
      const double v = e[0];
      return twox ? e[DX] + v : v;
    };
    auto row = [&](int iy, int iz) {
      const int lzh = iz / P < BZ ? iz / P : BZ - 1, k = iz - P * lzh;
      const int lyh = iy / P < BY ? iy / P : BY - 1, j = iy - P * lyh;
      const bool twoy = j == 0 && lyh > 0;
      const double* e = ex + (lzh * BY + lyh) * BX * D::ELEM + (k * N + j) * N;
      auto ysum = [&](const double* f) {
        const double v = xsum(f);
        return twoy ? xsum(f + DY) + v : v;
      };
      double s = ysum(e);
      if (k == 0 && lzh > 0) s = ysum(e + DZ) + s;
      if (ix == 0 || iy == 0 || iz == 0 || ix == nbx - 1 || iy == nby - 1 || iz == nbz - 1) {
        st_keep(part + (iz * NBY + iy) * ROW3 + lane, s, pol_keep);
      } else {
        const int dof = 3 * (node0 + npx * (iy + npy * iz)) + lane;
        if constexpr (kRes) {  // f = r - s load; constrained: 0 (operator.hpp:175-179)
          if (prm.load) s -= prm.load_scale * prm.load[dof];
          if (bmask && fixed(dof, gx0 + ix, gy0 + iy, gz0 + iz)) s = 0.0;
        } else if (bmask && fixed(dof, gx0 + ix, gy0 + iy, gz0 + iz)) {  // pass x through (operator.hpp:212-214)
          s = fb >= 0 ? Xc[c * D::NBP + (iz * D::NBYP + iy) * D::NBXP + ix] : prm.x[dof];
        }
        prm.y[dof] = s;
      }
    };
    if (full) {  // compile-time row walk (constant divisors, unrolled)
      constexpr int RPW = (NBY * D::NBZ + WARPS - 1) / WARPS;
#pragma unroll(RPW <= 6 ? RPW : 1)
      for (int t = 0; t < RPW; ++t) {
        const int r = warp + t * WARPS;
        if (r < NBY * D::NBZ) row(r % NBY, r / NBY);
      }
    } else {
      for_rows(nby, nbz, row);
    }
  }
  // (the next iteration's first barrier orders these slab reads before the
  // slabs are rewritten)
  HXG_PHASE(8);
  }  // brick loop
#if HXG_EXPERIMENT == 4
  if (tid == 0)
    for (int i = 0; i < 10; ++i) atomicAdd(&g_phase_cycles[i], (unsigned long long)ph[i]);
#endif
}

// Brick-boundary sums (the deterministic second half of scatter_add,
// mesh.hpp:105-116), brick-centric: a brick owns the nodes of its block that
// are not on its upper faces (unless the box ends there); of those, the ones
// on the block boundary were left as per-brick partials by the brick kernel.
// Each is summed over its <= 8 sharing bricks in increasing brick order
// (q = i0 + 2 i1 + 4 i2, brick lo_d + i_d).  One CTA per brick, one thread
// per owned boundary node (its three components together); nodes are
// enumerated compactly: rows (iy, iz) on a boundary plane are boundary along
// their whole length, the other rows only at ix = 0 (and the far face of the
// box).  The index math is all brick-local.
template <int P, int Q, int MODE = kJacobian>
__global__ void __launch_bounds__(kFixupThreads, HXG_FIXUP_MINB) fused_fixup_kernel(const __grid_constant__ FusedParams prm) {
  using D = FDims<P, Q>;
  constexpr int BX = D::BX, BY = D::BY, BZ = D::BZ;
  constexpr int PB0 = P * BX, PB1 = P * BY, PB2 = P * BZ;
  constexpr int NB3 = D::NB * 3;
  const QLayout& lay = prm.lay;
  const BoxDev& box = prm.box;
  const int npx = box.npd[0], npy = box.npd[1];
  const unsigned long long pol = policy_evict_first();
  const int fb = prm.face_bits;
  // Offset of sharing brick o = o0 + 2 o1 + 4 o2 (o_d = 1: the lower
  // neighbour along d) relative to this brick's partial of the same node:
  // brick index - (o0 + nb0 (o1 + nb1 o2)), local coordinate + o_d P B_d.
  __shared__ long long off[8];
  if (threadIdx.x < 8) {
    const int o0 = threadIdx.x & 1, o1 = (threadIdx.x >> 1) & 1, o2 = threadIdx.x >> 2;
    off[threadIdx.x] = -(long long)(o0 + lay.nb[0] * (o1 + lay.nb[1] * o2)) * NB3 +
                       3 * ((o2 * PB2 * D::NBY + o1 * PB1) * D::NBX + o0 * PB0);
  }
  __syncthreads();
  for (int bi = blockIdx.x; bi < prm.nbricks; bi += gridDim.x) {
    const int b = prm.blist ? prm.blist[prm.brick0 + bi] : prm.brick0 + bi;
    const int cx = b % lay.nb[0], cy = (b / lay.nb[0]) % lay.nb[1], cz = b / (lay.nb[0] * lay.nb[1]);
    const bool lx = cx == lay.nb[0] - 1, ly = cy == lay.nb[1] - 1, lz = cz == lay.nb[2] - 1;
    const int fnx = lx ? P * (box.cells[0] - cx * BX) + 1 : D::NBX;
    const int fny = ly ? P * (box.cells[1] - cy * BY) + 1 : D::NBY;
    const int fnz = lz ? P * (box.cells[2] - cz * BZ) + 1 : D::NBZ;
    const int nox = lx ? fnx : fnx - 1, noy = ly ? fny : fny - 1, noz = lz ? fnz : fnz - 1;
    const int nbx = lx ? 2 : 1, nby = ly ? 2 : 1, nbz = lz ? 2 : 1;  // boundary coords per axis
    const int iyc = noy - nby, izc = noz - nbz;                        // interior coords
    const int rowsA = nbz * noy + izc * nby;
    const int entA = rowsA * nox, entB = izc * iyc * nbx;  // nodes (3 components each)
    // small exact divisions through float reciprocals (t, r < 2^12)
    const float rnox = 1.0f / (float)nox, rnby = 1.0f / (float)nby, rnbx = 1.0f / (float)nbx,
                riyc = 1.0f / (float)(iyc > 0 ? iyc : 1);
    const int gx0 = PB0 * cx, gy0 = PB1 * cy, gz0 = PB2 * cz;
    const double* pbase = prm.partial + (size_t)b * NB3;
    const int sb0 = cx > 0, sb1 = (cy > 0) << 1, sb2 = (cz > 0) << 2;
    for (int t = threadIdx.x; t < entA + entB; t += kFixupThreads) {
      int ix, iy, iz;
      if (t < entA) {
        const int r = (int)(((float)t + 0.5f) * rnox);
        ix = t - r * nox;
        if (r < nbz * noy) {
          const bool up = r >= noy;
          iz = up ? fnz - 1 : 0;
          iy = up ? r - noy : r;
        } else {
          const int q = r - nbz * noy;
          const int qz = (int)(((float)q + 0.5f) * rnby);
          iz = 1 + qz;
          iy = q - qz * nby ? fny - 1 : 0;
        }
      } else {
        const int u = t - entA, r = (int)(((float)u + 0.5f) * rnbx);
        ix = u - r * nbx ? fnx - 1 : 0;
        const int rz = (int)(((float)r + 0.5f) * riyc);
        iz = 1 + rz;
        iy = 1 + (r - rz * iyc);
      }
      const int gx = gx0 + ix, gy = gy0 + iy, gz = gz0 + iz;
      if (prm.ifilter) {  // the partitioned apply's split around the interface exchange
        const int fi = prm.iface;
        const bool on = ((fi & 1) && gx == 0) || ((fi & 2) && gx == npx - 1) || ((fi & 4) && gy == 0) ||
                        ((fi & 8) && gy == npy - 1) || ((fi & 16) && gz == 0) ||
                        ((fi & 32) && gz == box.npd[2] - 1);
        if (on != (prm.ifilter == 1)) continue;
      }
      // sharing bricks: the lower neighbour along d when the node sits on the
      // block's low plane and the brick is not the first along d; summed in
      // increasing brick order (q = i0 + 2 i1 + 4 i2, i_d = s_d - o_d)
      const int sidx = (ix == 0 ? sb0 : 0) | (iy == 0 ? sb1 : 0) | (iz == 0 ? sb2 : 0);
      const double* a0 = pbase + ((iz * D::NBY + iy) * D::NBX + ix) * 3;
      double sum[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q & ~sidx) continue;
        const double* a = a0 + off[sidx - q];
        double v[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
          v[c] = HXG_FIXUP_LD == 1 ? __ldg(a + c) : HXG_FIXUP_LD == 2 ? a[c] : ld_once(a + c, pol);
#pragma unroll
        for (int c = 0; c < 3; ++c) sum[c] += v[c];
      }
      const size_t dof0 = 3 * ((size_t)gx + (size_t)npx * (gy + (size_t)npy * gz));
      const bool ffix = fb > 0 && (((fb & 1) && gx == 0) || ((fb & 2) && gx == npx - 1) ||
                                   ((fb & 4) && gy == 0) || ((fb & 8) && gy == npy - 1) ||
                                   ((fb & 16) && gz == 0) || ((fb & 32) && gz == box.npd[2] - 1));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const size_t dof = dof0 + c;
        const bool fixed = fb >= 0 ? ffix : prm.mask && prm.mask[dof];
        double s = sum[c];
        if (MODE == kResidual) {  // f = r - s load; constrained: 0 (operator.hpp:175-179)
          if (prm.load) s -= prm.load_scale * prm.load[dof];
          prm.y[dof] = fixed ? 0.0 : s;
        } else {
          prm.y[dof] = fixed ? prm.x[dof] : s;  // pass x through (operator.hpp:212-214)
        }
      }
    }
  }
}

// Fix-up grid over a launch's bricks.
inline unsigned fixup_grid(int nbricks) {
  return (unsigned)(nbricks < kFixupMaxGrid ? (nbricks > 0 ? nbricks : 1) : kFixupMaxGrid);
}

// Persistent grid: every resident CTA slot of the device, capped by the work.
template <class K>
unsigned persistent_grid(K kernel, int threads, size_t smem, int work) {
  static int sms = 0;
  if (!sms) HXG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int per_sm = 0;
  HXG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  long long g = (long long)(per_sm > 0 ? per_sm : 1) * sms;
  if (g > work) g = work;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

#if HXG_EXPERIMENT == 4
extern "C" int hxg_debug_phase_cycles(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 10);
  if (reset) {
    unsigned long long z[10] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
  return 0;
}
#endif

// The fused kernel for the operator's storage: Current for every (P, Q);
// the initial variants on the fine-level pairs Q = P + 1.
template <int P, int Q>
void (*select_fused(int storage))(FusedParams) {
  if constexpr (Q == P + 1) {
    switch (storage) {
      case kStorageInitialNative: return fused_jacobian_kernel<P, Q, kStorageInitialNative>;
      case kStorageInitialTuned: return fused_jacobian_kernel<P, Q, kStorageInitialTuned>;
      case kStorageInitialAD: return fused_jacobian_kernel<P, Q, kStorageInitialAD>;
      default: break;
    }
  }
  if (storage != kStorageCurrent)
    throw Error(HXG_ERR_UNSUPPORTED, "fused initial-storage kernels cover q = p + 1");
  return fused_jacobian_kernel<P, Q, kStorageCurrent>;
}

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
  prm.face_bits = op.face_bits();
  prm.tab = op.tab_.p;
  prm.state = op.state_->data.p;
  prm.geo = op.geometry_ ? op.geometry_->data.p : nullptr;
  if (op.perturb_ != 0.0 && !prm.geo)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "the perturbation hook needs geometric factors");
  prm.mu = op.mu_;
  prm.lambda = op.lambda_;
  prm.perturb = op.perturb_;
  for (size_t i = 0; i < op.interp_.size(); ++i) prm.B[i] = op.interp_[i];
  for (size_t i = 0; i < op.deriv_.size(); ++i) prm.Bd[i] = op.deriv_[i];
  dispatch_pq(op.p_, op.q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    using D = FDims<P, Q>;
    size_t need = (size_t)op.lay_.num_bricks() * D::NB * 3;
    if (op.partial_.n != need) op.partial_.alloc(need);
    prm.partial = op.partial_.p;
    size_t smem = sizeof(double) * D::SMEM;
    auto k = select_fused<P, Q>(op.storage_);
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
    prm.brick0 = 0;
    prm.nbricks = (int)op.lay_.num_bricks();
#if HXG_BRICK_PDL
    {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(persistent_grid(k, D::T, smem, prm.nbricks));
      cfg.blockDim = dim3(D::T);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = op.stream_;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      HXG_CUDA(cudaLaunchKernelEx(&cfg, k, prm));
    }
#else
    k<<<persistent_grid(k, D::T, smem, prm.nbricks), D::T, smem, op.stream_>>>(prm);
#endif
    HXG_CUDA(cudaGetLastError());
    if (op.split_evt_) {
      HXG_CUDA(cudaEventRecord(op.split_evt_, op.stream_));
      op.split_evt_ = nullptr;
    }
    const unsigned fg = HXG_SKIP_FIXUP ? 0 : fixup_grid(prm.nbricks);
    if (fg) {
#if HXG_FIXUP_PDL
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(fg);
      cfg.blockDim = dim3(kFixupThreads);
      cfg.stream = op.stream_;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      HXG_CUDA(cudaLaunchKernelEx(&cfg, fused_fixup_kernel<P, Q>, prm));
#else
      fused_fixup_kernel<P, Q><<<fg, kFixupThreads, 0, op.stream_>>>(prm);
#endif
    }
    HXG_CUDA(cudaGetLastError());
  });
}

void fused_jacobian_split(Operator& op, const double* du, double* y, int iface, cudaStream_t side,
                          const std::function<void()>& exchange) {
  if (op.storage_ != kStorageCurrent && op.q_ != op.p_ + 1)
    throw Error(HXG_ERR_UNSUPPORTED, "split apply: fused path only");
  const QLayout& lay = op.lay_;
  const int nbr = (int)lay.num_bricks();
  if (op.blist_iface_ != iface) {  // brick lists: interface layer first, then the rest
    std::vector<int> a, b;
    for (int k = 0; k < nbr; ++k) {
      const int bx = k % lay.nb[0], by = (k / lay.nb[0]) % lay.nb[1], bz = k / (lay.nb[0] * lay.nb[1]);
      const bool on = ((iface & 1) && bx == 0) || ((iface & 2) && bx == lay.nb[0] - 1) ||
                      ((iface & 4) && by == 0) || ((iface & 8) && by == lay.nb[1] - 1) ||
                      ((iface & 16) && bz == 0) || ((iface & 32) && bz == lay.nb[2] - 1);
      (on ? a : b).push_back(k);
    }
    op.blist_na_ = (int)a.size();
    a.insert(a.end(), b.begin(), b.end());
    op.blist_.upload(a);
    op.blist_iface_ = iface;
    if (!op.ev_a_) {
      HXG_CUDA(cudaEventCreateWithFlags(&op.ev_a_, cudaEventDisableTiming));
      HXG_CUDA(cudaEventCreateWithFlags(&op.ev_x_, cudaEventDisableTiming));
    }
  }
  FusedParams prm{};
  prm.box = op.box_;
  prm.lay = op.lay_;
  prm.x = du;
  prm.y = y;
  prm.mask = op.mask();
  prm.face_bits = op.face_bits();
  prm.tab = op.tab_.p;
  prm.state = op.state_->data.p;
  prm.geo = op.geometry_ ? op.geometry_->data.p : nullptr;
  if (op.perturb_ != 0.0 && !prm.geo)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "the perturbation hook needs geometric factors");
  prm.mu = op.mu_;
  prm.lambda = op.lambda_;
  prm.perturb = op.perturb_;
  prm.blist = op.blist_.p;
  prm.iface = iface;
  for (size_t i = 0; i < op.interp_.size(); ++i) prm.B[i] = op.interp_[i];
  for (size_t i = 0; i < op.deriv_.size(); ++i) prm.Bd[i] = op.deriv_[i];
  const int na = op.blist_na_, nb = nbr - na;
  dispatch_pq(op.p_, op.q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    using D = FDims<P, Q>;
    size_t need = (size_t)op.lay_.num_bricks() * D::NB * 3;
    if (op.partial_.n != need) op.partial_.alloc(need);
    prm.partial = op.partial_.p;
    size_t smem = sizeof(double) * D::SMEM;
    auto k = select_fused<P, Q>(op.storage_);
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
    cudaStream_t s = op.stream_;
    // 1. the interface layer and its interface-node sums
    FusedParams pa = prm;
    pa.brick0 = 0;
    pa.nbricks = na;
    if (na > 0) {
      k<<<persistent_grid(k, D::T, smem, na), D::T, smem, s>>>(pa);
      pa.ifilter = 1;
      fused_fixup_kernel<P, Q><<<fixup_grid(na), kFixupThreads, 0, s>>>(pa);
      HXG_CUDA(cudaGetLastError());
    }
    HXG_CUDA(cudaEventRecord(op.ev_a_, s));
    // 2. the interior bricks and every other boundary sum (enqueued before the
    // exchange, so a host-staged communicator blocking in exchange() still
    // overlaps with them)
    FusedParams pb = prm;
    pb.brick0 = na;
    pb.nbricks = nb;
    if (nb > 0) k<<<persistent_grid(k, D::T, smem, nb), D::T, smem, s>>>(pb);
    pb.brick0 = 0;
    pb.nbricks = nbr;
    pb.ifilter = 2;
    fused_fixup_kernel<P, Q><<<fixup_grid(nbr), kFixupThreads, 0, s>>>(pb);
    HXG_CUDA(cudaGetLastError());
    // 3. the exchange on the side stream, behind step 1 only
    HXG_CUDA(cudaStreamWaitEvent(side, op.ev_a_, 0));
    exchange();
    HXG_CUDA(cudaEventRecord(op.ev_x_, side));
    HXG_CUDA(cudaStreamWaitEvent(s, op.ev_x_, 0));
  });
}

// Fused residual (operator.hpp:146-180): one brick pass writing the state
// and f = r(u) - s load (constrained entries 0); the caller reads back the
// first inverted point.
void fused_residual(Operator& op, const double* u, double* f) {
  if (op.storage_ != kStorageCurrent || !op.geometry_)
    throw Error(HXG_ERR_UNSUPPORTED, "fused residual: Current storage with geometric factors");
  FusedParams prm{};
  prm.box = op.box_;
  prm.lay = op.lay_;
  prm.x = u;
  prm.y = f;
  prm.mask = op.mask();
  prm.face_bits = op.face_bits();
  prm.tab = op.tab_.p;
  prm.state = nullptr;
  prm.state_out = op.state_->data.p;
  prm.geo = op.geometry_->data.p;
  prm.geo_box = op.geometry_->box && HXG_RES_BOX_GEO;
  for (int d = 0; d < 3; ++d) prm.geo_g[d] = op.geometry_->g[d];
  prm.geo_jac = op.geometry_->jac;
  for (int i = 0; i < kMaxQ; ++i) prm.geo_qw[i] = op.geometry_->qw[i];
  prm.load = op.load_.n ? op.load_.p : nullptr;
  prm.load_scale = op.load_scale_;
  prm.fail = op.fail_.p;
  prm.mu = op.mu_;
  prm.lambda = op.lambda_;
  for (size_t i = 0; i < op.interp_.size(); ++i) prm.B[i] = op.interp_[i];
  for (size_t i = 0; i < op.deriv_.size(); ++i) prm.Bd[i] = op.deriv_[i];
  dispatch_pq(op.p_, op.q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    using D = FDims<P, Q>;
    size_t need = (size_t)op.lay_.num_bricks() * D::NB * 3;
    if (op.partial_.n != need) op.partial_.alloc(need);
    prm.partial = op.partial_.p;
    size_t smem = sizeof(double) * D::SMEM;
    auto k = prm.geo_box ? fused_jacobian_kernel<P, Q, kStorageCurrent, kResidualBox>
                         : fused_jacobian_kernel<P, Q, kStorageCurrent, kResidual>;
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
    prm.brick0 = 0;
    prm.nbricks = (int)op.lay_.num_bricks();
    k<<<persistent_grid(k, D::T, smem, prm.nbricks), D::T, smem, op.stream_>>>(prm);
    HXG_CUDA(cudaGetLastError());
    fused_fixup_kernel<P, Q, kResidual><<<fixup_grid(prm.nbricks), kFixupThreads, 0, op.stream_>>>(prm);
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
  prm.face_bits = op.face_bits();
  prm.tab = op.tab_.p;
  prm.state = op.state_->data.p;
  prm.geo = op.geometry_ ? op.geometry_->data.p : nullptr;
  if (op.perturb_ != 0.0 && !prm.geo)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "the perturbation hook needs geometric factors");
  prm.mu = op.mu_;
  prm.lambda = op.lambda_;
  prm.perturb = op.perturb_;
  for (size_t i = 0; i < op.interp_.size(); ++i) prm.B[i] = op.interp_[i];
  for (size_t i = 0; i < op.deriv_.size(); ++i) prm.Bd[i] = op.deriv_[i];
  dispatch_pq(op.p_, op.q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    using D = FDims<P, Q>;
    size_t need = (size_t)op.lay_.num_bricks() * D::NB * 3;
    if (op.partial_.n != need) op.partial_.alloc(need);
    prm.partial = op.partial_.p;
    size_t smem = sizeof(double) * D::SMEM;
    auto k = select_fused<P, Q>(op.storage_);
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
    const int nbz = op.lay_.nb[2], layer = op.lay_.nb[0] * op.lay_.nb[1];
    const int pb2 = P * D::BZ, npz = op.box_.npd[2];
    const size_t plane = (size_t)op.box_.npd[0] * op.box_.npd[1] * 3;
    // chunks of brick layers: enough to overlap the two PCIe directions with
    // little pipeline fill (HXG_HOST_CHUNKS overrides, for measurements)
    static const int env_chunks = [] {
      const char* e = std::getenv("HXG_HOST_CHUNKS");
      return e ? std::atoi(e) : 0;
    }();
    int want = env_chunks > 0 ? env_chunks : kHostChunks;
    if (want > HostPipe::kMaxChunks) want = HostPipe::kMaxChunks;
    const int C = nbz < want ? nbz : want;
    // HXG_PIPE_TRACE=1: per-chunk stage times to stderr (measurement only)
    static const bool trace = std::getenv("HXG_PIPE_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto tmark = [&](cudaStream_t st) {
      if (!trace) return;
      cudaEvent_t e;
      HXG_CUDA(cudaEventCreate(&e));
      HXG_CUDA(cudaEventRecord(e, st));
      tev.push_back(e);
    };
    const auto t_host0 = std::chrono::steady_clock::now();
    tmark(op.stream_);
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
      tmark(pp.h2d);
    }
    for (int i = 0; i < C; ++i) {
      const int lb = (int)((long long)i * nbz / C), le = (int)((long long)(i + 1) * nbz / C);
      HXG_CUDA(cudaStreamWaitEvent(pp.comp, pp.in_ready[i], 0));
      FusedParams pc = prm;
      pc.brick0 = lb * layer;
      pc.nbricks = (le - lb) * layer;
      // a fraction of the SMs is enough to keep up with PCIe and leaves the
      // copy engines' memory traffic less contended (HXG_PIPE_GRID_PCT)
      static const int grid_pct = [] {
        const char* e = std::getenv("HXG_PIPE_GRID_PCT");
        return e ? std::atoi(e) : kPipeGridPct;
      }();
      unsigned g = persistent_grid(k, D::T, smem, pc.nbricks);
      g = grid_pct > 0 && grid_pct < 100 ? (g * (unsigned)grid_pct + 99) / 100 : g;
      k<<<g, D::T, smem, pp.comp>>>(pc);
      HXG_CUDA(cudaGetLastError());
      const int zs = i == 0 ? 0 : pb2 * lb;
      const int ze = i == C - 1 ? npz : pb2 * le;
      fused_fixup_kernel<P, Q><<<fixup_grid(pc.nbricks), kFixupThreads, 0, pp.comp>>>(pc);
      HXG_CUDA(cudaGetLastError());
      HXG_CUDA(cudaEventRecord(pp.out_ready[i], pp.comp));
      tmark(pp.comp);
      HXG_CUDA(cudaStreamWaitEvent(pp.d2h, pp.out_ready[i], 0));
      HXG_CUDA(cudaMemcpyAsync(yh + zs * plane, pp.y.p + zs * plane,
                               (size_t)(ze - zs) * plane * sizeof(double), cudaMemcpyDeviceToHost,
                               pp.d2h));
      tmark(pp.d2h);
    }
    HXG_CUDA(cudaEventRecord(pp.done_evt, pp.d2h));
    HXG_CUDA(cudaStreamWaitEvent(op.stream_, pp.done_evt, 0));
    const auto t_host1 = std::chrono::steady_clock::now();
    HXG_CUDA(cudaStreamSynchronize(pp.d2h));
    if (trace) {
      HXG_CUDA(cudaDeviceSynchronize());
      std::fprintf(stderr, "[pipe] C=%d enqueue %.1f us |", C,
                   std::chrono::duration<double, std::micro>(t_host1 - t_host0).count());
      for (size_t i = 1; i < tev.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tev[0], tev[i]);
        std::fprintf(stderr, " %.0f", ms * 1e3);
      }
      std::fprintf(stderr, " (us: h2d x C, then comp/d2h per chunk)\n");
      for (auto e : tev) cudaEventDestroy(e);
    }
  });
}

}  // namespace hxg
