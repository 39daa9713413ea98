// Partitioned (multi-GPU) composition of the hot path: the
// box is cut into px x py x pz contiguous element blocks, one per rank; each
// rank holds every lattice node of its block, so the only shared entries are
// the node planes between neighbouring blocks.  The reference is
// single-process; the paper runs the same operator distributed,
// summing shared nodes after every apply (A = P^T E^T B^T D B E P,
// PAPER.md:224-228, :316).
//
//  * Comm: the communicator the library calls -- a table of two collective
//    entry points (grouped neighbour exchange, all-reduce) over device
//    buffers, stream-ordered.  Built in: NCCL (libnccl.so.2 resolved at
//    runtime, ncclSend/ncclRecv groups and ncclAllReduce on the operator's
//    stream).  Callers may supply their own table (the multi-process tests
//    on one GPU use gloo through it).
//  * Partition: block geometry, interface sums (x, then y, then z planes:
//    nodes on partition edges / corners collect all contributions, bitwise
//    identical on every rank holding them), interface scaling for the
//    transfers, owned-entry masks (a shared node belongs to the lower block
//    in every direction) and owned-entry dots (one all-reduce each).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <vector>

#include "common.hpp"
#include "hexmg_b200.h"
#include "operator.hpp"
#include "vector.hpp"

namespace hxg {

class Comm {
 public:
  Comm(int rank, int world, const hxg_comm_ops& ops) : rank_(rank), world_(world), ops_(ops) {}
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int world() const { return world_; }
  // Grouped exchange with up to 6 peers: send[i] (counts[i] doubles) to
  // peers[i], recv[i] from peers[i]; complete in stream order.
  virtual void exchange(int npeers, const int* peers, const double* const* send,
                        double* const* recv, const int64_t* counts, cudaStream_t s);
  // In-place all-reduce of `count` device doubles (op 0 sum, 1 max).
  virtual void allreduce(double* data, int64_t count, int op, cudaStream_t s);

 protected:
  int rank_, world_;
  hxg_comm_ops ops_{};
};

// NCCL communicator (ncclCommInitRank from a 128-byte unique id).
std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* unique_id);
void nccl_unique_id(void* out128);

// A node lattice of the partitioned box as this rank sees it: local nodes
// per direction, global nodes per direction, global index of local node 0.
// Order-p lattices: n = p cells + 1; h-multigrid levels of the p = 1 lattice
// (coarsened by 2^l): n = cells / 2^l + 1.
struct Lattice {
  int n[3] = {1, 1, 1};
  int g[3] = {1, 1, 1};
  long long off[3] = {0, 0, 0};
  long long size() const { return 3LL * n[0] * n[1] * n[2]; }
};

class Partition {
 public:
  // gcells: the whole box; dims: blocks per direction (rank = x fastest).
  Partition(Comm* comm, const int gcells[3], const int dims[3]);
  ~Partition() {
    if (host_) cudaFreeHost(host_);
  }
  Partition(const Partition&) = delete;
  Partition& operator=(const Partition&) = delete;
  Comm& comm() const { return *comm_; }
  int rank() const { return comm_->rank(); }
  const int* dims() const { return dims_; }
  const int* coords() const { return coords_; }
  const int* cells() const { return cells_; }  // local element counts
  const int* e0() const { return e0_; }        // first global element per direction
  const int* gcells() const { return gcells_; }
  int neighbour(int d, int step) const;  // rank, or -1 at the box boundary
  // faces of this block shared with a neighbour (bits -x,+x,-y,+y,-z,+z)
  int interface_faces() const {
    int bits = 0;
    for (int d = 0; d < 3; ++d) {
      if (neighbour(d, -1) >= 0) bits |= 1 << (2 * d);
      if (neighbour(d, +1) >= 0) bits |= 1 << (2 * d + 1);
    }
    return bits;
  }
  // Global Dirichlet faces (bit f: -x,+x,-y,+y,-z,+z) -> the ones on this block.
  int local_faces(int global_faces) const;

  // y (local L-vector of an order-p lattice) += the neighbours' partial sums
  // on the shared planes (x, y, z passes).  With mask (device), constrained
  // entries on the shared planes become x instead (identity rows).
  void exchange(int p, double* y, cudaStream_t s, const double* x = nullptr,
                const uint8_t* mask = nullptr);
  // y *= f on every shared plane (once per shared direction: a node on k
  // partition planes gets f^k), the multiplicity correction of the transfers.
  void scale_interfaces(int p, double* y, double f, cudaStream_t s);
  // 1 on the entries this rank owns (device, per order).
  const uint8_t* owned(int p);
  // Owned-entry dot, all-reduced over ranks.
  double dot(int p, const double* x, const double* y, cudaStream_t s);
  // Max over ranks of a host scalar (failure flags).
  double allreduce_max(double v, cudaStream_t s);
  // rough_seed (cg.hpp:138-147, mt19937(0x9e3779b9)) of the GLOBAL order-p
  // lattice vector restricted to this block, constrained entries zeroed.
  std::vector<double> global_seed_slice(int p, const std::vector<uint8_t>& local_mask) const;
  // Local node index -> global node index helpers (order p).
  void npd(int p, int out[3]) const;
  void global_npd(int p, int out[3]) const;

  // The same operations on an explicit lattice (the p-variants call these).
  Lattice lattice(int p) const;
  // h-level l of the p = 1 lattice; requires 2^l | the block's cells and
  // offsets (checked).
  Lattice h_lattice(int l) const;
  void exchange(const Lattice& L, double* y, cudaStream_t s, const double* x = nullptr,
                const uint8_t* mask = nullptr);
  void scale_interfaces(const Lattice& L, double* y, double f, cudaStream_t s);
  const uint8_t* owned(const Lattice& L);
  double dot(const Lattice& L, const double* x, const double* y, cudaStream_t s);
  std::vector<double> global_seed_slice(const Lattice& L, const std::vector<uint8_t>& local_mask) const;

 private:
  Comm* comm_;
  int gcells_[3], dims_[3], coords_[3], cells_[3], e0_[3];
  std::map<std::vector<int>, DevBuf<uint8_t>> owned_;
  DevBuf<double> buf_[4];  // send lo / hi, recv lo / hi
  DevBuf<double> scalar_;
  double* host_ = nullptr;  // pinned scalar
  DotWorkspace ws_;
};

}  // namespace hxg
