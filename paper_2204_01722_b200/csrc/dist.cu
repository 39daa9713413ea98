#include "dist.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <random>
#include <string>

namespace hxg {

// ---------------------------------------------------------------- Comm
void Comm::exchange(int npeers, const int* peers, const double* const* send, double* const* recv,
                    const int64_t* counts, cudaStream_t s) {
  if (npeers == 0) return;
  if (!ops_.exchange) throw Error(HXG_ERR_INVALID_ARGUMENT, "communicator has no exchange");
  const int rc = ops_.exchange(ops_.ctx, npeers, peers, send, recv, counts, s);
  if (rc) throw Error(HXG_ERR_GENERIC, "communicator exchange failed (" + std::to_string(rc) + ")");
}

void Comm::allreduce(double* data, int64_t count, int op, cudaStream_t s) {
  if (world_ == 1) return;
  if (!ops_.allreduce) throw Error(HXG_ERR_INVALID_ARGUMENT, "communicator has no all-reduce");
  const int rc = ops_.allreduce(ops_.ctx, data, count, op, s);
  if (rc) throw Error(HXG_ERR_GENERIC, "communicator all-reduce failed (" + std::to_string(rc) + ")");
}

namespace {

// NCCL entry points, resolved from the process's libnccl.so.2 (the one torch
// loaded, if any) so the library itself loads without NCCL.
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw Error(HXG_ERR_UNSUPPORTED, "libnccl.so.2 not found");
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) throw Error(HXG_ERR_UNSUPPORTED, std::string("NCCL symbol missing: ") + n);
    return p;
  };
  api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.Send = (decltype(api.Send))sym("ncclSend");
  api.Recv = (decltype(api.Recv))sym("ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
  api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  api.h = h;
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(HXG_ERR_GENERIC, std::string(what) + ": " + nccl().GetErrorString(r));
}

class NcclComm : public Comm {
 public:
  NcclComm(int rank, int world, const void* id) : Comm(rank, world, hxg_comm_ops{}) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(nccl().CommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  void exchange(int npeers, const int* peers, const double* const* send, double* const* recv,
                const int64_t* counts, cudaStream_t s) override {
    if (npeers == 0) return;
    auto& a = nccl();
    nccl_check(a.GroupStart(), "ncclGroupStart");
    for (int i = 0; i < npeers; ++i) {
      nccl_check(a.Send(send[i], (size_t)counts[i], ncclFloat64, peers[i], comm_, s), "ncclSend");
      nccl_check(a.Recv(recv[i], (size_t)counts[i], ncclFloat64, peers[i], comm_, s), "ncclRecv");
    }
    nccl_check(a.GroupEnd(), "ncclGroupEnd");
  }
  void allreduce(double* data, int64_t count, int op, cudaStream_t s) override {
    if (world_ == 1) return;
    nccl_check(nccl().AllReduce(data, data, (size_t)count, ncclFloat64, op ? ncclMax : ncclSum,
                                comm_, s),
               "ncclAllReduce");
  }

 private:
  ncclComm_t comm_ = nullptr;
};

// Node (g0, g1, g2) of plane i along direction d, entry t (component fastest).
__device__ __forceinline__ long long plane_dof(int d, int i, long long t, int nx, int ny) {
  const long long j = t / 3;
  const int c = (int)(t - 3 * j);
  long long gx, gy, gz;
  if (d == 0) {
    gx = i, gy = j % ny, gz = j / ny;
  } else if (d == 1) {
    gx = j % nx, gy = i, gz = j / nx;
  } else {
    gx = j % nx, gy = j / nx, gz = i;
  }
  return 3 * (gx + nx * (gy + (long long)ny * gz)) + c;
}

__global__ void pack_plane(const double* __restrict__ y, int d, int i, int nx, int ny,
                           long long count, double* __restrict__ buf) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x)
    buf[t] = y[plane_dof(d, i, t, nx, ny)];
}

// plane = own + received (a + b == b + a bitwise: both sides agree);
// with a mask, constrained entries are the identity row's x instead of a sum
// (operator.hpp:212-214 on every block holding them).
__global__ void add_plane(double* __restrict__ y, int d, int i, int nx, int ny, long long count,
                          const double* __restrict__ own, const double* __restrict__ recv,
                          const double* __restrict__ x, const uint8_t* __restrict__ mask) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x) {
    const long long dof = plane_dof(d, i, t, nx, ny);
    y[dof] = mask && mask[dof] ? x[dof] : own[t] + recv[t];
  }
}

__global__ void scale_plane(double* __restrict__ y, int d, int i, int nx, int ny, long long count,
                            double f) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x)
    y[plane_dof(d, i, t, nx, ny)] *= f;
}

__global__ void owned_kernel(uint8_t* m, int nx, int ny, int nz, int lox, int loy, int loz) {
  const long long n = 3LL * nx * ny * nz;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long node = t / 3;
    const int gx = (int)(node % nx), gy = (int)((node / nx) % ny), gz = (int)(node / ((long long)nx * ny));
    m[t] = !((lox && gx == 0) || (loy && gy == 0) || (loz && gz == 0));
  }
}

inline int grid_for_count(long long n) {
  long long g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  return g < 1 ? 1 : (int)g;
}

void split(int n, int parts, int i, int& size, int& offset) {
  const int base = n / parts, extra = n % parts;
  size = base + (i < extra ? 1 : 0);
  offset = i * base + (i < extra ? i : extra);
  if (base < 1) throw Error(HXG_ERR_INVALID_ARGUMENT, "more blocks than element layers");
}

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* unique_id) {
  return std::make_unique<NcclComm>(rank, world, unique_id);
}

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

// ----------------------------------------------------------- Partition
Partition::Partition(Comm* comm, const int gcells[3], const int dims[3]) : comm_(comm) {
  const int world = dims[0] * dims[1] * dims[2];
  if (world != comm->world())
    throw Error(HXG_ERR_INVALID_ARGUMENT, "partition blocks != communicator size");
  const int r = comm->rank();
  coords_[0] = r % dims[0];
  coords_[1] = (r / dims[0]) % dims[1];
  coords_[2] = r / (dims[0] * dims[1]);
  for (int d = 0; d < 3; ++d) {
    gcells_[d] = gcells[d];
    dims_[d] = dims[d];
    split(gcells[d], dims[d], coords_[d], cells_[d], e0_[d]);
  }
  scalar_.alloc(1);
  HXG_CUDA(cudaMallocHost(&host_, sizeof(double)));
}

int Partition::neighbour(int d, int step) const {
  int c[3] = {coords_[0], coords_[1], coords_[2]};
  c[d] += step;
  if (c[d] < 0 || c[d] >= dims_[d]) return -1;
  return c[0] + dims_[0] * (c[1] + dims_[1] * c[2]);
}

int Partition::local_faces(int global_faces) const {
  int bits = 0;
  for (int d = 0; d < 3; ++d) {
    if ((global_faces >> (2 * d) & 1) && coords_[d] == 0) bits |= 1 << (2 * d);
    if ((global_faces >> (2 * d + 1) & 1) && coords_[d] == dims_[d] - 1) bits |= 1 << (2 * d + 1);
  }
  return bits;
}

void Partition::npd(int p, int out[3]) const {
  for (int d = 0; d < 3; ++d) out[d] = p * cells_[d] + 1;
}
void Partition::global_npd(int p, int out[3]) const {
  for (int d = 0; d < 3; ++d) out[d] = p * gcells_[d] + 1;
}

Lattice Partition::lattice(int p) const {
  Lattice L;
  for (int d = 0; d < 3; ++d) {
    L.n[d] = p * cells_[d] + 1;
    L.g[d] = p * gcells_[d] + 1;
    L.off[d] = (long long)p * e0_[d];
  }
  return L;
}

Lattice Partition::h_lattice(int l) const {
  Lattice L;
  const int f = 1 << l;
  for (int d = 0; d < 3; ++d) {
    if (cells_[d] % f || e0_[d] % f || gcells_[d] % f)
      throw Error(HXG_ERR_INVALID_ARGUMENT, "h-lattice: block not aligned to the coarsening");
    L.n[d] = cells_[d] / f + 1;
    L.g[d] = gcells_[d] / f + 1;
    L.off[d] = e0_[d] / f;
  }
  return L;
}

void Partition::exchange(int p, double* y, cudaStream_t s, const double* x, const uint8_t* mask) {
  exchange(lattice(p), y, s, x, mask);
}

void Partition::exchange(const Lattice& L, double* y, cudaStream_t s, const double* x,
                         const uint8_t* mask) {
  if (comm_->world() == 1) return;
  const int* n = L.n;
  for (int d = 0; d < 3; ++d) {
    const int lo = neighbour(d, -1), hi = neighbour(d, +1);
    if (lo < 0 && hi < 0) continue;
    const long long count = 3LL * n[0] * n[1] * n[2] / n[d];
    for (auto& b : buf_)
      if (b.n < (size_t)count) b.alloc((size_t)count);
    int peers[2];
    const double* send[2];
    double* recv[2];
    int64_t counts[2];
    int np = 0;
    if (lo >= 0) {
      pack_plane<<<grid_for_count(count), 256, 0, s>>>(y, d, 0, n[0], n[1], count, buf_[0].p);
      peers[np] = lo, send[np] = buf_[0].p, recv[np] = buf_[2].p, counts[np] = count, ++np;
    }
    if (hi >= 0) {
      pack_plane<<<grid_for_count(count), 256, 0, s>>>(y, d, n[d] - 1, n[0], n[1], count, buf_[1].p);
      peers[np] = hi, send[np] = buf_[1].p, recv[np] = buf_[3].p, counts[np] = count, ++np;
    }
    HXG_CUDA(cudaGetLastError());
    comm_->exchange(np, peers, send, recv, counts, s);
    if (lo >= 0)
      add_plane<<<grid_for_count(count), 256, 0, s>>>(y, d, 0, n[0], n[1], count, buf_[0].p, buf_[2].p,
                                                      x, mask);
    if (hi >= 0)
      add_plane<<<grid_for_count(count), 256, 0, s>>>(y, d, n[d] - 1, n[0], n[1], count, buf_[1].p,
                                                      buf_[3].p, x, mask);
    HXG_CUDA(cudaGetLastError());
  }
}

void Partition::scale_interfaces(int p, double* y, double f, cudaStream_t s) {
  scale_interfaces(lattice(p), y, f, s);
}

void Partition::scale_interfaces(const Lattice& L, double* y, double f, cudaStream_t s) {
  const int* n = L.n;
  for (int d = 0; d < 3; ++d) {
    const long long count = 3LL * n[0] * n[1] * n[2] / n[d];
    if (neighbour(d, -1) >= 0)
      scale_plane<<<grid_for_count(count), 256, 0, s>>>(y, d, 0, n[0], n[1], count, f);
    if (neighbour(d, +1) >= 0)
      scale_plane<<<grid_for_count(count), 256, 0, s>>>(y, d, n[d] - 1, n[0], n[1], count, f);
  }
  HXG_CUDA(cudaGetLastError());
}

const uint8_t* Partition::owned(int p) { return owned(lattice(p)); }

const uint8_t* Partition::owned(const Lattice& L) {
  const std::vector<int> key{L.n[0], L.n[1], L.n[2]};
  auto it = owned_.find(key);
  if (it != owned_.end()) return it->second.p;
  DevBuf<uint8_t>& m = owned_[key];
  const long long total = L.size();
  m.alloc((size_t)total);
  owned_kernel<<<grid_for_count(total), 256>>>(m.p, L.n[0], L.n[1], L.n[2], neighbour(0, -1) >= 0,
                                               neighbour(1, -1) >= 0, neighbour(2, -1) >= 0);
  HXG_CUDA(cudaGetLastError());
  HXG_CUDA(cudaDeviceSynchronize());
  return m.p;
}

double Partition::dot(int p, const double* x, const double* y, cudaStream_t s) {
  return dot(lattice(p), x, y, s);
}

double Partition::dot(const Lattice& L, const double* x, const double* y, cudaStream_t s) {
  const uint8_t* m = comm_->world() > 1 ? owned(L) : nullptr;
  double* r = dot_masked_device(x, y, m, L.size(), ws_, 0, s);
  comm_->allreduce(r, 1, 0, s);
  HXG_CUDA(cudaMemcpyAsync(host_, r, sizeof(double), cudaMemcpyDeviceToHost, s));
  HXG_CUDA(cudaStreamSynchronize(s));
  return *host_;
}

double Partition::allreduce_max(double v, cudaStream_t s) {
  if (comm_->world() == 1) return v;
  *host_ = v;
  HXG_CUDA(cudaMemcpyAsync(scalar_.p, host_, sizeof(double), cudaMemcpyHostToDevice, s));
  comm_->allreduce(scalar_.p, 1, 1, s);
  HXG_CUDA(cudaMemcpyAsync(host_, scalar_.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  HXG_CUDA(cudaStreamSynchronize(s));
  return *host_;
}

std::vector<double> Partition::global_seed_slice(int p, const std::vector<uint8_t>& mask) const {
  return global_seed_slice(lattice(p), mask);
}

std::vector<double> Partition::global_seed_slice(const Lattice& L,
                                                 const std::vector<uint8_t>& mask) const {
  const int* n = L.n;
  const int* g = L.g;
  const long long x0 = L.off[0], y0 = L.off[1], z0 = L.off[2];
  std::vector<double> v(3 * (size_t)n[0] * n[1] * n[2]);
  std::mt19937 rng(0x9e3779b9u);
  long long pos = 0;  // global entries consumed so far
  size_t k = 0;
  for (int lz = 0; lz < n[2]; ++lz)
    for (int ly = 0; ly < n[1]; ++ly) {
      const long long g0 = 3 * (x0 + (long long)g[0] * ((y0 + ly) + (long long)g[1] * (z0 + lz)));
      rng.discard((unsigned long long)(g0 - pos));
      for (int t = 0; t < 3 * n[0]; ++t) v[k++] = 2.0 * (rng() * (1.0 / 4294967296.0)) - 1.0;
      pos = g0 + 3LL * n[0];
    }
  if (!mask.empty())
    for (size_t i = 0; i < v.size(); ++i)
      if (mask[i]) v[i] = 0.0;
  return v;
}

}  // namespace hxg
