// Transports of the sharded fit (see comm.h).
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

namespace rtd {

namespace {

void cu(cudaError_t e, const char* where) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw CommError{std::string("CUDA error ") + cudaGetErrorString(e) + " in " + where};
  }
}

// ------------------------------------------------------------------ NCCL, resolved at run time
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer the libnccl.so.2 already in the process (torch's), else the loader's search path
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
#define RTD_SYM(f)                                                        \
  api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f));         \
  if (!api.f) {                                                           \
    api.error = "libnccl.so.2 lacks nccl" #f;                             \
    return;                                                               \
  }
    RTD_SYM(GetUniqueId)
    RTD_SYM(CommInitRank)
    RTD_SYM(CommDestroy)
    RTD_SYM(AllGather)
    RTD_SYM(Send)
    RTD_SYM(Recv)
    RTD_SYM(GroupStart)
    RTD_SYM(GroupEnd)
    RTD_SYM(GetErrorString)
#undef RTD_SYM
  });
  if (!api.error.empty()) throw CommError{api.error};
  return api;
}

void nc(ncclResult_t r, const char* where) {
  if (r != ncclSuccess) throw CommError{std::string("NCCL error ") + nccl().GetErrorString(r) + " in " + where};
}

class NcclComm final : public Comm {
 public:
  NcclComm(const void* id, int rank, int world) : Comm(rank, world) {
    ncclUniqueId uid;
    static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
    memcpy(&uid, id, sizeof(uid));
    nc(nccl().CommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  void allgather_dev(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    nc(nccl().AllGather(send, recv, bytes, ncclChar, comm_, st), "ncclAllGather");
    cu(cudaStreamSynchronize(st), "allgather");
  }
  void alltoallv_dev(const void* send, const size_t* sb, const size_t* so, void* recv, const size_t* rb,
                     const size_t* ro, cudaStream_t st) override {
    nc(nccl().GroupStart(), "ncclGroupStart");
    for (int s = 0; s < world_; s++) {
      if (sb[s]) nc(nccl().Send((const char*)send + so[s], sb[s], ncclChar, s, comm_, st), "ncclSend");
      if (rb[s]) nc(nccl().Recv((char*)recv + ro[s], rb[s], ncclChar, s, comm_, st), "ncclRecv");
    }
    nc(nccl().GroupEnd(), "ncclGroupEnd");
    cu(cudaStreamSynchronize(st), "alltoallv");
  }
  void allgather_host(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    if (dev_cap_ < bytes * (world_ + 1)) {
      if (dev_) cudaFree(dev_);
      dev_ = nullptr;
      dev_cap_ = 0;
      cu(cudaMalloc(&dev_, bytes * (world_ + 1)), "cudaMalloc (allgather staging)");
      dev_cap_ = bytes * (world_ + 1);
    }
    char* s = (char*)dev_;
    char* r = s + bytes;
    cu(cudaMemcpyAsync(s, send, bytes, cudaMemcpyHostToDevice, st), "allgather h2d");
    allgather_dev(s, r, bytes, st);
    cu(cudaMemcpyAsync(recv, r, bytes * world_, cudaMemcpyDeviceToHost, st), "allgather d2h");
    cu(cudaStreamSynchronize(st), "allgather_host");
  }
  const char* kind() const override { return "nccl"; }

 private:
  ncclComm_t comm_ = nullptr;
  void* dev_ = nullptr;
  size_t dev_cap_ = 0;
};

// ------------------------------------------------------------------ caller callbacks on host buffers
class HostComm final : public Comm {
 public:
  HostComm(const rtdetmcd_transport& t, int rank, int world) : Comm(rank, world), t_(t) {}
  void allgather_host(const void* send, void* recv, size_t bytes, cudaStream_t) override {
    if (t_.allgather(t_.user, send, recv, bytes) != 0) throw CommError{"transport allgather failed"};
  }
  void allgather_dev(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    std::vector<char> s(bytes), r(bytes * world_);
    cu(cudaMemcpyAsync(s.data(), send, bytes, cudaMemcpyDeviceToHost, st), "allgather d2h");
    cu(cudaStreamSynchronize(st), "allgather d2h");
    allgather_host(s.data(), r.data(), bytes, st);
    cu(cudaMemcpyAsync(recv, r.data(), r.size(), cudaMemcpyHostToDevice, st), "allgather h2d");
    cu(cudaStreamSynchronize(st), "allgather h2d");
  }
  void alltoallv_dev(const void* send, const size_t* sb, const size_t* so, void* recv, const size_t* rb,
                     const size_t* ro, cudaStream_t st) override {
    size_t stot = 0, rtot = 0;
    for (int s = 0; s < world_; s++) {
      stot = std::max(stot, so[s] + sb[s]);
      rtot = std::max(rtot, ro[s] + rb[s]);
    }
    std::vector<char> hs(stot), hr(rtot);
    cu(cudaMemcpyAsync(hs.data(), send, stot, cudaMemcpyDeviceToHost, st), "alltoallv d2h");
    cu(cudaStreamSynchronize(st), "alltoallv d2h");
    if (t_.alltoallv(t_.user, hs.data(), sb, so, hr.data(), rb, ro) != 0) throw CommError{"transport alltoallv failed"};
    cu(cudaMemcpyAsync(recv, hr.data(), rtot, cudaMemcpyHostToDevice, st), "alltoallv h2d");
    cu(cudaStreamSynchronize(st), "alltoallv h2d");
  }
  const char* kind() const override { return "host"; }

 private:
  rtdetmcd_transport t_;
};

}  // namespace

Comm* make_nccl_comm(const void* unique_id, int rank, int world) { return new NcclComm(unique_id, rank, world); }
Comm* make_host_comm(const rtdetmcd_transport& t, int rank, int world) { return new HostComm(t, rank, world); }

void nccl_unique_id(void* out) {
  ncclUniqueId uid;
  nc(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  memcpy(out, &uid, sizeof(uid));
}

}  // namespace rtd
