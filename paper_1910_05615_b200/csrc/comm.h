// Inter-rank exchanges of the sharded fit (§4 partition + global standardisation,
// PAPER.md:849-874 aggregation, PAPER.md:975-995 distributed reweighting).  One process per GPU;
// the paper's master thread becomes "every rank runs the same deterministic fold of all-gathered
// records", so the only collectives are an all-gather and an all-to-all(v) of bytes.
//
// Two transports behind one interface:
//   NcclComm      -- NCCL over NVLink / NVSwitch on device buffers, enqueued on the context stream;
//                    libnccl.so.2 is dlopen'ed (the copy torch already loaded, else the system one),
//                    so the library has no link-time NCCL dependency;
//   HostComm      -- caller-supplied callbacks on host buffers (rtdetmcd_transport: e.g. gloo, MPI,
//                    or threads of one process); device data is staged through host memory.
// Every call is collective: all ranks call it in the same order with matching sizes.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "rtdetmcd.h"

namespace rtd {

struct CommError {
  std::string msg;
};

class Comm {
 public:
  Comm(int rank, int world) : rank_(rank), world_(world) {}
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int world() const { return world_; }
  // all-gather of `bytes` per rank; send / recv (world * bytes, rank order) DEVICE buffers; complete on return
  virtual void allgather_dev(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
  // all-to-all-v of DEVICE buffers: send_bytes[s] bytes from send + send_offs[s] go to rank s, recv_bytes[s]
  // bytes from rank s land at recv + recv_offs[s]; complete on return
  virtual void alltoallv_dev(const void* send, const size_t* send_bytes, const size_t* send_offs, void* recv,
                             const size_t* recv_bytes, const size_t* recv_offs, cudaStream_t st) = 0;
  // all-gather of HOST buffers (small records, status words)
  virtual void allgather_host(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
  virtual const char* kind() const = 0;

 protected:
  int rank_, world_;
};

// NCCL communicator for `world` ranks (id from rtdetmcd_nccl_unique_id on one rank, shared by the caller)
Comm* make_nccl_comm(const void* unique_id, int rank, int world);
// callbacks of the caller (copied)
Comm* make_host_comm(const rtdetmcd_transport& t, int rank, int world);
// 128-byte ncclUniqueId
void nccl_unique_id(void* out);

}  // namespace rtd
