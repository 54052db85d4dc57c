// comm.h — collectives of the partitioned (multi-GPU) solve path.
//
// The reference has no inter-process communication; the
// partitioned solve adds exactly two kinds of traffic:
//   * halo exchange: interface-node partial sums of every EBE product, one
//     point-to-point message per neighbouring partition (NCCL send/recv over
//     NVLink, grouped so all neighbours go at once);
//   * all-reduce: the per-column fp64 sums of every dot product (and the
//     replicated level-2 restriction), NCCL all-reduce.
// Two backends implement the same interface:
//   * NcclComm   — one process per GPU; NCCL is resolved at run time (dlopen),
//                  so the library also loads where NCCL is absent, and inside a
//                  torch process it binds the NCCL torch already loaded;
//   * ThreadComm — P ranks as P host threads of one process (any devices,
//                  including one shared GPU): the same SPMD solve code,
//                  exchanging through device copies + host barriers. Used to
//                  exercise the partitioned path on a single B200.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

namespace tsg {

struct Comm {
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual int device() const = 0;
  // in-place sums over ranks; every rank receives the identical result
  virtual void allreduce_sum(double* d, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_sum(float* d, size_t n, cudaStream_t s) = 0;
  // point-to-point: to neighbour nbr[k] send sbuf[k] (sbytes[k]) and receive
  // rbytes[k] into rbuf[k]; device buffers, ordered on stream s
  virtual void exchange(int nn, const int* nbr, void* const* sbuf, const size_t* sbytes, void* const* rbuf,
                        const size_t* rbytes, cudaStream_t s) = 0;
  virtual void barrier() = 0;
  // HOST bytes from `root` to every rank (setup data built once, e.g. level 2)
  virtual void broadcast(void* host, size_t n, int root) = 0;
  // a rank failed: peers blocked in (or entering) a collective fail too instead of waiting forever
  virtual void abort() {}
  virtual const char* kind() const = 0;
};

// ---- NCCL (one process per GPU) ---------------------------------------------
constexpr int kNcclIdBytes = 128;
bool nccl_available(std::string* why = nullptr);
void nccl_unique_id(unsigned char id[kNcclIdBytes]);
std::unique_ptr<Comm> make_nccl_comm(int nranks, int rank, const unsigned char id[kNcclIdBytes], int device);

// ---- in-process ranks (threads) ---------------------------------------------
struct ThreadWorld;  // shared by the P rank objects of one group
std::shared_ptr<ThreadWorld> make_thread_world(int nranks);
std::unique_ptr<Comm> make_thread_comm(const std::shared_ptr<ThreadWorld>& w, int rank, int device);

}  // namespace tsg

// the communicator behind an ABI handle (abi.cpp)
struct ts_comm;
namespace tsg {
Comm* comm_of(ts_comm* c);
}  // namespace tsg
