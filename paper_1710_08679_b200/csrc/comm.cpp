// comm.cpp — NCCL (dlopen) and in-process thread backends of tsg::Comm.
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

#include "ts_common.h"

namespace tsg {

// ============================================================ NCCL backend
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // prefer the NCCL already mapped into the process (torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.Send && a.Recv && a.GroupStart &&
           a.GroupEnd && a.Broadcast && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks required symbols";
    return a;
  }();
  return api;
}

#define TS_NCCL(x)                                                                            \
  do {                                                                                        \
    ncclResult_t r_ = (x);                                                                    \
    if (r_ != ncclSuccess) fail(TS_ERR_NCCL, std::string(#x) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

class NcclComm final : public Comm {
 public:
  NcclComm(int nranks, int rank, const unsigned char id[kNcclIdBytes], int device)
      : n_(nranks), r_(rank), dev_(device) {
    const NcclApi& a = nccl();
    if (!a.ok) fail(TS_ERR_NCCL, "nccl: " + a.why);
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == kNcclIdBytes, "ncclUniqueId size");
    std::memcpy(uid.internal, id, kNcclIdBytes);
    TS_CUDA(cudaSetDevice(device));
    TS_NCCL(a.CommInitRank(&comm_, nranks, uid, rank));
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  int rank() const override { return r_; }
  int size() const override { return n_; }
  int device() const override { return dev_; }
  void allreduce_sum(double* d, size_t n, cudaStream_t s) override {
    if (n_ > 1) TS_NCCL(nccl().AllReduce(d, d, n, ncclFloat64, ncclSum, comm_, s));
  }
  void allreduce_sum(float* d, size_t n, cudaStream_t s) override {
    if (n_ > 1) TS_NCCL(nccl().AllReduce(d, d, n, ncclFloat32, ncclSum, comm_, s));
  }
  void exchange(int nn, const int* nbr, void* const* sbuf, const size_t* sbytes, void* const* rbuf,
                const size_t* rbytes, cudaStream_t s) override {
    if (nn == 0) return;
    const NcclApi& a = nccl();
    TS_NCCL(a.GroupStart());
    for (int k = 0; k < nn; ++k) {
      if (sbytes[k]) TS_NCCL(a.Send(sbuf[k], sbytes[k], ncclChar, nbr[k], comm_, s));
      if (rbytes[k]) TS_NCCL(a.Recv(rbuf[k], rbytes[k], ncclChar, nbr[k], comm_, s));
    }
    TS_NCCL(a.GroupEnd());
  }
  void barrier() override {
    double* d = nullptr;
    TS_CUDA(cudaMalloc(&d, sizeof(double)));
    TS_CUDA(cudaMemset(d, 0, sizeof(double)));
    allreduce_sum(d, 1, nullptr);
    TS_CUDA(cudaDeviceSynchronize());
    cudaFree(d);
  }
  void broadcast(void* host, size_t n, int root) override {
    if (n_ == 1 || n == 0) return;
    void* d = nullptr;
    TS_CUDA(cudaMalloc(&d, n));
    struct Free {
      void* p;
      ~Free() { cudaFree(p); }
    } guard{d};
    if (r_ == root) TS_CUDA(cudaMemcpy(d, host, n, cudaMemcpyHostToDevice));
    TS_NCCL(nccl().Broadcast(d, d, n, ncclChar, root, comm_, nullptr));
    TS_CUDA(cudaStreamSynchronize(nullptr));
    if (r_ != root) TS_CUDA(cudaMemcpy(host, d, n, cudaMemcpyDeviceToHost));
  }
  const char* kind() const override { return "nccl"; }

 private:
  int n_, r_, dev_;
  ncclComm_t comm_ = nullptr;
};

}  // namespace

bool nccl_available(std::string* why) {
  const NcclApi& a = nccl();
  if (why) *why = a.why;
  return a.ok;
}

void nccl_unique_id(unsigned char id[kNcclIdBytes]) {
  const NcclApi& a = nccl();
  if (!a.ok) fail(TS_ERR_NCCL, "nccl: " + a.why);
  ncclUniqueId uid;
  TS_NCCL(a.GetUniqueId(&uid));
  std::memcpy(id, uid.internal, kNcclIdBytes);
}

std::unique_ptr<Comm> make_nccl_comm(int nranks, int rank, const unsigned char id[kNcclIdBytes], int device) {
  if (nranks < 1 || rank < 0 || rank >= nranks) validation("comm: rank out of range");
  return std::make_unique<NcclComm>(nranks, rank, id, device);
}

// ============================================================ thread backend
struct ThreadWorld {
  explicit ThreadWorld(int n)
      : n(n), dev(n, 0), sptr(size_t(n) * n, nullptr), sbytes(size_t(n) * n, 0), hd(n), hf(n) {}
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<int> dev;
  std::vector<const void*> sptr;  // [from][to]
  std::vector<size_t> sbytes;
  std::vector<std::vector<double>> hd;
  std::vector<std::vector<float>> hf;
  const void* bcast = nullptr;
  bool aborted = false;
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) fail(TS_ERR_NCCL, "thread comm: a peer rank failed");
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
      if (gen == g) {  // woken by an abort, not by the last arrival
        --arrived;
        fail(TS_ERR_NCCL, "thread comm: a peer rank failed");
      }
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

namespace {

class ThreadComm final : public Comm {
 public:
  ThreadComm(std::shared_ptr<ThreadWorld> w, int rank, int device) : w_(std::move(w)), r_(rank), dev_(device) {
    w_->dev[rank] = device;
  }
  int rank() const override { return r_; }
  int size() const override { return w_->n; }
  int device() const override { return dev_; }
  template <typename T>
  void sum(T* d, size_t n, cudaStream_t s, std::vector<std::vector<T>>& slots) {
    if (w_->n == 1) return;
    std::vector<T>& mine = slots[r_];
    mine.resize(n);
    TS_CUDA(cudaMemcpyAsync(mine.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    TS_CUDA(cudaStreamSynchronize(s));
    w_->wait();
    std::vector<T> tot(n, T(0));
    for (int q = 0; q < w_->n; ++q)  // rank order on every rank: identical results
      for (size_t i = 0; i < n; ++i) tot[i] += slots[q][i];
    w_->wait();
    TS_CUDA(cudaMemcpyAsync(d, tot.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
    TS_CUDA(cudaStreamSynchronize(s));
  }
  void allreduce_sum(double* d, size_t n, cudaStream_t s) override { sum(d, n, s, w_->hd); }
  void allreduce_sum(float* d, size_t n, cudaStream_t s) override { sum(d, n, s, w_->hf); }
  void exchange(int nn, const int* nbr, void* const* sbuf, const size_t* sbytes, void* const* rbuf,
                const size_t* rbytes, cudaStream_t s) override {
    TS_CUDA(cudaStreamSynchronize(s));  // packed send buffers complete
    for (int k = 0; k < nn; ++k) {
      w_->sptr[size_t(r_) * w_->n + nbr[k]] = sbuf[k];
      w_->sbytes[size_t(r_) * w_->n + nbr[k]] = sbytes[k];
    }
    w_->wait();
    for (int k = 0; k < nn; ++k) {
      const size_t idx = size_t(nbr[k]) * w_->n + r_;
      if (w_->sbytes[idx] != rbytes[k]) {
        w_->abort();
        fail(TS_ERR_VALIDATION, "thread comm: halo size mismatch");
      }
      if (rbytes[k])
        TS_CUDA(cudaMemcpyPeerAsync(rbuf[k], dev_, w_->sptr[idx], w_->dev[nbr[k]], rbytes[k], s));
    }
    TS_CUDA(cudaStreamSynchronize(s));
    w_->wait();  // peers may now reuse their send buffers
  }
  void barrier() override { w_->wait(); }
  void broadcast(void* host, size_t n, int root) override {
    if (w_->n == 1 || n == 0) return;
    if (r_ == root) w_->bcast = host;
    w_->wait();
    if (r_ != root) std::memcpy(host, w_->bcast, n);
    w_->wait();  // the root's buffer stays valid until every copy is done
  }
  void abort() override { w_->abort(); }
  const char* kind() const override { return "thread"; }

 private:
  std::shared_ptr<ThreadWorld> w_;
  int r_, dev_;
};

}  // namespace

std::shared_ptr<ThreadWorld> make_thread_world(int nranks) {
  if (nranks < 1 || nranks > 64) validation("comm: thread world size must be in [1, 64]");
  return std::make_shared<ThreadWorld>(nranks);
}

std::unique_ptr<Comm> make_thread_comm(const std::shared_ptr<ThreadWorld>& w, int rank, int device) {
  if (!w || rank < 0 || rank >= w->n) validation("comm: rank out of range");
  return std::make_unique<ThreadComm>(w, rank, device);
}

}  // namespace tsg
