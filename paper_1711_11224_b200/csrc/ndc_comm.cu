// z-slab transports (ndc_plan.h Transport):
//  * NcclTransport -- one process per GPU, grouped ncclSend/ncclRecv for the p_z-plane
//    halos (the plan issues them on its comm stream, overlapped with compute) and
//    ncclAllGather for the per-rank f64 partials (plan stream), over NVLink / NVSwitch.
//    Both go through ONE communicator: NCCL runs the operations of a communicator in
//    the order they are issued, whatever user stream each is enqueued on, and every rank
//    issues the same sequence (identical host decisions), so the order is the same on
//    all ranks -- no cross-communicator ordering hazard.  The price is that a scalar
//    all-gather waits for a halo exchange issued before it (config 5 at 8 ranks: ~0.6 ms
//    of NVLink time against a ~0.6 s iteration).
//    libnccl.so.2 is opened at run time (the unsharded path never needs it; when torch
//    has already loaded its bundled NCCL the same library object is reused).
//  * LocalTransport -- several slab ranks driven by host threads of one process (tests
//    and single-node emulation on fewer GPUs): halos are device-to-device copies issued
//    by the receiving rank after a host barrier on the stream it is given; no kernel ever
//    waits on another.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "ndc_plan.h"

namespace ndc {
namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // NDC_NCCL_LIBRARY: an explicit libnccl path (a process that will also load another
    // NCCL -- e.g. a framework's bundled copy -- must use that same library: the dynamic
    // linker shares one libnccl.so.2 per process by soname)
    void* h = nullptr;
    if (const char* path = std::getenv("NDC_NCCL_LIBRARY")) h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    api.lib = h;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(h, "ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(h, "ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
    api.GetErrorString =
        reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.lib || !api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv ||
      !api.GroupStart || !api.GroupEnd || !api.AllGather)
    fail(NDC_ERR_NCCL, "libnccl.so.2 not loadable");
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(NDC_ERR_NCCL, std::string(what) + ": " +
                           (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

class NcclTransport final : public Transport {
 public:
  NcclTransport(int device, int rank, int world, const unsigned char id[128])
      : rank_(rank), world_(world) {
    if (world < 1 || rank < 0 || rank >= world) fail(NDC_ERR_ARGUMENT, "bad rank / world");
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
    std::memcpy(uid.internal, id, 128);
    check_nccl(nccl().CommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclTransport() override {
    if (comm_ && nccl().CommDestroy) nccl().CommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  void exchange(const float* send_lo, float* recv_lo, const float* send_hi, float* recv_hi,
                size_t count, cudaStream_t s) override {
    auto& api = nccl();
    check_nccl(api.GroupStart(), "ncclGroupStart");
    if (send_lo) check_nccl(api.Send(send_lo, count, ncclFloat32, rank_ - 1, comm_, s), "ncclSend");
    if (recv_lo) check_nccl(api.Recv(recv_lo, count, ncclFloat32, rank_ - 1, comm_, s), "ncclRecv");
    if (send_hi) check_nccl(api.Send(send_hi, count, ncclFloat32, rank_ + 1, comm_, s), "ncclSend");
    if (recv_hi) check_nccl(api.Recv(recv_hi, count, ncclFloat32, rank_ + 1, comm_, s), "ncclRecv");
    check_nccl(api.GroupEnd(), "ncclGroupEnd");
  }
  void allgather(const double* in, double* out, size_t n, cudaStream_t s) override {
    check_nccl(nccl().AllGather(in, out, n, ncclFloat64, comm_, s), "ncclAllGather");
  }

 private:
  int rank_, world_;
  ncclComm_t comm_ = nullptr;
};

}  // namespace

// In-process group of slab ranks (one host thread per rank).
struct LocalGroup {
  explicit LocalGroup(int w) : world(w), slots(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
  struct Slot {
    const float* send_lo = nullptr;
    const float* send_hi = nullptr;
    const double* gin = nullptr;
  };
  int world;
  std::vector<Slot> slots;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
};

namespace {

class LocalTransport final : public Transport {
 public:
  LocalTransport(LocalGroup* g, int rank) : g_(g), rank_(rank) {}
  int rank() const override { return rank_; }
  int world() const override { return g_->world; }
  void exchange(const float* send_lo, float* recv_lo, const float* send_hi, float* recv_hi,
                size_t count, cudaStream_t s) override {
    check_cuda(cudaStreamSynchronize(s), "halo: producer sync");
    g_->slots[rank_].send_lo = send_lo;
    g_->slots[rank_].send_hi = send_hi;
    g_->barrier();
    if (recv_lo)
      check_cuda(cudaMemcpyAsync(recv_lo, g_->slots[rank_ - 1].send_hi, count * 4,
                                 cudaMemcpyDefault, s),
                 "halo copy");
    if (recv_hi)
      check_cuda(cudaMemcpyAsync(recv_hi, g_->slots[rank_ + 1].send_lo, count * 4,
                                 cudaMemcpyDefault, s),
                 "halo copy");
    check_cuda(cudaStreamSynchronize(s), "halo: consumer sync");
    g_->barrier();  // senders may reuse their planes only after every pull landed
  }
  void allgather(const double* in, double* out, size_t n, cudaStream_t s) override {
    check_cuda(cudaStreamSynchronize(s), "gather: producer sync");
    g_->slots[rank_].gin = in;
    g_->barrier();
    for (int r = 0; r < g_->world; ++r)
      check_cuda(cudaMemcpyAsync(out + r * n, g_->slots[r].gin, n * 8, cudaMemcpyDefault, s),
                 "gather copy");
    check_cuda(cudaStreamSynchronize(s), "gather: consumer sync");
    g_->barrier();
  }

 private:
  LocalGroup* g_;
  int rank_;
};

}  // namespace

std::unique_ptr<Transport> make_nccl_transport(int device, int rank, int world,
                                               const unsigned char id[128]) {
  return std::make_unique<NcclTransport>(device, rank, world, id);
}

LocalGroup* new_local_group(int world) { return new LocalGroup(world); }
void delete_local_group(LocalGroup* g) { delete g; }

std::unique_ptr<Transport> make_local_transport(LocalGroup* g, int rank) {
  if (!g || rank < 0 || rank >= g->world) fail(NDC_ERR_ARGUMENT, "bad local group rank");
  return std::make_unique<LocalTransport>(g, rank);
}

void nccl_unique_id(unsigned char out[128]) {
  ncclUniqueId uid;
  check_nccl(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out, uid.internal, 128);
}

}  // namespace ndc
