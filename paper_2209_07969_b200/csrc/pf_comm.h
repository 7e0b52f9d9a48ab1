// pf_comm.h — communication layer of the row-strip decomposition.
//
// Two implementations of the same two operations, both stream-ordered from the solver's view:
//   allreduce(d_buf, n)   FP64 sum of n device scalars over all strips (identical result on
//                         every rank)
//   halo(vec, comps)      every rank receives its ghost node rows (lower / upper neighbour)
//                         from their owners; rows are contiguous ranges (row-compact layout)
// * NcclComm: ncclAllReduce / grouped ncclSend+ncclRecv over NVLink / NVSwitch.  NCCL is
//   dlopen'ed at first use (the torch-bundled libnccl.so.2 when PFB200_NCCL_LIB points to it),
//   so the single-GPU library has no link-time NCCL dependency.
// * HostComm: an in-process emulation for several strips driven by several host threads on
//   ONE GPU (tests): device->host copies, a host barrier, rank-ordered host sums, host->device
//   copies.  No kernel ever waits on another kernel; all waiting happens on the host.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "nccl.h"

namespace pfb {

struct HaloSpec {
  int rank = 0, nranks = 1;
  long long send_lo_start = 0, send_lo_count = 0, recv_lo_start = 0, recv_lo_count = 0;
  long long send_hi_start = 0, send_hi_count = 0, recv_hi_start = 0, recv_hi_count = 0;
  bool has_lo() const { return rank > 0 && send_lo_count > 0; }
  bool has_hi() const { return rank < nranks - 1 && send_hi_count > 0; }
};

struct Comm {
  HaloSpec spec;
  virtual ~Comm() {}
  // returns an error string or empty
  virtual std::string allreduce(double* d_buf, int n, cudaStream_t s) = 0;
  virtual std::string halo(double* vec, int comps, cudaStream_t s) = 0;
  virtual bool capturable() const { return false; }  // may be recorded into a CUDA graph
};

// ---------------------------------------------------------------------------------------
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    return api;
  }
  std::string load() {
    if (lib) return "";
    const char* path = getenv("PFB200_NCCL_LIB");
    const char* cands[] = {path, "libnccl.so.2", "libnccl.so"};
    for (const char* c : cands) {
      if (!c) continue;
      lib = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
      if (lib) break;
    }
    if (!lib) return std::string("cannot dlopen NCCL: ") + dlerror();
#define PFB_SYM(name, field)                                     \
  field = reinterpret_cast<decltype(field)>(dlsym(lib, name));   \
  if (!field) return std::string("NCCL symbol missing: ") + name;
    PFB_SYM("ncclGetUniqueId", GetUniqueId)
    PFB_SYM("ncclCommInitRank", CommInitRank)
    PFB_SYM("ncclCommDestroy", CommDestroy)
    PFB_SYM("ncclAllReduce", AllReduce)
    PFB_SYM("ncclSend", Send)
    PFB_SYM("ncclRecv", Recv)
    PFB_SYM("ncclGroupStart", GroupStart)
    PFB_SYM("ncclGroupEnd", GroupEnd)
    PFB_SYM("ncclGetErrorString", GetErrorString)
#undef PFB_SYM
    return "";
  }
};

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  bool capturable() const override { return true; }
  ~NcclComm() override {
    if (comm) NcclApi::get().CommDestroy(comm);
  }
  std::string check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return "";
    return std::string(what) + ": " + NcclApi::get().GetErrorString(r);
  }
  std::string init(const unsigned char* id_bytes) {
    NcclApi& api = NcclApi::get();
    std::string e = api.load();
    if (!e.empty()) return e;
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    return check(api.CommInitRank(&comm, spec.nranks, id, spec.rank), "ncclCommInitRank");
  }
  std::string allreduce(double* d_buf, int n, cudaStream_t s) override {
    return check(NcclApi::get().AllReduce(d_buf, d_buf, (size_t)n, ncclDouble, ncclSum, comm, s),
                 "ncclAllReduce");
  }
  std::string halo(double* vec, int comps, cudaStream_t s) override {
    NcclApi& api = NcclApi::get();
    std::string e = check(api.GroupStart(), "ncclGroupStart");
    if (!e.empty()) return e;
    if (spec.has_lo()) {
      e += check(api.Send(vec + spec.send_lo_start * comps, spec.send_lo_count * comps,
                          ncclDouble, spec.rank - 1, comm, s), "ncclSend lo");
      e += check(api.Recv(vec + spec.recv_lo_start * comps, spec.recv_lo_count * comps,
                          ncclDouble, spec.rank - 1, comm, s), "ncclRecv lo");
    }
    if (spec.has_hi()) {
      e += check(api.Send(vec + spec.send_hi_start * comps, spec.send_hi_count * comps,
                          ncclDouble, spec.rank + 1, comm, s), "ncclSend hi");
      e += check(api.Recv(vec + spec.recv_hi_start * comps, spec.recv_hi_count * comps,
                          ncclDouble, spec.rank + 1, comm, s), "ncclRecv hi");
    }
    e += check(api.GroupEnd(), "ncclGroupEnd");
    return e;
  }
};

// ---------------------------------------------------------------------------------------
struct HostGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int waiting = 0;
  long long generation = 0;
  std::vector<std::vector<double>> red, out_lo, out_hi;
  explicit HostGroup(int nranks) : n(nranks), red(nranks), out_lo(nranks), out_hi(nranks) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++waiting == n) {
      waiting = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct HostComm : Comm {
  HostGroup* g = nullptr;
  static std::string cu(cudaError_t e) { return e == cudaSuccess ? "" : cudaGetErrorString(e); }
  std::string allreduce(double* d_buf, int n, cudaStream_t s) override {
    std::vector<double> mine(n);
    std::string e = cu(cudaMemcpyAsync(mine.data(), d_buf, n * sizeof(double),
                                       cudaMemcpyDeviceToHost, s));
    e += cu(cudaStreamSynchronize(s));
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->red[spec.rank] = mine;
    }
    g->barrier();
    std::vector<double> sum(n, 0.0);
    for (int r = 0; r < g->n; ++r)
      for (int i = 0; i < n; ++i) sum[i] += g->red[r][i];  // rank order: deterministic
    g->barrier();
    e += cu(cudaMemcpyAsync(d_buf, sum.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    e += cu(cudaStreamSynchronize(s));
    return e;
  }
  std::string halo(double* vec, int comps, cudaStream_t s) override {
    std::string e;
    auto pull = [&](std::vector<double>& dst, long long start, long long count) {
      dst.resize(count * comps);
      e += cu(cudaMemcpyAsync(dst.data(), vec + start * comps, count * comps * sizeof(double),
                              cudaMemcpyDeviceToHost, s));
    };
    if (spec.has_lo()) pull(g->out_lo[spec.rank], spec.send_lo_start, spec.send_lo_count);
    if (spec.has_hi()) pull(g->out_hi[spec.rank], spec.send_hi_start, spec.send_hi_count);
    e += cu(cudaStreamSynchronize(s));
    g->barrier();
    if (spec.has_lo()) {
      const std::vector<double>& src = g->out_hi[spec.rank - 1];
      e += cu(cudaMemcpyAsync(vec + spec.recv_lo_start * comps, src.data(),
                              src.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    if (spec.has_hi()) {
      const std::vector<double>& src = g->out_lo[spec.rank + 1];
      e += cu(cudaMemcpyAsync(vec + spec.recv_hi_start * comps, src.data(),
                              src.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    e += cu(cudaStreamSynchronize(s));
    g->barrier();
    return e;
  }
};

}  // namespace pfb
