// comm.h — the collectives of the row-partitioned path (block vectors partitioned
// by rows) behind one interface:
//   * allreduce_sum_f64  — the step's single Gram allreduce (the "sync" of PAPER.md:154, 234),
//                          ||B||_F^2 and the explicit-residual norm;
//   * allreduce_max_i32  — the X0 != 0 flag;
//   * allgather_i64      — row ranges and ghost counts at create time;
//   * exchange           — grouped point-to-point: the halo of the SpMM and the ghost-plan lists.
// NcclComm is the product (one process per GPU, NCCL over NVLink / NVSwitch).  LoopComm runs P
// ranks as P host threads on ONE device for testing the multi-rank path: every collective is a
// host rendezvous plus stream-event dependencies and plain copies / one reduction kernel, so no
// kernel ever waits on another rank's kernel (B200_PROFILING.md: no spinning cross-rank kernels
// on one GPU).  Sums run over ranks in rank order, so every rank gets identical bits.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace lsba {

struct P2POp {          // one peer of a grouped exchange (bytes; either side may be 0)
  int peer;
  const void* send;
  size_t send_bytes;
  void* recv;
  size_t recv_bytes;
};

class Comm {
 public:
  virtual ~Comm() {}
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // Each returns 0 on success, else an error (message in err): 1 = CUDA, 2 = NCCL.
  virtual int allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) = 0;
  virtual int allreduce_max_i32(int* buf, size_t count, cudaStream_t s) = 0;
  virtual int allgather_i64(const int64_t* send, int64_t* recv, size_t count, cudaStream_t s) = 0;
  virtual int exchange(const std::vector<P2POp>& ops, cudaStream_t s) = 0;
  std::string err;
};

// ------------------------------------------------------------------------------------ NCCL
class NcclComm : public Comm {
 public:
  ncclComm_t comm = nullptr;
  int r = 0, p = 1;
  // f2: device-API state for the Gram allreduce folded into the Gram's tail (gram7.cuh)
  bool devar = false;
  ncclDevComm dcomm{};
  ncclDevComm* d_dcomm = nullptr;   // device copy read by the Gram kernel
  ncclWindow_t win = nullptr;
  void* wbuf = nullptr;
  ~NcclComm() override {
    if (d_dcomm) cudaFree(d_dcomm);
    if (devar) ncclDevCommDestroy(comm, &dcomm);
    if (win) ncclCommWindowDeregister(comm, win);
    if (wbuf) ncclMemFree(wbuf);
    if (comm) ncclCommDestroy(comm);
  }
  // Collective over the ranks: a symmetric window of `bytes` and a device communicator with one
  // LSA barrier.  Returns 0 and leaves devar false (plain ncclAllReduce) when the ranks do not
  // all share one NVLink load/store domain.
  int init_devar(size_t bytes) {
    bytes = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    if (int e = check(ncclMemAlloc(&wbuf, bytes))) return e;
    if (int e = check(ncclCommWindowRegister(comm, wbuf, bytes, &win, NCCL_WIN_COLL_SYMMETRIC))) return e;
    ncclDevCommRequirements reqs;
    std::memset(&reqs, 0, sizeof reqs);
    reqs.lsaBarrierCount = 1;
    if (int e = check(ncclDevCommCreate(comm, &reqs, &dcomm))) return e;
    if (cudaMalloc((void**)&d_dcomm, sizeof dcomm) != cudaSuccess ||
        cudaMemcpy(d_dcomm, &dcomm, sizeof dcomm, cudaMemcpyHostToDevice) != cudaSuccess) {
      err = "CUDA: device communicator copy";
      ncclDevCommDestroy(comm, &dcomm);
      return 1;
    }
    devar = (dcomm.lsaSize == p);
    return 0;
  }
  int init(const ncclUniqueId& uid, int nranks, int rank) {
    r = rank;
    p = nranks;
    return check(ncclCommInitRank(&comm, nranks, uid, rank));
  }
  int rank() const override { return r; }
  int size() const override { return p; }
  int allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) override {
    return check(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, comm, s));
  }
  int allreduce_max_i32(int* buf, size_t count, cudaStream_t s) override {
    return check(ncclAllReduce(buf, buf, count, ncclInt, ncclMax, comm, s));
  }
  int allgather_i64(const int64_t* send, int64_t* recv, size_t count, cudaStream_t s) override {
    return check(ncclAllGather(send, recv, count, ncclInt64, comm, s));
  }
  int exchange(const std::vector<P2POp>& ops, cudaStream_t s) override {
    if (ops.empty()) return 0;
    if (int e = check(ncclGroupStart())) return e;
    for (const P2POp& o : ops) {
      if (o.send_bytes) {
        if (int e = check(ncclSend(o.send, o.send_bytes, ncclUint8, o.peer, comm, s))) { ncclGroupEnd(); return e; }
      }
      if (o.recv_bytes) {
        if (int e = check(ncclRecv(o.recv, o.recv_bytes, ncclUint8, o.peer, comm, s))) { ncclGroupEnd(); return e; }
      }
    }
    return check(ncclGroupEnd());
  }

 private:
  int check(ncclResult_t r_) {
    if (r_ == ncclSuccess) return 0;
    err = std::string("NCCL: ") + ncclGetErrorString(r_);
    return 2;
  }
};

// ------------------------------------------------------------------------------------ loopback
constexpr int kLoopMaxRanks = 16;
struct LoopPtrs { const void* p[kLoopMaxRanks]; };

template <typename T, bool MAX>
__global__ void k_loop_reduce(size_t count, int P, LoopPtrs src, T* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    T acc = static_cast<const T*>(src.p[0])[i];
    for (int q = 1; q < P; ++q) {            // rank order: identical bits on every rank
      const T v = static_cast<const T*>(src.p[q])[i];
      acc = MAX ? (v > acc ? v : acc) : acc + v;
    }
    out[i] = acc;
  }
}

struct LoopGroup {
  explicit LoopGroup(int P_) : P(P_), slot(P_) {}
  ~LoopGroup() {
    for (Slot& s : slot) {
      if (s.ev1) cudaEventDestroy(s.ev1);
      if (s.ev2) cudaEventDestroy(s.ev2);
      if (s.scratch) cudaFree(s.scratch);
    }
  }
  struct Slot {
    const void* send = nullptr;
    std::vector<P2POp> ops;
    cudaEvent_t ev1 = nullptr, ev2 = nullptr;
    void* scratch = nullptr;
    size_t scap = 0;
  };
  int P;
  std::vector<Slot> slot;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

class LoopComm : public Comm {
 public:
  LoopComm(LoopGroup* g_, int r_) : g(g_), r(r_) {}
  int init() {
    LoopGroup::Slot& me = g->slot[r];
    if (!me.ev1 && cuda(cudaEventCreateWithFlags(&me.ev1, cudaEventDisableTiming))) return 1;
    if (!me.ev2 && cuda(cudaEventCreateWithFlags(&me.ev2, cudaEventDisableTiming))) return 1;
    return 0;
  }
  int rank() const override { return r; }
  int size() const override { return g->P; }

  int allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) override {
    return reduce<double, false>(buf, count, s);
  }
  int allreduce_max_i32(int* buf, size_t count, cudaStream_t s) override {
    return reduce<int, true>(buf, count, s);
  }
  int allgather_i64(const int64_t* send, int64_t* recv, size_t count, cudaStream_t s) override {
    LoopGroup::Slot& me = g->slot[r];
    me.send = send;
    if (cuda(cudaEventRecord(me.ev1, s))) return 1;
    g->barrier();
    for (int q = 0; q < g->P; ++q) {
      if (q != r && cuda(cudaStreamWaitEvent(s, g->slot[q].ev1, 0))) return 1;
      if (count && cuda(cudaMemcpyAsync(recv + (size_t)q * count, g->slot[q].send, sizeof(int64_t) * count,
                                        cudaMemcpyDeviceToDevice, s))) return 1;
    }
    return finish(s);
  }
  int exchange(const std::vector<P2POp>& ops, cudaStream_t s) override {
    LoopGroup::Slot& me = g->slot[r];
    me.ops = ops;
    if (cuda(cudaEventRecord(me.ev1, s))) return 1;
    g->barrier();
    for (const P2POp& o : ops) {
      if (!o.recv_bytes) continue;
      const LoopGroup::Slot& peer = g->slot[o.peer];
      const P2POp* match = nullptr;
      for (const P2POp& po : peer.ops)
        if (po.peer == r) match = &po;
      if (!match || match->send_bytes != o.recv_bytes) {
        err = "loopback exchange: unmatched send/recv sizes";
        g->barrier();
        return 1;
      }
      if (cuda(cudaStreamWaitEvent(s, peer.ev1, 0))) return 1;
      if (cuda(cudaMemcpyAsync(o.recv, match->send, o.recv_bytes, cudaMemcpyDeviceToDevice, s))) return 1;
    }
    return finish(s);
  }

 private:
  LoopGroup* g;
  int r;
  int cuda(cudaError_t e) {
    if (e == cudaSuccess) return 0;
    err = std::string("CUDA (loopback comm): ") + cudaGetErrorString(e);
    return 1;
  }
  // second rendezvous: nobody reuses a buffer a peer still reads
  int finish(cudaStream_t s) {
    LoopGroup::Slot& me = g->slot[r];
    if (cuda(cudaEventRecord(me.ev2, s))) return 1;
    g->barrier();
    for (int q = 0; q < g->P; ++q)
      if (q != r && cuda(cudaStreamWaitEvent(s, g->slot[q].ev2, 0))) return 1;
    return 0;
  }
  template <typename T, bool MAX>
  int reduce(T* buf, size_t count, cudaStream_t s) {
    LoopGroup::Slot& me = g->slot[r];
    if (me.scap < count * sizeof(T)) {
      if (me.scratch) cudaFree(me.scratch);
      me.scratch = nullptr;
      me.scap = 0;
      if (cuda(cudaMalloc(&me.scratch, count * sizeof(T)))) return 1;
      me.scap = count * sizeof(T);
    }
    me.send = buf;
    if (cuda(cudaEventRecord(me.ev1, s))) return 1;
    g->barrier();
    LoopPtrs src{};
    for (int q = 0; q < g->P; ++q) {
      src.p[q] = g->slot[q].send;
      if (q != r && cuda(cudaStreamWaitEvent(s, g->slot[q].ev1, 0))) return 1;
    }
    if (count) {
      const int grid = (int)std::min<size_t>((count + 255) / 256, 1024);
      k_loop_reduce<T, MAX><<<grid, 256, 0, s>>>(count, g->P, src, static_cast<T*>(me.scratch));
      if (cuda(cudaGetLastError())) return 1;
    }
    if (int e = finish(s)) return e;
    if (count && cuda(cudaMemcpyAsync(buf, me.scratch, count * sizeof(T), cudaMemcpyDeviceToDevice, s))) return 1;
    return 0;
  }
};

}  // namespace lsba
