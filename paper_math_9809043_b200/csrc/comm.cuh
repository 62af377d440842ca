// comm.cuh — the z-slab collectives of the distributed solver.
//
//   halo       after a sweep / prolongation / lift: the boundary xy-planes of a level
//              vector go into the neighbours' ghost planes (depth 1; depth 2 for the
//              y-restricted temporary the z-restriction reads).
//   allreduce  one fp64 CG scalar (r.z, p.Ap, ||r||^2, ||b||^2): allgather of the
//              per-rank partials, then a fixed-order sum on device -> identical bits on
//              every rank, so every rank takes the same stop decisions.
//   gather     the slabs of the first replicated level (restricted RHS at solve time,
//              faces at setup) into the full array on every rank.
//
// Backends: NCCL (one process per GPU, NVLink/NVSwitch; ncclSend/Recv, ncclAllGather,
// ncclBroadcast, all enqueued on the context's stream) and LOOPBACK (P ranks as host
// threads of one process on one GPU, each with its own context and stream; exchanges are
// device copies between the contexts' buffers fenced by host barriers).  Loopback runs
// the full decomposition on a single GPU so it can be parity-tested; only the transport
// differs from NCCL.  No kernel ever waits on another rank's kernel.
#pragma once
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <vector>

#ifdef MSS_WITH_NCCL
#include <nccl.h>
#endif

#include "internal.cuh"
#include "kernels.cuh"

namespace mss {

struct Comm {
  int rank = 0, size = 1;
  double* gbuf = nullptr;   // device [size] allgather buffer (NCCL allreduce)
  virtual ~Comm() {}
  // v: interior pointer of a ghosted level vector (plane elements per xy-plane, nzl local
  // planes); copies `depth` boundary planes into the neighbours' ghost planes.
  virtual int halo(cudaStream_t st, double* v, int64_t plane, int nzl, int depth) {
    return exch(st, v, v - depth * plane, v + (int64_t)(nzl - depth) * plane, v + (int64_t)nzl * plane,
                (size_t)plane * depth);
  }
  // general neighbour exchange: send_lo -> rank-1 (lands in its recv_hi), send_hi -> rank+1
  // (lands in its recv_lo); n elements each way.
  virtual int exch(cudaStream_t st, const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi,
                   size_t n) = 0;
  virtual int allreduce_sum(cudaStream_t st, double* dev_val) = 0;
  // full: array of the replicated level; segment r is [off[r], off[r] + len[r]) (elements),
  // each rank has filled its own segment.
  virtual int gather(cudaStream_t st, double* full, const std::vector<int64_t>& off,
                     const std::vector<int64_t>& len) = 0;
  virtual int barrier(cudaStream_t st) = 0;
};

// ---------------------------------------------------------------------------- loopback
struct LoopGroup {
  int size;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<double*> ptr;
  std::vector<const double*> lo, hi;
  std::vector<double> val;
  int refs = 0;
  explicit LoopGroup(int n) : size(n), ptr(n, nullptr), lo(n, nullptr), hi(n, nullptr), val(n, 0.0) {}
  bool broken = false;
  // host barrier; false if a rank failed to arrive within 300 s (the group is then
  // broken and every later collective fails instead of hanging)
  bool wait() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const long long g = gen;
    if (++arrived == size) {
      arrived = 0;
      gen++;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct LoopComm : Comm {
  LoopGroup* g;
  LoopComm(LoopGroup* grp, int r) : g(grp) {
    rank = r;
    size = grp->size;
  }
  int exch(cudaStream_t st, const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi,
           size_t n) override {
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSS_ECUDA;
    g->lo[rank] = send_lo;
    g->hi[rank] = send_hi;
    if (!g->wait()) return MSS_EINVAL;
    const size_t bytes = sizeof(double) * n;
    if (rank > 0 && cudaMemcpyAsync(recv_lo, g->hi[rank - 1], bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return MSS_ECUDA;
    if (rank < size - 1 && cudaMemcpyAsync(recv_hi, g->lo[rank + 1], bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return MSS_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSS_ECUDA;
    if (!g->wait()) return MSS_EINVAL;   // nobody overwrites a boundary plane before every neighbour copied it
    return MSS_OK;
  }
  int allreduce_sum(cudaStream_t st, double* dev_val) override {
    double h = 0.0;
    if (cudaMemcpyAsync(&h, dev_val, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess) return MSS_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSS_ECUDA;
    g->val[rank] = h;
    if (!g->wait()) return MSS_EINVAL;
    double s = 0.0;
    for (int i = 0; i < size; ++i) s += g->val[i];
    if (!g->wait()) return MSS_EINVAL;
    if (cudaMemcpyAsync(dev_val, &s, sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess) return MSS_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSS_ECUDA;
    return MSS_OK;
  }
  int gather(cudaStream_t st, double* full, const std::vector<int64_t>& off, const std::vector<int64_t>& len) override {
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSS_ECUDA;
    g->ptr[rank] = full;
    if (!g->wait()) return MSS_EINVAL;
    for (int q = 0; q < size; ++q) {
      if (q == rank || len[q] == 0) continue;
      if (cudaMemcpyAsync(full + off[q], g->ptr[q] + off[q], sizeof(double) * len[q], cudaMemcpyDeviceToDevice, st) !=
          cudaSuccess)
        return MSS_ECUDA;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSS_ECUDA;
    if (!g->wait()) return MSS_EINVAL;
    return MSS_OK;
  }
  int barrier(cudaStream_t st) override {
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSS_ECUDA;
    return g->wait() ? MSS_OK : MSS_EINVAL;
  }
};

// ---------------------------------------------------------------------------- NCCL
#ifdef MSS_WITH_NCCL
struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  int exch(cudaStream_t st, const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi,
           size_t n) override {
    // a failed call inside the group still closes it, so later collectives are not absorbed
    if (ncclGroupStart() != ncclSuccess) return MSS_ENCCL;
    bool ok = true;
    if (rank > 0) {
      ok = ok && ncclSend(send_lo, n, ncclDouble, rank - 1, c, st) == ncclSuccess;
      ok = ok && ncclRecv(recv_lo, n, ncclDouble, rank - 1, c, st) == ncclSuccess;
    }
    if (rank < size - 1) {
      ok = ok && ncclSend(send_hi, n, ncclDouble, rank + 1, c, st) == ncclSuccess;
      ok = ok && ncclRecv(recv_hi, n, ncclDouble, rank + 1, c, st) == ncclSuccess;
    }
    const bool closed = ncclGroupEnd() == ncclSuccess;
    return (ok && closed) ? MSS_OK : MSS_ENCCL;
  }
  int allreduce_sum(cudaStream_t st, double* dev_val) override {
    if (ncclAllGather(dev_val, gbuf, 1, ncclDouble, c, st) != ncclSuccess) return MSS_ENCCL;
    k_sum_ordered<<<1, 32, 0, st>>>(gbuf, size, dev_val);
    return cudaGetLastError() == cudaSuccess ? MSS_OK : MSS_ECUDA;
  }
  int gather(cudaStream_t st, double* full, const std::vector<int64_t>& off, const std::vector<int64_t>& len) override {
    if (ncclGroupStart() != ncclSuccess) return MSS_ENCCL;
    bool ok = true;
    for (int q = 0; q < size && ok; ++q) {
      if (len[q] == 0) continue;
      ok = ncclBroadcast(full + off[q], full + off[q], len[q], ncclDouble, q, c, st) == ncclSuccess;
    }
    const bool closed = ncclGroupEnd() == ncclSuccess;
    return (ok && closed) ? MSS_OK : MSS_ENCCL;
  }
  int barrier(cudaStream_t st) override {
    // an allreduce of one element is the cheapest stream-ordered barrier
    if (ncclAllReduce(gbuf, gbuf, 1, ncclDouble, ncclSum, c, st) != ncclSuccess) return MSS_ENCCL;
    return cudaStreamSynchronize(st) == cudaSuccess ? MSS_OK : MSS_ECUDA;
  }
};
#endif

}  // namespace mss
