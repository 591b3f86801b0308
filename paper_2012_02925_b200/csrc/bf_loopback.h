// bf_loopback.h — in-process stand-in for the NCCL calls of the multi-rank path.
//
// The device runtime moves halo messages with ncclGroupStart / ncclSend /
// ncclRecv / ncclGroupEnd and sums residuals with ncclAllGather (bf_runtime.cu
// nccl_exchange, rank_allgather).  This header gives the same five entry points
// with NCCL's stream semantics for ranks that are threads of ONE process (one
// host thread per rank, any GPUs, several ranks may share one GPU):
//
//   * Send / Recv inside a group are matched per (sender, receiver) pair in
//     issue order, as NCCL matches them;
//   * a receive is a device-to-device copy on the receiver's stream, ordered
//     after the sender's stream reached the send (event), and the sender's
//     stream is ordered after the copy (the send "completes" when the data
//     has moved, so the sender may refill its buffer afterwards);
//   * AllGather concatenates every rank's buffer in rank order, with the same
//     two-sided stream ordering.
//
// So the runtime's exchange / overlap / allgather code runs unchanged with
// this transport bound instead of libnccl — which is how the NCCL path is
// exercised on a one-GPU machine (tests/test_gpu_loopback.py).  Host threads
// block only inside GroupEnd / AllGather, after posting all of their own sends,
// so ranks that issue the same sequence of collectives cannot deadlock; a
// timeout (BF_LOOPBACK_TIMEOUT seconds, default 120) or bf_loopback_abort()
// turns a missing peer into an error instead of a hang.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

namespace bf_lb {

struct Post {                     // one send waiting for its receive
  const void* buf = nullptr;
  size_t bytes = 0;
  cudaEvent_t ready = nullptr;    // sender's stream reached the send
  cudaEvent_t consumed = nullptr; // receiver's copy done (recorded on its stream)
  bool done = false;
};

struct Gather {                   // one AllGather generation
  std::vector<const void*> buf;
  std::vector<cudaEvent_t> ready, done;
  int posted = 0, copied = 0, left = 0;
};

struct World {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<std::shared_ptr<Post>>> box;   // (src, dst)
  std::map<long long, Gather> gathers;
  bool aborted = false;
  double timeout_s = 120.0;
  explicit World(int nranks) : n(nranks) {
    if (const char* e = std::getenv("BF_LOOPBACK_TIMEOUT")) timeout_s = std::atof(e);
  }
};

struct Rank {                     // what a loopback ncclComm_t points to
  World* w = nullptr;
  int rank = 0;
  long long gen = 0;              // AllGather calls made by this rank
};

inline Rank* as_rank(ncclComm_t c) { return reinterpret_cast<Rank*>(c); }

struct Op {
  bool send;
  void* buf;
  size_t bytes;
  int peer;
  Rank* r;
  cudaStream_t s;
};

inline thread_local std::vector<Op> t_ops;
inline thread_local int t_depth = 0;

// wait on w->cv until pred() holds; false on abort / timeout
template <class Pred>
bool wait_for(World* w, std::unique_lock<std::mutex>& lk, Pred pred) {
  const auto until = std::chrono::steady_clock::now() +
                     std::chrono::milliseconds((long long)(w->timeout_s * 1000.0));
  while (!pred()) {
    if (w->aborted) return false;
    if (w->cv.wait_until(lk, until) == std::cv_status::timeout && !pred()) {
      w->aborted = true;   // a peer is gone: release every waiter
      w->cv.notify_all();
      return false;
    }
  }
  return !w->aborted;
}

inline cudaEvent_t new_event() {
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}

inline ncclResult_t flush(std::vector<Op>& ops) {
  if (ops.empty()) return ncclSuccess;
  World* w = ops[0].r->w;
  std::vector<std::pair<const Op*, std::shared_ptr<Post>>> sent;
  // 1. post every send (never blocks)
  for (const Op& op : ops) {
    if (!op.send) continue;
    auto p = std::make_shared<Post>();
    p->buf = op.buf;
    p->bytes = op.bytes;
    p->ready = new_event();
    if (cudaEventRecord(p->ready, op.s) != cudaSuccess) return ncclUnhandledCudaError;
    {
      std::lock_guard<std::mutex> lk(w->m);
      w->box[{op.r->rank, op.peer}].push_back(p);
    }
    sent.emplace_back(&op, p);
  }
  w->cv.notify_all();
  // 2. every receive: take the peer's oldest unmatched send, copy on our stream
  for (const Op& op : ops) {
    if (op.send) continue;
    std::shared_ptr<Post> p;
    {
      std::unique_lock<std::mutex> lk(w->m);
      auto& q = w->box[{op.peer, op.r->rank}];
      if (!wait_for(w, lk, [&] { return !q.empty(); })) return ncclSystemError;
      p = q.front();
      q.pop_front();
    }
    if (p->bytes != op.bytes) return ncclInvalidUsage;   // NCCL: truncation error
    if (cudaStreamWaitEvent(op.s, p->ready, 0) != cudaSuccess) return ncclUnhandledCudaError;
    if (op.bytes && cudaMemcpyAsync(op.buf, p->buf, op.bytes, cudaMemcpyDefault, op.s) !=
                        cudaSuccess)
      return ncclUnhandledCudaError;
    cudaEvent_t c = new_event();
    if (cudaEventRecord(c, op.s) != cudaSuccess) return ncclUnhandledCudaError;
    {
      std::lock_guard<std::mutex> lk(w->m);
      p->consumed = c;
      p->done = true;
    }
    w->cv.notify_all();
  }
  // 3. a send completes when its receiver copied it
  for (auto& [op, p] : sent) {
    {
      std::unique_lock<std::mutex> lk(w->m);
      if (!wait_for(w, lk, [&] { return p->done; })) return ncclSystemError;
    }
    if (cudaStreamWaitEvent(op->s, p->consumed, 0) != cudaSuccess) return ncclUnhandledCudaError;
    cudaEventDestroy(p->ready);      // released once the queued waits completed
    cudaEventDestroy(p->consumed);
  }
  return ncclSuccess;
}

inline ncclResult_t GroupStart() {
  ++t_depth;
  return ncclSuccess;
}

inline ncclResult_t GroupEnd() {
  if (t_depth <= 0) return ncclInvalidUsage;
  if (--t_depth > 0) return ncclSuccess;
  std::vector<Op> ops;
  ops.swap(t_ops);
  return flush(ops);
}

inline size_t type_bytes(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

inline ncclResult_t enqueue(bool send, const void* buf, size_t count, ncclDataType_t t, int peer,
                            ncclComm_t comm, cudaStream_t s) {
  Rank* r = as_rank(comm);
  if (!r || peer < 0 || peer >= r->w->n) return ncclInvalidArgument;
  t_ops.push_back(Op{send, const_cast<void*>(buf), count * type_bytes(t), peer, r, s});
  if (t_depth == 0) {   // outside a group: a group of one
    std::vector<Op> ops;
    ops.swap(t_ops);
    return flush(ops);
  }
  return ncclSuccess;
}

inline ncclResult_t Send(const void* buf, size_t count, ncclDataType_t t, int peer,
                         ncclComm_t comm, cudaStream_t s) {
  return enqueue(true, buf, count, t, peer, comm, s);
}

inline ncclResult_t Recv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                         cudaStream_t s) {
  return enqueue(false, buf, count, t, peer, comm, s);
}

inline ncclResult_t AllGather(const void* sendbuf, void* recvbuf, size_t count, ncclDataType_t t,
                              ncclComm_t comm, cudaStream_t s) {
  Rank* r = as_rank(comm);
  if (!r) return ncclInvalidArgument;
  World* w = r->w;
  const size_t bytes = count * type_bytes(t);
  const long long g = r->gen++;
  cudaEvent_t ready = new_event();
  if (cudaEventRecord(ready, s) != cudaSuccess) return ncclUnhandledCudaError;
  std::vector<const void*> bufs;
  std::vector<cudaEvent_t> readies;
  {
    std::unique_lock<std::mutex> lk(w->m);
    Gather& G = w->gathers[g];
    if (G.buf.empty()) {
      G.buf.assign(w->n, nullptr);
      G.ready.assign(w->n, nullptr);
      G.done.assign(w->n, nullptr);
      G.left = w->n;
    }
    G.buf[r->rank] = sendbuf;
    G.ready[r->rank] = ready;
    G.posted += 1;
    w->cv.notify_all();
    if (!wait_for(w, lk, [&] { return w->gathers[g].posted == w->n; })) return ncclSystemError;
    bufs = w->gathers[g].buf;
    readies = w->gathers[g].ready;
  }
  for (int q = 0; q < w->n; ++q) {
    if (cudaStreamWaitEvent(s, readies[q], 0) != cudaSuccess) return ncclUnhandledCudaError;
    if (bytes && cudaMemcpyAsync(static_cast<char*>(recvbuf) + (size_t)q * bytes, bufs[q], bytes,
                                 cudaMemcpyDefault, s) != cudaSuccess)
      return ncclUnhandledCudaError;
  }
  cudaEvent_t done = new_event();
  if (cudaEventRecord(done, s) != cudaSuccess) return ncclUnhandledCudaError;
  std::vector<cudaEvent_t> dones;
  {
    std::unique_lock<std::mutex> lk(w->m);
    Gather& G = w->gathers[g];
    G.done[r->rank] = done;
    G.copied += 1;
    w->cv.notify_all();
    if (!wait_for(w, lk, [&] { return w->gathers[g].copied == w->n; })) return ncclSystemError;
    dones = w->gathers[g].done;
  }
  // our send buffer may be refilled only after every rank copied it
  for (int q = 0; q < w->n; ++q)
    if (cudaStreamWaitEvent(s, dones[q], 0) != cudaSuccess) return ncclUnhandledCudaError;
  {
    std::lock_guard<std::mutex> lk(w->m);
    Gather& G = w->gathers[g];
    if (--G.left == 0) {   // every rank has queued its waits: release the events
      for (auto e : G.ready) cudaEventDestroy(e);
      for (auto e : G.done) cudaEventDestroy(e);
      w->gathers.erase(g);
    }
  }
  return ncclSuccess;
}

inline const char* GetErrorString(ncclResult_t r) {
  switch (r) {
    case ncclSuccess: return "no error";
    case ncclUnhandledCudaError: return "loopback transport: CUDA call failed";
    case ncclSystemError: return "loopback transport: peer rank did not arrive (timeout/abort)";
    case ncclInvalidUsage: return "loopback transport: mismatched send/recv sizes or group nesting";
    case ncclInvalidArgument: return "loopback transport: invalid argument";
    default: return "loopback transport error";
  }
}

inline void abort(World* w) {
  std::lock_guard<std::mutex> lk(w->m);
  w->aborted = true;
  w->cv.notify_all();
}

}  // namespace bf_lb
